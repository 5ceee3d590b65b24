"""Time reduce-added split-K schedules of the decode projections, fixed split counts against
stream-K ranges (gemm.cu Sched.sk), with L2 flushed before each launch (median of reps).

    python tools/gemm_sk_probe.py --model qwen3-4b --m 64 128
"""

import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_18521_b200 import _capi  # noqa: E402
from tools.gemm_bench import MODEL_SHAPES  # noqa: E402


def time_code(W, A, out, N, K, M, code, reps):
    ms = C.c_float()
    st = _capi.lib().ab_debug_gemm_time(C.c_void_p(W.data_ptr()), C.c_void_p(A.data_ptr()), C.c_void_p(out.data_ptr()),
                                        None, N, K, M, code, 2 | 128 | 1024, reps, C.byref(ms))
    return None if st else ms.value * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen3-4b")
    ap.add_argument("--m", type=int, nargs="+", default=[64, 128, 256])
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--shapes", nargs="+", default=["qkv", "o", "down", "gate_up"])
    a = ap.parse_args()
    res = []
    for name in a.shapes:
        N, K, _ = MODEL_SHAPES[a.model][name]
        W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        for M in a.m:
            A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
            row = {"shape": name, "N": N, "K": K, "M": M, "weight_MB": N * K * 2 / 1e6, "codes": {}}
            for swap, lgs in ((1, (5, 6, 7, 8)), (0, (7, 8))):
                for lg in lgs:
                    if swap and (1 << lg) > max(256, M) * 2:
                        continue
                    tile = f"{'swap' if swap else 'noswap'}{1 << lg}"
                    for sp in (2, 3, 4, 5, 6, 7, 8, 12):
                        t = time_code(W, A, out, N, K, M, 0x8000 | swap | (lg << 1) | (sp << 5), a.reps)
                        if t:
                            row["codes"][f"{tile}_red{sp}"] = round(t, 2)
                    t = time_code(W, A, out, N, K, M, 0x10000 | 0x8000 | swap | (lg << 1) | (1 << 5), a.reps)
                    if t:
                        row["codes"][f"{tile}_sk"] = round(t, 2)
            best = min(row["codes"].items(), key=lambda kv: kv[1])
            sk = {k: v for k, v in row["codes"].items() if k.endswith("_sk")}
            bsk = min(sk.items(), key=lambda kv: kv[1]) if sk else None
            row["best"] = best
            row["best_sk"] = bsk
            row["best_TBps"] = round(N * K * 2 / (best[1] * 1e-6) / 1e12, 2)
            print(json.dumps({k: v for k, v in row.items() if k != "codes"}), flush=True)
            res.append(row)
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/gemm_sk_probe_{a.model}.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
