"""Time every valid schedule of the tcgen05 GEMM on the decode shapes (cluster-8 split plans),
next to the schedule the cost model picks, to calibrate choose_sched (gemm.cu).

    python tools/gemm_sched_sweep.py [--m 64 128 256 ...] [--shapes qkv o down]
"""

import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_18521_b200 import _capi  # noqa: E402

SHAPES = {"qkv": (2048, 1536, 0), "o": (1536, 1536, 2), "gate_up": (17920, 1536, 3), "down": (1536, 8960, 2)}


def decode(c):
    if c == 0:
        return None
    return {"swap": c & 1, "t": 1 << ((c >> 1) & 15), "sp": (c >> 5) & 31}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, nargs="+", default=[64, 128, 192, 256, 384, 512, 768, 1024])
    ap.add_argument("--shapes", nargs="+", default=["qkv", "o", "down"])
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--cluster", type=int, default=8, choices=[1, 2, 8],
                    help="plan cluster size (2: plain, not pair; 1: TMA reduce-add split-K for fp32 residual GEMMs)")
    args = ap.parse_args()
    lib = _capi.lib()
    ncl = C.c_int()
    _capi.call("ab_debug_gemm_clusters", args.cluster, C.byref(ncl))
    cs = args.cluster
    flag = {8: 16, 2: 512, 1: 1024}[cs]
    for name in args.shapes:
        N, K, epi = SHAPES[name]
        W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        for M in args.m:
            A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            out = torch.zeros(M, N if epi != 3 else N // 2, device="cuda",
                              dtype=torch.float32 if epi in (1, 2) else torch.bfloat16)
            bias = torch.zeros(N, device="cuda", dtype=torch.bfloat16) if epi == 0 else None
            auto = lib.ab_debug_gemm_sched(N, K, M, 256, cs, ncl.value, 0, epi)
            res = []
            for swap in (1, 0):
                for t in ((32, 64, 128, 256) if swap else (128, 256)):
                    for sp in ((1, 2, 4, 8) if cs != 2 else (1, 2)):
                        code = swap | ((t.bit_length() - 1) << 1) | (sp << 5)
                        if cs == 1 and sp > 1:
                            if epi != 2:
                                continue
                            code |= 0x8000
                        if lib.ab_debug_gemm_sched(N, K, M, 256, cs, ncl.value, 0x40000000 | code, epi) == 0:
                            continue
                        ms = C.c_float()
                        _capi.call("ab_debug_gemm_time", C.c_void_p(W.data_ptr()), C.c_void_p(A.data_ptr()),
                                   C.c_void_p(out.data_ptr()), C.c_void_p(bias.data_ptr()) if bias is not None else None,
                                   N, K, M, code, epi + flag + 128, args.reps, C.byref(ms))
                        res.append((round(ms.value * 1e3, 1), code))
            res.sort()
            a = [r for r in res if r[1] == (auto & 0x3ff)]
            print(json.dumps({"shape": name, "M": M, "auto": decode(auto), "auto_us": a[0][0] if a else None,
                              "best": [(us, decode(c)) for us, c in res[:3]]}), flush=True)


if __name__ == "__main__":
    main()
