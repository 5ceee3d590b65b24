"""Time the tcgen05 GEMM (ab_debug_gemm) on decoder shapes, next to torch/cuBLAS.

    python tools/gemm_bench.py [--m 1024 64] [--reps 20]
"""

import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_18521_b200 import _capi  # noqa: E402

MODEL_SHAPES = {  # name: (N, K, epi)   decode projections per model shape
    "qwen2.5-1.5b": {
        "qkv": (2048, 1536, 0),
        "o": (1536, 1536, 2),
        "gate_up": (17920, 1536, 3),
        "down": (1536, 8960, 2),
        "lm_head": (151936, 1536, 1),
    },
    "qwen3-4b": {
        "qkv": (6144, 2560, 2),
        "o": (2560, 4096, 2),
        "gate_up": (19456, 2560, 3),
        "down": (2560, 9728, 2),
        "lm_head": (151936, 2560, 1),
    },
}
SHAPES = MODEL_SHAPES["qwen2.5-1.5b"]


def run(N, K, M, epi, bn, reps, split, cublas=True):
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    flags, epi = epi & ~15, epi & 15
    bias = torch.zeros(N, device="cuda", dtype=torch.bfloat16) if epi == 0 else None
    if epi == 3:
        out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
    elif epi == 0:
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    else:
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    code = epi + flags + (16 if split else 0) + (32 if bn == 0 else 0)  # bn 0: schedule table (decode path)
    args = (C.c_void_p(W.data_ptr()), C.c_void_p(A.data_ptr()), C.c_void_p(out.data_ptr()),
            C.c_void_p(bias.data_ptr()) if bias is not None else None, N, K, M, bn or 256, code)
    msv = C.c_float()
    _capi.call("ab_debug_gemm_time", *args, reps, C.byref(msv))  # device-timed, L2 flushed, median
    ms = msv.value
    if not cublas:
        return {"us": round(ms * 1e3, 1)}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    # cuBLAS reference for the same contraction
    for _ in range(3):
        torch.matmul(A, W.t())
    cts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        torch.matmul(A, W.t())
        b.record()
        torch.cuda.synchronize()
        cts.append(a.elapsed_time(b))
    cts.sort()
    cms = cts[len(cts) // 2]
    flops = 2.0 * M * N * K
    wbytes = N * K * 2
    return {"us": round(ms * 1e3, 1), "TFLOP/s": round(flops / ms / 1e9, 1), "W GB/s": round(wbytes / ms / 1e6, 1),
            "cublas_us": round(cms * 1e3, 1), "cublas_TFLOP/s": round(flops / cms / 1e9, 1)}


def sweep(args):
    """Time every fixed schedule (swap / tile / split-K) per shape and row count."""
    for name, (N, K, epi) in SHAPES.items():
        for M in args.m:
            res = []
            for swap in (1, 0):
                for t in ((32, 64, 128, 256) if swap else (128, 256)):
                    if not swap and (N % 128 or (epi == 3 and (t != 256 or N % 256))):
                        continue
                    for sp in (1, 2, 4, 8):  # split-K <= the debug cluster size (8)
                        if K // 64 < 2 * sp:
                            continue
                        lg = t.bit_length() - 1
                        code = swap | (lg << 1) | (sp << 5)
                        r = run(N, K, M, epi | 16 | 128, code, args.reps, False, cublas=False)
                        res.append((r["us"], swap, t, sp))
            r = run(N, K, M, epi | 256 | 128, 0x4000, args.reps, False, cublas=False)  # CTA pair
            res.append((r["us"], 2, 256, 1))  # swap column 2 = CTA pair
            auto = run(N, K, M, epi, 0, args.reps, True)
            res.sort()
            floor = min(r[0] for r in res)  # invalid codes launch an empty kernel: drop them
            res = [r for r in res if r[0] > floor + 0.5] or res
            print(json.dumps({"shape": name, "M": M, "auto_us": auto["us"], "cublas_us": auto["cublas_us"],
                              "best": res[:4]}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, nargs="+", default=[1024, 256, 64, 8])
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--bn", type=int, nargs="+", default=[0], help="activation tile width; 0 = automatic (as the decode path)")
    ap.add_argument("--split", type=int, default=1)
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--pair", action="store_true", help="time the CTA-pair plans (cluster of 2)")
    ap.add_argument("--model", default="qwen2.5-1.5b", choices=sorted(MODEL_SHAPES))
    ap.add_argument("--mode", type=int, default=0, help="2: operand fill only, 4: MMA only (debug timing)")
    args = ap.parse_args()
    global SHAPES
    SHAPES = MODEL_SHAPES[args.model]
    if args.mode:
        _capi.call("ab_debug_gemm_trace", args.mode, None)
    if args.sweep:
        return sweep(args)
    res = []
    for name, (N, K, epi) in SHAPES.items():
        for M in args.m:
            for bn in args.bn:
                r = run(N, K, M, epi | (256 if args.pair else 0), bn, args.reps, bool(args.split) and not args.pair)
                r.update({"shape": name, "M": M, "BN": bn})
                res.append(r)
                print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
