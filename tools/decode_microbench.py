"""Per-kernel decode timing at a fixed live batch and context (kernel tuning aid).

    python tools/decode_microbench.py --model qwen2.5-1.5b --batch 1024 --ctx 1400 --iters 16

Builds the engine, admits `batch` samples of a long trace, decodes until the
context reaches `ctx`, then profiles `iters` iterations (every launch timed with
CUDA events) and prints per-kernel average time, algorithmic GB/s and TFLOP/s.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2509_18521_b200 as pb  # noqa: E402
from paper_2509_18521_b200.rollouts import RolloutSample  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-1.5b")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--ctx", type=int, default=1400)
    ap.add_argument("--prompt", type=int, default=256)
    ap.add_argument("--iters", type=int, default=16)
    ap.add_argument("--page", type=int, default=64)
    ap.add_argument("--kv-pages", type=int, default=0)
    ap.add_argument("--det", action="store_true", help="deterministic GEMM plans only (no reduce-add split-K)")
    ap.add_argument("--ncu", action="store_true",
                    help="bracket only the profiled iterations with cudaProfilerStart/Stop "
                         "(run under ncu --profile-from-start off)")
    args = ap.parse_args()
    spec = pb.PRESETS[args.model]
    if args.layers:
        spec = spec.truncated(args.layers)
    l_max = max(4096, args.ctx + args.iters + 8)
    eng = pb.LengthDrivenEngine(pb.EngineConfig(max_slots=args.batch, l_max=l_max), model=spec,
                                sampling=pb.SamplingConfig(temperature=0.8), prompt_len=args.prompt,
                                page_size=args.page, kv_pages=args.kv_pages, max_handles=max(4096, 2 * args.batch),
                                max_groups=args.batch, nondeterministic_gemm=not args.det)
    eng.begin_step(0)
    for i in range(args.batch):
        s = RolloutSample(i // 8, i % 8)
        s.target_length = l_max
        eng.submit(s)
    t0 = time.perf_counter()
    warm = max(1, args.ctx - args.prompt)
    eng.decode_iterations(warm)
    t1 = time.perf_counter()
    if args.ncu:
        import torch

        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        eng.decode_iterations(args.iters)
        eng.stats()
        torch.cuda.profiler.stop()
        print(json.dumps({"ncu_window_iters": args.iters, "batch": args.batch, "ctx": args.ctx}))
        return
    # steady state at the target context: un-instrumented graph replays, device clock around them
    c0 = eng.clock
    eng.decode_iterations(args.iters)
    steady_ms = 1e3 * (eng.clock - c0) / args.iters
    t1 = time.perf_counter()
    eng.profile(True, 1)
    for _ in range(args.iters):  # one host chunk per iteration: each replays the profiled graph
        eng.decode_iterations(1)
    t2 = time.perf_counter()
    ks = eng.kernel_stats()
    tot = sum(k["ms"] for k in ks)
    rows = []
    for k in sorted(ks, key=lambda k: -k["ms"]):
        us = 1e3 * k["ms"] / max(k["launches"], 1)
        rows.append({"kernel": k["name"], "share": round(k["ms"] / tot, 4), "avg_us": round(us, 2),
                     "GB/s": round(k["bytes"] / (k["ms"] * 1e-3) / 1e9, 1) if k["ms"] else None,
                     "TFLOP/s": round(k["flops"] / (k["ms"] * 1e-3) / 1e12, 1) if k["flops"] else None})
    out = {"model": spec.name, "batch": args.batch, "ctx": args.ctx, "warm_iters": warm,
           "warm_s": round(t1 - t0, 2), "warm_ms_per_iter": round(1e3 * (t1 - t0) / warm, 3),
           "steady_ms_per_iter": round(steady_ms, 3),
           "profiled_ms_per_iter": round(1e3 * (t2 - t1) / args.iters, 3),
           "note": "steady: graph replays at ctx..ctx+iters with no instrumentation (device clock); kernels: "
                   "CUDA events around every kernel of the profiled graph (breaks PDL overlap, so the "
                   "per-kernel times include launch gaps)", "kernels": rows}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
