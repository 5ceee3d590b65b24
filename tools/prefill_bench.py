"""Prefill / re-prefill throughput of the engine (tuning aid for SURVEY §8 f1).

    python tools/prefill_bench.py --model qwen2.5-1.5b --samples 64 --gen 2000 [--ncu]

Admits `samples` samples (groups of 8, 256-token prompts), decodes `gen` iterations, aborts, bumps the
version and resubmits: the resubmit plus the admitting iteration re-prefill samples x gen rows (plus the
groups' prompts).  Prints the re-prefill wall time and rows/s (the timed span includes one decode
iteration).  --ncu brackets only the resubmit with cudaProfilerStart/Stop.
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
    ap.add_argument("--samples", type=int, default=64)
    ap.add_argument("--gen", type=int, default=2000)
    ap.add_argument("--ncu", action="store_true")
    args = ap.parse_args()
    import torch

    spec = pb.PRESETS[args.model]
    eng = pb.LengthDrivenEngine(pb.EngineConfig(max_slots=max(64, args.samples), l_max=args.gen + 64), model=spec,
                                prompt_len=256, page_size=64, max_handles=4096, max_groups=1024,
                                kv_resume="reprefill", nondeterministic_gemm=True)
    eng.begin_step(0)
    samples = []
    for i in range(args.samples):
        s = RolloutSample(i // 8, i % 8)
        s.target_length = args.gen + 32
        eng.submit(s)
        samples.append(s)
    eng.decode_iterations(args.gen)
    paused = eng.abort_active()
    eng.begin_step(1)
    st0 = eng.stats()
    torch.cuda.synchronize()
    if args.ncu:
        torch.cuda.profiler.start()
    t0 = time.perf_counter()
    for p in paused:
        eng.submit(p)
    eng._flush()
    # the rebuild happens when the resumed samples are admitted (admission-time re-prefill): one
    # decode iteration admits them all (S >= samples)
    eng.decode_iterations(1)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if args.ncu:
        torch.cuda.profiler.stop()
    st1 = eng.stats()
    rows = st1.reprefill_tokens - st0.reprefill_tokens
    prompt_rows = st1.prefill_tokens - st0.prefill_tokens
    print(json.dumps({"model": spec.name, "samples": len(paused), "reprefill_rows": rows, "prompt_rows": prompt_rows,
                      "seconds": round(t1 - t0, 4), "rows_per_s": round((rows + prompt_rows) / (t1 - t0), 1),
                      "reprefill_seconds": round(st1.reprefill_seconds - st0.reprefill_seconds, 4)}))
    eng.close()


if __name__ == "__main__":
    main()
