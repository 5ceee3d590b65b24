"""Create one engine with decode-GEMM autotuning on (AB_AUTOTUNE_LOG=1 prints the chosen
schedule per row count; =2 also every candidate before it runs) and report the tuning time.

    python tools/autotune_probe.py --model qwen2.5-1.5b --slots 1024 [--det]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2509_18521_b200 as pb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-1.5b")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--slots", type=int, default=1024)
    ap.add_argument("--det", action="store_true")
    args = ap.parse_args()
    spec = pb.PRESETS[args.model]
    if args.layers:
        spec = spec.truncated(args.layers)
    t0 = time.perf_counter()
    eng = pb.LengthDrivenEngine(pb.EngineConfig(max_slots=args.slots, l_max=4096), model=spec, prompt_len=256,
                                page_size=64, kv_pages=4096, max_handles=max(4096, 2 * args.slots),
                                max_groups=args.slots, nondeterministic_gemm=not args.det, gemm_autotune=False)
    t1 = time.perf_counter()
    eng.close()
    eng = pb.LengthDrivenEngine(pb.EngineConfig(max_slots=args.slots, l_max=4096), model=spec, prompt_len=256,
                                page_size=64, kv_pages=4096, max_handles=max(4096, 2 * args.slots),
                                max_groups=args.slots, nondeterministic_gemm=not args.det, gemm_autotune=True)
    t2 = time.perf_counter()
    print(f"create without tuning {t1 - t0:.2f} s, with tuning {t2 - t1:.2f} s", flush=True)
    eng.close()


if __name__ == "__main__":
    main()
