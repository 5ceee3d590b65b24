#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --workload C1 --steps 2 --warmup 3 --sync-steps 2 --no-cpu --out gpurun_out/runs_c1 > gpurun_out/bench_c1.log 2>&1
timeout 1200 python bench.py --steps 3 --warmup 3 --sync-steps 1 --no-cpu --kv-resume retain > gpurun_out/bench_retain.log 2>&1
timeout 2000 python bench.py --workload C3 --steps 2 --warmup 1 --sync-steps 1 --no-cpu > gpurun_out/bench_c3.log 2>&1
