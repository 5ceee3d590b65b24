#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 3 --warmup 3 --sync-steps 1 > gpurun_out/bench.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_b1024_c1400.csv python tools/decode_microbench.py --batch 1024 --ctx 1400 --iters 2 --ncu \
  > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_b64_c3000.csv python tools/decode_microbench.py --batch 64 --ctx 3000 --iters 2 --ncu \
  > gpurun_out/ncu_launch64.log 2>&1
timeout 1200 python bench.py --steps 3 --warmup 3 --sync-steps 1 --no-cpu --kv-resume retain > gpurun_out/bench_retain.log 2>&1
timeout 2000 python bench.py --workload C3 --steps 2 --warmup 1 --sync-steps 1 --no-cpu > gpurun_out/bench_c3.log 2>&1
