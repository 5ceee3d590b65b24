#!/bin/bash
# full GPU tests, ncu launch lists of one decode iteration at b = 1024 and 64 (C2) and 64 (C3), C2 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for cfg in "1024 1400 qwen2.5-1.5b" "64 3000 qwen2.5-1.5b" "64 3000 qwen3-4b"; do
  set -- $cfg
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_$3_b$1.csv python tools/decode_microbench.py --model $3 --batch $1 --ctx $2 --iters 2 --ncu \
    > gpurun_out/ncu_launch_$3_b$1.log 2>&1
done
timeout 1500 python bench.py --steps 3 --warmup 3 --sync-steps 1 > gpurun_out/bench.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log
