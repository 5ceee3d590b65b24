#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/pytest_kernels.log
timeout 900 python tools/gemm_bench.py --sweep --m 1024 512 256 128 64 16 --reps 7 > gpurun_out/gemm_sweep.jsonl 2>&1
for cfg in "1024 1400" "256 2000" "64 3000"; do
  set -- $cfg
  timeout 300 python tools/decode_microbench.py --batch $1 --ctx $2 --iters 16 > gpurun_out/micro_b$1.json 2>&1
done
