#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
for cfg in "1024 1400" "256 2000" "64 3000"; do
  set -- $cfg
  timeout 400 python tools/decode_microbench.py --batch $1 --ctx $2 --iters 16 > gpurun_out/micro_b$1.json 2>&1
done
timeout 400 python tools/decode_microbench.py --model qwen3-4b --batch 64 --ctx 3000 --iters 16 > gpurun_out/micro_c3_b64.json 2>&1
timeout 300 python tools/gemm_trace.py 6144 2560 64 $((0x904d)) $((2+1024+128)) > gpurun_out/trace_c3_qkv.log 2>&1
