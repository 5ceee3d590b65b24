#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_model_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_model.log
export AB_AUTOTUNE_LOG=1
for cfg in "1024 1400" "256 2000" "64 3000"; do
  set -- $cfg
  timeout 400 python tools/decode_microbench.py --batch $1 --ctx $2 --iters 16 > gpurun_out/micro_b$1.json 2> gpurun_out/tune_b$1.log
done
timeout 400 python tools/decode_microbench.py --model qwen3-4b --batch 64 --ctx 3000 --iters 16 > gpurun_out/micro_c3_b64.json 2> gpurun_out/tune_c3.log
