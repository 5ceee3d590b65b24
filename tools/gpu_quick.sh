#!/bin/bash
# Quick check after a decode-path change: model/engine GPU tests + the decode microbench at 4 batch sizes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_model_gpu.py tests/test_engine_gpu.py -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_quick.log
for cfg in "1024 1400" "512 1600" "256 2000" "64 3000"; do
  set -- $cfg
  timeout 300 python tools/decode_microbench.py --batch $1 --ctx $2 --iters 16 > gpurun_out/micro_b$1.json 2>&1
done
tail -3 gpurun_out/pytest_quick.log
