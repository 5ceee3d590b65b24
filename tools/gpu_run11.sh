#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_model_gpu.py tests/test_engine_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_model.log
for et in 0 1; do
  for cfg in "1024 1400" "256 2000" "64 3000"; do
    set -- $cfg
    AB_GEMM_TRIGGER=$et timeout 400 python tools/decode_microbench.py --batch $1 --ctx $2 --iters 4 > gpurun_out/gt${et}_b$1.json 2>&1
  done
  AB_GEMM_TRIGGER=$et timeout 400 python tools/decode_microbench.py --model qwen3-4b --batch 64 --ctx 3000 --iters 4 > gpurun_out/gt${et}_c3.json 2>&1
done
grep -H warm_ms gpurun_out/gt*.json
