#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_model_gpu.py tests/test_engine_gpu.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_model.log
export AB_AUTOTUNE_LOG=1
timeout 300 python tools/prefill_bench.py --samples 64 --gen 2000 > gpurun_out/prefill_c2.log 2> gpurun_out/prefill_c2.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_prefill.csv python tools/prefill_bench.py --samples 16 --gen 1000 --ncu > gpurun_out/ncu_prefill.log 2>&1
unset AB_AUTOTUNE_LOG
for cfg in "1024 1400" "64 3000"; do
  set -- $cfg
  timeout 400 python tools/decode_microbench.py --batch $1 --ctx $2 --iters 16 > gpurun_out/micro_b$1.json 2>&1
done
