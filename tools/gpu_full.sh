#!/bin/bash
# Full check: GPU tests, smoke, bench (C2), microbench at the step's typical batch sizes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for cfg in "1024 1400" "512 1600" "256 2000" "64 3000"; do
  set -- $cfg
  timeout 300 python tools/decode_microbench.py --batch $1 --ctx $2 --iters 16 > gpurun_out/micro_b$1.json 2>&1
done
timeout 1500 python bench.py ${BENCH_ARGS:---steps 3 --warmup 3 --sync-steps 1} > gpurun_out/bench.log 2>&1
