#!/bin/bash
# ncu --set full of the re-prefill kernels (flash prefill attention + the prefill GEMMs), inside the
# prefill bench's profiler window (16 resumed samples x 1000 carried tokens).
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"k_prefill_flash|k_gemm_tc" -s 260 -c 6 -o gpurun_out/prof_reprefill \
  python tools/prefill_bench.py --samples 16 --gen 1000 --ncu > gpurun_out/ncu_reprefill.log 2>&1
