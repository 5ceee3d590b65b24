#!/bin/bash
mkdir -p gpurun_out
for mask in 6 14 2 4; do
  for cfg in "1024 1400" "256 2000" "64 3000"; do
    set -- $cfg
    AB_PDL_MASK=$mask timeout 400 python tools/decode_microbench.py --batch $1 --ctx $2 --iters 4 > gpurun_out/pdl_m${mask}_b$1.json 2>&1
  done
done
grep -H warm_ms gpurun_out/pdl_m*.json
