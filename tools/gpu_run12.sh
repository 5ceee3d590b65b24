#!/bin/bash
mkdir -p gpurun_out
for it in 2 3 4 6; do
  for cfg in "1024 1400 qwen2.5-1.5b" "256 2000 qwen2.5-1.5b" "64 3000 qwen2.5-1.5b" "64 3000 qwen3-4b"; do
    set -- $cfg
    AB_ATT_ITEMS=$it timeout 400 python tools/decode_microbench.py --model $3 --batch $1 --ctx $2 --iters 4 > gpurun_out/ai${it}_$3_b$1.json 2>&1
  done
done
for f in gpurun_out/ai*.json; do python -c "
import json,sys
d=json.load(open('$f')); a=[k for k in d['kernels'] if k['kernel']=='attention'][0]
print('$f', d['warm_ms_per_iter'], a['avg_us'])"; done
