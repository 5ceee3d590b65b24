#!/bin/bash
# ncu --set full of the decode attention kernel at a fixed (batch, ctx), inside the microbench's
# cudaProfilerStart/Stop window: tools/gpu_ncu_attn.sh BATCH CTX [tag]
mkdir -p gpurun_out
B=${1:-1024}; CTX=${2:-1400}; TAG=${3:-attn}
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:k_decode_attn -c 2 -o gpurun_out/prof_${TAG}_b${B}_c${CTX} \
  python tools/decode_microbench.py --batch $B --ctx $CTX --iters 1 --ncu > gpurun_out/ncu_${TAG}_b${B}.log 2>&1
