#!/bin/bash
# ncu --set full of single tcgen05 GEMM launches: tools/gpu_ncu_gemm.sh "N K M BN EPI" ...
mkdir -p gpurun_out
i=0
for args in "$@"; do
  i=$((i+1))
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 1 -c 1 -o gpurun_out/gemm_$i python tools/gemm_one.py $args > gpurun_out/ncu_gemm_$i.log 2>&1
done
