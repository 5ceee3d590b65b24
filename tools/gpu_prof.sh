#!/bin/bash
# Profiling call: per-kernel launch list + one full capture of each hot kernel, inside a
# cudaProfilerStart/Stop window of tools/decode_microbench.py at fixed (batch, ctx).
mkdir -p gpurun_out
for cfg in "1024 1400" "448 1100"; do
  set -- $cfg
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_b$1_c$2.csv python tools/decode_microbench.py --batch $1 --ctx $2 --iters 2 --ncu \
    > gpurun_out/ncu_launch_b$1.log 2>&1
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_gemm_tc|k_decode_attn|k_sample" -c 7 -o gpurun_out/prof_b$1_c$2 \
    python tools/decode_microbench.py --batch $1 --ctx $2 --iters 1 --ncu > gpurun_out/ncu_full_b$1.log 2>&1
  timeout 600 python tools/decode_microbench.py --batch $1 --ctx $2 --iters 16 > gpurun_out/micro_b$1_c$2.json 2>&1
done
