#!/bin/bash
# Round evidence call: bench (clocks sampled inside bench.py), ncu launch list + full captures at a fixed
# decode point (b=1024, ctx=1400, inside the microbench's profiler window), microbench at three points.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python bench.py ${BENCH_ARGS:---steps 3 --warmup 3 --sync-steps 1} > gpurun_out/bench.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_b1024_c1400.csv python tools/decode_microbench.py --batch 1024 --ctx 1400 --iters 2 --ncu \
  > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"k_decode_attn|k_sample" -c 3 -o gpurun_out/prof_attn_b1024_c1400 \
  python tools/decode_microbench.py --batch 1024 --ctx 1400 --iters 1 --ncu > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:k_gemm_tc -c 5 -o gpurun_out/prof_gemm_b1024_c1400 \
  python tools/decode_microbench.py --batch 1024 --ctx 1400 --iters 1 --ncu > gpurun_out/ncu_gemm.log 2>&1
for cfg in "1024 1400" "256 2000" "64 3000"; do
  set -- $cfg
  timeout 300 python tools/decode_microbench.py --batch $1 --ctx $2 --iters 16 > gpurun_out/micro_b$1.json 2>&1
done
