#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/gemm_trace.py 6144 2560 64 $((0x904d)) $((2+1024+128)) > gpurun_out/trace_c3_qkv.log 2>&1
timeout 120 python tools/gemm_trace.py 19456 2560 64 $((0x830)) $((3+16+128)) > gpurun_out/trace_c3_gu.log 2>&1
timeout 120 python tools/gemm_trace.py 2560 9728 64 $((0x908d)) $((2+1024+128)) > gpurun_out/trace_c3_down.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:k_rope_kv_f32 -c 1 -o gpurun_out/prof_rope_b1024 \
  python tools/decode_microbench.py --batch 1024 --ctx 1400 --iters 1 --ncu > gpurun_out/ncu_rope.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:k_gemm_tc -c 8 -o gpurun_out/prof_gemm_c3_b64 \
  python tools/decode_microbench.py --model qwen3-4b --batch 64 --ctx 3000 --iters 1 --ncu > gpurun_out/ncu_gemm_c3.log 2>&1
for cfg in "1024 1400" "64 3000"; do
  set -- $cfg
  timeout 400 python tools/decode_microbench.py --batch $1 --ctx $2 --iters 16 > gpurun_out/micro_b$1.json 2>&1
done
