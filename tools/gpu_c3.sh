#!/bin/bash
# C3 (Qwen3-4B shape, <= 64 live rows) decode evidence: microbench, ncu launch list, GEMMs vs cuBLAS.
mkdir -p gpurun_out
timeout 400 python tools/decode_microbench.py --model qwen3-4b --batch 64 --ctx 3000 --iters 16 > gpurun_out/micro_c3_b64.json 2>&1
timeout 400 python tools/decode_microbench.py --model qwen3-4b --batch 16 --ctx 6000 --iters 16 > gpurun_out/micro_c3_b16.json 2>&1
timeout 400 python tools/gemm_bench.py --model qwen3-4b --m 64 32 8 > gpurun_out/gemm_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 1200 --csv --log-file gpurun_out/launches_c3.csv python tools/decode_microbench.py --model qwen3-4b --batch 64 --ctx 3000 --iters 4 > gpurun_out/ncu_launch_c3.log 2>&1
