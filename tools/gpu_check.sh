#!/bin/bash
# One gpurun call: GPU tests, smoke, raw clocks, a short C2 bench, an ncu launch list and one full capture.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks.csv &
CP=$!
timeout 1200 python bench.py ${BENCH_ARGS:---steps 3 --warmup 3 --sync-steps 1} > gpurun_out/bench.log 2>&1
kill $CP
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60000 -c 3000 --csv --log-file gpurun_out/launches.csv python tools/decode_microbench.py --batch 1024 --ctx 1400 --iters 4 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 20 -c 2 -o gpurun_out/prof_attn python tools/decode_microbench.py --batch 1024 --ctx 1400 --iters 2 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/*.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_sample" -s 60 -c 8 -o gpurun_out/prof_gemm python tools/decode_microbench.py --batch 1024 --ctx 1400 --iters 1 > gpurun_out/ncu_gemm.log 2>&1
timeout 300 python tools/decode_microbench.py --batch 1024 --ctx 1400 --iters 16 > gpurun_out/micro_b1024.json 2>&1
timeout 300 python tools/decode_microbench.py --batch 256 --ctx 2000 --iters 16 > gpurun_out/micro_b256.json 2>&1
