mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_model_gpu.py -m gpu -q -x 2>&1 | tail -25 > gpurun_out/pytest_model.log
timeout 300 python tools/decode_microbench.py --batch 1024 --ctx 1400 --iters 16 > gpurun_out/micro_b1024.json 2>&1
timeout 300 python tools/decode_microbench.py --batch 64 --ctx 3000 --iters 16 > gpurun_out/micro_b64.json 2>&1
timeout 400 python tools/decode_microbench.py --model qwen3-4b --batch 64 --ctx 3000 --iters 16 > gpurun_out/micro_c3_b64.json 2>&1
timeout 900 python tools/gemm_bench.py --model qwen3-4b --sweep --m 64 16 --reps 7 > gpurun_out/sweep_c3.log 2>&1
timeout 600 python tools/gemm_bench.py --sweep --m 256 64 --reps 7 > gpurun_out/sweep_c2.log 2>&1
