# round-2 validation batch: GEMM epilogue / SwiGLU pass changes
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_kernels_gpu.py tests/test_model_gpu.py tests/test_replay_model_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest3.log 2>&1; echo rc=$? >> gpurun_out/pytest3.log
AB_AUTOTUNE_LOG=1 timeout 600 python tools/decode_microbench.py --model qwen3-4b --batch 64 --ctx 3000 --iters 32 > gpurun_out/micro_c3_b64.log 2>&1
AB_AUTOTUNE_LOG=1 timeout 600 python tools/decode_microbench.py --model qwen2.5-1.5b --batch 384 --ctx 1350 --iters 32 > gpurun_out/micro_c2_b384.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_swiglu|k_gemm" -c 6 \
  -o gpurun_out/prof_c3_b64_gemms python tools/decode_microbench.py --model qwen3-4b --batch 64 --ctx 3000 --iters 1 --ncu > gpurun_out/ncu_c3_gemms.log 2>&1
bash tools/gpu.sh launches 64 3000 qwen3-4b
bash tools/gpu.sh launches 384 1350 qwen2.5-1.5b
tail -3 gpurun_out/pytest3.log
