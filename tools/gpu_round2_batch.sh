# round-2 validation batch (gpurun from the repo root): GPU tests of the changed paths, steady-state
# decode microbenchmarks, the attention ncu capture at the bench's operating point, a short C2 bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_sampler.py tests/test_kernels_gpu.py tests/test_model_gpu.py tests/test_replay_model_gpu.py tests/test_dp_gpu.py tests/test_engine_gpu.py tests/test_replay_gpu.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest3.log 2>&1; echo rc=$? >> gpurun_out/pytest3.log
AB_AUTOTUNE_LOG=1 timeout 600 python tools/decode_microbench.py --model qwen3-4b --batch 64 --ctx 3000 --iters 32 > gpurun_out/micro_c3_b64.log 2>&1
timeout 600 python tools/decode_microbench.py --model qwen2.5-1.5b --batch 384 --ctx 1350 --iters 32 > gpurun_out/micro_c2_b384.log 2>&1
timeout 600 python tools/decode_microbench.py --model qwen2.5-1.5b --batch 64 --ctx 3000 --iters 32 > gpurun_out/micro_c2_b64.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_decode_attn -c 3 \
  -o gpurun_out/prof_attn_b384_c1350 python tools/decode_microbench.py --batch 384 --ctx 1350 --iters 1 --ncu > gpurun_out/ncu_attn_b384.log 2>&1
python tools/ncu_attn_point.py gpurun_out/prof_attn_b384_c1350.ncu-rep --b 384 --ctx 1350 > gpurun_out/attn_point.log 2>&1
timeout 1500 python bench.py --steps 4 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err
tail -3 gpurun_out/pytest3.log
