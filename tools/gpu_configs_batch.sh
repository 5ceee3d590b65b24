# GPU tests of the KV-release change, then the C4 over-provision sweep (GSPO, N'/N = 1.5 / 2 / 3) and C3
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_replay_model_gpu.py tests/test_model_gpu.py tests/test_engine_gpu.py tests/test_dp_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_kv.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/pytest_kv.log
run() { tag=$1; shift; timeout 2400 python bench.py --no-cpu "$@" > gpurun_out/cfg_${tag}.log 2> gpurun_out/cfg_${tag}.err; echo "$tag rc=$?"; tail -n 1 gpurun_out/cfg_${tag}.err; }
for x in 2 1.5 3; do run C4_$x --workload C4 --over-provision $x --steps 3 --warmup 3 --sync-steps 2; done
