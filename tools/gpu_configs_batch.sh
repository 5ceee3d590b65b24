# Bench lines for BASELINE.json configs[2..4] on one B200 (per-engine shares of the 8-GPU configs):
# C4 over-provision sweep (GSPO, N'/N = 1.5 / 2 / 3), C3 (DAPO, recycling); launch lists after the changes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_k.log 2>&1; tail -1 gpurun_out/pytest_k.log
bash tools/gpu.sh launches 64 3000 qwen3-4b
bash tools/gpu.sh launches 384 1350 qwen2.5-1.5b
run() { tag=$1; shift; timeout 2400 python bench.py --no-cpu "$@" > gpurun_out/cfg_${tag}.log 2> gpurun_out/cfg_${tag}.err; echo "$tag rc=$?"; }
for x in 1.5 2 3; do run C4_$x --workload C4 --over-provision $x --steps 3 --warmup 3 --sync-steps 2; done
run C3 --workload C3 --steps 3 --warmup 3 --sync-steps 2
