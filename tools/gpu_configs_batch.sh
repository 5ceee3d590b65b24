# Bench lines for BASELINE.json configs[2..4] on one B200 (per-engine shares of the 8-GPU configs):
# C3 (DAPO, recycling), the C4 over-provision sweep (GSPO, N'/N = 1.5 / 2 / 3), C5 (R1-Distill-7B shape);
# the multi-rank bench path at world 2 on this one GPU; launch lists / autotune choices after the changes
mkdir -p gpurun_out
bash tools/gpu.sh dp2 --workload C1 --steps 3 --warmup 3 --sync-steps 2
run() { tag=$1; shift; timeout 2400 python bench.py --no-cpu "$@" > gpurun_out/cfg_${tag}.log 2> gpurun_out/cfg_${tag}.err; echo "$tag rc=$?"; }
run C3 --workload C3 --steps 3 --warmup 3 --sync-steps 2
for x in 1.5 2 3; do run C4_$x --workload C4 --over-provision $x --steps 3 --warmup 3 --sync-steps 2; done
run C5 --workload C5 --steps 3 --warmup 3 --sync-steps 2
bash tools/gpu.sh launches 64 3000 qwen3-4b
bash tools/gpu.sh launches 384 1350 qwen2.5-1.5b
AB_AUTOTUNE_LOG=1 timeout 600 python tools/decode_microbench.py --model qwen2.5-1.5b --batch 384 --ctx 1350 --iters 16 > gpurun_out/micro_c2_b384.log 2>&1
