# full GPU suite + smoke + the default bench line + sampler ncu (gpurun from the repo root)
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
for B in 384 64; do
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_sample -c 2 \
  -o gpurun_out/prof_sampler_b$B python tools/decode_microbench.py --batch $B --ctx 1350 --iters 1 --ncu > gpurun_out/ncu_sampler_b$B.log 2>&1
done
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
