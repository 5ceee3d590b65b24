# K1 sampler: parity tests + ncu of the split kernels at b = 384 and 64 (C2 shape)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_sampler.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_sampler.log 2>&1; tail -3 gpurun_out/pytest_sampler.log
for B in 384 64; do
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_sample -c 2 \
  -o gpurun_out/prof_sampler_b$B python tools/decode_microbench.py --batch $B --ctx 1350 --iters 1 --ncu > gpurun_out/ncu_sampler_b$B.log 2>&1
done
