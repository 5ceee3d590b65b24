mkdir -p gpurun_out
timeout 3300 python bench.py --no-cpu --workload C4 --over-provision 3 --steps 3 --warmup 3 --sync-steps 2 > gpurun_out/cfg_C4_3.log 2> gpurun_out/cfg_C4_3.err; echo "C4_3 rc=$?"; tail -n 1 gpurun_out/cfg_C4_3.err
