# final round-2 evidence: full GPU suite, smoke, the default bench line, memcheck on the engine paths
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider -m gpu \
  tests/test_engine_gpu.py -k "exactly_once or abort or advantages or clipped or resume_segments" > gpurun_out/sanitize_memcheck_engine.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_memcheck_engine.log
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider -m gpu \
  tests/test_sampler.py -k "151936 and 48" > gpurun_out/sanitize_memcheck_sampler.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_memcheck_sampler.log
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider -m gpu \
  tests/test_sampler.py tests/test_attention_gpu.py -k "151936 and 48 or b64 and c3 and page64" > gpurun_out/sanitize_synccheck.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_synccheck.log
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/smoke.log; tail -n 3 gpurun_out/sanitize_*.log
