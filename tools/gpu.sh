#!/bin/bash
# One documented entry point for the GPU-box runs (invoked through gpurun from the repo root):
#   gpurun --timeout T -- 'bash tools/gpu.sh MODE [args]'
# Outputs land in gpurun_out/ (scratch; summaries worth keeping are copied into profiles/).
#   tests [pytest -k expr]   pytest -m gpu (optionally filtered), full log + per-test report dir
#   smoke                    __graft_entry__ build + smoke
#   bench [bench.py args]    one bench line
#   launches B CTX [preset]  ncu launch list (gpu__time_duration) of decode iterations at (batch, ctx)
#   ncu_attn B CTX           ncu --set full of the decode attention kernel
#   sanitize                 compute-sanitizer racecheck + memcheck on the engine / attention tests
#                            (closed on the GPU pool since round 2 session 3)
#   forcedp [bench args]     plain vs --force-dp (world-1 lockstep wrapper) decisions, compared
#   dp2 [bench args]         bench.py at world 2 on one GPU (gloo host collectives, IPC exchange)
set -u
mkdir -p gpurun_out
export AB_TEST_REPORT_DIR=gpurun_out/test_reports
MODE=${1:-tests}
shift || true
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
case "$MODE" in
  tests)
    if [ $# -gt 0 ]; then K=(-k "$*"); else K=(); fi
    timeout 3000 python -m pytest tests -m gpu -q -x -p no:cacheprovider -rs "${K[@]}" > gpurun_out/pytest_gpu.log 2>&1
    echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
    tail -5 gpurun_out/pytest_gpu.log ;;
  smoke)
    timeout 900 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
    echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -3 gpurun_out/smoke.log ;;
  bench)
    timeout 3000 python bench.py "$@" > gpurun_out/bench.log 2> gpurun_out/bench.err
    echo "bench rc=$?" >> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.log ;;
  launches)
    B=${1:-1024}; CTX=${2:-1400}; PRESET=${3:-qwen2.5-1.5b}
    timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${PRESET}_b${B}_c${CTX}.csv \
      python tools/decode_microbench.py --model $PRESET --batch $B --ctx $CTX --iters 2 --ncu \
      > gpurun_out/launches_${PRESET}_b${B}.log 2>&1
    python tools/launch_summary.py gpurun_out/launches_${PRESET}_b${B}_c${CTX}.csv | tail -30 ;;
  ncu_attn)
    bash tools/gpu_ncu_attn.sh "$@" ;;
  sanitize)
    for tool in racecheck memcheck; do
      timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider \
        -m gpu tests/test_attention_gpu.py -k "b64 and c3 and page64 or mixed7 and c5" \
        > gpurun_out/sanitize_${tool}_attention.log 2>&1
      echo "rc=$?" >> gpurun_out/sanitize_${tool}_attention.log
      timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider \
        -m gpu tests/test_engine_gpu.py tests/test_replay_model_gpu.py -k "c1_tiny and april and reprefill or exactly_once or advantages" \
        > gpurun_out/sanitize_${tool}_engine.log 2>&1
      echo "rc=$?" >> gpurun_out/sanitize_${tool}_engine.log
    done
    tail -n 3 gpurun_out/sanitize_*.log ;;
  forcedp)
    # the lockstep DP wrapper at world 1 must make the plain engine's decisions (same iterations and
    # carried tokens per step): two short bench runs, decisions compared by tools/compare_forcedp.py
    timeout 1200 python bench.py --steps 3 --warmup 2 --no-sync --no-cpu "$@" > gpurun_out/forcedp_plain.log 2>&1
    timeout 1200 python bench.py --steps 3 --warmup 2 --no-sync --no-cpu --force-dp "$@" > gpurun_out/forcedp_dp.log 2>&1
    python tools/compare_forcedp.py gpurun_out/forcedp_plain.log gpurun_out/forcedp_dp.log | tee gpurun_out/forcedp_compare.txt ;;
  dp2)
    # the multi-rank bench path at world 2 on ONE GPU: two torchrun ranks pinned to cuda:0, gloo host
    # collectives, device-side lockstep exchange through CUDA IPC (scaling is not measurable here)
    AB_BENCH_DEVICE=0 AB_BENCH_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --no-cpu --kv-pages ${KVP:-30000} "$@" \
      > gpurun_out/dp2_bench.log 2> gpurun_out/dp2_bench.err
    echo "dp2 rc=$?" >> gpurun_out/dp2_bench.err; tail -c 2500 gpurun_out/dp2_bench.log ;;
  *) echo "unknown mode $MODE"; exit 2 ;;
esac
