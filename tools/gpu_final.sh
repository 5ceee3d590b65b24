#!/bin/bash
# Round-end evidence: GPU tests, smoke, C2 bench (default: KV re-prefill), then the ncu captures and
# microbench points of tools/gpu_round.sh.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
bash tools/gpu_round.sh
timeout 400 python tools/decode_microbench.py --batch 512 --ctx 1600 --iters 16 > gpurun_out/micro_b512.json 2>&1
timeout 400 python tools/decode_microbench.py --model qwen3-4b --batch 64 --ctx 3000 --iters 16 > gpurun_out/micro_c3_b64.json 2>&1
timeout 300 python tools/prefill_bench.py --samples 64 --gen 2000 > gpurun_out/prefill_c2.log 2>&1
