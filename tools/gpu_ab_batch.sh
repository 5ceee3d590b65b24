# A/B: attention work-cursor prefetch (AB_ATT_PREFETCH) and the 128-row prefill attention blocks
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_model_gpu.py tests/test_attention_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_ab.log 2>&1; echo rc=$? >> gpurun_out/pytest_ab.log
AB_ATT_PREFETCH=1 timeout 1200 python -m pytest tests/test_attention_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_ab_pf.log 2>&1; echo rc=$? >> gpurun_out/pytest_ab_pf.log
for PF in 0 1; do
  AB_ATT_PREFETCH=$PF timeout 600 python tools/decode_microbench.py --model qwen2.5-1.5b --batch 384 --ctx 1350 --iters 32 > gpurun_out/ab_c2_b384_pf$PF.log 2>&1
  AB_ATT_PREFETCH=$PF timeout 600 python tools/decode_microbench.py --model qwen3-4b --batch 64 --ctx 3000 --iters 32 > gpurun_out/ab_c3_b64_pf$PF.log 2>&1
  AB_ATT_PREFETCH=$PF timeout 600 python tools/decode_microbench.py --model qwen2.5-1.5b --batch 1024 --ctx 1400 --iters 16 > gpurun_out/ab_c2_b1024_pf$PF.log 2>&1
done
timeout 600 python tools/prefill_bench.py --samples 64 --gen 2000 > gpurun_out/prefill_bench.log 2>&1
timeout 600 python tools/prefill_bench.py --samples 256 --gen 1000 > gpurun_out/prefill_bench2.log 2>&1
tail -2 gpurun_out/pytest_ab.log gpurun_out/pytest_ab_pf.log; cat gpurun_out/prefill_bench*.log | tail -2
for f in gpurun_out/ab_*.log; do python -c "
import json,sys; s=open('$f').read(); d=json.loads(s[s.rfind(chr(10)+'{')+1:]); print('$f', d['steady_ms_per_iter'])"; done
timeout 2400 python bench.py --no-cpu --workload C4 --over-provision 2 --steps 3 --warmup 3 --sync-steps 2 > gpurun_out/cfg_C4_2.log 2> gpurun_out/cfg_C4_2.err; echo "C4_2 rc=$?"; tail -2 gpurun_out/cfg_C4_2.err
