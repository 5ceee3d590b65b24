#!/bin/bash
# GEMM iteration call: kernel numerics, tcgen05 GEMM schedules vs cuBLAS on the decode shapes, decode microbench.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/pytest_kernels.log
python -c "
import ctypes as C, sys; sys.path.insert(0, '.')
from paper_2509_18521_b200 import _capi
for cs in (1, 2, 4, 8, 16):
    n = C.c_int()
    try:
        _capi.call('ab_debug_gemm_clusters', cs, C.byref(n)); print('cluster', cs, 'max clusters', n.value)
    except Exception as e: print('cluster', cs, e)
" > gpurun_out/clusters.txt 2>&1
timeout 300 python tools/gemm_trace.py 1536 1536 8 256 50 > gpurun_out/trace1.txt 2>&1
timeout 900 python tools/gemm_bench.py --sweep --m 1024 512 256 128 64 16 --reps 7 > gpurun_out/gemm_sweep.jsonl 2>&1
timeout 300 python tools/decode_microbench.py --batch 1024 --ctx 1400 --iters 16 > gpurun_out/micro_b1024.json 2>&1
timeout 300 python tools/decode_microbench.py --batch 256 --ctx 2000 --iters 16 > gpurun_out/micro_b256.json 2>&1
timeout 300 python tools/decode_microbench.py --batch 64 --ctx 3000 --iters 16 > gpurun_out/micro_b64.json 2>&1
