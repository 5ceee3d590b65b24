# per-CTA timelines (tools/gemm_trace.py) of the small decode projections under reduce-add schedules
mkdir -p gpurun_out
E=$((2|128|1024))
tr() { echo "== $*"; timeout 120 python tools/gemm_trace.py "$@" 2>&1 | head -40; }
{
tr 1536 1536 384 $((0x8000|1|(7<<1)|(4<<5))) $E      # C2 O, swap an128 red4
tr 1536 1536 384 $((0x18000|1|(7<<1)|(1<<5))) $E     # C2 O, swap an128 stream-K
tr 2048 1536 384 $((0x8000|1|(7<<1)|(3<<5))) $E      # C2 QKV (reduce-add into fp32), an128 red3
tr 6144 2560 64 $((0x8000|1|(6<<1)|(3<<5))) $E       # C3 QKV, an64 red3
tr 19456 2560 64 $((0x18000|1|(6<<1)|(1<<5))) $E     # C3 gate-up (fp32 workspace), an64 stream-K
} > gpurun_out/gemm_traces.txt 2>&1
tail -5 gpurun_out/gemm_traces.txt
