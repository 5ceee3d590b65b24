# steady decode iteration time vs the attention work-items-per-CTA and PDL-mask knobs
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 300 python tools/decode_microbench.py --iters 32 $MB > gpurun_out/knob_$tag.log 2>&1;
        python -c "
import json; s=open('gpurun_out/knob_$tag.log').read(); d=json.loads(s[s.rfind(chr(10)+'{')+1:]); print('$tag', d['steady_ms_per_iter'])"; }
MB="--model qwen2.5-1.5b --batch 384 --ctx 1350"
for it in 2 3 4 6; do run c2_items$it AB_ATT_ITEMS=$it; done
for pm in 6 2 4 14; do run c2_pdl$pm AB_PDL_MASK=$pm; done
MB="--model qwen3-4b --batch 64 --ctx 3000"
for it in 2 3 4 6; do run c3_items$it AB_ATT_ITEMS=$it; done
for pm in 6 2 4 14; do run c3_pdl$pm AB_PDL_MASK=$pm; done
