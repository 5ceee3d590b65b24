#!/bin/bash
mkdir -p gpurun_out
for z in 0 1; do
  if [ $z = 1 ]; then export AB_ROPE_NOZERO=1; fi
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none --csv -k regex:k_rope \
    --log-file gpurun_out/rope_nozero$z.csv python tools/decode_microbench.py --batch 1024 --ctx 1400 --iters 1 --ncu > /dev/null 2>&1
  timeout 400 python tools/decode_microbench.py --batch 1024 --ctx 1400 --iters 4 > gpurun_out/rope_micro_nozero$z.json 2>&1
done
