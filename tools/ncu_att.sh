#!/bin/bash
# ncu of chain attention launches (config 3): final event (launches 384-385) and a middle one
mkdir -p gpurun_out
for v in 1 0; do
  for s in 384 192; do
    LB_ATT_GROUP=$v timeout 600 ncu --set full --clock-control none -k regex:chain_attn -s $s -c 1 \
      -o gpurun_out/att_g${v}_s${s} python tools/llm_step.py --config 3 > gpurun_out/att_ncu_g${v}_s${s}.log 2>&1
  done
done
ls gpurun_out/*.ncu-rep
