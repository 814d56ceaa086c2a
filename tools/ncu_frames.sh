#!/bin/bash
# ncu --set full capture of one frames_small_kernel launch (config 2) + source-line export
# usage: tools/ncu_frames.sh TAG [variant]
TAG=${1:-x}; VAR=${2:-}
mkdir -p gpurun_out
[ -n "$VAR" ] && export LB_LIB_VARIANT=$VAR
timeout 900 ncu --set full --import-source on --clock-control none -k regex:frames_small -c 1 \
  -o gpurun_out/${TAG}_frames python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  --no-llm --no-wer --no-parity > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
