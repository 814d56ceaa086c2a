#!/bin/bash
# close kernel: parity subset, config-2 step time, and one ncu --set full capture with source
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -m gpu -x -q -k "config2_full_batch or random or worlds or beam_900 or edge" 2>&1 | tail -1
bash tools/ab_env.sh LB_DUMMY "x" 3
timeout 600 ncu --set full --import-source on --clock-control none -k regex:close_kernel -c 1 \
  -o gpurun_out/close3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  --no-llm --no-wer --no-parity > gpurun_out/close_ncu.log 2>&1; tail -1 gpurun_out/close_ncu.log
