#!/bin/bash
# K1 eight-lanes-per-row (LB_LSM_ROWS=1, default) vs warp-per-row (0): parity tests, config-2
# step time, ncu duration of both forms
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -m gpu -x -q -k "prologue or raw" 2>&1 | tail -1
bash tools/ab_env.sh LB_LSM_ROWS "0 1" 3
for v in 0 1; do
  LB_LSM_ROWS=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:log_softmax -c 2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-llm --no-wer --no-parity 2>/dev/null | grep -E "log_softmax|gpu__time" | sed "s/^/rows=$v /"
done
