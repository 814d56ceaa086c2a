#!/bin/bash
# K1 row-per-thread (LB_LSM_ROWS=1) vs warp-per-row (0): parity tests + config-2 step time
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -m gpu -x -q -k "prologue or raw" 2>&1 | tail -1
bash tools/ab_env.sh LB_LSM_ROWS "0 1" 3
