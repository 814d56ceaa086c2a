#!/bin/bash
# A/B an environment knob on the config-2 bench: tools/ab_env.sh VAR "v1 v2 ..." [rounds]
VAR=$1; VALS=$2; R=${3:-2}
for rnd in $(seq 1 $R); do for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --no-llm --no-wer --no-cpu-baseline --no-e2e --no-parity --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$VAR=$v', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
done; done
