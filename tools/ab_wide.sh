#!/bin/bash
# A/B of the general frames kernel (beam 256 / 900) between library variants
mkdir -p gpurun_out
for v in $1; do
  LB_LIB_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wide or beam_900 or 4096 or vocab_64 or fallback" 2>&1 | tail -1 | sed "s/^/$v tests: /"
done
for rnd in 1 2; do for v in $1; do for k in 256 900; do
  LB_LIB_VARIANT=$v timeout 600 python bench.py --beam $k --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-llm --no-wer --no-parity 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v beam $k', round(d['ms_per_step'],2), d['layout'] if 'layout' in d else '')"
done; done; done
