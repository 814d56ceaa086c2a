#!/bin/bash
# A/B of the streaming e2e (config 2): LB_STREAM_OVERLAP=1 (pipelined searches share the SMs)
# vs 0 (searches back to back, copies and host assembly overlapped)
for rnd in 1 2; do for v in 1 0; do
  LB_STREAM_OVERLAP=$v timeout 300 python bench.py --no-llm --no-wer --no-cpu-baseline --no-parity --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('overlap=$v', 'device', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), 'single', round(d['e2e']['single_call']['value']/1e6,2), d['clocks']['sm_mhz'])"
done; done
