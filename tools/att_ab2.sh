python -m pytest tests/test_llm.py -m gpu -x -q 2>&1 | tail -1
for kh in 4 2 1; do LB_ATT_KH=$kh timeout 600 ncu --metrics gpu__time_duration.sum -k regex:chain_attn -s 384 -c 1 python tools/llm_step.py --config 3 2>/dev/null | grep -E "chain_attn|gpu__time" | sed "s/^/KH=$kh /"; done
for v in 1 0; do LB_ATT_GROUP=$v python tools/prof_llm.py --config 3 2>/dev/null | grep -E "chain_attn|total device" ; done
for v in 1 0 1 0; do LB_ATT_GROUP=$v python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/att_c3_$v.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/att_c3_$v.json').read().strip().splitlines()[-1]);print('group=$v', d['ms_per_step'], d['clocks']['sm_mhz'], d.get('parity_check')[:10])"; done
