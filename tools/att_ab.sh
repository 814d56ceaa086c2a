python -m pytest tests/test_llm.py -m gpu -x -q > gpurun_out/att_llm.log 2>&1; tail -2 gpurun_out/att_llm.log
python -m pytest tests/test_full_size.py -m gpu -x -q -k "config3 or config5" > gpurun_out/att_full.log 2>&1; tail -2 gpurun_out/att_full.log
for v in 1 0 1 0; do LB_ATT_GROUP=$v python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/att_c3_$v.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/att_c3_$v.json').read().strip().splitlines()[-1]);print('group=$v', d['ms_per_step'], d['clocks']['sm_mhz'], d.get('parity_check'))"; done
