mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g6_tests.log 2>&1; tail -5 gpurun_out/g6_tests.log; grep -E "^(FAILED|ERROR)|Error" gpurun_out/g6_tests.log | head -20
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-wer > gpurun_out/g6_c1.json 2> gpurun_out/g6_c1.err; python -c "
import json;d=json.loads(open('gpurun_out/g6_c1.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['gpu_launches'],d['parity_check'],d['llm'])"; tail -5 gpurun_out/g6_c1.err
