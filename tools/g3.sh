mkdir -p gpurun_out
timeout 600 python bench.py --no-llm > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err; tail -c 600 gpurun_out/g3_bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/g3_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["parity_check"], d["cpu_baseline"])
PY
timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-wer --no-cpu-baseline --no-e2e > gpurun_out/g3_c3.json 2> gpurun_out/g3_c3.err; tail -c 400 gpurun_out/g3_c3.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:frames_small -c 1 -o gpurun_out/frames_r2a python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-llm --no-wer --no-parity > gpurun_out/g3_ncu.log 2>&1; tail -3 gpurun_out/g3_ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2a.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-llm --no-wer --no-parity > /dev/null 2>&1; tail -3 gpurun_out/launches_r2a.csv
