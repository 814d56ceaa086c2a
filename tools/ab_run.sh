# usage: bash tools/ab_run.sh TAG "variant1 variant2 ..."   (variants built by tools/ab_variants.py)
TAG=$1; VARS=$2
mkdir -p gpurun_out
for v in $VARS; do
  LB_LIB_VARIANT=$v timeout 600 python -m pytest tests/test_full_size.py -m gpu -x -q -k "config2_full_batch or per_frame" > gpurun_out/${TAG}_${v}_tests.log 2>&1
  echo "$v tests: $(tail -1 gpurun_out/${TAG}_${v}_tests.log)"
done
AB_ROUNDS=${AB_ROUNDS:-3} python tools/ab_variants.py run "python bench.py --no-llm --no-wer --no-cpu-baseline --no-e2e --no-parity --steps 20 --warmup 3" $VARS 2>&1 | tee gpurun_out/${TAG}_ab.txt
for v in $VARS; do
  LB_LIB_VARIANT=$v timeout 300 python bench.py --phases --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-llm --no-wer --no-parity > gpurun_out/${TAG}_${v}_ph.json 2>/dev/null
done
python - <<PY
import json
for v in "$VARS".split():
    try:
        d=json.loads(open(f"gpurun_out/${TAG}_{v}_ph.json").read().strip().splitlines()[-1])
        ph=d["phase_cycles_per_frame"]; print(v, {k:round(x) for k,x in ph.items()})
    except Exception as e: print(v, "ERR", e)
PY
