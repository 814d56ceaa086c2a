#!/bin/bash
# dev loop on the GPU box: parity tests of the search kernels + one config-2 bench line (+phases)
# usage: tools/gpu_check.sh TAG [pytest -k expr]
TAG=${1:-x}; K=${2:-}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_tests.log 2>&1
else
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1
fi
tail -3 gpurun_out/${TAG}_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-llm --no-wer > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 300 python bench.py --phases --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-llm --no-wer > gpurun_out/${TAG}_ph.json 2>&1
python - <<PY
import json
for f in ("gpurun_out/${TAG}_bench.json","gpurun_out/${TAG}_ph.json"):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "ms/step", round(d["ms_per_step"],3), "kernel_ms", d.get("roofline",{}).get("kernel_ms"))
        ph=d.get("phase_cycles_per_frame")
        if ph: print({k:round(v) for k,v in ph.items()})
    except Exception as e: print(f, "ERR", e)
PY
