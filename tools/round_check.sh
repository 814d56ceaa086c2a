#!/bin/bash
# full verification on the GPU box: build, all GPU tests, smoke, default bench, phase split
TAG=${1:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1
tail -3 gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -c 600 gpurun_out/${TAG}_bench.json
timeout 300 python bench.py --phases --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-llm --no-wer > gpurun_out/${TAG}_ph.json 2>&1
