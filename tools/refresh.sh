#!/bin/bash
# measurement refresh on one B200: frame-kernel ncu capture + launch list, default bench,
# reference arm, config 3, phase split.  usage: tools/refresh.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:frames_small -c 1 \
  -o gpurun_out/${TAG}_frames python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  --no-llm --no-wer --no-parity > gpurun_out/${TAG}_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --no-e2e --no-llm --no-wer --no-parity > gpurun_out/${TAG}_launches.log 2>&1
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err
timeout 1200 python bench.py --config 3 > gpurun_out/${TAG}_config3.json 2> gpurun_out/${TAG}_config3.err
timeout 300 python bench.py --phases --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-llm --no-wer --no-parity > gpurun_out/${TAG}_ph.json 2>&1
for f in bench reference config3 ph; do tail -c 300 gpurun_out/${TAG}_$f.json; echo; done
