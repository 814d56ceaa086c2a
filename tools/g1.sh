set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g1_tests.log 2>&1; tail -3 gpurun_out/g1_tests.log
timeout 600 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; tail -c 3000 gpurun_out/g1_bench.json
timeout 300 python bench.py --phases --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-llm --no-wer > gpurun_out/g1_ph.json 2>&1; tail -c 1500 gpurun_out/g1_ph.json
