mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g4_tests.log 2>&1; tail -3 gpurun_out/g4_tests.log
grep -E "Error|error|FAILED|assert" gpurun_out/g4_tests.log | head -20
bash tools/ab_run.sh ab2 "ns nons pc96 pc128"
