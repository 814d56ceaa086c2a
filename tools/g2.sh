mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_full_size.py tests/test_multiproc.py -m gpu -x -q --durations=0 > gpurun_out/g2_tests.log 2>&1; tail -30 gpurun_out/g2_tests.log
