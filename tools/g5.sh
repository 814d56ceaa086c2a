mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tiny_char_lm.py tests/test_llm.py -m gpu -x -q > gpurun_out/g5_tests.log 2>&1; tail -15 gpurun_out/g5_tests.log
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-wer > gpurun_out/g5_c1.json 2> gpurun_out/g5_c1.err; tail -c 2500 gpurun_out/g5_c1.json; tail -5 gpurun_out/g5_c1.err
