bash tools/refresh.sh r2e
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2e_tests.log 2>&1; tail -1 gpurun_out/r2e_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1; tail -1 gpurun_out/r2e_smoke.log
