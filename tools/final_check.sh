bash tools/refresh.sh ${TAG:-r2f}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG:-r2f}_tests.log 2>&1; tail -1 gpurun_out/${TAG:-r2f}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-r2f}_smoke.log 2>&1; tail -1 gpurun_out/${TAG:-r2f}_smoke.log
