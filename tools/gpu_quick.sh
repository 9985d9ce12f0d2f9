mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?; tail -2 gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu.py -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python tools/ab_vcycle.py C3 ${AB_ARGS} > gpurun_out/ab.log 2>&1; echo ab rc $?
cat gpurun_out/ab.log
