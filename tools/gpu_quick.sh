mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python tools/ab_vcycle.py C3 > gpurun_out/ab.log 2>&1; echo ab rc $?
cat gpurun_out/ab.log
