mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep "Model name"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
tail -5 gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu.py -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -40 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc $?
tail -20 gpurun_out/bench1.err; cat gpurun_out/bench1.json
