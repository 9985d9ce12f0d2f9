mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "asmsp or edge" > gpurun_out/pytest_asmsp.log 2>&1; echo pytest rc $?; tail -2 gpurun_out/pytest_asmsp.log
timeout 1500 python tools/asmsp_sequence.py --config C4 --steps 8 --mu 0 50 1000 --out gpurun_out/asmsp_c4.json > gpurun_out/asmsp_c4.log 2>&1; echo asmsp rc $?
grep '^{"mu"' gpurun_out/asmsp_c4.log
