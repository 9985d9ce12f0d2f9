mkdir -p gpurun_out
nproc
timeout 1500 python tools/asmsp_sequence.py --config C4 --steps 6 --mu 0 10 30 --out gpurun_out/asmsp_c4.json > gpurun_out/asmsp_c4.log 2>&1; echo asmsp rc $?
tail -4 gpurun_out/asmsp_c4.log
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --kernel-reps 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5 rc $?
tail -3 gpurun_out/bench_c5.err
