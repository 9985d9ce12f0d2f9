# Round-end evidence (profiles/r02): bench line, ncu launch list of the bench command,
# launch list (+DRAM bytes) of one full solve, one --set full capture of a BILU color launch
# and one of a level-0 PGS-MC color launch.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
$NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"mspk|sell_|bilu_|bsr_|cgs_|dcgs_|pcol_|gemv|restrict|prolong|gather|scale" -c 600 --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
echo bench-launches rc $?
python tools/profile_solve.py > gpurun_out/prof_plain.log 2>&1 && \
$NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches_solve.csv python tools/profile_solve.py > gpurun_out/ncu_l.log 2>&1
echo launches rc $?
python tools/profile_solve.py --kernel arnoldi_step15 > gpurun_out/prof_plain2.log 2>&1
$NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:"bilu_meta4" -s 12 -c 1 \
  -o gpurun_out/full_bilu python tools/profile_solve.py --kernel arnoldi_step15 > gpurun_out/ncu_f.log 2>&1
echo full rc $?
$NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:"sell_row_uniform" -s 4 -c 1 \
  -o gpurun_out/full_gs python tools/profile_solve.py --kernel arnoldi_step15 > gpurun_out/ncu_g.log 2>&1
echo full-gs rc $?
ls -la gpurun_out
