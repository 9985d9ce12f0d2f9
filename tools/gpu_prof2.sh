mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python tools/profile_solve.py --kernel vcycle > gpurun_out/prof_plain.log 2>&1 && \
$NCU --profile-from-start off --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches_vcycle.csv python tools/profile_solve.py --kernel vcycle > gpurun_out/ncu_v.log 2>&1
echo vcycle rc $?
python tools/profile_solve.py --kernel bilu > gpurun_out/prof_plain2.log 2>&1 && \
$NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:"bilu_block" -c 4 -o gpurun_out/prof_bilu python tools/profile_solve.py --kernel bilu > gpurun_out/ncu_b.log 2>&1
echo bilu rc $?
python tools/profile_solve.py --kernel cgs2_step15 > gpurun_out/prof_plain3.log 2>&1 && \
$NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:"cgs_|bsr_spmv" -c 4 -o gpurun_out/prof_cgs python tools/profile_solve.py --kernel cgs2_step15 > gpurun_out/ncu_c.log 2>&1
echo cgs rc $?
