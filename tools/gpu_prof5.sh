mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python tools/profile_solve.py --kernel cgs2_step25 > gpurun_out/prof_plain.log 2>&1 && \
$NCU --profile-from-start off --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_cgs25.csv python tools/profile_solve.py --kernel cgs2_step25 > gpurun_out/ncu_c.log 2>&1
echo rc $?
