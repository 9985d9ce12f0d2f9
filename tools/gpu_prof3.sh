mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python tools/profile_solve.py --kernel arnoldi_step15 > gpurun_out/prof_plain.log 2>&1 && \
$NCU --profile-from-start off --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches_step.csv python tools/profile_solve.py --kernel arnoldi_step15 > gpurun_out/ncu_s.log 2>&1
echo step rc $?
