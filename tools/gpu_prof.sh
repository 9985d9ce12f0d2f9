mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python tools/profile_solve.py > gpurun_out/prof_plain.log 2>&1 && \
$NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_solve.py > gpurun_out/ncu_launch.log 2>&1
echo launch rc $?
$NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:"bilu_color|bsr_spmv|pgs_color|multidot|multiaxpy|gemv" -c 14 -o gpurun_out/prof_full python tools/profile_solve.py > gpurun_out/ncu_full.log 2>&1
echo full rc $?
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
