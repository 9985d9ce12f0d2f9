# per-launch ncu list of one graph-replayed a9 apply (C3): duration, DRAM bytes, grid, warps active
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for t in ${BILU_META:-1 0}; do
  MSP_BILU_META=$t $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --log-file gpurun_out/bilu_launches_meta$t.csv python tools/profile_solve.py --kernel bilu > gpurun_out/bilu_l$t.log 2>&1
  echo meta$t rc $?
done
