# per-launch ncu list of one graph-replayed a9 apply (reps=2 -> 3 replays) for TMA on/off
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for t in 1 0; do
  MSP_BILU_TMA=$t $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__shared_mem_per_block_dynamic,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem \
    --clock-control none --csv --log-file gpurun_out/bilu_launches_tma$t.csv python tools/profile_solve.py --kernel bilu > gpurun_out/bilu_l$t.log 2>&1
  echo tma$t rc $?
done
