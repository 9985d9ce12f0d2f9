# ncu --set full of the BILU color kernels (graph-replayed a9 via time_kernel), with source
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python tools/profile_solve.py --kernel bilu > gpurun_out/prof_plain.log 2>&1
echo plain rc $?
$NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:"bilu_block" -c 16 \
  -o gpurun_out/prof_bilu python tools/profile_solve.py --kernel bilu > gpurun_out/ncu_bilu.log 2>&1
echo full rc $?
tail -3 gpurun_out/ncu_bilu.log
