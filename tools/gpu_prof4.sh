mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python tools/profile_solve.py --kernel bilu > gpurun_out/prof_plain.log 2>&1 && \
$NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:"bilu_block" -s 3 -c 3 -o gpurun_out/prof_bilu2 python tools/profile_solve.py --kernel bilu > gpurun_out/ncu_b2.log 2>&1
echo rc $?
