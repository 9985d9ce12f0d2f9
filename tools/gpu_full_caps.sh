# --set full captures per kernel family, first launches of a graph-replayed Arnoldi step
# (j = 15): FAMS="regex:count;regex:count" (keep each call's reports under gpurun's 64 MiB)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python tools/profile_solve.py --kernel arnoldi_step15 > gpurun_out/prof_plain.log 2>&1 || exit 1
IFS=';' read -ra FS <<< "${FAMS}"
for fam in "${FS[@]}"; do
  rx="${fam%%:*}"; cnt="${fam##*:}"; tag=$(echo "$rx" | tr -c 'a-z0-9\n' '_' | cut -c1-20)
  $NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:"$rx" -c $cnt \
    -o gpurun_out/full_$tag python tools/profile_solve.py --kernel arnoldi_step15 > gpurun_out/ncu_f_$tag.log 2>&1
  echo "full $rx rc $?"
done
ls -la gpurun_out/*.ncu-rep
