# A/B of (compile flags | environment) variants on the C3 bench:
#   bash tools/gpu_ab_build_env.sh "-DX=1|" "|MSP_Y=2" ...   -> gpurun_out/abc_C3_<i>.json
mkdir -p gpurun_out
i=0
for spec in "$@"; do
  flags="${spec%%|*}"; envs="${spec#*|}"
  MSP_NVCC_EXTRA="$flags" python -c "import __graft_entry__ as g; g.build_product(force=True)" > gpurun_out/abb_build_$i.log 2>&1 || { echo "build $i failed"; i=$((i+1)); continue; }
  env $envs X_=1 timeout 600 python bench.py --no-cpu-baseline --steps ${AB_STEPS:-3} --warmup 3 2>gpurun_out/abc_C3_$i.err | tail -1 > gpurun_out/abc_C3_$i.json
  echo "variant $i [$spec] rc $?"
  i=$((i+1))
done
