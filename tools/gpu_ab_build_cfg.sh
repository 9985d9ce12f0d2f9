# A/B of compile-time variants on a given config: CFG=C5 bash tools/gpu_ab_build_cfg.sh "" "-DX=1" ...
mkdir -p gpurun_out
i=0
for flags in "$@"; do
  MSP_NVCC_EXTRA="$flags" python -c "import __graft_entry__ as g; g.build_product(force=True)" > gpurun_out/abb_build_$i.log 2>&1 || { echo "build $i failed"; continue; }
  for c in ${CFGS:-C3}; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --steps ${AB_STEPS:-3} --warmup 3 2>gpurun_out/abc_${c}_$i.err | tail -1 > gpurun_out/abc_${c}_$i.json
    echo "variant $i [$flags] $c rc $?"
  done
  i=$((i+1))
done
