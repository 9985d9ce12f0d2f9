# A/B of compile-time variants on the C3 bench: bash tools/gpu_ab_build.sh "-DX=1" "-DX=2" ...
# (each variant rebuilt on the box with MSP_NVCC_EXTRA; "" = the default build)
mkdir -p gpurun_out
i=0
for flags in "$@"; do
  MSP_NVCC_EXTRA="$flags" python -c "import __graft_entry__ as g; g.build_product(force=True)" > gpurun_out/abb_build_$i.log 2>&1 || { echo "build $i failed"; continue; }
  timeout 400 python bench.py --no-cpu-baseline --steps ${AB_STEPS:-5} --warmup 3 2>gpurun_out/ab_b$i.err | tail -1 > gpurun_out/ab_b$i.json
  echo "variant $i [$flags] rc $?"
  i=$((i+1))
done
