# A/B of compile-time kernel variants: VARIANTS="tag1:flags1;tag2:flags2" (flags -> nvcc)
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  tag="${v%%:*}"; flags="${v#*:}"
  MSP_NVCC_EXTRA="$flags" python -c "import __graft_entry__ as g; g.build_product(force=True)" > gpurun_out/build_$tag.log 2>&1 || { echo "build $tag failed"; tail -20 gpurun_out/build_$tag.log; continue; }
  echo "== $tag ($flags)"
  timeout 300 python tools/ab_vcycle.py C3 ${AB_ARGS} 2>&1 | grep -E "^\S|bilu|msp_apply|vcycle|a4_|cgs2_step|solve_ms"
done
