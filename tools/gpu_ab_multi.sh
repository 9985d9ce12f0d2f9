# A/B of several environment settings on the C3 bench: bash tools/gpu_ab_multi.sh "A=1 B=2" "A=2" ...
# writes gpurun_out/abm_<i>.json
mkdir -p gpurun_out
i=0
for e in "$@"; do
  env $e timeout 400 python bench.py --no-cpu-baseline --steps ${AB_STEPS:-5} --warmup 3 2>gpurun_out/abm_$i.err | tail -1 > gpurun_out/abm_$i.json
  echo "variant $i [$e] rc $?"
  i=$((i+1))
done
