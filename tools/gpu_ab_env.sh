# A/B of an environment switch on the C3 bench: bash tools/gpu_ab_env.sh VAR "v1 v2 ..." [bench args]
# writes gpurun_out/ab_<VAR>_<v>.json (one bench line each)
mkdir -p gpurun_out
var=$1; vals=$2; shift 2
for v in $vals; do
  env $var=$v timeout 400 python bench.py --no-cpu-baseline "$@" 2>gpurun_out/ab_${var}_$v.err | tail -1 > gpurun_out/ab_${var}_$v.json
  echo "$var=$v rc $?"
done
