# A/B an environment switch on bench.py, alternating order, same box.
# usage: bash tools/ab_env.sh VAR "v1 v2" REPS TAG bench-args...
var=$1; vals=$2; reps=$3; tag=$4; shift 4
for r in $(seq 1 $reps); do
  for v in $vals; do
    env $var=$v timeout 900 python bench.py "$@" > gpurun_out/ab_${tag}_${var}_${v}_$r.json 2>/dev/null
    echo "$var=$v rep=$r rc=$?"
  done
done
