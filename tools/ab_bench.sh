#!/bin/bash
# A/B the in-tree kernel builds on c2: tools/ab_bench.sh [CONFIG] NAME... ("base" = libflycoo.so);
# prints ms per sweep and per-mode ms for each build, twice in alternating order.
cfg=2
if [[ "$1" =~ ^[0-9]+$ ]]; then cfg=$1; shift; fi
for rep in 1 2; do
  for n in "$@"; do
    lib=libflycoo_$n.so; [ "$n" = base ] && lib=libflycoo.so
    FLYCOO_LIB=$lib python bench.py --config $cfg --steps ${STEPS:-30} --warmup 5 --no-cpu-baseline --no-e2e ${NNZ:+--nnz $NNZ} 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', round(d['ms_per_step'],4), d['config']['mode_ms'], round(d['roofline']['frac'],4))"
  done
done
