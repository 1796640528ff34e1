#!/bin/bash
# A/B: fibre reuse kernel (tools/experiments/pack_fibre_reuse.patch, built as libflycoo_reuse.so with
# -DPACK_REUSE=1) x lexicographic input order, c2.  FLYCOO_EXP_LEXSORT was a temporary bench.py knob
# (sort the generated COO by its flattened coordinate before build_device_sharded); removed after the run.
run() { # lib lexsort tag
  FLYCOO_LIB=$1 FLYCOO_EXP_LEXSORT=$2 python bench.py --config 2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null |
   python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$3', round(d['ms_per_step'],4), d['config']['mode_ms'], round(d['roofline']['frac'],4))"
}
for rep in 1 2; do
run libflycoo.so 0 base_draw
run libflycoo.so 1 base_lex
run libflycoo_reuse.so 0 reuse_draw
run libflycoo_reuse.so 1 reuse_lex
done
