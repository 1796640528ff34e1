#!/bin/bash
# Accumulator-tile (m) sweep: tools/tile_sweep.sh CONFIG STEPS BYTES...  (FLYCOO_ACC_TILE_BYTES)
cfg=$1; steps=$2; shift 2
for b in "$@"; do
  FLYCOO_ACC_TILE_BYTES=$b python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$cfg', $b, d['config']['params_m'], round(d['ms_per_step'],3), d['config']['mode_ms'])"
done
