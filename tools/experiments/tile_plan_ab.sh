timeout 900 python -m pytest tests/test_gpu_tile_plan.py -x -q -m gpu 2>&1 | tail -15
b() { env $1 python bench.py --config ${2:-2} --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],4), d['config']['mode_ms'], round(d['roofline']['frac'],4))"; }
for r in 1 2; do
b FLYCOO_TILE_PLAN=0
b FLYCOO_TILE_PLAN=1
done
