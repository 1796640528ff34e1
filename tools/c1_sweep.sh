for t in 1024 2048 4096 8192; do
  for ch in 2048 4096 8192; do
    r=$(FLYCOO_ACC_TILE_BYTES=$t FLYCOO_CHUNK=$ch timeout 300 python bench.py --config 1 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['config']['mode_ms'], d['config']['params_m'])")
    echo "tile=$t chunk=$ch $r"
  done
done
