# Round evidence on one B200: smoke, GPU tests, every bench line, the
# reference arm, a 2-rank self-launched functional run.
# usage (from the repo root, under gpurun): bash tools/gpu_round_run.sh TAG
tag=${1:-r2}
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -q -m gpu --durations=12 > gpurun_out/${tag}_gpu_tests.log 2>&1; echo tests=$?
python bench.py > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench_c2.err; echo bench=$?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${tag}_bench_reference_arm.json 2> gpurun_out/${tag}_bench_ref.err; echo ref=$?
for c in 1 3 4 5; do
  s=30; [ $c = 1 ] && s=100; [ $c -ge 4 ] && s=10
  timeout 1200 python bench.py --config $c --steps $s --warmup 3 > gpurun_out/${tag}_bench_c$c.json 2> gpurun_out/${tag}_bench_c$c.err; echo c$c=$?
done
FLYCOO_PG_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/${tag}_selflaunch_2ranks.json 2> gpurun_out/${tag}_selflaunch.err; echo self=$?
