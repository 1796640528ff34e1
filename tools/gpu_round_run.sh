# Round-end evidence on one B200: GPU tests, smoke, every bench line.
# usage (from the repo root, under gpurun): bash tools/gpu_round_run.sh TAG
tag=${1:-r1}
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -q -m gpu --durations=8 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
python bench.py > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_reference_arm.json 2> gpurun_out/bench_ref.err; echo ref=$?
for c in 1 3 4 5; do
  s=30; [ $c = 1 ] && s=100; [ $c -ge 4 ] && s=10
  timeout 1200 python bench.py --config $c --steps $s --warmup 3 > gpurun_out/${tag}_bench_c$c.json 2> gpurun_out/bench_c$c.err; echo c$c=$?
done
