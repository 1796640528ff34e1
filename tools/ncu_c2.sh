# ncu evidence for one bench config on one B200 (run under gpurun from the repo root)
# usage: bash tools/ncu_c2.sh TAG [CONFIG] [KERNEL_REGEX]
tag=${1:-r2}; cfg=${2:-2}; kre=${3:-mode_pass_pack}
args="--config $cfg --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $args > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py $args > gpurun_out/${tag}_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$kre -s 3 -c 3 \
    -o gpurun_out/${tag}_prof python bench.py $args > gpurun_out/${tag}_ncu.log 2>&1
echo ncu_rc=$?
