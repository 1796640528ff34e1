# Final ncu evidence (one GPU): c2 launch list + full capture of the three
# mode passes (-> profiles/traffic.json), and one c4 mode-0 pass.
# usage (from the repo root, under gpurun): bash tools/ncu_round.sh TAG
tag=${1:-r2g}
args2="--config 2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
args4="--config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $args2 > gpurun_out/${tag}_plain_c2.log 2>&1 && \
python bench.py $args4 > gpurun_out/${tag}_plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py $args2 > gpurun_out/${tag}_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mode_pass_pack -s 3 -c 3 \
    -o gpurun_out/${tag}_c2 python bench.py $args2 > gpurun_out/${tag}_ncu_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mode_pass_pack -s 3 -c 1 \
    -o gpurun_out/${tag}_c4 python bench.py $args4 > gpurun_out/${tag}_ncu_c4.log 2>&1
echo ncu_rc=$?
