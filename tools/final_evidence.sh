bash tools/ncu_round.sh r2w
for t in c2 c4; do ncu -i gpurun_out/r2w_$t.ncu-rep --page raw --csv > gpurun_out/r2w_${t}_raw.csv 2>/dev/null; done
python tools/traffic_from_ncu.py gpurun_out/r2w_c2_raw.csv 2 "ncu --set full (profiles/r2w_ncu_c2_pack_kernel.txt, bench.py --config 2 --steps 2 --warmup 1): dram__bytes_read.sum + dram__bytes_write.sum" && cp profiles/traffic.json gpurun_out/traffic.json
bash tools/gpu_round_run.sh r2x
