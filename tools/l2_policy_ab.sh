# c4 with the selective L2 policy on the WIDE kernel's gathers (FLYCOO_L2_HOT_MB)
for mb in 0 60 100 0 60 100; do
  FLYCOO_L2_HOT_MB=$mb timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/l2pol_c4_${mb}_$RANDOM.json 2> /dev/null; echo "mb=$mb rc=$?"
done
