"""Per-kernel share of an ncu launch list (gpu__time_duration.sum CSV).
usage: python profiles/launch_shares.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    if len(r) > vi:
        agg[r[ki][:100]][0] += 1
        agg[r[ki][:100]][1] += float(r[vi].replace(",", ""))
tot = sum(v for _, v in agg.values())
print(f"{'launches':>8} {'total us':>10} {'share':>6}  kernel")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:8d} {v / 1e3:10.1f} {100 * v / tot:5.1f}%  {k}")
# the timed step (one sweep) launches only the mode passes and the K2 reduce;
# the rest is the generator and the layout build (untimed, reported as gen_s
# / build_s)
step = {k: cv for k, cv in agg.items() if "mode_pass" in k or "reduce_level" in k}
st = sum(v for _, v in step.values())
if st:
    print("\nshares within the sweep (mode passes + K2):")
    for k, (c, v) in sorted(step.items(), key=lambda x: -x[1][1]):
        print(f"{c:8d} {v / 1e3:10.1f} {100 * v / st:5.1f}%  {k}")
