"""Warp-level instructions executed (and stall samples) per CUDA source line.
usage: ncu -i X.ncu-rep --page source --csv --print-source=cuda,sass > s.csv
       python profiles/ncu_insts.py s.csv ELEMENTS [top]
ELEMENTS (the kernel's nonzeros) turns counts into instructions per element."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
nel = float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fname, agg = None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Line No", "") or not r[0].isdigit():
        continue
    try:
        ins = int(r[7]) if r[7] not in ("-", "") else 0
        samp = int(r[4]) if r[4] not in ("-", "") else 0
    except (ValueError, IndexError):
        continue
    agg.append((ins, samp, fname, int(r[0]), r[1].strip()[:88]))
ti = sum(a[0] for a in agg) or 1
ts = sum(a[1] for a in agg) or 1
print(f"warp instructions {ti}  = {ti / nel:.2f} per element;  stall samples {ts}")
print(" inst%  inst/el  stall%  line")
for ins, samp, f, ln, src in sorted(agg, reverse=True)[:top]:
    print(f"{100 * ins / ti:5.1f}% {ins / nel:7.3f} {100 * samp / ts:6.1f}%  {f}:{ln}  {src}")
