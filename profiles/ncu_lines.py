"""Aggregate ncu source-page warp-stall samples per CUDA source line.
usage: ncu -i X.ncu-rep --page source --csv --print-source=cuda,sass > s.csv
       python profiles/ncu_lines.py s.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, func, hdr = None, None, None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "":
        continue
    try:
        samp = int(r[4]) if r[4] not in ("-", "") else 0
    except ValueError:
        continue
    key = (fname, int(r[0]), r[1].strip()[:90])
    agg[key] = agg.get(key, 0) + samp
tot = sum(agg.values()) or 1
print(f"total samples {tot}")
for (f, ln, src), s in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * s / tot:5.1f}% {f}:{ln:4d}  {src}")
