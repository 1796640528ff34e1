"""Write profiles/traffic.json (the bench's roofline.traffic) from an ncu
capture of bench.py: DRAM bytes (read + write) per mode-pass launch, stamped
with the workload and a hash of the CUDA sources so bench.py refuses it for
any other kernel build or config.

usage: ncu -i gpurun_out/X.ncu-rep --page raw --csv > raw.csv
       python tools/traffic_from_ncu.py raw.csv CONFIG "<capture description>"
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2309_09131_b200.params import device_params  # noqa: E402
from paper_2309_09131_b200.synth import CONFIGS  # noqa: E402


def scale(v: str, unit: str) -> float:
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v) * mult[unit]


def main():
    raw, cfg_index, what = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    rows = list(csv.reader(open(raw)))
    h, units = rows[0], rows[1]
    ik, ir, iw = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    per, names = [], []
    for r in rows[2:]:
        if "mode_pass" not in r[ik]:
            continue
        per.append(scale(r[ir], units[ir]) + scale(r[iw], units[iw]))
        names.append(r[ik])
    if not per:
        sys.exit("no mode_pass kernels in the capture")
    cfg = CONFIGS[cfg_index]
    params = device_params(cfg["dims"], cfg["nnz"], cfg["rank"])
    out = {"config": cfg_index, "nnz": cfg["nnz"], "params_m": list(params.m), "params_g": params.g,
           "kernel_sources": bench.kernel_sources_hash(), "kernels": names,
           "dram_bytes_per_launch": sum(per) / len(per), "per_launch": per,
           "source": f"ncu --set full ({what}): dram__bytes_read.sum + dram__bytes_write.sum"}
    (ROOT / "profiles" / "traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
