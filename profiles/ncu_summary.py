"""Print the key metrics of every kernel in an ncu report (raw page CSV).
usage: ncu -i X.ncu-rep --page raw --csv > raw.csv; python profiles/ncu_summary.py raw.csv"""
import csv
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "l1tex__lsu_writeback_active_mem_lgds.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "launch__grid_size"]
rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
units = rows[1]
for r in rows[2:]:
    print("-" * 60)
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"  {k:72s} {r[i]} {units[i]}")
    st = []
    for i, k in enumerate(h):
        if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
            try:
                st.append((float(r[i].replace(",", "")), k.split("stalled_")[-1]))
            except ValueError:
                pass
    def num(k):
        return float(r[h.index(k)].replace(",", "")) if k in h and r[h.index(k)] else None
    sec, req = (num("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
                num("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"))
    if sec and req:
        print(f"  {'derived: global-load sectors per request':72s} {sec / req:.2f}")
    dr, dw, t = (num("dram__bytes_read.sum"), num("dram__bytes_write.sum"),
                 num("gpu__time_duration.sum"))
    if dr is not None and dw is not None and t:
        # dram__bytes in the units ncu printed (Gbyte / Mbyte) over ms
        ur = units[h.index("dram__bytes_read.sum")]
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(ur, 1.0)
        tu = units[h.index("gpu__time_duration.sum")]
        ts = {"ms": 1e-3, "us": 1e-6, "s": 1.0, "ns": 1e-9}.get(tu, 1e-3)
        print(f"  {'derived: achieved DRAM GB/s':72s} {(dr + dw) * scale / (t * ts) / 1e9:.0f}")
    tot = sum(v for v, _ in st) or 1
    print("  stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in sorted(st, reverse=True)[:8]))
