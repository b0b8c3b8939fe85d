"""Markdown summary of an ncu --set full report (per kernel): time, DRAM bytes,
cache hit rates, issue efficiency, occupancy.  Usage: ncu_summary.py REPORT [title]"""
import csv, subprocess, sys
rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum", "lts__t_bytes.sum"]
col = {k: hdr.index(k) for k in want if k in hdr}
kn = hdr.index("Kernel Name")
print(f"### {title}\n")
print("| kernel | " + " | ".join(f"{k} [{units[col[k]]}]" for k in col) + " |")
print("|---|" + "---|" * len(col))
for r in data:
    name = r[kn].split("(")[0].split("::")[-1]
    print(f"| {name} | " + " | ".join(r[col[k]] for k in col) + " |")
