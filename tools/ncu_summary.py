"""Condense ncu raw CSV exports (gpurun_out/ncu_cfg_*.csv) into one table: per capture the kernel, its duration,
DRAM bytes and throughput, registers and achieved occupancy. usage: python tools/ncu_summary.py FILES... > out.csv"""
import csv
import os
import sys

COLS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
w = csv.writer(sys.stdout)
w.writerow(["capture"] + COLS)
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    if len(rows) < 3:
        continue
    h = rows[0]
    cells = []
    for c in COLS:  # value and its unit (ncu picks the unit per capture)
        if c not in h:
            cells.append("")
            continue
        i = h.index(c)
        cells.append(f"{rows[2][i]} {rows[1][i]}".strip())
    w.writerow([os.path.basename(f)[8:-4]] + cells)
