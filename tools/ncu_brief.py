"""Condensed view of an ncu raw CSV (one kernel): time, DRAM, instructions, issue/warps active, occupancy
limits, stall breakdown (per issue-active), registers and shared memory. usage: ncu_brief.py raw.csv"""
import csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
d = dict(zip(hdr, rows[2]))
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.per_second", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__shared_mem_per_block_static",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "sm__cycles_elapsed.avg.per_second"]
for k in keys:
    print(f"{k:60s} {d.get(k, '-')}")
st = {k.split("stalled_")[1].replace("_per_issue_active.ratio", ""): float(v) for k, v in d.items()
      if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
print("stalls/issue:", ", ".join(f"{k} {v:.2f}" for k, v in sorted(st.items(), key=lambda x: -x[1]) if v > 0.05))
