"""Headline metrics + stall mix of an ncu report: python tools/ncu_brief.py report.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    print(d.get("Kernel Name", "")[:90])
    for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
              "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
              "launch__grid_size"]:
        print(f"  {k:60s} {d.get(k)}")
    st = [(k, float(d[k] or 0)) for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    st.sort(key=lambda x: -x[1])
    print("  stalls/issue:", ", ".join(f"{k[34:-29]}={x:.2f}" for k, x in st[:8]))
