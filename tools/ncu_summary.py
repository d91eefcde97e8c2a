"""Print key metrics, stall mix and the hottest SASS lines of an ncu report.
usage: python tools/ncu_summary.py <report.ncu-rep> [n_units_for_per_unit_counts]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
for m in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed.avg.per_cycle_active", "dram__bytes_read.sum", "launch__registers_per_thread",
          "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
          "smsp__thread_inst_executed_per_inst_executed.ratio"]:
    if m in h:
        print(f"{m:60s} {r[2][h.index(m)]:>16s} {r[1][h.index(m)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ie, ss, sc, ad = (h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source"),
                  h.index("Address"))
tot = sum(int(x[ie] or 0) for x in rows[2:])
st = sum(int(x[ss] or 0) for x in rows[2:]) or 1
print(f"instructions {tot:.4g} ({tot / units:.1f} per unit)")
cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
mix = sorted(((sum(float(x[i] or 0) for x in rows[2:]) / st * 100, h[i]) for i in cols), reverse=True)[:8]
print("stalls:", ", ".join(f"{n[6:]} {v:.1f}%" for v, n in mix))
hot = sorted(rows[2:], key=lambda x: -int(x[ss] or 0))[:15]
for x in hot:
    print(f"  {x[ad][-5:]} exec/unit {int(x[ie] or 0) / units:7.3f} stall {100 * int(x[ss] or 0) / st:5.1f}%  {x[sc][:80]}")
