"""Summarise ncu reports and bench JSON lines into profiles/ (committed evidence).

usage: python tools/summarize_profiles.py <evidence dir> <round tag>
  reads  <dir>/full_*.ncu-rep, <dir>/launches_default.csv, <dir>/bench_*.json
  writes profiles/<tag>_ncu_<name>.csv   (key metrics of each full capture)
         profiles/<tag>_launches_default.csv (per-launch device times, kernel shares)
         profiles/<tag>_bench.jsonl       (the bench lines)
         profiles/ncu_traffic.json        (DRAM bytes per launch of the dominant kernels)
         profiles/ncu_kernels.json        (per capture <workload>_<mode>: instructions, DRAM bytes, IPC,
                                           pipe utilisation per launch -- read by bench.py's roofline)
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__thread_inst_executed_per_inst_executed.ratio",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def stall_summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    h = rows[1]
    cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    ia = h.index("Warp Stall Sampling (All Samples)")

    def num(x):
        try:
            return float(x or 0)
        except ValueError:
            return 0.0

    # a report with several kernels repeats the function / header rows: sum the numeric ones
    data = [r for r in rows[2:] if len(r) == len(h) and r[ia] != h[ia]]
    tot = sum(num(r[ia]) for r in data) or 1.0
    return {h[i][6:]: round(100 * sum(num(r[i]) for r in data) / tot, 1) for i in cols}


def main():
    src, tag = sys.argv[1], sys.argv[2]
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    traffic_path = os.path.join(prof, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    kern_path = os.path.join(prof, "ncu_kernels.json")
    kernels = json.load(open(kern_path)) if os.path.exists(kern_path) else {}
    for rep in sorted(glob.glob(os.path.join(src, "full_*.ncu-rep"))):
        name = os.path.basename(rep)[5:-8]
        h, units, data = ncu_raw(rep)
        with open(os.path.join(prof, f"{tag}_ncu_{name}.csv"), "w") as f:
            wr = csv.writer(f)
            wr.writerow(["kernel", "metric", "value", "unit"])
            for row in data:
                kern = row[h.index("Kernel Name")][:80]
                for m in METRICS:
                    if m in h:
                        wr.writerow([kern, m, row[h.index(m)], units[h.index(m)]])
            for k, v in stall_summary(rep).items():
                wr.writerow([kern, f"stall_pct.{k}", v, "%"])
        row = data[0]
        rd = float(row[h.index("dram__bytes_read.sum")]) * SCALE.get(units[h.index("dram__bytes_read.sum")], 1)
        wb = float(row[h.index("dram__bytes_write.sum")]) * SCALE.get(units[h.index("dram__bytes_write.sum")], 1)
        key = name
        ent = {"kernel": row[h.index("Kernel Name")][:60], "dram_bytes_per_launch": rd + wb,
               "source": f"profiles/{tag}_ncu_{name}.csv"}
        if name == "c4":  # tools/gpu_evidence*.sh captures c4 on 1e7 points; bench c4 runs 1e8
            key = "c4_1e7pts"
            ent["note"] = "captured on a 1e7-point launch (bench c4 uses 1e8); not used as the bench traffic"
        traffic[key] = ent
        print(f"{name}: {rd + wb:.3e} DRAM bytes per launch")

        def num(m):
            return float(row[h.index(m)]) if m in h and row[h.index(m)] not in ("", "n/a") else None
        kernels[name] = {
            "kernel": row[h.index("Kernel Name")][:60], "source": f"profiles/{tag}_ncu_{name}.csv",
            "duration_ms": num("gpu__time_duration.sum") * (1e-3 if units[h.index("gpu__time_duration.sum")] == "us"
                                                             else 1.0),
            "inst_per_launch": num("smsp__inst_executed.sum"), "dram_bytes_per_launch": rd + wb,
            "ipc": num("sm__inst_executed.avg.per_cycle_active"),
            "alu_pct": num("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "fma_pct": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "fp64_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "lsu_pct": num("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
            "lts_pct": num("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "dram_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
        }
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    json.dump(kernels, open(kern_path, "w"), indent=1, sort_keys=True)
    for lc in sorted(glob.glob(os.path.join(src, "launches_*.csv"))):
        summarize_launches(lc, os.path.join(prof, f"{tag}_{os.path.basename(lc)}"))
    write_bench(src, prof, tag)


def summarize_launches(lc, dst):
    if os.path.exists(lc):
        lines = [ln for ln in open(lc) if not ln.startswith("==")]
        rows = list(csv.reader(lines))
        h = rows[0]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        per = {}
        for r in rows[1:]:
            k = r[ki].split("(")[0].replace("void ", "")[:60]
            if "fp64_probe" in k or "at::" in k:
                continue  # bench's roofline probe / torch fills: outside the timed steps
            per.setdefault(k, [0, 0.0])
            per[k][0] += 1
            per[k][1] += float(r[vi])
        tot = sum(v[1] for v in per.values())
        with open(dst, "w") as f:
            wr = csv.writer(f)
            wr.writerow(["kernel", "launches", "total_ns", "share"])
            for k, (n, ns) in sorted(per.items(), key=lambda x: -x[1][1]):
                wr.writerow([k, n, int(ns), f"{ns / tot:.4f}"])


def write_bench(src, prof, tag):
    with open(os.path.join(prof, f"{tag}_bench.jsonl"), "w") as f:
        for b in sorted(glob.glob(os.path.join(src, "bench_*.json"))):
            txt = open(b).read().strip().splitlines()
            if txt:
                d = json.loads(txt[-1])
                d["_file"] = os.path.basename(b)
                f.write(json.dumps(d) + "\n")


if __name__ == "__main__":
    main()
