"""Per-source-line executed warp instructions (and stall samples) of an ncu report:
python tools/ncu_lineprof.py report.ncu-rep [divisor] [min_per_unit]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
mn = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
f = None
cur = None
seen = set()
agg = {}
stall = {}
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 7 and r[0] not in ("", "Line No"):
        cur = (f, int(r[0]), r[1][:80])
    elif len(r) > 7 and r[0] == "" and r[2].startswith("0x"):
        a = int(r[2], 16)
        if a in seen:
            continue
        seen.add(a)
        n = int(r[7]) if r[7] not in ("-", "") else 0
        agg[cur] = agg.get(cur, 0) + n
        stall[cur] = stall.get(cur, 0) + (int(r[4]) if r[4] not in ("-", "") else 0)
tot = sum(agg.values())
st = sum(stall.values())
print(f"total warp instructions {tot:.0f} = {tot / div:.1f} per unit; stall samples {st}")
for k in sorted(agg, key=lambda k: (k[0], k[1])):
    if agg[k] / div >= mn or stall[k] > 0.01 * st:
        print(f"{agg[k] / div:8.2f} {100.0 * stall[k] / max(st, 1):5.1f}%  {k[0]}:{k[1]}  {k[2]}")
