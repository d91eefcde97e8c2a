"""Per CUDA source line: instructions executed and stall samples of one ncu report.
usage: python tools/ncu_lines.py <report.ncu-rep> [units] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, rows, hdr = "", [], None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0] and len(r) >= len(hdr) - 2:
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            rows.append((int(r[ie] or 0), int(r[ss] or 0), f"{fname}:{r[0]}", r[1][:80]))
        except ValueError:
            pass
tot = sum(x[0] for x in rows) or 1
st = sum(x[1] for x in rows) or 1
print(f"total instructions {tot:.4g} ({tot / units:.1f} per unit), stall samples {st}")
for ie, ss, loc, src in sorted(rows, key=lambda x: -x[0])[:top]:
    print(f"{ie / units:9.1f} {100 * ie / tot:5.1f}% stall {100 * ss / st:5.1f}%  {loc:28s} {src}")
