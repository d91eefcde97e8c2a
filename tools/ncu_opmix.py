"""Executed warp instructions per SASS opcode (first mnemonic token) of an ncu
report's SASS source page: python tools/ncu_opmix.py report.ncu-rep [units]"""
import csv
import collections
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
ie = hdr.index("Instructions Executed")
agg = collections.Counter()
for r in rows:
    if len(r) <= ie or not r[0].startswith("0x"):
        continue
    s = r[1].strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1] if " " in s else s
    op = s.split()[0].rstrip(";") if s else "?"
    agg[op] += int(r[ie] or 0)
tot = sum(agg.values()) or 1
print(f"total {tot:.4g} ({tot / units:.1f} per unit)")
for op, n in agg.most_common(45):
    print(f"{n / units:9.2f} {100 * n / tot:5.1f}%  {op}")
