"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel.
usage: python tools/launch_summary.py <launches.csv> [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg, cnt = collections.OrderedDict(), collections.Counter()
for r in rows[i + 1:]:
    if len(r) > vi:
        k = r[ki][:100]
        agg[k] = agg.get(k, 0.0) + float(r[vi].replace(",", ""))
        cnt[k] += 1
tot = sum(agg.values())
print(f"{sys.argv[1]}: total {tot / 1e3:.1f} us over {sum(cnt.values())} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"  {v / 1e3:9.1f} us {100 * v / tot:5.1f}% x{cnt[k]:<4d} {k}")
