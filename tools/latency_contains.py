"""Latency of the drop-in single-point calls (contains / count_crossings) through
the C-ABI: mean microseconds per call over a warm loop (polygon cached on the
device by content after the first call)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_04316_b200 import Engine  # noqa: E402
from paper_2306_04316_b200 import workloads as W  # noqa: E402

eng = Engine(devices=[0])
out = {}
for nv in (4, 1000, 100_000):
    poly = W.star_polygon(nv)
    pts = W.uniform_points(2000, W.bounds(poly), 3)
    for mode in (0, 1, 2):
        eng.contains(pts[0], poly, mode)
        t0 = time.perf_counter()
        for p in pts:
            try:
                eng.contains(p, poly, mode)
            except Exception:
                pass
        out[f"contains n={nv} mode={mode}"] = (time.perf_counter() - t0) / len(pts) * 1e6
    t0 = time.perf_counter()
    for p in pts[:500]:
        eng.count_crossings(p[None, :], poly.vx, poly.vy, 0)
    out[f"count_crossings_c1 n={nv}"] = (time.perf_counter() - t0) / 500 * 1e6
print(json.dumps({"unit": "us per call", **{k: round(v, 1) for k, v in out.items()}}))
