"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck): every
kernel family, every mode, bucketed and unbucketed, CSR with oversize
polygons, count_crossings, multi-shard.  Exits non-zero on a parity failure."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import adversarial  # noqa: E402
import oracle  # noqa: E402
from paper_2306_04316_b200 import Engine  # noqa: E402
from paper_2306_04316_b200 import workloads as W  # noqa: E402

bad = 0
with Engine(devices=[0]) as eng, Engine(devices=[0, 0]) as eng2:
    poly, xy = W.config2(300, n_points=9_001)
    for bucket in (0, 1):
        eng.set_bucketing(bucket)
        for mode in (0, 1, 2):
            for pre in (True, False):
                r = eng.classify(xy, poly, mode, prefilter=pre)
                w, _ = oracle.port_classify(xy, poly.vx, poly.vy, poly.ring_off, mode, prefilter=pre)
                bad += int(not np.array_equal(r.verdicts, w))
    eng.set_bucketing(-1)
    for name, p, pts in adversarial.cases()[:6]:
        for mode in (0, 1, 2):
            r = eng2.classify(pts, p, mode)
            w, _ = oracle.port_classify(pts, p.vx, p.vy, p.ring_off, mode)
            bad += int(not np.array_equal(r.verdicts, w))
    s = W.degenerate(300, seed=3)
    for mode in (0, 1, 2):
        r = eng2.classify_csr(s, mode)
        w, _ = oracle.port_classify_csr(s, mode)
        bad += int(not np.array_equal(r.verdicts, w))
    big = W.star_polygon(2000, seed=3)
    c, d = eng.count_crossings(xy[:500], big.vx, big.vy, 0)
    wc, _ = oracle.port_count_crossings(xy[:500], big.vx, big.vy, 0)
    bad += int(not np.array_equal(c, wc))
print("sanitize cases:", "OK" if bad == 0 else f"{bad} mismatches")
sys.exit(1 if bad else 0)
