"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel family and mode -- the single-polygon scan (key scan
+ candidate flushes, bucketed by the radix sort and unbucketed, prefilter on /
off), the literal exact path (PC_OPT_EXACT), the small-call kernel (contains,
count_crossings), the CSR tile kernel with oversize polygons deferred to the
warp kernel, the opt-in segment tree, multi-shard contexts, prefilter_bbox /
scatter_verdicts and the CSV reader / writer.  Every result is checked against
the C restatement (test infrastructure); exits non-zero on a mismatch."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import adversarial  # noqa: E402
import oracle  # noqa: E402
from paper_2306_04316_b200 import Engine  # noqa: E402
from paper_2306_04316_b200 import workloads as W  # noqa: E402
from paper_2306_04316_b200.engine import CsrSet, Polygon  # noqa: E402

bad = 0


def same(tag, got, want):
    global bad
    if not np.array_equal(got, want):
        bad += 1
        print("MISMATCH", tag, int((np.asarray(got) != np.asarray(want)).sum()))


def big_csr():
    """A CSR set mixing footprints with a few >96-vertex polygons (deferred to pip_csr_warp_kernel)."""
    s = W.footprints(200, seed=5)
    stars = [W.star_polygon(n, seed=k) for k, n in enumerate((150, 400))]
    vx, vy, ro, pro = [s.vx], [s.vy], list(s.ring_off), list(s.poly_ring_off)
    xy, pt_off = [s.xy], list(s.pt_off)
    for k, p in enumerate(stars):
        base = ro[-1]
        vx.append(p.vx)
        vy.append(p.vy)
        ro.append(base + len(p.vx))
        pro.append(pro[-1] + 1)
        pts = W.uniform_points(300, W.bounds(p), 11 + k)
        xy.append(pts)
        pt_off.append(pt_off[-1] + len(pts))
    return CsrSet(np.concatenate(xy), np.array(pt_off, np.uint64), np.concatenate(vx), np.concatenate(vy),
                  np.array(ro, np.uint64), np.array(pro, np.uint64))


with Engine(devices=[0]) as eng, Engine(devices=[0, 0]) as eng2:
    # the scan: bucketed / unbucketed, many candidates per CTA (flushes), prefilter on / off
    for poly, xy in (W.config2(300, n_points=9_001), W.config2(5000, n_points=12_345),
                     (W.fractal_polygon(20_000, seed=3), W.uniform_points(20_000, (-1.3, -1.3, 1.3, 1.3), 4))):
        for bucket in (0, 1):
            eng.set_bucketing(bucket)
            for mode in (0, 1, 2):
                for pre in (True, False):
                    r = eng.classify(xy, poly, mode, prefilter=pre)
                    w, _ = oracle.port_classify(xy, poly.vx, poly.vy, poly.ring_off, mode, prefilter=pre, threads=8)
                    same(("scan", len(poly.vx), bucket, mode, pre), r.verdicts, w)
    eng.set_bucketing(-1)
    # adversarial cases through a 2-shard context
    for name, p, pts in adversarial.cases()[:8]:
        for mode in (0, 1, 2):
            r = eng2.classify(pts, p, mode)
            w, _ = oracle.port_classify(pts, p.vx, p.vy, p.ring_off, mode)
            same(("adv", name, mode), r.verdicts, w)
    # small calls: contains-sized batches and count_crossings (small and large n)
    poly, xy = W.config2(1000, n_points=5000)
    for mode in (0, 1, 2):
        r = eng.classify(xy[:700], poly, mode)
        w, _ = oracle.port_classify(xy[:700], poly.vx, poly.vy, poly.ring_off, mode)
        same(("small", mode), r.verdicts, w)
    for n in (300, 5000):
        for mode in (0, 1):
            c, d = eng.count_crossings(xy[:n], poly.vx, poly.vy, mode)
            wc, wd = oracle.port_count_crossings(xy[:n], poly.vx, poly.vy, mode)
            same(("count", n, mode), d, wd)
            same(("count", n, mode), c[wd == 0], wc[wd == 0])
    # CSR: footprints + oversize polygons; degenerate grids with duplicates (2 shards)
    for s, e in ((big_csr(), eng), (W.degenerate(300, seed=3), eng2)):
        for mode in (0, 1, 2):
            r = e.classify_csr(s, mode)
            w, _ = oracle.port_classify_csr(s, mode, threads=8)
            same(("csr", s.n_polys, mode), r.verdicts, w)
    # the literal exact path
    eng.set_exact(True)
    poly, xy = W.config2(300, n_points=9_001)
    for mode in (0, 1, 2):
        r = eng.classify(xy, poly, mode)
        w, _ = oracle.port_classify(xy, poly.vx, poly.vy, poly.ring_off, mode)
        same(("exact", mode), r.verdicts, w)
        s = W.degenerate(200, seed=4)
        r = eng.classify_csr(s, mode)
        w, _ = oracle.port_classify_csr(s, mode)
        same(("exact csr", mode), r.verdicts, w)
    eng.set_exact(False)
    # the opt-in segment tree
    eng.set_tree(1)
    poly, xy = W.config2(6000, n_points=30_000)
    for mode in (0, 1):
        r = eng.classify(xy, poly, mode)
        w, _ = oracle.port_classify(xy, poly.vx, poly.vy, poly.ring_off, mode, threads=8)
        same(("tree", mode), r.verdicts, w)
    eng.set_tree(0)
    # prefilter_bbox / scatter_verdicts
    box = (-0.5, -0.5, 0.6, 0.7)
    pts, idx, _ = eng.prefilter_bbox(xy[:20_000], box)
    inb = (xy[:20_000, 0] >= box[0]) & (xy[:20_000, 0] <= box[2]) & (xy[:20_000, 1] >= box[1]) & (xy[:20_000, 1] <= box[3])
    same(("prefilter",), idx, np.nonzero(inb)[0].astype(idx.dtype))
    v = np.arange(len(idx), dtype=np.uint8) % 4
    out = eng.scatter_verdicts(idx, v, 20_000)
    ref = np.full(20_000, 1, np.uint8)
    ref[idx.astype(np.int64)] = v
    same(("scatter",), out, ref)
    # CSV reader / writer
    lines = "".join(f"{i},{float(x)!r},{float(y)!r}\n" for i, (x, y) in enumerate(xy[:3000]))
    text = ("id,lon,lat\n" + lines).encode()
    got = eng.parse_points_csv(text, len("id,lon,lat\n"), 1, 2)[0]
    same(("csv",), got.reshape(-1, 2), xy[:3000])
    from paper_2306_04316_b200.engine import make_records
    recs = make_records(np.arange(3000, dtype=np.uint64), xy[:3000], np.zeros(3000, np.uint8))
    txt = eng.format_results_csv(recs)
    same(("emit rows",), np.array([bytes(txt).count(b"\n")]), np.array([3001]))
print("sanitize cases:", "OK" if bad == 0 else f"{bad} mismatches")
sys.exit(1 if bad else 0)
