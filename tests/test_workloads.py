"""CPU tests of the seeded workload generators."""
import numpy as np

from paper_2306_04316_b200 import workloads as W


def test_star_polygon_shape_and_determinism():
    a = W.star_polygon(1000)
    b = W.star_polygon(1000)
    assert np.array_equal(a.vx, b.vx) and len(a.vx) == 1001
    assert a.vx[0] == a.vx[-1] and a.vy[0] == a.vy[-1]
    r = np.hypot(a.vx[:-1], a.vy[:-1])
    assert r.min() >= 0.5 - 1e-12 and r.max() <= 1.0 + 1e-12
    th = np.arctan2(a.vy[:-1], a.vx[:-1]) % (2 * np.pi)
    assert np.allclose(np.sort(th), th, atol=1e-9)  # sorted angles


def test_points_chunked_determinism_independent_of_threads():
    a = W.uniform_points(3_000_000, (-1, -2, 1, 2), 5, threads=1)
    b = W.uniform_points(3_000_000, (-1, -2, 1, 2), 5, threads=7)
    assert np.array_equal(a, b)
    assert a[:, 0].min() >= -1 and a[:, 0].max() < 1 and a[:, 1].min() >= -2


def test_fractal_polygon_simple_star():
    p = W.fractal_polygon(20_000)
    r = np.hypot(p.vx[:-1], p.vy[:-1])
    assert r.min() >= 0.8 - 1e-9 and r.max() <= 1.2 + 1e-9


def test_footprints_layout():
    s = W.footprints(5000)
    assert s.n_polys == 5000 and s.n_points == 5000 * 64
    assert np.array_equal(s.pt_off, np.arange(5001, dtype=np.uint64) * 64)
    nv = np.diff(s.ring_off.astype(np.int64))
    assert nv.min() >= 5 and nv.max() <= 17  # 4..16 distinct + closing vertex
    assert set(np.unique(nv)) <= {5, 7, 9, 11, 13, 15, 17}
    assert 5.0 - 0.01 < s.vy.min() and s.vy.max() < 6.0 + 0.01
    assert -0.51 < s.vx.min() and s.vx.max() < 0.51


def test_degenerate_layout():
    s = W.degenerate(4000, allow_dups=True)
    nv = np.diff(s.ring_off.astype(np.int64))
    assert nv.min() >= 5 and nv.max() <= 65
    assert np.all(s.vx == np.round(s.vx * 2) / 2)  # grid coordinates
    dup = (np.diff(s.vx) == 0) & (np.diff(s.vy) == 0)
    assert dup.sum() > 100  # consecutive duplicates present (P8)
    assert (np.diff(s.poly_ring_off.astype(np.int64)) == 2).sum() > 50  # some polygons with holes
    s2 = W.degenerate(4000, allow_dups=False)
    starts = s2.ring_off[:-1].astype(np.int64)
    ends = s2.ring_off[1:].astype(np.int64)
    for a, b in zip(starts[:500], ends[:500]):
        x, y = s2.vx[a:b], s2.vy[a:b]
        assert not np.any((np.diff(x) == 0) & (np.diff(y) == 0))
