"""Segment-tree C1 / C2 path for single polygons (pip_tree.cu, PC_OPT_TREE) against
the reference, bit-exact: forced on for every input shape (stars of many
sizes, the adversarial cases, points on vertices / vertex y-levels / edges,
overlapping holes and self-intersecting rings -- the verified-order fallback --,
no bbox prefilter), and on vs off on the sweep's large polygons."""
import numpy as np
import pytest

import adversarial
import oracle
from paper_2306_04316_b200 import workloads as W
from paper_2306_04316_b200.engine import Polygon

pytestmark = pytest.mark.gpu
THREADS = 16


MODES = (0, 1)  # C1, C2 (the tree's modes)


def _check(engine, xy, poly, prefilter=True, source=None, modes=MODES):
    for mode in modes:
        _check1(engine, xy, poly, mode, prefilter, source)


def _check1(engine, xy, poly, mode, prefilter, source):
    got = engine.classify(xy, poly, mode, prefilter=prefilter)
    if source is None:
        source = "reference" if prefilter and oracle.ref_available() else "port"
    if source == "reference":
        want_v, want_s = oracle.ref_classify(xy, poly.vx, poly.vy, poly.ring_off, mode)
    else:
        want_v, want_s = oracle.port_classify(xy, poly.vx, poly.vy, poly.ring_off, mode, prefilter=prefilter,
                                              threads=THREADS)
    assert np.array_equal(got.verdicts, want_v), f"{int((got.verdicts != want_v).sum())} of {len(xy)} differ"
    assert np.array_equal(got.stats, want_s)


@pytest.fixture
def tree_on(engine):
    engine.set_tree(1)
    yield engine
    engine.set_tree(-1)


@pytest.mark.parametrize("n", [10, 100, 1000, 20_000])
def test_stars(tree_on, n):
    poly = W.star_polygon(n, seed=n)
    xy = W.uniform_points(60_000, W.bounds(poly), n + 1)
    _check(tree_on, xy, poly)
    _check(tree_on, xy, poly, prefilter=False)


def test_adversarial_cases(tree_on):
    for name, poly, xy in adversarial.cases():
        src = "port" if name == adversarial.cases()[-1][0] else None  # duplicate vertices: the C restatement
        _check(tree_on, np.ascontiguousarray(xy), poly, source=src)


def test_points_on_vertices_levels_and_edges(tree_on):
    poly = W.star_polygon(5000, seed=7)
    rng = np.random.default_rng(8)
    vx, vy = poly.vx, poly.vy
    k = rng.integers(0, len(vx) - 1, 4000)
    t = rng.random(4000)
    on_edge = np.stack([vx[k] + t * (vx[k + 1] - vx[k]), vy[k] + t * (vy[k + 1] - vy[k])], 1)
    levels = np.stack([rng.uniform(-1, 1, 4000), vy[k]], 1)              # exactly on vertex y-levels
    near = levels + np.stack([np.zeros(4000), rng.choice([-1, 1], 4000) * np.spacing(np.abs(levels[:, 1]))], 1)
    verts = np.stack([vx, vy], 1)
    xy = np.ascontiguousarray(np.concatenate([on_edge, levels, near, verts, W.uniform_points(20_000, W.bounds(poly), 9)]))
    _check(tree_on, xy, poly)


def test_vertex_y_clusters(tree_on):
    """Vertices whose y differ below 2^-32 of the polygon's height (the vertex
    keys' radix sort orders the top 32 of their 53 bits and fixes up such runs
    on the full key), with points on, between and just off those y-levels."""
    from paper_2306_04316_b200.engine import Polygon
    rng = np.random.default_rng(21)
    base = W.star_polygon(6000, seed=21)
    vx, vy = base.vx.copy(), base.vy.copy()
    # snap to a coarse grid of levels, then spread inside each level by < 2^-32
    vy[:-1] = np.round(vy[:-1] * 64) / 64 + rng.integers(0, 8, len(vy) - 1) * 1e-12
    vy[-1] = vy[0]
    poly = Polygon(vx, vy, base.ring_off)
    lv = np.unique(vy)
    y = np.concatenate([lv, lv + 5e-13, np.nextafter(lv, np.inf), np.nextafter(lv, -np.inf)])
    xy = np.stack([rng.uniform(-1, 1, len(y)), y], 1)
    xy = np.ascontiguousarray(np.concatenate([xy, W.uniform_points(30_000, W.bounds(poly), 22)]))
    _check(tree_on, xy, poly)


def test_overlapping_holes_and_self_intersections(tree_on):
    rng = np.random.default_rng(12)
    rings = [np.stack([np.cos(t) * 100, np.sin(t) * 100], 1) for t in [np.linspace(0, 2 * np.pi, 3001)]]
    rings[0][-1] = rings[0][0]
    for _ in range(120):  # overlapping square holes: edges cross inside node ranges
        cx, cy = rng.uniform(-60, 60, 2)
        rings.append(np.array([(cx, cy), (cx + 9, cy), (cx + 9, cy + 9), (cx, cy + 9), (cx, cy)]))
    holed = Polygon.from_rings(rings)
    _check(tree_on, W.uniform_points(100_000, (-110, -110, 110, 110), 13), holed)
    # a random-order ring: thousands of crossings
    p = rng.uniform(-1, 1, (2000, 2))
    p = np.concatenate([p, p[:1]])
    tangled = Polygon.from_rings([p])
    _check(tree_on, W.uniform_points(50_000, (-1, -1, 1, 1), 14), tangled)


@pytest.mark.parametrize("n", [100_000, 1_000_000])
def test_sweep_tree_vs_scan(engine, n):
    """Auto mode on the sweep's big polygons: tree and scan paths agree on all
    1e6 points, and a seeded subsample agrees with the reference."""
    poly, xy = W.config2(n)
    for mode in MODES:
        engine.set_tree(1)
        a = engine.classify(xy, poly, mode)
        engine.set_tree(0)
        b = engine.classify(xy, poly, mode)
        engine.set_tree(-1)
        assert np.array_equal(a.verdicts, b.verdicts)
        idx = np.random.default_rng(n).choice(len(xy), 3000, replace=False)
        sub = np.ascontiguousarray(xy[idx])
        want_v, _ = oracle.ref_classify(sub, poly.vx, poly.vy, poly.ring_off, mode)
        assert np.array_equal(a.verdicts[idx], want_v)


def test_fuzz_random_polygons(tree_on):
    """200 random polygons (simple stars, random-order rings, grids with holes,
    integer coordinates for exact ties), each with points on its vertices, its
    vertex y-levels, edge midpoints and uniform points, forced through the tree."""
    rng = np.random.default_rng(77)
    for t in range(200):
        kind = t % 4
        n = int(rng.integers(4, 60))
        if kind == 0:  # star
            ang = np.sort(rng.uniform(0, 2 * np.pi, n))
            r = rng.uniform(0.3, 1.0, n)
            ring = np.stack([r * np.cos(ang), r * np.sin(ang)], 1)
        elif kind == 1:  # random order: self-intersecting
            ring = rng.uniform(-1, 1, (n, 2))
        elif kind == 2:  # integer grid (horizontal edges, ties everywhere)
            ring = rng.integers(-5, 6, (n, 2)).astype(np.float64)
            keep = np.concatenate([[True], np.any(ring[1:] != ring[:-1], axis=1)])
            ring = ring[keep]
            if len(ring) < 3 or np.all(ring[0] == ring[-1]):
                continue
        else:  # tiny extent far from the origin
            ang = np.sort(rng.uniform(0, 2 * np.pi, n))
            ring = np.stack([1e3 + 1e-6 * np.cos(ang), -7.5 + 1e-6 * np.sin(ang)], 1)
        ring = np.concatenate([ring, ring[:1]])
        rings = [ring]
        if kind == 2 and t % 8 == 2:
            rings.append(np.array([[0., 0.], [1., 0.], [1., 1.], [0., 1.], [0., 0.]]))
        poly = Polygon.from_rings(rings)
        vx, vy = poly.vx, poly.vy
        x0, x1, y0, y1 = vx.min(), vx.max(), vy.min(), vy.max()
        pts = [np.stack([vx, vy], 1), np.stack([(vx[:-1] + vx[1:]) / 2, (vy[:-1] + vy[1:]) / 2], 1),
               np.stack([rng.uniform(x0, x1, len(vy)), vy], 1),
               np.stack([rng.uniform(x0, x1, 300), rng.uniform(y0, y1, 300)], 1)]
        xy = np.ascontiguousarray(np.concatenate(pts))
        _check(tree_on, xy, poly, source="port")
