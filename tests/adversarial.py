"""Hand-built edge-case inputs shared by the CPU oracle tests, the golden
fixture generator and the GPU parity tests.  Each case is (name, Polygon,
points (n,2) float64).  They target SURVEY §8 parity rules P2-P8: vertices and
edges on the ray, horizontal edges, bbox boundaries, product underflow and
overflow in the straddle test, signed zeros, holes, and (P8) duplicate
consecutive vertices."""
from __future__ import annotations

import numpy as np

from paper_2306_04316_b200.engine import Polygon

SQUARE = [(0, 0), (1, 0), (1, 1), (0, 1), (0, 0)]
DIAMOND = [(0, 0), (2, 2), (4, 0), (2, -2), (0, 0)]


def _grid_points(x0, x1, y0, y1, k):
    xs = np.linspace(x0, x1, k)
    ys = np.linspace(y0, y1, k)
    X, Y = np.meshgrid(xs, ys)
    return np.stack([X.ravel(), Y.ravel()], 1)


def _special_points(poly: Polygon, rng, n_rand=512):
    """Vertices, edge midpoints, vertex y-levels with various x, bbox corners, random."""
    with np.errstate(all="ignore"):
        return _special_points_impl(poly, rng, n_rand)


def _special_points_impl(poly: Polygon, rng, n_rand):
    vx, vy = poly.vx, poly.vy
    pts = [np.stack([vx, vy], 1)]
    mid = np.stack([(vx[:-1] + vx[1:]) / 2, (vy[:-1] + vy[1:]) / 2], 1)
    pts.append(mid)
    x0, x1 = vx.min(), vx.max()
    y0, y1 = vy.min(), vy.max()
    with np.errstate(over="ignore"):
        w = x1 - x0 if np.isfinite(x1 - x0) else max(abs(x0), abs(x1))
    w = max(w, 1e-300)
    for y in np.unique(vy):
        pts.append(np.array([[x0 - w, y], [x0, y], [(x0 + x1) / 2, y], [x1, y], [x1 + w, y]]))
    pts.append(np.array([[x0, y0], [x0, y1], [x1, y0], [x1, y1]]))
    cx, hx = x0 / 2 + x1 / 2, (x1 / 2 - x0 / 2) * 1.2
    cy, hy = y0 / 2 + y1 / 2, (y1 / 2 - y0 / 2) * 1.2
    pts.append(np.stack([cx + hx * rng.uniform(-1, 1, n_rand), cy + hy * rng.uniform(-1, 1, n_rand)], 1))
    with np.errstate(over="ignore", invalid="ignore"):
        out = np.concatenate(pts)
    return np.ascontiguousarray(np.clip(out, -1.79e308, 1.79e308), dtype=np.float64)


def cases(include_dups: bool = True):
    rng = np.random.default_rng(2306)
    out = []
    sq = Polygon.from_rings([SQUARE])
    out.append(("unit_square_grid", sq, _grid_points(-1, 2, -1, 2, 25)))
    out.append(("unit_square_special", sq, _special_points(sq, rng)))
    dm = Polygon.from_rings([DIAMOND])
    out.append(("diamond", dm, _special_points(dm, rng)))
    hole = [(0.25, 0.25), (0.75, 0.25), (0.75, 0.75), (0.25, 0.75), (0.25, 0.25)]
    holed = Polygon.from_rings([SQUARE, hole])
    out.append(("square_with_hole", holed, _special_points(holed, rng)))
    # integer-grid comb with horizontal runs and collinear vertices
    comb = [(0, 0), (6, 0), (6, 3), (5, 3), (5, 1), (4, 1), (4, 3), (2, 3), (2, 1), (1, 1), (1, 3), (0, 3),
            (0, 2), (0, 0)]
    cp = Polygon.from_rings([comb])
    out.append(("comb", cp, _special_points(cp, rng, 2048)))
    # product underflow (P4): all y around 1e-300 -> f_prev*f_next underflows to 0
    tiny = np.array(SQUARE, np.float64) * 1e-300 + np.array([0.0, 2e-300])
    tp = Polygon.from_rings([tiny])
    pts = _special_points(tp, rng)
    pts = np.concatenate([pts, np.stack([rng.uniform(-1e-300, 2e-300, 256), rng.uniform(1e-300, 4e-300, 256)], 1),
                          np.array([[0.5e-300, 0.0], [0.5e-300, 5e-324], [0.5e-300, -5e-324]])])
    out.append(("tiny_underflow", tp, np.ascontiguousarray(pts)))
    # subnormal coordinates
    sub = np.array(SQUARE, np.float64) * 4e-323
    sp = Polygon.from_rings([sub])
    out.append(("subnormal", sp, _special_points(sp, rng)))
    # overflow (P4): |coords| ~ 1e308, differences overflow to inf
    huge = np.array([(-1, -1), (1, -1), (1, 1), (-1, 1), (-1, -1)], np.float64) * 1.5e308
    hp = Polygon.from_rings([huge])
    hpts = _special_points(hp, rng)
    hpts = np.concatenate([hpts, np.array([[0.0, 0.0], [1e308, -1.7e308], [-1.7e308, 1.5e308], [0.0, 1.5e308]])])
    out.append(("huge_overflow", hp, np.ascontiguousarray(np.clip(hpts, -1.79e308, 1.79e308))))
    # signed zeros
    sz = Polygon.from_rings([[(-0.0, -1.0), (1.0, -0.0), (0.0, 1.0), (-1.0, 0.0), (-0.0, -1.0)]])
    zp = np.array([[0.0, 0.0], [-0.0, -0.0], [0.0, -0.0], [-0.0, 0.0], [1.0, 0.0], [1.0, -0.0], [-1.0, -0.0],
                   [0.5, -0.0], [-2.0, 0.0], [-2.0, -0.0]], np.float64)
    out.append(("signed_zero", sz, np.ascontiguousarray(np.concatenate([zp, _special_points(sz, rng)]))))
    # near-degenerate slivers: nearly horizontal edges (tiny dy), nearly collinear
    sl = [(0, 0), (10, 1e-12), (10, 1e-12 + 1e-15), (0, 3e-16), (0, 0)]
    slp = Polygon.from_rings([sl])
    out.append(("sliver", slp, _special_points(slp, rng, 4096)))
    # large coordinates with small extents (lon/lat-like cancellation)
    base = np.array([(0.0, 0.0), (3e-4, 1e-4), (2e-4, 4e-4), (-1e-4, 2e-4), (0.0, 0.0)]) + np.array([179.9999, 5.5])
    bp = Polygon.from_rings([base])
    out.append(("lonlat_small", bp, _special_points(bp, rng, 4096)))
    if include_dups:
        # P8: consecutive duplicate vertices (rejected by the reference Ring)
        dup = [(0, 0), (2, 0), (2, 0), (2, 2), (1, 2), (1, 2), (0, 2), (0, 0)]
        dpp = Polygon.from_rings([dup])
        out.append(("dup_vertices", dpp, _special_points(dpp, rng)))
    return out
