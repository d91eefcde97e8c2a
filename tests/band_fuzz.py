"""Band-targeted inputs for the fast path's certified shortcuts (test helper).

The fast kernels decide a (point, edge) side test in fp32 on polygon-local
coordinates and trust the sign only outside a band |s| <= 2^-20 (DESIGN.md
§3.4); their straddle filters trust keys only off ties.  These generators put
points exactly where those arguments are tight: at local side values of
±(0.25 .. 4) bands from random edges (both sides), on the edges' y-levels, and
at ±(0.5 .. 2) tol from edges for Robust mode.

Local map (pip_device.cuh local_map_from_bbox): L = (v - bbox_min) * s with
s = 2^-e per axis, W = m 2^e, m in [1/2, 1).  For edge a -> b the local normal
is N = (Lb.y - La.y, -(Lb.x - La.x)); a point La + t (Lb - La) + u 2^-20 N/|N|^2
has local side value u 2^-20.
"""
from __future__ import annotations

import numpy as np

BAND = 2.0 ** -20


def _pow2_scale(extent):
    _, e = np.frexp(np.asarray(extent, np.float64))
    return np.ldexp(1.0, -e)


def edge_list(vx, vy, ring_off):
    """(a_idx, b_idx) of every edge (within rings)."""
    a = []
    for r in range(len(ring_off) - 1):
        lo, hi = int(ring_off[r]), int(ring_off[r + 1])
        if hi - lo >= 2:
            a.append(np.arange(lo, hi - 1, dtype=np.int64))
    a = np.concatenate(a) if a else np.zeros(0, np.int64)
    return a, a + 1


def near_edge_points(vx, vy, a, b, bbox, n, rng, tol=None):
    """n points near random edges (a[k] -> b[k]) of one polygon with outer bbox
    (x0, y0, x1, y1): side-band offsets (tol None) or ±(0.5..2) tol offsets."""
    x0, y0, x1, y1 = bbox
    sx, sy = _pow2_scale(x1 - x0), _pow2_scale(y1 - y0)
    k = rng.integers(0, len(a), n)
    ax, ay, bx, by = vx[a[k]], vy[a[k]], vx[b[k]], vy[b[k]]
    t = rng.random(n)
    sign = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    if tol is None:
        # local side value u * 2^-20, |u| log-uniform in [1/4, 4]
        u = sign * np.exp2(rng.uniform(-2.0, 2.0, n))
        lax, lay = (ax - x0) * sx, (ay - y0) * sy
        lbx, lby = (bx - x0) * sx, (by - y0) * sy
        nxl, nyl = lby - lay, -(lbx - lax)
        n2 = nxl * nxl + nyl * nyl
        with np.errstate(divide="ignore", invalid="ignore"):
            off = np.where(n2 > 0, u * BAND / n2, 0.0)
        lpx = lax + t * (lbx - lax) + off * nxl
        lpy = lay + t * (lby - lay) + off * nyl
        px, py = x0 + lpx / sx, y0 + lpy / sy
    else:
        # world distance (0.5 .. 2) tol from the segment, perpendicular
        dx, dy = bx - ax, by - ay
        ln = np.hypot(dx, dy)
        d = sign * tol * rng.uniform(0.5, 2.0, n)
        with np.errstate(divide="ignore", invalid="ignore"):
            ux, uy = np.where(ln > 0, -dy / ln, 0.0), np.where(ln > 0, dx / ln, 0.0)
        px, py = ax + t * dx + d * ux, ay + t * dy + d * uy
    # a share of the points sits exactly on a vertex's y-level (key ties)
    lvl = rng.random(n) < 0.1
    py = np.where(lvl, ay, py)
    return np.stack([px, py], axis=1)


def bbox_of(vx, vy, ring_off):
    lo, hi = int(ring_off[0]), int(ring_off[1])
    return float(vx[lo:hi].min()), float(vy[lo:hi].min()), float(vx[lo:hi].max()), float(vy[lo:hi].max())


def csr_near_edge(s, per_poly, rng, tol=None):
    """A CSR set with the same polygons as s and per_poly near-edge points each."""
    from paper_2306_04316_b200.engine import CsrSet
    P = s.n_polys
    pts = np.empty((P, per_poly, 2), np.float64)
    vx, vy = s.vx, s.vy
    # vectorised over polygons: pick an edge of each polygon's rings uniformly
    r0 = s.poly_ring_off[:-1].astype(np.int64)
    r1 = s.poly_ring_off[1:].astype(np.int64)
    v0 = s.ring_off[r0].astype(np.int64)
    v1 = s.ring_off[r1].astype(np.int64)
    ov1 = s.ring_off[r0 + 1].astype(np.int64)  # outer ring end
    # outer bbox per polygon
    x0 = np.minimum.reduceat(vx, v0)
    x1 = np.maximum.reduceat(vx, v0)
    y0 = np.minimum.reduceat(vy, v0)
    y1 = np.maximum.reduceat(vy, v0)
    # reduceat spans to the next polygon's start: restrict to the outer ring
    # (holes lie inside it for these generators, so the polygon span is the outer box)
    del ov1
    sx, sy = _pow2_scale(x1 - x0), _pow2_scale(y1 - y0)
    for j in range(per_poly):
        # random vertex index in [v0, v1 - 1); edges that cross a ring end are
        # skipped by re-drawing to the previous vertex (a closed ring repeats its first vertex)
        k = v0 + (rng.random(P) * (v1 - v0 - 1)).astype(np.int64)
        ax, ay, bx, by = vx[k], vy[k], vx[k + 1], vy[k + 1]
        t = rng.random(P)
        sign = np.where(rng.random(P) < 0.5, -1.0, 1.0)
        if tol is None:
            u = sign * np.exp2(rng.uniform(-2.0, 2.0, P))
            lax, lay = (ax - x0) * sx, (ay - y0) * sy
            lbx, lby = (bx - x0) * sx, (by - y0) * sy
            nxl, nyl = lby - lay, -(lbx - lax)
            n2 = nxl * nxl + nyl * nyl
            with np.errstate(divide="ignore", invalid="ignore"):
                off = np.where(n2 > 0, u * BAND / n2, 0.0)
            px = x0 + (lax + t * (lbx - lax) + off * nxl) / sx
            py = y0 + (lay + t * (lby - lay) + off * nyl) / sy
        else:
            dx, dy = bx - ax, by - ay
            ln = np.hypot(dx, dy)
            d = sign * tol * rng.uniform(0.5, 2.0, P)
            with np.errstate(divide="ignore", invalid="ignore"):
                ux, uy = np.where(ln > 0, -dy / ln, 0.0), np.where(ln > 0, dx / ln, 0.0)
            px, py = ax + t * dx + d * ux, ay + t * dy + d * uy
        lvl = rng.random(P) < 0.1
        py = np.where(lvl, ay, py)
        pts[:, j, 0] = px
        pts[:, j, 1] = py
    pt_off = (np.arange(P + 1, dtype=np.uint64) * per_poly).astype(np.uint64)
    return CsrSet(pts.reshape(-1, 2), pt_off, s.vx, s.vy, s.ring_off, s.poly_ring_off)
