"""The five BASELINE.json configs as seeded synthetic inputs.

The paper's Google Open Buildings / GADM Ghana data is not
available; these stand in for it with the shapes, sizes and distributions
BASELINE.json names.  Generation runs in libpolycast_workloads.so
(std::mt19937_64, the reference's 53-bit mapping), so a (config, seed) pair
yields identical bytes on every machine with this image.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native
from .engine import CsrSet, Polygon

SEED = 20230607  # arXiv 2306.04316
SWEEP_N = (10, 100, 1000, 10_000, 100_000, 1_000_000)


def _p(a):
    return a.ctypes.data


def star_polygon(n: int, seed: int = SEED, rmin=0.5, rmax=1.0) -> Polygon:
    """c1/c2: vertex k at angle 2*pi*k/n, radius uniform in [rmin, rmax]; closed ring."""
    vx = np.empty(n + 1, np.float64)
    vy = np.empty(n + 1, np.float64)
    _native.workloads_lib().wl_star(n, seed, rmin, rmax, _p(vx), _p(vy))
    return Polygon(vx, vy)


def fractal_polygon(n: int = 200_000, seed: int = SEED, amp: float = 0.2, terms: int = 128, threads=0) -> Polygon:
    """c4: star polygon with 1/f-noise radius 1 + amp*nu(theta), simple (r > 0)."""
    vx = np.empty(n + 1, np.float64)
    vy = np.empty(n + 1, np.float64)
    _native.workloads_lib().wl_fractal_star(n, seed, amp, terms, _p(vx), _p(vy), threads)
    return Polygon(vx, vy)


def uniform_points(n: int, box, seed: int, threads=0) -> np.ndarray:
    xy = np.empty((n, 2), np.float64)
    x0, y0, x1, y1 = box
    _native.workloads_lib().wl_uniform_points(n, x0, y0, x1, y1, seed, _p(xy), threads)
    return xy


def uniform_points_range(lo: int, hi: int, box, seed: int, threads=0) -> np.ndarray:
    """Points [lo, hi) of uniform_points(n, box, seed) for any n >= hi (one rank's shard)."""
    xy = np.empty((max(hi - lo, 0), 2), np.float64)
    x0, y0, x1, y1 = box
    _native.workloads_lib().wl_uniform_points_range(lo, hi, x0, y0, x1, y1, seed, _p(xy), threads)
    return xy


def bounds(poly: Polygon):
    """Tight box of the outer ring (== bbox_of)."""
    b = np.empty(4, np.float64)
    nv = int(poly.ring_off[1])
    _native.workloads_lib().wl_bounds(_p(poly.vx), _p(poly.vy), nv, _p(b))
    return tuple(float(v) for v in b)


def _csr(kind: int, n_polys: int, seed: int, pts_per_poly: int, allow_dups: bool, threads=0) -> CsrSet:
    lib = _native.workloads_lib()
    h = lib.wl_csr_new(kind, n_polys, seed, pts_per_poly, int(allow_dups), threads)
    try:
        np_, nr, nv, npt = (C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64())
        lib.wl_csr_sizes(h, C.byref(np_), C.byref(nr), C.byref(nv), C.byref(npt))
        vx = np.empty(nv.value, np.float64)
        vy = np.empty(nv.value, np.float64)
        ring_off = np.empty(nr.value + 1, np.uint64)
        poly_ring_off = np.empty(np_.value + 1, np.uint64)
        xy = np.empty((npt.value, 2), np.float64)
        pt_off = np.empty(np_.value + 1, np.uint64)
        lib.wl_csr_copy(h, _p(vx), _p(vy), _p(ring_off), _p(poly_ring_off), _p(xy), _p(pt_off))
    finally:
        lib.wl_csr_free(h)
    return CsrSet(xy, pt_off, vx, vy, ring_off, poly_ring_off)


def footprints(n_polys: int = 1_000_000, seed: int = SEED, pts_per_poly: int = 64, threads=0) -> CsrSet:
    """c3: rotated rectangles / L- and staircase shapes (4-16 vertices, sides
    10-50 m) in lon/lat degrees around (0, 5.5); 64 points each (half uniform in
    the bbox, half within +-5 m of a vertex); CSR by polygon id."""
    return _csr(3, n_polys, seed, pts_per_poly, False, threads)


def degenerate(n_polys: int = 100_000, seed: int = SEED, allow_dups: bool = True, threads=0) -> CsrSet:
    """c5: integer-grid polygons (4-64 vertices: horizontal edges, collinear and
    duplicate consecutive vertices, concave notches, optional hole); ~100 points
    each, half exactly on vertices/edges/vertex y-levels, half uniform."""
    return _csr(5, n_polys, seed, 0, allow_dups, threads)


# ---- the configs by name ---------------------------------------------------

def config1(seed=SEED):
    """c1: star n=1000, 1e6 points uniform in [-1,1]^2."""
    poly = star_polygon(1000, seed)
    return poly, uniform_points(1_000_000, (-1.0, -1.0, 1.0, 1.0), seed + 1)


def config2(n: int, seed=SEED, n_points=1_000_000):
    """c2: star polygon with n vertices, 1e6 points uniform in its bounding box."""
    poly = star_polygon(n, seed)
    return poly, uniform_points(n_points, bounds(poly), seed + 2 + n)


def config4(seed=SEED, n_points=100_000_000, threads=0, shard=None):
    """c4: 200,000-vertex fractal star, 1e8 points uniform in its bbox;
    shard = (lo, hi) generates only points [lo, hi) of the same sequence."""
    poly = fractal_polygon(200_000, seed, threads=threads)
    if shard is not None:
        return poly, uniform_points_range(shard[0], shard[1], bounds(poly), seed + 4, threads)
    return poly, uniform_points(n_points, bounds(poly), seed + 4, threads)
