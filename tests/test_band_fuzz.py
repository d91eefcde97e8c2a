"""Band-targeted fuzz (GPU): >= 1e8 points placed where the fast path's
certificates are tight, each compared bit-exactly against BOTH the C
restatement of the reference (oracle/build/libpip_oracle.so, all host threads,
pinned to the unmodified reference in test_oracle.py) and the literal GPU loop
(PC_OPT_EXACT).

Points sit at local side values of ±(1/4 .. 4) fp32 bands (2^-20, DESIGN.md
§3.4) from random edges, 10% of them exactly on a vertex's y-level (filter-key
ties), over random stars, a lon/lat star near (0°, 5.5°), a fractal star, the
c3 footprints and the c5 integer grids; Robust mode additionally at
±(0.5 .. 2) tol from edges for tol = 1e-12 (the default) and coarser
tolerances.  Point budget per mode (C1 / C2 / Robust-band): 5.5e7 single-polygon
+ 4.2e7 CSR = 9.7e7, plus 3.2e7 Robust ±tol points, i.e. > 1e8 in all.
"""
import os

import numpy as np
import pytest

import band_fuzz as BF
import oracle
from paper_2306_04316_b200 import Engine
from paper_2306_04316_b200 import workloads as W
from paper_2306_04316_b200.engine import Polygon

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 8
MODES = (0, 1, 2)


@pytest.fixture(scope="module")
def exact_engine():
    eng = Engine(devices=[0])
    eng.set_exact(True)
    yield eng
    eng.close()


def lonlat_star(n, seed):
    p = W.star_polygon(n, seed)
    # ~0.05 degree footprint around (0, 5.5): lon/lat cancellation in p - a
    return Polygon(p.vx * 0.05, 5.5 + p.vy * 0.05)


SINGLE_CASES = {
    # name: (polygon builder, n points, seed)
    "star64": (lambda: W.star_polygon(64, 11), 20_000_000, 101),
    "star1000": (lambda: W.star_polygon(1000, 12), 20_000_000, 102),
    "lonlat1000": (lambda: lonlat_star(1000, 13), 10_000_000, 103),
    "fractal20k": (lambda: W.fractal_polygon(20_000, 14), 5_000_000, 104),
}


def single_points(name, tol=None):
    build, n, seed = SINGLE_CASES[name]
    poly = build()
    a, b = BF.edge_list(poly.vx, poly.vy, poly.ring_off)
    rng = np.random.default_rng(seed + (0 if tol is None else 7))
    xy = BF.near_edge_points(poly.vx, poly.vy, a, b, BF.bbox_of(poly.vx, poly.vy, poly.ring_off), n, rng, tol)
    return poly, xy


def _cmp(tag, got, want_v, want_s, ref_bits):
    from paper_2306_04316_b200.engine import verdicts_to_bits
    # got: fast Result (bits); want_v/want_s: port oracle; ref_bits: exact Result
    mode = tag[1]
    ib, ab = verdicts_to_bits(want_v, mode)
    bad_o = int(np.count_nonzero(got.inside_bits != ib)) + int(np.count_nonzero(got.aux_bits != ab))
    bad_x = int(np.count_nonzero(got.inside_bits != ref_bits.inside_bits)) + int(
        np.count_nonzero(got.aux_bits != ref_bits.aux_bits))
    assert bad_o == 0, f"{tag}: {bad_o} words differ from the oracle"
    assert bad_x == 0, f"{tag}: {bad_x} words differ from the exact GPU loop"
    assert np.array_equal(got.stats, want_s), tag


@pytest.mark.parametrize("name", sorted(SINGLE_CASES))
@pytest.mark.parametrize("mode", MODES)
def test_band_single(engine, exact_engine, name, mode):
    poly, xy = single_points(name)
    got = engine.classify(xy, poly, mode, verdicts=False)
    ex = exact_engine.classify(xy, poly, mode, verdicts=False)
    want_v, want_s = oracle.port_classify(xy, poly.vx, poly.vy, poly.ring_off, mode, threads=THREADS)
    _cmp((name, mode), got, want_v, want_s, ex)


@pytest.mark.parametrize("name,tol", [("star1000", 1e-12), ("star1000", 1e-6), ("lonlat1000", 1e-12),
                                      ("lonlat1000", 1e-9), ("star64", 1e-3)])
def test_band_robust_tol(engine, exact_engine, name, tol):
    poly, xy = single_points(name, tol=tol)
    xy = xy[:4_000_000]
    got = engine.classify(xy, poly, 2, tol, verdicts=False)
    ex = exact_engine.classify(xy, poly, 2, tol, verdicts=False)
    want_v, want_s = oracle.port_classify(xy, poly.vx, poly.vy, poly.ring_off, 2, tol, threads=THREADS)
    _cmp((name, 2, tol), got, want_v, want_s, ex)


CSR_CASES = {
    "footprints": (lambda: W.footprints(1_000_000, seed=21, pts_per_poly=0), 32, 201),
    "grids": (lambda: W.degenerate(200_000, seed=22), 50, 202),
}


def csr_points(name, tol=None):
    build, per, seed = CSR_CASES[name]
    s = build()
    return BF.csr_near_edge(s, per, np.random.default_rng(seed + (0 if tol is None else 7)), tol)


@pytest.mark.parametrize("name", sorted(CSR_CASES))
@pytest.mark.parametrize("mode", MODES)
def test_band_csr(engine, exact_engine, name, mode):
    s = csr_points(name)
    got = engine.classify_csr(s, mode, verdicts=False)
    ex = exact_engine.classify_csr(s, mode, verdicts=False)
    want_v, want_s = oracle.port_classify_csr(s, mode, threads=THREADS)
    _cmp((name, mode), got, want_v, want_s, ex)


@pytest.mark.parametrize("tol", [1e-12, 1e-9])
def test_band_csr_robust_tol(engine, exact_engine, tol):
    s = csr_points("footprints", tol=tol)
    got = engine.classify_csr(s, 2, tol, verdicts=False)
    ex = exact_engine.classify_csr(s, 2, tol, verdicts=False)
    want_v, want_s = oracle.port_classify_csr(s, 2, tol, threads=THREADS)
    _cmp(("footprints", 2, tol), got, want_v, want_s, ex)
