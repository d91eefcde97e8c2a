"""The reference's acceptance checks 1 and 2 (proj/tests/acceptance/acceptance.cpp
:109-212) through the GPU path, on exactly the reference's inputs: its 50-polygon
corpus (5..500 vertices, convex / star-shaped; :82-99) x 1e5 points each, built by
the reference's own generators, and its independent winding-number oracle
(proj/tests/support/winding_oracle.hpp) -- both through oracle/_ref
(ref_accept_shim.cpp, test infrastructure).  The per-point contains() loop of
the reference becomes one batched contains-semantics call (no bbox
prefilter) per polygon and mode.

Check 1: Robust vs the winding oracle, points either side calls Boundary skipped,
         compared + skipped = 5e6, zero mismatches.
Check 2: off-grid mode agreement: points within 1e-9 of a vertex y skipped, and
         points Robust calls Boundary; C1 and C2 must equal Robust and C2 must not
         raise DegenerateEdge (Error).
"""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2306_04316_b200.engine import Polygon

pytestmark = pytest.mark.gpu
N_POLY, N_PTS = 50, 100_000
INSIDE, OUTSIDE, BOUNDARY, ERROR = 0, 1, 2, 3


@pytest.fixture(scope="module")
def corpus():
    if not oracle.ref_available() or not hasattr(oracle.ref(), "ref_corpus_polygon"):
        pytest.skip("oracle/_ref built without the acceptance shim")
    lib = oracle.ref()
    lib.ref_corpus_polygon.argtypes = [C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64]
    lib.ref_corpus_polygon.restype = C.c_uint64
    lib.ref_corpus_points.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
    lib.ref_winding_oracle.argtypes = [C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p]
    out = []
    for idx in range(N_POLY):
        vx, vy = np.zeros(600), np.zeros(600)
        nv = lib.ref_corpus_polygon(idx, vx.ctypes.data, vy.ctypes.data, 600)
        poly = Polygon(vx[:nv].copy(), vy[:nv].copy())
        xy = np.zeros((N_PTS, 2))
        lib.ref_corpus_points(idx, N_PTS, xy.ctypes.data)
        out.append((idx, poly, xy))
    return lib, out


def test_check1_robust_vs_winding_oracle(engine, corpus):
    lib, polys = corpus
    compared = skipped = mismatches = 0
    for idx, poly, xy in polys:
        robust = engine.classify(xy, poly, 2, prefilter=False, bits=False).verdicts
        want = np.zeros(N_PTS, np.uint8)
        lib.ref_winding_oracle(idx, xy.ctypes.data, N_PTS, want.ctypes.data)
        skip = (robust == BOUNDARY) | (want == BOUNDARY)
        skipped += int(skip.sum())
        compared += int((~skip).sum())
        mismatches += int((robust[~skip] != want[~skip]).sum())
    assert compared + skipped == N_POLY * N_PTS
    assert mismatches == 0, f"robust/oracle mismatches: {mismatches}"


def test_check2_mode_agreement_off_grid(engine, corpus):
    _, polys = corpus
    compared = mismatches = degenerate = 0
    for idx, poly, xy in polys:
        ys = np.sort(poly.vy)
        pos = np.searchsorted(ys, xy[:, 1])
        near = np.zeros(N_PTS, bool)
        for off in (0, -1):  # the lower_bound element and its predecessor (acceptance.cpp:167-172)
            j = np.clip(pos + off, 0, len(ys) - 1)
            ok = (pos + off >= 0) & (pos + off < len(ys))
            near |= ok & (np.abs(ys[j] - xy[:, 1]) <= 1e-9)
        robust = engine.classify(xy, poly, 2, prefilter=False, bits=False).verdicts
        keep = ~near & (robust != BOUNDARY)
        c1 = engine.classify(xy, poly, 0, prefilter=False, bits=False).verdicts
        c2 = engine.classify(xy, poly, 1, prefilter=False, bits=False).verdicts
        compared += int(keep.sum())
        degenerate += int((keep & (c2 == ERROR)).sum())
        ok2 = keep & (c2 != ERROR)
        mismatches += int(((c1 != robust) | (c2 != robust))[ok2].sum())
    assert compared > 0.9 * N_POLY * N_PTS
    assert degenerate == 0, f"DegenerateEdge raised for {degenerate} filtered points"
    assert mismatches == 0, f"mode disagreements: {mismatches}"
