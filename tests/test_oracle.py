"""CPU tests of the checkers: the C restatement (oracle/pip_oracle.c) is pinned
against the reference's own known-answer tests and against the unmodified
reference (oracle/_ref) on every duplicate-free input; both are pinned against
the committed golden vectors (tests/golden/golden_v1.npz)."""
import os

import numpy as np
import pytest

import oracle
from paper_2306_04316_b200 import workloads as W
from paper_2306_04316_b200.engine import CsrSet, Polygon

import adversarial

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz")
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
SQ = Polygon.from_rings([adversarial.SQUARE])
IN, OUT, BND, ERR = 0, 1, 2, 3


def port_contains(p, poly, mode):
    v, _ = oracle.port_classify(np.array([p], float), poly.vx, poly.vy, poly.ring_off, mode, prefilter=False)
    return int(v[0])


def test_port_unit_square_kats():
    # geometry_test.cpp:95-121 via verdicts; acceptance check 3 truth table
    counts, err = oracle.port_count_crossings(np.array([[0.5, 0.5], [-1.0, 0.5], [2.0, 0.5]]), SQ.vx, SQ.vy, 0)
    assert list(counts) == [1, 2, 0] and not err.any()
    counts, err = oracle.port_count_crossings(np.array([[0.5, 0.5], [-1.0, 0.5], [0.5, 0.0]]), SQ.vx, SQ.vy, 1)
    assert list(counts[:2]) == [1, 2] and list(err) == [0, 0, 1]
    for mode in (0, 1, 2):
        assert port_contains((0.5, 0.5), SQ, mode) == IN
        assert port_contains((5.0, 5.0), SQ, mode) == OUT
    assert port_contains((1.0, 0.5), SQ, 2) == BND
    assert port_contains((0.5, 0.0), SQ, 1) == ERR
    assert port_contains((0.5, 0.0), SQ, 2) == BND
    # vertex-on-ray double count (geometry_test.cpp:145-160)
    dm = Polygon.from_rings([adversarial.DIAMOND])
    c, _ = oracle.port_count_crossings(np.array([[-3.0, 0.0]]), dm.vx, dm.vy, 0)
    assert c[0] == 4
    assert port_contains((-3.0, 0.0), dm, 0) == OUT
    assert port_contains((2.0, 0.0), dm, 2) == IN


def test_port_prefilter_semantics_p3():
    # contains(C1) of (-1,1) is Inside (3 crossings) but classify_batch is Outside
    assert port_contains((-1.0, 1.0), SQ, 0) == IN
    v, _ = oracle.port_classify(np.array([[-1.0, 1.0]]), SQ.vx, SQ.vy, SQ.ring_off, 0, prefilter=True)
    assert v[0] == OUT


def test_port_batch_probes():
    # batch_test.cpp:65-85, acceptance check 9
    v, st = oracle.port_classify(np.array([[0.5, 0.5], [1.5, 0.5], [0.5, -0.5], [-0.5, 0.5]]), SQ.vx, SQ.vy,
                                 SQ.ring_off, 2)
    assert list(v) == [IN, OUT, OUT, OUT] and list(st) == [1, 3, 0, 0]
    v, st = oracle.port_classify(np.array([[0.5, 0.0], [0.5, 0.5], [-2.0, 0.5]]), SQ.vx, SQ.vy, SQ.ring_off, 1)
    assert list(v) == [ERR, IN, OUT] and st[3] == 1
    v, _ = oracle.port_classify(np.array([[0.5, 0.0], [-5.0, 0.0], [0.5, 0.5]]), SQ.vx, SQ.vy, SQ.ring_off, 1)
    assert list(v) == [ERR, OUT, IN]


def test_port_p8_duplicate_vertices():
    # a zero-length edge on the ray: C1 counts it (+1), C2 -> Error, Robust never Boundary/count
    ring = Polygon.from_rings([[(0, 0), (2, 0), (2, 1), (2, 1), (0, 1), (0, 0)]])
    c, _ = oracle.port_count_crossings(np.array([[1.0, 1.0]]), ring.vx, ring.vy, 0)
    # edges on y=1: (2,1)->(2,1) zero-length: product 0 -> straddle, n=(0,0), side=0 -> counted
    assert c[0] >= 1
    v, _ = oracle.port_classify(np.array([[-1.0, 1.0]]), ring.vx, ring.vy, ring.ring_off, 1, prefilter=False)
    assert v[0] == ERR


@needs_ref
def test_ref_shim_kats():
    assert oracle.ref_count_crossings((0.5, 0.5), SQ.vx, SQ.vy, 0) == 1
    assert oracle.ref_count_crossings((-1.0, 0.5), SQ.vx, SQ.vy, 1) == 2
    assert oracle.ref_count_crossings((0.5, 0.0), SQ.vx, SQ.vy, 1) is None
    assert oracle.ref_contains((1.0, 0.5), SQ.vx, SQ.vy, SQ.ring_off, 2) == BND
    assert oracle.ref_contains((-1.0, 1.0), SQ.vx, SQ.vy, SQ.ring_off, 0) == IN
    with pytest.raises(oracle.RefError):
        oracle.ref_classify(np.zeros((1, 2)), [0, 1, 1, 0], [0, 0, 0, 0], [0, 4], 0)  # duplicate vertex


@needs_ref
@pytest.mark.parametrize("name,poly,xy", [c for c in adversarial.cases(include_dups=False)],
                         ids=[c[0] for c in adversarial.cases(include_dups=False)])
def test_port_matches_reference_adversarial(name, poly, xy):
    for mode in (0, 1, 2):
        rv, rs = oracle.ref_classify(xy, poly.vx, poly.vy, poly.ring_off, mode)
        pv, ps = oracle.port_classify(xy, poly.vx, poly.vy, poly.ring_off, mode)
        assert np.array_equal(rv, pv) and np.array_equal(rs, ps), (name, mode)
        # contains() semantics, per point through the reference
        sub = xy[:: max(1, len(xy) // 300)]
        want = [oracle.ref_contains(p, poly.vx, poly.vy, poly.ring_off, mode) for p in sub]
        got, _ = oracle.port_classify(sub, poly.vx, poly.vy, poly.ring_off, mode, prefilter=False)
        assert list(got) == want, (name, mode)


@needs_ref
def test_port_matches_reference_configs():
    cases = [W.config2(n, n_points=20_000) for n in (10, 100, 1000)]
    poly = W.fractal_polygon(20_000)
    cases.append((poly, W.uniform_points(5000, W.bounds(poly), 3)))
    for poly, xy in cases:
        for mode in (0, 1, 2):
            rv, rs = oracle.ref_classify(xy, poly.vx, poly.vy, poly.ring_off, mode)
            pv, ps = oracle.port_classify(xy, poly.vx, poly.vy, poly.ring_off, mode, threads=4)
            assert np.array_equal(rv, pv) and np.array_equal(rs, ps)


@needs_ref
def test_port_matches_reference_csr():
    for s in (W.footprints(3000), W.degenerate(1500, allow_dups=False)):
        for mode in (0, 1, 2):
            rv, rs = oracle.ref_classify_csr(s, mode)
            pv, ps = oracle.port_classify_csr(s, mode, threads=4)
            assert np.array_equal(rv, pv) and np.array_equal(rs, ps)


def _golden():
    g = np.load(GOLDEN)
    return g, [str(n) for n in g["__names__"]]


def test_golden_vectors_pin_port():
    g, names = _golden()
    assert len(names) >= 15
    for name in names:
        kind = str(g[f"{name}/kind"])
        for mode in (0, 1, 2):
            if kind == "single":
                v, st = oracle.port_classify(g[f"{name}/xy"], g[f"{name}/vx"], g[f"{name}/vy"], g[f"{name}/ring_off"],
                                             mode)
                cv, _ = oracle.port_classify(g[f"{name}/xy"], g[f"{name}/vx"], g[f"{name}/vy"],
                                             g[f"{name}/ring_off"], mode, prefilter=False)
                assert np.array_equal(cv, g[f"{name}/contains{mode}"]), (name, mode)
            else:
                s = CsrSet(*(g[f"{name}/{k}"] for k in ("xy", "pt_off", "vx", "vy", "ring_off", "poly_ring_off")))
                v, st = oracle.port_classify_csr(s, mode)
            assert np.array_equal(v, g[f"{name}/verdicts{mode}"]), (name, mode)
            assert np.array_equal(st, g[f"{name}/stats{mode}"]), (name, mode)


@needs_ref
def test_golden_vectors_pin_reference():
    g, names = _golden()
    for name in names:
        if str(g[f"{name}/source"]) != "reference":
            continue
        for mode in (0, 1, 2):
            if str(g[f"{name}/kind"]) == "single":
                v, _ = oracle.ref_classify(g[f"{name}/xy"], g[f"{name}/vx"], g[f"{name}/vy"], g[f"{name}/ring_off"],
                                           mode)
            else:
                s = CsrSet(*(g[f"{name}/{k}"] for k in ("xy", "pt_off", "vx", "vy", "ring_off", "poly_ring_off")))
                v, _ = oracle.ref_classify_csr(s, mode)
            assert np.array_equal(v, g[f"{name}/verdicts{mode}"]), (name, mode)
