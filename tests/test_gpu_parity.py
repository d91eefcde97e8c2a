"""GPU parity: libpolycast_cuda.so (through the C-ABI) vs the oracle, bit-exact.

Checker: the unmodified reference (oracle/_ref/libpolycast_ref.so, built from
/root/reference and shipped prebuilt) wherever it can express the input, the C
restatement (oracle/build/libpip_oracle.so, pinned to the reference in
test_oracle.py) for duplicate-vertex inputs (P8) and for large CSR sets.
Sizes: full BASELINE configs where the checker finishes in seconds, seeded
subsamples of the same inputs otherwise, plus size-independent properties at
full size.
"""
import os

import numpy as np
import pytest

import adversarial
import oracle
from paper_2306_04316_b200 import CrossingMode, DegenerateEdge, Engine, unpack_bits, verdicts_to_bits
from paper_2306_04316_b200 import workloads as W
from paper_2306_04316_b200.engine import Classification, CsrSet, Polygon

pytestmark = pytest.mark.gpu
MODES = (0, 1, 2)
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz")
THREADS = os.cpu_count() or 8


def check_single(xy, poly, mode, got, prefilter=True, source=None):
    if source is None:
        source = "reference" if oracle.ref_available() and prefilter else "port"
    if source == "reference":
        want_v, want_s = oracle.ref_classify(xy, poly.vx, poly.vy, poly.ring_off, mode)
    else:
        want_v, want_s = oracle.port_classify(xy, poly.vx, poly.vy, poly.ring_off, mode, prefilter=prefilter,
                                              threads=THREADS)
    assert np.array_equal(got.verdicts, want_v), f"mode {mode}: {(got.verdicts != want_v).sum()} verdicts differ"
    assert np.array_equal(got.stats, want_s)
    ib, ab = verdicts_to_bits(want_v, mode)
    if got.inside_bits is not None:
        assert np.array_equal(got.inside_bits, ib) and np.array_equal(got.aux_bits, ab)


# ---- golden vectors -----------------------------------------------------------

def test_golden_vectors(engine):
    g = np.load(GOLDEN)
    for name in (str(n) for n in g["__names__"]):
        for mode in MODES:
            if str(g[f"{name}/kind"]) == "single":
                poly = Polygon(g[f"{name}/vx"], g[f"{name}/vy"], g[f"{name}/ring_off"])
                xy = g[f"{name}/xy"]
                r = engine.classify(xy, poly, mode)
                assert np.array_equal(r.verdicts, g[f"{name}/verdicts{mode}"]), (name, mode)
                assert np.array_equal(r.stats, g[f"{name}/stats{mode}"]), (name, mode)
                r0 = engine.classify(xy, poly, mode, prefilter=False)
                assert np.array_equal(r0.verdicts, g[f"{name}/contains{mode}"]), (name, mode, "contains")
            else:
                s = CsrSet(*(g[f"{name}/{k}"] for k in ("xy", "pt_off", "vx", "vy", "ring_off", "poly_ring_off")))
                r = engine.classify_csr(s, mode)
                assert np.array_equal(r.verdicts, g[f"{name}/verdicts{mode}"]), (name, mode)
                assert np.array_equal(r.stats, g[f"{name}/stats{mode}"]), (name, mode)


@pytest.mark.parametrize("case", adversarial.cases(), ids=[c[0] for c in adversarial.cases()])
def test_adversarial(engine, case):
    name, poly, xy = case
    src = "port" if name == "dup_vertices" else None
    for mode in MODES:
        check_single(xy, poly, mode, engine.classify(xy, poly, mode), source=src)
        check_single(xy, poly, mode, engine.classify(xy, poly, mode, prefilter=False), prefilter=False)


# ---- KATs through the Python mirror of the reference API ------------------------

def test_reference_kats(engine):
    sq = Polygon.from_rings([adversarial.SQUARE])
    for mode in (CrossingMode.C1, CrossingMode.C2, CrossingMode.Robust):
        assert engine.contains((0.5, 0.5), sq, mode) == Classification.Inside
        assert engine.contains((5.0, 5.0), sq, mode) == Classification.Outside
    assert engine.contains((1.0, 0.5), sq, CrossingMode.Robust) == Classification.Boundary
    with pytest.raises(DegenerateEdge):
        engine.contains((0.5, 0.0), sq, CrossingMode.C2)
    counts, deg = engine.count_crossings([[0.5, 0.5], [-1.0, 0.5], [2.0, 0.5]], sq.vx, sq.vy, CrossingMode.C1)
    assert list(counts) == [1, 2, 0] and not deg.any()
    dm = Polygon.from_rings([adversarial.DIAMOND])
    counts, _ = engine.count_crossings([[-3.0, 0.0]], dm.vx, dm.vy, CrossingMode.C1)
    assert counts[0] == 4
    r = engine.classify_batch([[0.5, 0.0], [0.5, 0.5], [-2.0, 0.5]], sq, CrossingMode.C2)
    assert list(r.verdicts) == [3, 0, 1] and r.stats[3] == 1


def test_count_crossings_vs_reference(engine):
    rng = np.random.default_rng(5)
    for n in (5, 37, 400, 3000):
        poly = W.star_polygon(n, seed=n)
        xy = W.uniform_points(3000, W.bounds(poly), n)
        xy[:200] = np.stack([rng.choice(poly.vx, 200), rng.choice(poly.vy, 200)], 1)  # rays through vertices
        for mode in (0, 1):
            c, d = engine.count_crossings(xy, poly.vx, poly.vy, mode)
            wc, wd = oracle.port_count_crossings(xy, poly.vx, poly.vy, mode)
            assert np.array_equal(d, wd)
            assert np.array_equal(c[wd == 0], wc[wd == 0])
            if oracle.ref_available():
                for i in range(0, 3000, 97):
                    want = oracle.ref_count_crossings(xy[i], poly.vx, poly.vy, mode)
                    assert (want is None) == bool(d[i])
                    if want is not None:
                        assert c[i] == want


# ---- configs ----------------------------------------------------------------------

def test_config1_full(engine):
    poly, xy = W.config1()
    for mode in MODES:
        check_single(xy, poly, mode, engine.classify_batch(xy, poly, mode))


@pytest.mark.parametrize("n", W.SWEEP_N)
def test_config2_sweep(engine, n):
    poly, xy = W.config2(n)
    for mode in MODES:
        got = engine.classify_batch(xy, poly, mode)
        assert int(got.stats.sum()) == len(xy)
        if n <= 10_000:
            check_single(xy, poly, mode, got)
        else:  # seeded subsample keeps the CPU checker to seconds
            idx = np.random.default_rng(n + mode).choice(len(xy), 20_000 if n == 100_000 else 2_000, replace=False)
            sub = np.ascontiguousarray(xy[idx])
            want_v, _ = (oracle.ref_classify(sub, poly.vx, poly.vy, poly.ring_off, mode) if oracle.ref_available()
                         else oracle.port_classify(sub, poly.vx, poly.vy, poly.ring_off, mode, threads=THREADS))
            assert np.array_equal(got.verdicts[idx], want_v)


def test_config3_footprints(engine):
    s = W.footprints(200_000)
    for mode in MODES:
        got = engine.classify_csr(s, mode)
        want_v, want_s = oracle.port_classify_csr(s, mode, threads=THREADS)
        assert np.array_equal(got.verdicts, want_v) and np.array_equal(got.stats, want_s)
        ib, ab = verdicts_to_bits(want_v, mode)
        assert np.array_equal(got.inside_bits, ib) and np.array_equal(got.aux_bits, ab)
    if oracle.ref_available():
        s = W.footprints(20_000, seed=77)
        for mode in MODES:
            want_v, _ = oracle.ref_classify_csr(s, mode)
            assert np.array_equal(engine.classify_csr(s, mode).verdicts, want_v)


def test_config4_subsample(engine):
    poly = W.fractal_polygon(200_000)
    xy = W.uniform_points(1_000_000, W.bounds(poly), 4)
    for mode in MODES:
        got = engine.classify_batch(xy, poly, mode)
        idx = np.random.default_rng(mode).choice(len(xy), 10_000, replace=False)
        sub = np.ascontiguousarray(xy[idx])
        want_v, _ = (oracle.ref_classify(sub, poly.vx, poly.vy, poly.ring_off, mode) if oracle.ref_available()
                     else oracle.port_classify(sub, poly.vx, poly.vy, poly.ring_off, mode, threads=THREADS))
        assert np.array_equal(got.verdicts[idx], want_v)
        assert int(got.stats.sum()) == len(xy)


def test_config5_degenerate_full(engine):
    s = W.degenerate(100_000, allow_dups=True)
    assert s.n_points > 9_000_000
    for mode in MODES:
        got = engine.classify_csr(s, mode)
        want_v, want_s = oracle.port_classify_csr(s, mode, threads=THREADS)
        assert np.array_equal(got.verdicts, want_v), f"mode {mode}: {(got.verdicts != want_v).sum()} differ"
        assert np.array_equal(got.stats, want_s)
    if oracle.ref_available():
        s = W.degenerate(10_000, allow_dups=False, seed=5)
        for mode in MODES:
            want_v, _ = oracle.ref_classify_csr(s, mode)
            assert np.array_equal(engine.classify_csr(s, mode).verdicts, want_v)


def test_config5_as_single_polygons(engine):
    """Each degenerate polygon (with duplicates and holes) through the single-polygon kernel."""
    s = W.degenerate(300, allow_dups=True, seed=9)
    for p in range(0, 300, 7):
        r0, r1 = int(s.poly_ring_off[p]), int(s.poly_ring_off[p + 1])
        v0, v1 = int(s.ring_off[r0]), int(s.ring_off[r1])
        poly = Polygon(s.vx[v0:v1], s.vy[v0:v1], s.ring_off[r0:r1 + 1] - s.ring_off[r0])
        xy = np.ascontiguousarray(s.xy[int(s.pt_off[p]):int(s.pt_off[p + 1])])
        for mode in MODES:
            check_single(xy, poly, mode, engine.classify(xy, poly, mode), source="port")
            check_single(xy, poly, mode, engine.classify(xy, poly, mode, prefilter=False), prefilter=False)


# ---- sizes, layouts, sharding --------------------------------------------------

@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 4095, 100_003])
def test_ragged_point_counts(engine, n):
    poly = W.star_polygon(777)
    xy = W.uniform_points(max(n, 1), (-1.1, -1.1, 1.1, 1.1), n)[:n]
    for mode in MODES:
        got = engine.classify(xy, poly, mode)
        assert len(got.verdicts) == n and int(got.stats.sum()) == n
        if n:
            check_single(xy, poly, mode, got)


def test_many_holes_and_huge_ring(engine):
    rng = np.random.default_rng(3)
    rings = [np.stack([np.cos(t) * 100, np.sin(t) * 100], 1) for t in [np.linspace(0, 2 * np.pi, 5001)]]
    rings[0][-1] = rings[0][0]
    for k in range(150):  # 150 small square holes
        cx, cy = rng.uniform(-60, 60, 2)
        h = [(cx, cy), (cx + 1, cy), (cx + 1, cy + 1), (cx, cy + 1), (cx, cy)]
        rings.append(np.array(h))
    poly = Polygon.from_rings(rings)
    xy = W.uniform_points(200_000, (-110, -110, 110, 110), 8)
    for mode in MODES:
        check_single(xy, poly, mode, engine.classify(xy, poly, mode))
    # a 1e6-edge ring with few points: exercises the edge-chunk split
    big = W.star_polygon(1_000_000)
    xy = W.uniform_points(3000, W.bounds(big), 9)
    for mode in MODES:
        check_single(xy, big, mode, engine.classify(xy, big, mode))


@pytest.mark.parametrize("shards", [2, 3])
def test_multi_shard_identical(shards):
    """Shard logic across 'GPUs' (here: 2 or 3 logical devices on one GPU, each
    enqueued from its own host thread) gives bit-identical output -- the
    reference's determinism check at 1e6 points (acceptance.cpp:345-357,
    batch_test.cpp:87-105): a star, 1e6 points of configs[3], a CSR set."""
    poly, xy = W.config2(1000, n_points=300_017)
    p4, x4 = W.config4(n_points=1_000_000)
    s = W.degenerate(20_000, allow_dups=True, seed=3)
    with Engine(devices=[0]) as one, Engine(devices=[0] * shards) as many:
        assert many.device_count == shards
        for mode in MODES:
            for P, X in ((poly, xy), (p4, x4)):
                a, b = one.classify_batch(X, P, mode), many.classify_batch(X, P, mode)
                assert np.array_equal(a.verdicts, b.verdicts) and np.array_equal(a.inside_bits, b.inside_bits)
                assert np.array_equal(a.aux_bits, b.aux_bits) and np.array_equal(a.stats, b.stats)
            a, b = one.classify_csr(s, mode), many.classify_csr(s, mode)
            assert np.array_equal(a.verdicts, b.verdicts) and np.array_equal(a.inside_bits, b.inside_bits)
            assert np.array_equal(a.aux_bits, b.aux_bits) and np.array_equal(a.stats, b.stats)


@pytest.mark.parametrize("n_verts", [1000, 20_000])  # scan kernel / segment tree
def test_chunked_upload_matches_one_piece(engine, n_verts):
    """Host-API shards above 2 x 2^23 points upload in 2^23-point chunks, each
    classified while the next uploads (pip_capi.cu); the result must equal the
    device-pointer call on the whole array (one piece), bit for bit, and a
    subsample must match the reference."""
    import torch
    n = 2 * (1 << 23) + 12_345  # three chunks, the last one ragged
    poly = W.star_polygon(n_verts)
    xy = W.uniform_points(n, W.bounds(poly), 17)
    dev = torch.device("cuda:0")
    d_xy = torch.from_numpy(xy).to(dev)
    d_vx, d_vy = torch.from_numpy(poly.vx).to(dev), torch.from_numpy(poly.vy).to(dev)
    d_ro = torch.from_numpy(poly.ring_off.view(np.int64)).to(dev)
    nw = (n + 31) // 32
    for mode in (0, 1):
        host = engine.classify_batch(xy, poly, mode)
        d_in = torch.empty(nw, dtype=torch.int32, device=dev)
        d_aux = torch.empty(nw, dtype=torch.int32, device=dev)
        d_st = torch.empty(4, dtype=torch.int64, device=dev)
        d_v = torch.empty(n, dtype=torch.uint8, device=dev)
        engine.classify_dev(0, torch.cuda.current_stream().cuda_stream, d_xy, n, d_vx, d_vy, d_ro, poly.n_rings,
                            poly.n_verts, mode, 1e-12, True, d_in, d_aux, d_st, d_v)
        torch.cuda.synchronize()
        assert np.array_equal(d_in.cpu().numpy().view(np.uint32), host.inside_bits)
        assert np.array_equal(d_aux.cpu().numpy().view(np.uint32), host.aux_bits)
        assert np.array_equal(d_v.cpu().numpy(), host.verdicts)
        assert np.array_equal(d_st.cpu().numpy().view(np.uint64), host.stats)
        # chunk seams and a random subsample against the reference
        idx = np.unique(np.concatenate([np.arange(0, 64), (1 << 23) + np.arange(-64, 64),
                                        (2 << 23) + np.arange(-64, 64), np.arange(n - 64, n),
                                        np.random.default_rng(5).integers(0, n, 20_000)]))
        sub = np.ascontiguousarray(xy[idx])
        want_v, _ = (oracle.ref_classify(sub, poly.vx, poly.vy, poly.ring_off, mode) if oracle.ref_available()
                     else oracle.port_classify(sub, poly.vx, poly.vy, poly.ring_off, mode, threads=THREADS))
        assert np.array_equal(host.verdicts[idx], want_v)


def test_device_pointer_api_matches_host_api(engine):
    import torch
    poly, xy = W.config2(1000, n_points=123_457)
    dev = torch.device("cuda:0")
    d_xy = torch.from_numpy(xy).to(dev)
    d_vx, d_vy = torch.from_numpy(poly.vx).to(dev), torch.from_numpy(poly.vy).to(dev)
    d_ro = torch.from_numpy(poly.ring_off.view(np.int64)).to(dev)
    nw = (len(xy) + 31) // 32
    for mode in MODES:
        d_in = torch.empty(nw, dtype=torch.int32, device=dev)
        d_aux = torch.empty(nw, dtype=torch.int32, device=dev)
        d_st = torch.empty(4, dtype=torch.int64, device=dev)
        d_v = torch.empty(len(xy), dtype=torch.uint8, device=dev)
        st = torch.cuda.current_stream().cuda_stream
        engine.classify_dev(0, st, d_xy, len(xy), d_vx, d_vy, d_ro, poly.n_rings, poly.n_verts, mode, 1e-12, True,
                            d_in, d_aux, d_st, d_v)
        torch.cuda.synchronize()
        host = engine.classify_batch(xy, poly, mode)
        assert np.array_equal(d_v.cpu().numpy(), host.verdicts)
        assert np.array_equal(d_in.cpu().numpy().view(np.uint32), host.inside_bits)
        assert np.array_equal(d_st.cpu().numpy().view(np.uint64), host.stats)
    s = W.footprints(10_000)
    t = {k: torch.from_numpy(getattr(s, k).view(np.int64) if getattr(s, k).dtype == np.uint64 else getattr(s, k))
         .to(dev) for k in ("xy", "pt_off", "vx", "vy", "ring_off", "poly_ring_off")}
    nw = (s.n_points + 31) // 32
    d_in = torch.empty(nw, dtype=torch.int32, device=dev)
    d_aux = torch.empty(nw, dtype=torch.int32, device=dev)
    d_st = torch.empty(4, dtype=torch.int64, device=dev)
    engine.classify_csr_dev(0, torch.cuda.current_stream().cuda_stream, t["xy"], t["pt_off"], s.n_polys, s.n_points,
                            t["vx"], t["vy"], t["ring_off"], t["poly_ring_off"], 0, 1e-12, d_in, d_aux, d_st)
    torch.cuda.synchronize()
    host = engine.classify_csr(s, 0)
    assert np.array_equal(d_in.cpu().numpy().view(np.uint32), host.inside_bits)


def test_bits_match_verdicts_and_launch_count(engine):
    poly, xy = W.config2(100, n_points=50_000)
    r = engine.classify_batch(xy, poly, CrossingMode.Robust)
    assert engine.last_launch_count >= 3  # prep, classify, finalize: native kernels ran
    inside = unpack_bits(r.inside_bits, len(xy))
    aux = unpack_bits(r.aux_bits, len(xy))
    assert np.array_equal(inside, r.verdicts == 0) and np.array_equal(aux, r.verdicts == 2)


def test_invalid_arguments_report_status(engine):
    from paper_2306_04316_b200 import DeviceError
    bad = Polygon(np.zeros(4), np.zeros(4), np.array([0, 2, 2], np.uint64))  # empty ring
    with pytest.raises(DeviceError) as e:
        engine.classify(np.zeros((4, 2)), bad, 0)
    assert e.value.status == 1
    with pytest.raises(DeviceError):
        engine.classify(np.zeros((4, 2)), Polygon.from_rings([adversarial.SQUARE]), 7)


@pytest.mark.parametrize("bucket", [0, 1])
def test_bucketing_modes_identical(bucket):
    """y-bucketing (pip_sort.cu) forced off / on: bit-identical to the reference, all modes,
    with and without the bbox prefilter, including points outside the box."""
    cases = [W.config2(1000, n_points=100_003), W.config2(64, n_points=50_001)]
    poly = W.star_polygon(300, seed=4)
    cases.append((poly, W.uniform_points(77_777, (-2.0, -2.0, 2.0, 2.0), 5)))  # many points outside the bbox
    for name, p, xy in adversarial.cases():
        cases.append((p, xy))
    with Engine(devices=[0]) as eng:
        eng.set_bucketing(bucket)
        for i, (poly, xy) in enumerate(cases):
            src = "port" if i == len(cases) - 1 else None  # last adversarial case has duplicate vertices
            for mode in MODES:
                check_single(xy, poly, mode, eng.classify(xy, poly, mode), source=src)
                check_single(xy, poly, mode, eng.classify(xy, poly, mode, prefilter=False), prefilter=False)


def _concat_csr(parts):
    """Concatenate CsrSets (offsets rebased)."""
    xy, vx, vy = [], [], []
    pt_off, ring_off, pring = [0], [0], [0]
    for s in parts:
        base_p, base_v, base_r = pt_off[-1], ring_off[-1], pring[-1]
        xy.append(s.xy)
        vx.append(s.vx)
        vy.append(s.vy)
        pt_off += [base_p + int(v) for v in s.pt_off[1:]]
        ring_off += [base_v + int(v) for v in s.ring_off[1:]]
        pring += [base_r + int(v) for v in s.poly_ring_off[1:]]
    return CsrSet(np.ascontiguousarray(np.concatenate(xy)), np.array(pt_off, np.uint64), np.concatenate(vx),
                  np.concatenate(vy), np.array(ring_off, np.uint64), np.array(pring, np.uint64))


def _single_as_csr(poly, xy):
    return CsrSet(np.ascontiguousarray(xy), np.array([0, len(xy)], np.uint64), poly.vx, poly.vy, poly.ring_off,
                  np.array([0, poly.n_rings], np.uint64))


def test_csr_oversize_and_mixed_polygons(engine):
    """CSR stages hold <=1024 points / 512 vertices / 128 rings; bigger polygons take the
    global-memory path.  Mix both, plus empty polygons and odd vertex offsets."""
    rng = np.random.default_rng(11)
    parts = [W.footprints(300, seed=1)]
    big = W.star_polygon(2000, seed=3)                         # > kVmax vertices
    parts.append(_single_as_csr(big, W.uniform_points(3000, W.bounds(big), 4)))  # > kPmax points
    parts.append(W.degenerate(200, seed=5))
    rings = [[(0, 0), (300, 0), (300, 300), (0, 300), (0, 0)]]
    for k in range(140):                                       # > kRmax rings
        x, y = 10 + 20 * (k % 14), 10 + 20 * (k // 14)
        rings.append([(x, y), (x + 5, y), (x + 5, y + 5), (x, y + 5), (x, y)])
    holed = Polygon.from_rings(rings)
    parts.append(_single_as_csr(holed, rng.uniform(-10, 310, (500, 2))))
    parts.append(CsrSet(np.zeros((0, 2)), np.array([0, 0], np.uint64), np.array([0., 1, 1, 0]),
                        np.array([0., 0, 1, 0]), np.array([0, 4], np.uint64), np.array([0, 1], np.uint64)))
    parts.append(W.footprints(500, seed=2, pts_per_poly=33))     # unaligned point runs
    s = _concat_csr(parts)
    for mode in MODES:
        got = engine.classify_csr(s, mode)
        want_v, want_s = oracle.port_classify_csr(s, mode, threads=THREADS)
        assert np.array_equal(got.verdicts, want_v), f"mode {mode}: {(got.verdicts != want_v).sum()} differ"
        assert np.array_equal(got.stats, want_s)


def test_bucketing_skewed_inputs(engine):
    """All points on a handful of y values / one bin (counting-sort edge cases), and
    points far outside the bbox with and without the prefilter."""
    rng = np.random.default_rng(21)
    poly = W.star_polygon(500, seed=8)
    n = 70_001
    xy = np.empty((n, 2))
    xy[:, 0] = rng.uniform(-1.2, 1.2, n)
    xy[:, 1] = rng.choice(np.array([0.0, 0.25, -0.5, poly.vy[3], poly.vy[77]]), n)
    xy[:1000, 1] = 1e300
    xy[1000:2000, 1] = -1e300
    engine.set_bucketing(1)
    try:
        for mode in MODES:
            check_single(xy, poly, mode, engine.classify(xy, poly, mode))
            check_single(xy, poly, mode, engine.classify(xy, poly, mode, prefilter=False), prefilter=False)
    finally:
        engine.set_bucketing(-1)


def _near_edge_points(s, deltas, ts=(0.25, 0.5, 0.75)):
    """Per polygon of CsrSet s: points on every outer-ring edge (a + t (b - a) in
    binary64) and nudged off it along the edge normal by each delta (relative to
    the polygon's bbox size), so that they fall inside, on and just outside the
    fp32 fast path's band (pip_csr_common.cuh)."""
    xy, pt_off = [], [0]
    for p in range(s.n_polys):
        r0 = int(s.poly_ring_off[p])
        v0, v1 = int(s.ring_off[r0]), int(s.ring_off[r0 + 1])
        x, y = s.vx[v0:v1], s.vy[v0:v1]
        size = max(x.max() - x.min(), y.max() - y.min())
        pts = []
        for i in range(len(x) - 1):
            ax, ay, bx, by = x[i], y[i], x[i + 1], y[i + 1]
            ln = np.hypot(bx - ax, by - ay) or 1.0
            nx, ny = (by - ay) / ln, (ax - bx) / ln
            for t in ts:
                px, py = ax + t * (bx - ax), ay + t * (by - ay)
                pts.append((px, py))
                for d in deltas:
                    pts.append((px + d * size * nx, py + d * size * ny))
                    pts.append((px - d * size * nx, py - d * size * ny))
            pts.append((ax, ay))                       # the vertex itself (tie)
            pts.append((ax + 0.3 * size, ay))          # on the vertex's y-level (tie)
        xy.extend(pts)
        pt_off.append(len(xy))
    return CsrSet(np.ascontiguousarray(np.array(xy, np.float64)), np.array(pt_off, np.uint64), s.vx, s.vy,
                  s.ring_off, s.poly_ring_off)


def test_csr_fast_path_band_and_ties(engine):
    """C1 CSR fast path (fp32 side test with a certified band, integer y keys):
    points on / within / just outside the band of every edge, vertex ties, for
    footprints in lon/lat degrees and for integer-grid polygons."""
    deltas = (1e-16, 1e-12, 1e-9, 2e-7, 4e-7, 1e-6, 3e-6, 1e-4)
    for base in (W.footprints(400, seed=31), W.degenerate(150, seed=32, allow_dups=False)):
        s = _near_edge_points(base, deltas)
        for mode in MODES:
            got = engine.classify_csr(s, mode)
            want_v, want_s = oracle.port_classify_csr(s, mode, threads=THREADS)
            assert np.array_equal(got.verdicts, want_v), f"mode {mode}: {(got.verdicts != want_v).sum()} differ"
            assert np.array_equal(got.stats, want_s)


def test_csr_fast_path_gates(engine):
    """Polygons where the fast path must switch itself off or route points to the
    exact path: the adversarial cases as CSR polygons (tiny / subnormal / huge
    extents, signed zeros, slivers), a hole poking outside the outer ring, and a
    polygon straddling y = 0 with points at |y| < 2^-400."""
    rng = np.random.default_rng(41)
    parts = []
    for name, poly, xy in adversarial.cases(include_dups=False):
        parts.append(_single_as_csr(poly, xy))
    out = [(0, 0), (4, 0), (4, 4), (0, 4), (0, 0)]
    hole = [(1, 1), (6, 1), (6, 3), (1, 3), (1, 1)]  # extends past the outer ring's bbox
    ph = Polygon.from_rings([out, hole])
    parts.append(_single_as_csr(ph, np.concatenate([rng.uniform(-1, 7, (800, 2)), adversarial._special_points(ph, rng)])))
    eq = [(-1.0, -1.0), (1.0, -1.0), (1.0, 1.0), (-1.0, 1.0), (-1.0, -1.0)]
    pe = Polygon.from_rings([eq, [(-0.5, -1e-310), (0.5, -1e-310), (0.5, 1e-310), (-0.5, 1e-310), (-0.5, -1e-310)]])
    ys = np.array([0.0, -0.0, 1e-320, -1e-320, 1e-310, -1e-310, 2e-310, 1e-130, 1e-121, 3e-121, -3e-121])
    exy = np.stack([np.repeat(np.linspace(-1.2, 1.2, 13), len(ys)), np.tile(ys, 13)], 1)
    parts.append(_single_as_csr(pe, np.concatenate([exy, rng.uniform(-1.2, 1.2, (500, 2))])))
    # footprints moved along x: |x| * s_x below / above the C2 fast-path gate (2^20)
    for shift in (100.0, 3000.0):
        fp = _near_edge_points(W.footprints(60, seed=int(shift)), (1e-12, 1e-9, 1e-6))
        parts.append(CsrSet(np.ascontiguousarray(fp.xy + [shift, 0.0]), fp.pt_off, fp.vx + shift, fp.vy, fp.ring_off,
                            fp.poly_ring_off))
    s = _concat_csr(parts)
    for mode in MODES:
        got = engine.classify_csr(s, mode)
        want_v, want_s = oracle.port_classify_csr(s, mode, threads=THREADS)
        assert np.array_equal(got.verdicts, want_v), f"mode {mode}: {(got.verdicts != want_v).sum()} differ"
        assert np.array_equal(got.stats, want_s)


# ---- GPU prefilter_bbox / scatter_verdicts ------------------------

def _prefilter_ref(xy, box):
    """batch.hpp:137-153 restated: closed-interval membership, input order kept."""
    x0, y0, x1, y1 = box
    m = (xy[:, 0] >= x0) & (xy[:, 0] <= x1) & (xy[:, 1] >= y0) & (xy[:, 1] <= y1)
    idx = np.nonzero(m)[0].astype(np.uint64)
    return xy[m], idx, len(xy) - len(idx)


@pytest.mark.parametrize("n", [0, 1, 31, 1000, 16385, 5_000_003])
def test_prefilter_bbox_matches_reference_loop(engine, n):
    rng = np.random.default_rng(n + 5)
    xy = rng.uniform(-2, 2, (n, 2))
    if n > 10:
        xy[:5] = [[1.0, 0.5], [-1.0, -1.0], [1.0, 1.0], [np.nan, 0.0], [0.0, np.inf]]  # edges, corner, NaN, inf
    for box in ((-1.0, -1.0, 1.0, 1.0), (0.0, 0.0, 0.0, 0.0), (-5.0, -5.0, 5.0, 5.0), (3.0, 3.0, 4.0, 4.0)):
        got_xy, got_idx, got_out = engine.prefilter_bbox(xy, box)
        want_xy, want_idx, want_out = _prefilter_ref(xy, box)
        assert got_out == want_out
        assert np.array_equal(got_idx, want_idx)
        assert np.array_equal(got_xy.view(np.uint64), want_xy.view(np.uint64))  # bit-identical points


def test_scatter_verdicts_and_cli_pipeline(engine):
    """CLI pipeline (polycast_cli.cpp:78-80): prefilter -> classify the in-box points ->
    scatter == classify_batch of the whole batch; plus the reference's error cases."""
    poly = W.star_polygon(300, seed=9)
    rng = np.random.default_rng(3)
    b = W.bounds(poly)
    xy = np.stack([rng.uniform(b[0] - 1, b[2] + 1, 200_001), rng.uniform(b[1] - 1, b[3] + 1, 200_001)], 1)
    box = (float(poly.vx.min()), float(poly.vy.min()), float(poly.vx.max()), float(poly.vy.max()))
    for mode in MODES:
        ixy, idx, n_out = engine.prefilter_bbox(xy, box)
        inbox = engine.classify(ixy, poly, mode, prefilter=False).verdicts
        full = engine.scatter_verdicts(idx, inbox, len(xy))
        assert np.array_equal(full, engine.classify(xy, poly, mode).verdicts)
        assert n_out == int((full == 1).sum()) - int((inbox == 1).sum())
    with pytest.raises(Exception):
        engine.prefilter_bbox(xy, (1.0, 0.0, 0.0, 1.0))  # BBox: min must not exceed max
    with pytest.raises(Exception):
        engine.scatter_verdicts(np.array([0, 7], np.uint64), np.zeros(2, np.uint8), 5)  # index out of range
    with pytest.raises(Exception):
        engine.scatter_verdicts(np.arange(6, dtype=np.uint64), np.zeros(6, np.uint8), 5)  # more verdicts than total
    assert np.array_equal(engine.scatter_verdicts(np.zeros(0, np.uint64), np.zeros(0, np.uint8), 4), np.ones(4))


def test_single_fast_side_band(engine):
    """Single-polygon C1 slow path (certified fp32 side test, LocalMap): points on,
    inside, at and just outside the band of every edge of a star polygon and of a
    lon/lat footprint-like polygon, with and without the bbox prefilter, bucketed
    and not."""
    deltas = (1e-16, 1e-12, 1e-9, 2e-7, 4e-7, 1e-6, 3e-6, 1e-4)
    ring = [(5.0 + 0.0004 * np.cos(t), 0.5 + 0.0003 * np.sin(t)) for t in np.linspace(0, 2 * np.pi, 41)[:-1]]
    far = [(1.0e6 + 1.5 * np.cos(t), 0.5 + 1.2 * np.sin(t)) for t in np.linspace(0, 2 * np.pi, 23)[:-1]]
    far2 = [(1.0e6 + 0.2 * np.cos(t), 0.5 + 0.15 * np.sin(t)) for t in np.linspace(0, 2 * np.pi, 23)[:-1]]
    # C2's fp32 test is gated on max|x| / W <= 2^20: `far` passes the gate, `far2` does not
    polys = [W.star_polygon(300, seed=12), Polygon.from_rings([ring + [ring[0]]]),
             Polygon.from_rings([far + [far[0]]]), Polygon.from_rings([far2 + [far2[0]]])]
    for poly in polys:
        s = _near_edge_points(_single_as_csr(poly, np.zeros((1, 2))), deltas)
        xy = s.xy
        for bucket in (0, 1):
            engine.set_bucketing(bucket)
            try:
                for mode in MODES:
                    check_single(xy, poly, mode, engine.classify(xy, poly, mode))
                    check_single(xy, poly, mode, engine.classify(xy, poly, mode, prefilter=False), prefilter=False)
            finally:
                engine.set_bucketing(-1)


def test_robust_tolerances(engine):
    """Robust mode's fp32 records are valid only while tol <= 2^-30 * min(W, H):
    tolerances on both sides of that gate (0, the default 1e-12, 1e-9, 1e-6, 1e-2)
    on a star polygon (W ~ 2) with near-edge points, against the reference."""
    poly = W.star_polygon(200, seed=14)
    s = _near_edge_points(_single_as_csr(poly, np.zeros((1, 2))), (1e-16, 1e-12, 1e-9, 1e-7, 1e-6, 1e-3))
    xy = s.xy
    for tol in (0.0, 1e-12, 1e-9, 1e-6, 1e-2):
        got = engine.classify(xy, poly, CrossingMode.Robust, boundary_tol=tol)
        want_v, want_s = oracle.ref_classify(xy, poly.vx, poly.vy, poly.ring_off, 2, tol=tol)
        assert np.array_equal(got.verdicts, want_v), (tol, int((got.verdicts != want_v).sum()))
        assert np.array_equal(got.stats, want_s)


def test_csr_robust_tolerances(engine):
    """CSR Robust fast path (pip_csr_tile.cu): keys of RN(p.y -+ tol) and the C2
    record, gated by tol * 2 * max(s_x, s_y) <= 2^-25.  Footprints (~1e-4 deg) and
    integer-grid polygons with points at distances around each tol from every edge
    (0.5, 0.99, 1.01, 2 tol) plus the usual band deltas; tolerances on both sides
    of the gate, against the C restatement (pinned to the reference)."""
    base_fp = W.footprints(150, seed=51)
    base_gr = W.degenerate(60, seed=52, allow_dups=False)
    for tol in (0.0, 1e-12, 1e-10, 1e-8, 1e-6, 1e-3):
        parts = []
        for base, size in ((base_fp, 3e-4), (base_gr, 30.0)):
            rel = tuple(f * tol / size for f in (0.5, 0.99, 1.01, 2.0)) if tol > 0 else ()
            parts.append(_near_edge_points(base, rel + (1e-13, 1e-9, 1e-6)))
        s = _concat_csr(parts)
        got = engine.classify_csr(s, CrossingMode.Robust, boundary_tol=tol)
        want_v, want_s = oracle.port_classify_csr(s, CrossingMode.Robust, tol=tol, threads=THREADS)
        assert np.array_equal(got.verdicts, want_v), (tol, int((got.verdicts != want_v).sum()))
        assert np.array_equal(got.stats, want_s)


def test_graph_replay_matches_direct_calls():
    """PC_OPT_GRAPH: the 2nd identical device-pointer call is captured, later ones
    replay the graph; results must equal direct (graph-off) calls, follow changed
    input contents at the same addresses, and survive scratch re-allocation
    (a bigger call in between invalidates the captured addresses)."""
    import torch
    dev = torch.device("cuda:0")
    poly, xy = W.config2(1000, n_points=200_000)
    big = W.uniform_points(3_000_000, W.bounds(poly), 5)
    t = {k: torch.from_numpy(v).to(dev) for k, v in (("vx", poly.vx), ("vy", poly.vy))}
    ro = torch.from_numpy(np.ascontiguousarray(poly.ring_off).view(np.int64)).to(dev)
    d_xy = torch.from_numpy(xy).to(dev)
    d_big = torch.from_numpy(big).to(dev)
    with Engine(devices=[0]) as g, Engine(devices=[0]) as direct:
        direct.set_graphs(False)
        for mode in MODES:
            def run(eng, pts, n):
                nw = (n + 31) // 32
                bits = torch.zeros(2 * nw, dtype=torch.int32, device=dev)
                st = torch.zeros(4, dtype=torch.int64, device=dev)
                s = torch.cuda.current_stream().cuda_stream
                eng.classify_dev(0, s, pts, n, t["vx"], t["vy"], ro, poly.n_rings, poly.n_verts, mode, 1e-12, True,
                                 bits[:nw], bits[nw:], st)
                torch.cuda.synchronize()
                return bits.cpu().numpy(), st.cpu().numpy()
            want = run(direct, d_xy, len(xy))
            for _ in range(4):  # direct, capture, replay, replay
                got = run(g, d_xy, len(xy))
                assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
            want_big = run(direct, d_big, len(big))
            got_big = run(g, d_big, len(big))  # grows the scratch: captured graphs are stale
            assert np.array_equal(got_big[0], want_big[0])
            d_xy.copy_(torch.flip(d_xy, [0]))  # new contents, same address
            want2 = run(direct, d_xy, len(xy))
            for _ in range(3):
                got2 = run(g, d_xy, len(xy))
                assert np.array_equal(got2[0], want2[0]) and np.array_equal(got2[1], want2[1])


@pytest.mark.parametrize("n_edges", [3, 63, 64, 65, 1023, 2047, 2048, 2049, 4095, 4097, 6143, 32767, 32769])
def test_scan_chunk_and_tile_boundaries(engine, n_edges):
    """Edge counts around the scan kernel's key tiles (2048), 4-word copy
    granularity, 64-edge chunks and the 32768-edge wave switch: the fast path
    equals the literal loop (PC_OPT_EXACT) on 300k y-ordered points, all modes."""
    poly = W.star_polygon(n_edges, seed=n_edges)
    xy = W.uniform_points(300_000, W.bounds(poly), n_edges + 1)
    with Engine(devices=[0]) as ex:
        ex.set_exact(True)
        for mode in MODES:
            a = engine.classify(xy, poly, mode, verdicts=False)
            b = ex.classify(xy, poly, mode, verdicts=False)
            assert np.array_equal(a.inside_bits, b.inside_bits) and np.array_equal(a.aux_bits, b.aux_bits), mode
            assert np.array_equal(a.stats, b.stats)
