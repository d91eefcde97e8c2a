"""the linearity fit of the benchmark harness.

Three implementations of the reference's least_squares_fit / error_report
(proj/include/polycast/bench.hpp:123-198) must agree:
  * the UNMODIFIED reference (oracle/_ref, ref_bench_shim.cpp),
  * the drop-in C++ header include/polycast/bench.hpp (tests/cpp/bench_shim.cpp),
  * bench.py's lsq_fit / error_rows (the fit on the GPU sweep timings).
Inputs: the paper's published timing tables (PAPER.md, Table-projection-small:
10 sizes x 6 implementations, and Table-projection-large for the error report)
and the GPU sweep timings of this round's committed bench line.  Tolerance:
1e-9 relative (the three restate the same operation order, so in practice the
results are bit-identical).  Also: random_batch (bench.hpp:62-80) bit-identical
to the reference's, and emit_report / read_samples_csv round trip.
"""
import ctypes as C
import glob
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

SHIM = os.path.join(ROOT, "tests", "cpp", "libbench_shim.so")
TOL = 1e-9

# PAPER.md Table-projection-small: points, then seconds per implementation
SMALL_N = [10, 1120, 2230, 3340, 4450, 5560, 6670, 7780, 8890, 10000]
SMALL = {
    "Algorithm_2": [0.000797, 0.085122, 0.160281, 0.218364, 0.289474, 0.366708, 0.424220, 0.497226, 0.572252, 0.639463],
    "Algorithm_1": [0.000678, 0.080887, 0.170801, 0.224381, 0.298039, 0.391248, 0.449986, 0.523772, 0.640621, 0.667802],
    "numba": [0.000455, 0.053803, 0.100509, 0.150193, 0.204831, 0.251546, 0.298660, 0.348369, 0.413792, 0.446130],
    "numba_p": [0.000193, 0.011901, 0.021441, 0.030485, 0.047858, 0.049396, 0.058415, 0.070565, 0.081335, 0.090945],
    "opencv": [0.000885, 0.060541, 0.119104, 0.176672, 0.239670, 0.283920, 0.331706, 0.387975, 0.448136, 0.494594],
    "shapely": [0.040110, 3.921390, 7.746753, 11.664765, 15.478461, 19.261769, 23.099383, 27.049710, 30.752390,
                34.666056],
}
# PAPER.md Table-lsq (the paper's own fit of the small table, 6 decimals)
PAPER_LSQ = {"Algorithm_2": (0.000063, 0.010103), "Algorithm_1": (0.000068, 0.004402), "numba": (0.000045, 0.001039),
             "numba_p": (0.000009, 0.001607), "opencv": (0.000049, 0.008094), "shapely": (0.003462, 0.041119)}
# PAPER.md Table-projection-large
LARGE_N = [1908647, 3807294, 5705941, 7604588, 9503235, 11401882, 13300529, 15199176, 17097823]
LARGE = {
    "Algorithm_2": [120.244296, 239.848545, 359.452793, 479.057041, 598.661289, 718.265538, 837.869786, 957.474034,
                    1077.078283],
    "numba_p": [17.027383, 33.963956, 50.900529, 67.837102, 84.773674, 101.710247, 118.646820, 135.583393, 152.519965],
}

_u64 = np.uint64


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


@pytest.fixture(scope="module")
def shims():
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = oracle.ref()
    if not hasattr(ref, "ref_least_squares_fit"):
        pytest.skip("oracle/_ref built without the bench shim (needs nlohmann json)")
    if not os.path.exists(SHIM):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp"), SHIM], check=True)
    ours = C.CDLL(SHIM)
    for lib, pre in ((ref, "ref"), (ours, "our")):
        f = getattr(lib, f"{pre}_least_squares_fit")
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        f.restype = C.c_int
        g = getattr(lib, f"{pre}_error_report")
        g.argtypes = [C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        g.restype = None
        h = getattr(lib, f"{pre}_random_batch")
        h.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
        h.restype = None
    ours.our_report_roundtrip.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_char_p, C.c_char_p]
    ours.our_report_roundtrip.restype = C.c_int
    return {"ref": ref, "our": ours}


def fit_c(lib, pre, x, t):
    n = np.ascontiguousarray(x, _u64)
    tt = np.ascontiguousarray(t, np.float64)
    s, i = C.c_double(), C.c_double()
    rc = getattr(lib, f"{pre}_least_squares_fit")(_p(n), _p(tt), len(n), C.byref(s), C.byref(i))
    return None if rc else (s.value, i.value)


def report_c(lib, pre, fit, x, t):
    n = np.ascontiguousarray(x, _u64)
    tt = np.ascontiguousarray(t, np.float64)
    pr, ab, rl = (np.zeros(len(n)) for _ in range(3))
    getattr(lib, f"{pre}_error_report")(fit[0], fit[1], _p(n), _p(tt), len(n), _p(pr), _p(ab), _p(rl))
    return pr, ab, rl


def close(a, b):
    return abs(a - b) <= TOL * max(abs(a), abs(b), 1e-300)


def three_fits(shims, x, t):
    r = fit_c(shims["ref"], "ref", x, t)
    o = fit_c(shims["our"], "our", x, t)
    p = bench.lsq_fit(x, t)
    for a, b in ((r, o), (r, p)):
        assert close(a[0], b[0]) and close(a[1], b[1]), (a, b)
    return r


@pytest.mark.parametrize("alg", sorted(SMALL))
def test_paper_small_table_fit(shims, alg):
    r = three_fits(shims, SMALL_N, SMALL[alg])
    # the paper's own fit (PAPER.md Table-lsq), rounded to 6 decimals there
    ps, pi = PAPER_LSQ[alg]
    assert abs(r[0] - ps) <= 5.01e-7 and abs(r[1] - pi) <= 5.01e-7 + 1e-6, (alg, r, (ps, pi))


@pytest.mark.parametrize("alg", sorted(LARGE))
def test_paper_large_table_error_report(shims, alg):
    fit = three_fits(shims, SMALL_N, SMALL[alg])
    pr_r, ab_r, rl_r = report_c(shims["ref"], "ref", fit, LARGE_N, LARGE[alg])
    pr_o, ab_o, rl_o = report_c(shims["our"], "our", fit, LARGE_N, LARGE[alg])
    rows = bench.error_rows(fit[0], fit[1], LARGE_N, LARGE[alg])
    for k, (p, a, rel) in enumerate(rows):
        for ref_v, our_v, py_v in ((pr_r[k], pr_o[k], p), (ab_r[k], ab_o[k], a), (rl_r[k], rl_o[k], rel)):
            assert close(ref_v, our_v) and close(ref_v, py_v), (alg, k, ref_v, our_v, py_v)


def test_degenerate_fit(shims):
    assert fit_c(shims["ref"], "ref", [5, 5, 5], [1.0, 2.0, 3.0]) is None
    assert fit_c(shims["our"], "our", [5, 5, 5], [1.0, 2.0, 3.0]) is None
    assert fit_c(shims["our"], "our", [5], [1.0]) is None
    with pytest.raises(ValueError):
        bench.lsq_fit([5, 5], [1.0, 2.0])


def _committed_sweeps():
    """GPU sweep timings from the committed bench lines (profiles/*_bench.jsonl)."""
    out = []
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r2*_bench.jsonl"))):
        for ln in open(f):
            d = json.loads(ln)
            sw = d.get("sweep")
            if sw and sw.get("kernel_ms"):
                out.append((os.path.basename(f), sw))
    return out


def test_gpu_sweep_fit_matches_reference(shims):
    sweeps = _committed_sweeps()
    if not sweeps:
        pytest.skip("no committed sweep timings yet")
    for name, sw in sweeps:
        labels = list(sw["kernel_ms"])
        n = [int(lb.split("=")[1]) for lb in labels]
        t = [sw["kernel_ms"][lb] / 1e3 for lb in labels]
        r = three_fits(shims, n, t)
        assert close(r[0], sw["fit"]["slope_s_per_edge"]) and close(r[1], sw["fit"]["intercept_s"]), name
        rows = report_c(shims["ref"], "ref", r, n, t)[2]
        for lb, rel in zip(labels, rows):
            assert close(rel, sw["fit"]["rel_err"][lb]), (name, lb)
        # the paper's O(n) claim: linear in n on the scan path
        assert sw["fit"]["r2"] >= 0.99, (name, sw["fit"]["r2"])


def test_random_batch_identical(shims):
    for box, n, seed in (((-1.0, -2.0, 3.0, 4.0), 1000, 7), ((0.0, 5.0, 1e-3, 5.001), 257, 2 ** 40 + 3)):
        b = np.ascontiguousarray(box, np.float64)
        a_r = np.zeros(2 * n)
        a_o = np.zeros(2 * n)
        shims["ref"].ref_random_batch(_p(b), n, seed, _p(a_r))
        shims["our"].our_random_batch(_p(b), n, seed, _p(a_o))
        assert np.array_equal(a_r.view(np.uint64), a_o.view(np.uint64))


def test_report_roundtrip(shims, tmp_path):
    n = np.ascontiguousarray(SMALL_N, _u64)
    t = np.ascontiguousarray(SMALL["numba"], np.float64)
    js, cs = str(tmp_path / "r.json"), str(tmp_path / "s.csv")
    assert shims["our"].our_report_roundtrip(_p(n), _p(t), len(n), js.encode(), cs.encode()) == len(n)
    doc = json.load(open(js))
    assert [s["n"] for s in doc["samples"]] == SMALL_N and len(doc["fits"]) == 1 and len(doc["errors"]) == len(n)
    flat = open(str(tmp_path / "r.csv")).read().splitlines()
    assert flat[0] == "n,algorithm,actual_s,predicted_s" and len(flat) == len(n) + 1
    assert all(not math.isnan(e["relative_error"]) for e in doc["errors"])
