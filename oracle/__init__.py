"""TEST INFRASTRUCTURE — the parity checkers.  Never the product path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.

  ref   oracle/_ref/libpolycast_ref.so — the UNMODIFIED reference implementation
        (proj/include/polycast/{geometry,batch}.hpp compiled from
        /root/reference by oracle/Makefile) behind a C-ABI shim.
  port  oracle/build/libpip_oracle.so — plain-C restatement over raw arrays
        (pip_oracle.c), pinned against `ref` and the reference's KATs in tests/,
        used where the reference types cannot express the input (P8).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libpolycast_ref.so")
PORT_LIB = os.path.join(HERE, "build", "libpip_oracle.so")

_vp = C.c_void_p


def _p(a):
    return None if a is None else a.ctypes.data


class RefError(RuntimeError):
    pass


_ref = None
_port = None


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_LIB)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_classify.argtypes = [_vp, C.c_uint64, _vp, _vp, _vp, C.c_uint32, C.c_int, C.c_double, C.c_uint64,
                                     _vp, _vp]
        lib.ref_prepare.argtypes = [_vp, C.c_uint64, _vp, _vp, _vp, C.c_uint32]
        lib.ref_prepare.restype = _vp
        lib.ref_prepared_free.argtypes = [_vp]
        lib.ref_run_prepared.argtypes = [_vp, C.c_int, C.c_double, C.c_uint64, _vp]
        lib.ref_contains.argtypes = [C.c_double, C.c_double, _vp, _vp, _vp, C.c_uint32, C.c_int, C.c_double]
        lib.ref_count_crossings.argtypes = [C.c_double, C.c_double, _vp, _vp, C.c_uint64, C.c_int, _vp]
        lib.ref_bbox_of.argtypes = [_vp, _vp, _vp, C.c_uint32, _vp]
        lib.ref_classify_csr.argtypes = [_vp, _vp, C.c_uint64, _vp, _vp, _vp, _vp, C.c_int, C.c_double, C.c_uint64,
                                         _vp, _vp]
        lib.ref_default_worker_count.restype = C.c_uint64
        if hasattr(lib, "ref_parse_double"):
            lib.ref_parse_double.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(C.c_double)]
            lib.ref_parse_double.restype = C.c_int
            lib.ref_read_points_csv.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, C.c_int,
                                                C.c_char, C.c_int, _vp, C.c_uint64, _vp, _vp, _vp, C.c_char_p,
                                                C.c_uint64]
            lib.ref_read_points_csv.restype = C.c_int
        if hasattr(lib, "ref_write_results_csv"):
            lib.ref_write_results_csv.argtypes = [C.c_char_p, _vp, _vp, _vp, C.c_uint64]
            lib.ref_write_results_csv.restype = C.c_int
        _ref = lib
    return _ref


def port():
    global _port
    if _port is None:
        lib = C.CDLL(PORT_LIB)
        lib.orc_classify.argtypes = [_vp, C.c_uint64, _vp, _vp, _vp, C.c_uint32, C.c_int, C.c_double, C.c_int, _vp,
                                     _vp, C.c_int]
        lib.orc_classify_csr.argtypes = [_vp, _vp, C.c_uint64, _vp, _vp, _vp, _vp, C.c_int, C.c_double, _vp, _vp,
                                         C.c_int]
        lib.orc_count_crossings.argtypes = [_vp, C.c_uint64, _vp, _vp, C.c_uint64, C.c_int, _vp, _vp]
        lib.orc_bbox.argtypes = [_vp, _vp, _vp, C.c_uint64, _vp]
        _port = lib
    return _port


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# ---- reference (unmodified polycast) ------------------------------------------

def ref_classify(xy, vx, vy, ring_off, mode, tol=1e-12, workers=0):
    """Reference classify_batch -> (verdicts uint8[n], stats uint64[4])."""
    xy, vx, vy, ro = _c(xy, np.float64), _c(vx, np.float64), _c(vy, np.float64), _c(ring_off, np.uint64)
    n = xy.size // 2
    v = np.empty(n, np.uint8)
    st = np.zeros(4, np.uint64)
    rc = ref().ref_classify(_p(xy), n, _p(vx), _p(vy), _p(ro), len(ro) - 1, int(mode), float(tol), workers, _p(v),
                            _p(st))
    if rc != 0:
        raise RefError(ref().ref_last_error().decode())
    return v, st


def ref_contains(p, vx, vy, ring_off, mode, tol=1e-12):
    """Reference contains(): 0 Inside, 1 Outside, 2 Boundary, 3 = DegenerateEdge thrown."""
    vx, vy, ro = _c(vx, np.float64), _c(vy, np.float64), _c(ring_off, np.uint64)
    r = ref().ref_contains(float(p[0]), float(p[1]), _p(vx), _p(vy), _p(ro), len(ro) - 1, int(mode), float(tol))
    if r < 0:
        raise RefError(ref().ref_last_error().decode())
    return r


def ref_count_crossings(p, vx, vy, mode):
    """Reference count_crossings_c1/_c2 -> count, or None when DegenerateEdge is thrown."""
    vx, vy = _c(vx, np.float64), _c(vy, np.float64)
    cnt = np.zeros(1, np.uint64)
    r = ref().ref_count_crossings(float(p[0]), float(p[1]), _p(vx), _p(vy), len(vx), int(mode), _p(cnt))
    if r == 3:
        return None
    if r != 0:
        raise RefError(ref().ref_last_error().decode())
    return int(cnt[0])


def ref_classify_csr(s, mode, tol=1e-12, threads=0):
    n = s.n_points
    v = np.empty(n, np.uint8)
    st = np.zeros(4, np.uint64)
    rc = ref().ref_classify_csr(_p(s.xy), _p(s.pt_off), s.n_polys, _p(s.vx), _p(s.vy), _p(s.ring_off),
                                _p(s.poly_ring_off), int(mode), float(tol), threads, _p(v), _p(st))
    if rc != 0:
        raise RefError(ref().ref_last_error().decode())
    return v, st


class RefPrepared:
    """Reference Polygon + PointBatch built once (outside any timer)."""

    def __init__(self, xy, vx, vy, ring_off):
        self._keep = [_c(xy, np.float64), _c(vx, np.float64), _c(vy, np.float64), _c(ring_off, np.uint64)]
        xy, vx, vy, ro = self._keep
        self.h = ref().ref_prepare(_p(xy), xy.size // 2, _p(vx), _p(vy), _p(ro), len(ro) - 1)
        if not self.h:
            raise RefError(ref().ref_last_error().decode())

    def run(self, mode, tol=1e-12, workers=0):
        st = np.zeros(4, np.uint64)
        ref().ref_run_prepared(self.h, int(mode), float(tol), workers, _p(st))
        return st

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_prepared_free(self.h)
            self.h = None


def host_threads() -> int:
    return int(ref().ref_default_worker_count()) if ref_available() else (os.cpu_count() or 1)


# ---- C restatement ----------------------------------------------------------------

def port_classify(xy, vx, vy, ring_off, mode, tol=1e-12, prefilter=True, threads=1):
    xy, vx, vy, ro = _c(xy, np.float64), _c(vx, np.float64), _c(vy, np.float64), _c(ring_off, np.uint64)
    n = xy.size // 2
    v = np.empty(n, np.uint8)
    st = np.zeros(4, np.uint64)
    port().orc_classify(_p(xy), n, _p(vx), _p(vy), _p(ro), len(ro) - 1, int(mode), float(tol), int(bool(prefilter)),
                        _p(v), _p(st), threads)
    return v, st


def port_classify_csr(s, mode, tol=1e-12, threads=1):
    n = s.n_points
    v = np.empty(n, np.uint8)
    st = np.zeros(4, np.uint64)
    port().orc_classify_csr(_p(s.xy), _p(s.pt_off), s.n_polys, _p(s.vx), _p(s.vy), _p(s.ring_off),
                            _p(s.poly_ring_off), int(mode), float(tol), _p(v), _p(st), threads)
    return v, st


def port_count_crossings(xy, vx, vy, mode):
    xy, vx, vy = _c(xy, np.float64), _c(vx, np.float64), _c(vy, np.float64)
    n = xy.size // 2
    counts = np.zeros(n, np.uint64)
    err = np.zeros(n, np.uint8)
    port().orc_count_crossings(_p(xy), n, _p(vx), _p(vy), len(vx), int(mode), _p(counts), _p(err))
    return counts, err


# ---- reference CSV reader / number parser (io.hpp; ref_io_shim.cpp) -----------------------

def ref_parse_double(cell: bytes):
    """(ok, value) of the reference's detail::parse_double (io.hpp:116-124)."""
    lib = ref()
    out = C.c_double(0.0)
    ok = lib.ref_parse_double(C.c_char_p(cell), C.c_uint64(len(cell)), C.byref(out))
    return bool(ok), out.value


def ref_read_points_csv(path, x=1, y=2, has_header=True, delim=",", lenient=False, cap=None):
    """The reference's read_points_csv (io.hpp:148-225) -> dict(kind, points, skipped, row, msg);
    x / y: column name (str) or index (int); kind 0 = ok, 1 CsvParseError, 2 ColumnMissing,
    3 FileNotFound, 4 IoError, 5 invalid_argument."""
    lib = ref()
    if cap is None:
        cap = os.path.getsize(path) // 2 + 16 if os.path.exists(path) else 16
    out = np.empty((cap, 2), np.float64)
    n, sk, row = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
    msg = C.create_string_buffer(1024)
    xs = x.encode() if isinstance(x, str) else None
    ys = y.encode() if isinstance(y, str) else None
    k = lib.ref_read_points_csv(str(path).encode(), xs, 0 if xs else int(x), ys, 0 if ys else int(y),
                                int(bool(has_header)), delim.encode(), int(bool(lenient)),
                                out.ctypes.data_as(C.c_void_p), C.c_uint64(cap), C.byref(n), C.byref(sk),
                                C.byref(row), msg, C.c_uint64(1024))
    return {"kind": k, "points": out[:min(n.value, cap)].copy(), "skipped": sk.value, "row": row.value,
            "msg": msg.value.decode(errors="replace")}


def ref_write_results_csv(path, index, xy, verdict):
    """The reference's write_results_csv (io.hpp:325-335) -> 0 ok, 4 IoError, 6 other."""
    idx = _c(index, np.uint64)
    xy = _c(xy, np.float64)
    v = _c(verdict, np.uint8)
    return ref().ref_write_results_csv(str(path).encode(), _p(idx), _p(xy), _p(v), len(v))
