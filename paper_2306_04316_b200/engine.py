"""Python host interface over the C-ABI (mirrors the reference's batch API).

Reference interface mirrored (names, argument meaning, error behaviour):
  classify_batch(batch, poly, mode, workers=0, boundary_tol=1e-12)
      proj/include/polycast/batch.hpp:184-230  -> Engine.classify_batch
  contains(p, poly, mode, boundary_tol)  geometry.hpp:281-300 -> Engine.contains
  count_crossings_c1/_c2(p, ring)        geometry.hpp:182-229 -> Engine.count_crossings
plus the CSR multi-polygon batch and device-pointer calls
for kernel-only timing.  Every call goes to libpolycast_cuda.so; there is no
CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _native

DEFAULT_BOUNDARY_TOL = 1e-12


class CrossingMode(IntEnum):  # geometry.hpp:107
    C1 = 0
    C2 = 1
    Robust = 2


class Verdict(IntEnum):  # batch.hpp:60
    Inside = 0
    Outside = 1
    Boundary = 2
    Error = 3


class Classification(IntEnum):  # geometry.hpp:96
    Inside = 0
    Outside = 1
    Boundary = 2


class DegenerateEdge(RuntimeError):
    """Mirrors polycast::DegenerateEdge (geometry.hpp:19-21)."""


class DeviceError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


# pc_result_record / polycast::ResultRecord (32 bytes)
RESULT_RECORD = np.dtype({"names": ["index", "x", "y", "verdict"], "formats": [np.uint64, np.float64, np.float64,
                                                                               np.uint8],
                          "offsets": [0, 8, 16, 24], "itemsize": 32})


def make_records(index, xy, verdict) -> np.ndarray:
    """Records for format_results_csv from an index array, (n, 2) points and verdict bytes."""
    n = len(verdict)
    xy = np.asarray(xy, np.float64).reshape(n, 2)
    recs = np.zeros(n, dtype=RESULT_RECORD)
    recs["index"], recs["x"], recs["y"], recs["verdict"] = index, xy[:, 0], xy[:, 1], verdict
    return recs


def _ptr(a) -> int | None:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags.c_contiguous
        return a.ctypes.data
    return int(a.data_ptr())  # torch tensor


@dataclass
class Polygon:
    """SoA polygon: closed rings [ring_off[r], ring_off[r+1]) of vx/vy; ring 0 outer."""
    vx: np.ndarray
    vy: np.ndarray
    ring_off: np.ndarray = field(default=None)

    def __post_init__(self):
        self.vx = np.ascontiguousarray(self.vx, dtype=np.float64)
        self.vy = np.ascontiguousarray(self.vy, dtype=np.float64)
        if self.ring_off is None:
            self.ring_off = np.array([0, len(self.vx)], dtype=np.uint64)
        self.ring_off = np.ascontiguousarray(self.ring_off, dtype=np.uint64)

    @classmethod
    def from_rings(cls, rings):
        """rings: list of sequences of (x, y), each closed (first == last)."""
        xs, ys, off = [], [], [0]
        for r in rings:
            r = np.asarray(r, dtype=np.float64).reshape(-1, 2)
            xs.append(r[:, 0])
            ys.append(r[:, 1])
            off.append(off[-1] + len(r))
        return cls(np.concatenate(xs), np.concatenate(ys), np.array(off, dtype=np.uint64))

    @property
    def n_rings(self) -> int:
        return len(self.ring_off) - 1

    @property
    def n_verts(self) -> int:
        return int(self.ring_off[-1])

    @property
    def n_edges(self) -> int:
        return self.n_verts - self.n_rings


@dataclass
class CsrSet:
    """Many polygons with their own points (CSR): see pc_classify_csr."""
    xy: np.ndarray            # (n_points, 2) float64
    pt_off: np.ndarray        # (P+1,) uint64
    vx: np.ndarray
    vy: np.ndarray
    ring_off: np.ndarray      # (R+1,) uint64 into vx/vy
    poly_ring_off: np.ndarray  # (P+1,) uint64 into rings

    @property
    def n_polys(self) -> int:
        return len(self.pt_off) - 1

    @property
    def n_points(self) -> int:
        return int(self.pt_off[-1] - self.pt_off[0])

    def edges_per_point(self) -> np.ndarray:
        """Point-edge tests each polygon's points cost (edges of all its rings)."""
        ring_edges = np.diff(self.ring_off.astype(np.int64)) - 1
        csum = np.concatenate([[0], np.cumsum(ring_edges)])
        pr = self.poly_ring_off.astype(np.int64)
        return csum[pr[1:]] - csum[pr[:-1]]

    def work(self) -> int:
        return int((np.diff(self.pt_off.astype(np.int64)) * self.edges_per_point()).sum())


@dataclass
class Result:
    verdicts: np.ndarray | None
    inside_bits: np.ndarray | None
    aux_bits: np.ndarray | None
    stats: np.ndarray  # inside, outside, boundary, error


class Engine:
    """A libpolycast_cuda context over one or more GPUs."""

    def __init__(self, num_gpus: int = 0, devices=None):
        self.lib = _native.load()
        h = C.c_void_p()
        if devices is not None:
            arr = (C.c_int * len(devices))(*devices)
            rc = self.lib.pc_create_devices(C.byref(h), arr, len(devices))
        else:
            rc = self.lib.pc_create(C.byref(h), num_gpus)
        if rc != _native.PC_OK or not h.value:
            raise DeviceError(rc, "pc_create failed: no usable CUDA device (there is no CPU fallback)")
        self.ctx = h

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.pc_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def device_count(self) -> int:
        return self.lib.pc_device_count(self.ctx)

    @property
    def last_launch_count(self) -> int:
        return int(self.lib.pc_last_launch_count(self.ctx))

    # ---- measurement hooks -----------------------------------------------------
    def set_option(self, option: int, value: int):
        self._check(self.lib.pc_set_option(self.ctx, int(option), int(value)), "pc_set_option")

    def set_bucketing(self, mode: int):
        """-1 auto, 0 off, 1 on (PC_OPT_BUCKET_POINTS); never changes results."""
        self.set_option(1, mode)

    def set_tree(self, mode: int):
        """0 off (default), 1 on (PC_OPT_TREE): the opt-in segment-tree path for C1/C2
        single polygons -- an extension outside the reference's linear scan; never
        changes results."""
        self.set_option(2, mode)

    def set_graphs(self, on: bool):
        """PC_OPT_GRAPH (default on): repeated identical device-pointer calls replay
        a captured CUDA graph."""
        self.set_option(4, int(bool(on)))

    def set_exact(self, on: bool):
        """PC_OPT_EXACT: run only the literal binary64 loop (pip_exact.cu), the
        full-size checker of the fast path."""
        self.set_option(3, int(bool(on)))

    def set_profiling(self, on: bool = True):
        self._check(self.lib.pc_set_profiling(self.ctx, int(bool(on))), "pc_set_profiling")

    def profile_take(self, dev_index: int = 0) -> list[float]:
        buf = (C.c_double * 4096)()
        k = self.lib.pc_profile_take(self.ctx, dev_index, buf, 4096)
        return [buf[i] for i in range(min(k, 4096))]

    def fp64_rate(self, dev_index: int = 0, ms: float = 200.0) -> float:
        out = C.c_double()
        self._check(self.lib.pc_measure_fp64_rate(self.ctx, dev_index, ms, C.byref(out)), "pc_measure_fp64_rate")
        return out.value

    def _check(self, rc, where):
        if rc != _native.PC_OK:
            raise DeviceError(rc, f"{where}: {self.lib.pc_last_error(self.ctx).decode()}")

    # ---- host-pointer API ---------------------------------------------------
    def classify(self, xy: np.ndarray, poly: Polygon, mode=CrossingMode.C1, boundary_tol=DEFAULT_BOUNDARY_TOL,
                 prefilter=True, verdicts=True, bits=True, out=None) -> Result:
        """`out` = optional (verdicts, inside_bits, aux_bits) preallocated (e.g. pinned) arrays."""
        xy = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, 2)
        n = len(xy)
        nw = (n + 31) // 32
        if out is not None:
            v, ib, ab = out
        else:
            v = np.empty(n, np.uint8) if verdicts else None
            ib = np.empty(nw, np.uint32) if bits else None
            ab = np.empty(nw, np.uint32) if bits else None
        st = np.zeros(4, np.uint64)
        rc = self.lib.pc_classify(self.ctx, _ptr(xy), n, _ptr(poly.vx), _ptr(poly.vy), _ptr(poly.ring_off),
                                  poly.n_rings, int(mode), float(boundary_tol), int(bool(prefilter)), _ptr(v),
                                  _ptr(ib), _ptr(ab), _ptr(st))
        self._check(rc, "pc_classify")
        return Result(v, ib, ab, st)

    def classify_batch(self, xy, poly: Polygon, mode=CrossingMode.C1, workers: int = 0,
                       boundary_tol=DEFAULT_BOUNDARY_TOL) -> Result:
        """batch.hpp:184 semantics (bbox prefilter); `workers` does not change the output."""
        del workers
        return self.classify(xy, poly, mode, boundary_tol, prefilter=True)

    def contains(self, p, poly: Polygon, mode=CrossingMode.C1, boundary_tol=DEFAULT_BOUNDARY_TOL):
        """geometry.hpp:281 semantics (no prefilter); C2 degenerate raises DegenerateEdge."""
        r = self.classify(np.array([p], np.float64), poly, mode, boundary_tol, prefilter=False, bits=False)
        v = int(r.verdicts[0])
        if v == Verdict.Error:
            raise DegenerateEdge("contains: horizontal edge lies on the query ray")
        return Classification(v)

    def classify_csr(self, s: CsrSet, mode=CrossingMode.C1, boundary_tol=DEFAULT_BOUNDARY_TOL,
                     verdicts=True, bits=True, out=None) -> Result:
        n = s.n_points
        nw = (n + 31) // 32
        if out is not None:
            v, ib, ab = out
        else:
            v = np.empty(n, np.uint8) if verdicts else None
            ib = np.empty(nw, np.uint32) if bits else None
            ab = np.empty(nw, np.uint32) if bits else None
        st = np.zeros(4, np.uint64)
        rc = self.lib.pc_classify_csr(self.ctx, _ptr(s.xy), _ptr(s.pt_off), s.n_polys, _ptr(s.vx), _ptr(s.vy),
                                      _ptr(s.ring_off), _ptr(s.poly_ring_off), int(mode), float(boundary_tol),
                                      _ptr(v), _ptr(ib), _ptr(ab), _ptr(st))
        self._check(rc, "pc_classify_csr")
        return Result(v, ib, ab, st)

    def count_crossings(self, xy, vx, vy, mode=CrossingMode.C1):
        """Per-point crossing counts of one closed ring; returns (counts, degenerate flags)."""
        xy = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, 2)
        vx = np.ascontiguousarray(vx, dtype=np.float64)
        vy = np.ascontiguousarray(vy, dtype=np.float64)
        n = len(xy)
        counts = np.zeros(n, np.uint64)
        deg = np.zeros(n, np.uint8)
        rc = self.lib.pc_count_crossings(self.ctx, _ptr(xy), n, _ptr(vx), _ptr(vy), len(vx), int(mode),
                                         _ptr(counts), _ptr(deg))
        self._check(rc, "pc_count_crossings")
        return counts, deg

    def prefilter_bbox(self, xy, box):
        """prefilter_bbox (batch.hpp:137-153) on the GPU: (inside_xy, original_indices,
        outside_count) for the closed box (min_x, min_y, max_x, max_y), input order kept."""
        xy = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, 2)
        b = np.ascontiguousarray(box, dtype=np.float64).reshape(4)
        n = len(xy)
        out = np.empty((n, 2), np.float64)
        idx = np.empty(n, np.uint64)
        k = C.c_uint64(0)
        rc = self.lib.pc_prefilter_bbox(self.ctx, _ptr(xy), n, _ptr(b), _ptr(out), _ptr(idx), C.byref(k))
        self._check(rc, "pc_prefilter_bbox")
        return out[:k.value], idx[:k.value], n - k.value

    def scatter_verdicts(self, original_indices, inbox_verdicts, n_total):
        """scatter_verdicts (batch.hpp:157-168) on the GPU: full-length verdicts, Outside where filtered."""
        idx = np.ascontiguousarray(original_indices, dtype=np.uint64)
        v = np.ascontiguousarray(inbox_verdicts, dtype=np.uint8)
        if len(idx) != len(v):
            raise ValueError("scatter_verdicts: verdict count does not match index map")
        out = np.empty(int(n_total), np.uint8)
        rc = self.lib.pc_scatter_verdicts(self.ctx, _ptr(idx), _ptr(v), len(v), int(n_total), _ptr(out))
        self._check(rc, "pc_scatter_verdicts")
        return out

    def parse_points_csv(self, text: bytes, data_start: int, x_col: int, y_col: int, delim: str = ","):
        """The data-row loop of read_points_csv on the GPU (pc_parse_points_csv):
        (xy float64 (n,2) of the good rows in file order, n_bad, byte offset of the
        first bad row's line or None, its kind (2 short row, 3 x cell, 4 y cell))."""
        buf = np.frombuffer(text, dtype=np.uint8) if len(text) else np.zeros(1, np.uint8)
        cap = (len(text) + 1) // 4 + 1  # a good row takes >= 4 bytes ("d,d\n") except the file's last
        out = np.empty((cap, 2), np.float64)  # untouched pages cost nothing
        n, bad, fb, kind = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0), C.c_uint32(0)
        rc = self.lib.pc_parse_points_csv(self.ctx, _ptr(buf), len(text), int(data_start), int(x_col), int(y_col),
                                          delim.encode(), _ptr(out), cap, C.byref(n), C.byref(bad), C.byref(fb),
                                          C.byref(kind))
        self._check(rc, "pc_parse_points_csv")
        first = None if fb.value == 2 ** 64 - 1 else fb.value
        return out[:n.value], bad.value, first, kind.value

    def format_results_csv(self, recs: np.ndarray) -> np.ndarray:
        """write_results_csv's text on the GPU (pc_format_results_csv) for records of
        dtype RESULT_RECORD (see make_records): header plus one "index,x,y,verdict"
        row per record, coordinates as printf("%.17g").  Returns the bytes (uint8)."""
        assert recs.dtype == RESULT_RECORD and recs.flags.c_contiguous
        n = len(recs)
        cap = 18 + 80 * n
        out = np.empty(cap, np.uint8)  # untouched pages past the text cost nothing
        ln = C.c_uint64(0)
        rc = self.lib.pc_format_results_csv(self.ctx, _ptr(recs) if n else None, n, _ptr(out), cap, C.byref(ln))
        self._check(rc, "pc_format_results_csv")
        return out[:ln.value]

    def format_results_csv_dev(self, dev_index, stream_ptr, d_recs, n, d_out, cap, d_len):
        rc = self.lib.pc_format_results_csv_dev(self.ctx, dev_index, stream_ptr, _ptr(d_recs), int(n), _ptr(d_out),
                                                int(cap), _ptr(d_len))
        self._check(rc, "pc_format_results_csv_dev")

    def parse_points_csv_dev(self, dev_index, stream_ptr, d_text, n_bytes, data_start, x_col, y_col, delim,
                             d_out_xy, cap_points, d_result):
        rc = self.lib.pc_parse_points_csv_dev(self.ctx, dev_index, stream_ptr, _ptr(d_text), int(n_bytes),
                                              int(data_start), int(x_col), int(y_col), delim.encode(),
                                              _ptr(d_out_xy), int(cap_points), _ptr(d_result))
        self._check(rc, "pc_parse_points_csv_dev")

    # ---- device-pointer API (torch tensors as HBM buffers) ------------------
    def classify_dev(self, dev_index, stream_ptr, d_xy, n, d_vx, d_vy, d_ring_off, n_rings, n_verts, mode,
                     boundary_tol, prefilter, d_inside, d_aux, d_stats, d_verdicts=None):
        rc = self.lib.pc_classify_dev(self.ctx, dev_index, stream_ptr, _ptr(d_xy), n, _ptr(d_vx), _ptr(d_vy),
                                      _ptr(d_ring_off), n_rings, n_verts, int(mode), float(boundary_tol),
                                      int(bool(prefilter)), _ptr(d_verdicts), _ptr(d_inside), _ptr(d_aux),
                                      _ptr(d_stats))
        self._check(rc, "pc_classify_dev")

    def classify_csr_dev(self, dev_index, stream_ptr, d_xy, d_pt_off, n_polys, n_points, d_vx, d_vy, d_ring_off,
                         d_poly_ring_off, mode, boundary_tol, d_inside, d_aux, d_stats, d_verdicts=None):
        rc = self.lib.pc_classify_csr_dev(self.ctx, dev_index, stream_ptr, _ptr(d_xy), _ptr(d_pt_off), n_polys,
                                          n_points, _ptr(d_vx), _ptr(d_vy), _ptr(d_ring_off), _ptr(d_poly_ring_off),
                                          int(mode), float(boundary_tol), _ptr(d_verdicts), _ptr(d_inside),
                                          _ptr(d_aux), _ptr(d_stats))
        self._check(rc, "pc_classify_csr_dev")


def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    """Bit plane (bit i%32 of word i//32) -> bool[n]."""
    b = np.unpackbits(words.view(np.uint8), bitorder="little")
    return b[:n].astype(bool)


def pack_bits(flags: np.ndarray) -> np.ndarray:
    n = len(flags)
    nw = (n + 31) // 32
    padded = np.zeros(nw * 32, np.uint8)
    padded[:n] = flags.astype(np.uint8)
    return np.packbits(padded, bitorder="little").view(np.uint32)


def verdicts_to_bits(verdicts: np.ndarray, mode) -> tuple[np.ndarray, np.ndarray]:
    aux_v = Verdict.Boundary if int(mode) == CrossingMode.Robust else Verdict.Error
    return pack_bits(verdicts == Verdict.Inside), pack_bits(verdicts == aux_v)
