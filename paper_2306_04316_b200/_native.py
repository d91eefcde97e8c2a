"""ctypes binding of libpolycast_cuda.so (include/polycast_cuda.h).

The shared library is built in-tree by ``make -C paper_2306_04316_b200`` (or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
or no GPU is usable, loading / context creation raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")
# POLYCAST_LIB_VARIANT=<dir> selects a build under lib/<dir>: "debug" is the
# checking build (device-side bounds checks, `make -C paper_2306_04316_b200 debug`)
CUDA_LIB = os.path.join(LIB_DIR, os.environ.get("POLYCAST_LIB_VARIANT", ""), "libpolycast_cuda.so")
WORKLOADS_LIB = os.path.join(LIB_DIR, "libpolycast_workloads.so")

PC_OK, PC_EINVAL, PC_ECUDA, PC_ENOMEM, PC_ENCCL = 0, 1, 2, 3, 4

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)
_vp = C.c_void_p

# name -> (restype, argtypes); every symbol declared in include/polycast_cuda.h
SIGNATURES = {
    "pc_create": (C.c_int, [C.POINTER(_vp), C.c_int]),
    "pc_create_devices": (C.c_int, [C.POINTER(_vp), C.POINTER(C.c_int), C.c_int]),
    "pc_destroy": (None, [_vp]),
    "pc_last_error": (C.c_char_p, [_vp]),
    "pc_device_count": (C.c_int, [_vp]),
    "pc_version": (C.c_char_p, []),
    "pc_classify": (C.c_int, [_vp, _vp, C.c_uint64, _vp, _vp, _vp, C.c_uint32, C.c_int, C.c_double, C.c_int,
                              _vp, _vp, _vp, _vp]),
    "pc_classify_csr": (C.c_int, [_vp, _vp, _vp, C.c_uint64, _vp, _vp, _vp, _vp, C.c_int, C.c_double,
                                  _vp, _vp, _vp, _vp]),
    "pc_count_crossings": (C.c_int, [_vp, _vp, C.c_uint64, _vp, _vp, C.c_uint64, C.c_int, _vp, _vp]),
    "pc_classify_dev": (C.c_int, [_vp, C.c_int, _vp, _vp, C.c_uint64, _vp, _vp, _vp, C.c_uint32, C.c_uint64,
                                  C.c_int, C.c_double, C.c_int, _vp, _vp, _vp, _vp]),
    "pc_classify_csr_dev": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, C.c_uint64, C.c_uint64, _vp, _vp, _vp, _vp,
                                      C.c_int, C.c_double, _vp, _vp, _vp, _vp]),
    "pc_prefilter_bbox": (C.c_int, [_vp, _vp, C.c_uint64, _vp, _vp, _vp, _vp]),
    "pc_scatter_verdicts": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_uint64, _vp]),
    "pc_prefilter_bbox_dev": (C.c_int, [_vp, C.c_int, _vp, _vp, C.c_uint64, _vp, _vp, _vp, _vp]),
    "pc_scatter_verdicts_dev": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, C.c_uint64, C.c_uint64, _vp, _vp]),
    "pc_parse_points_csv": (C.c_int, [_vp, _vp, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_char, _vp,
                                      C.c_uint64, _vp, _vp, _vp, _vp]),
    "pc_parse_points_csv_dev": (C.c_int, [_vp, C.c_int, _vp, _vp, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32,
                                          C.c_char, _vp, C.c_uint64, _vp]),
    "pc_format_results_csv": (C.c_int, [_vp, _vp, C.c_uint64, _vp, C.c_uint64, _vp]),
    "pc_format_results_csv_dev": (C.c_int, [_vp, C.c_int, _vp, _vp, C.c_uint64, _vp, C.c_uint64, _vp]),
    "pc_last_launch_count": (C.c_uint64, [_vp]),
    "pc_set_profiling": (C.c_int, [_vp, C.c_int]),
    "pc_set_option": (C.c_int, [_vp, C.c_int, C.c_int64]),
    "pc_profile_take": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_double), C.c_int]),
    "pc_measure_fp64_rate": (C.c_int, [_vp, C.c_int, C.c_double, C.POINTER(C.c_double)]),
}

_lib = None


def load() -> C.CDLL:
    """Loads libpolycast_cuda.so (no GPU needed to load; context creation needs one)."""
    global _lib
    if _lib is None:
        if not os.path.exists(CUDA_LIB):
            raise RuntimeError(
                f"{CUDA_LIB} is missing: build it with `make -C paper_2306_04316_b200` "
                "(there is no CPU fallback)")
        lib = C.CDLL(CUDA_LIB)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


_wl = None


def workloads_lib() -> C.CDLL:
    global _wl
    if _wl is None:
        if not os.path.exists(WORKLOADS_LIB):
            raise RuntimeError(f"{WORKLOADS_LIB} is missing: build with `make -C paper_2306_04316_b200`")
        lib = C.CDLL(WORKLOADS_LIB)
        lib.wl_star.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, _vp, _vp]
        lib.wl_star.restype = None
        lib.wl_fractal_star.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_int, _vp, _vp, C.c_int]
        lib.wl_fractal_star.restype = None
        lib.wl_uniform_points.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                          _vp, C.c_int]
        lib.wl_uniform_points.restype = None
        lib.wl_uniform_points_range.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                                C.c_double, C.c_uint64, _vp, C.c_int]
        lib.wl_uniform_points_range.restype = None
        lib.wl_bounds.argtypes = [_vp, _vp, C.c_uint64, _vp]
        lib.wl_bounds.restype = None
        lib.wl_csr_new.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int]
        lib.wl_csr_new.restype = _vp
        lib.wl_csr_sizes.argtypes = [_vp, _u64p, _u64p, _u64p, _u64p]
        lib.wl_csr_sizes.restype = None
        lib.wl_csr_copy.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp]
        lib.wl_csr_copy.restype = None
        lib.wl_csr_free.argtypes = [_vp]
        lib.wl_csr_free.restype = None
        _wl = lib
    return _wl
