"""polycast-b200: B200-native batched point-in-polygon (arXiv 2306.04316).

The product is libpolycast_cuda.so (sm_100a kernels + C-ABI, include/polycast_cuda.h)
and the drop-in C++ API in include/polycast/*.hpp.  This package holds the
build recipe, the ctypes binding used by tests and bench.py, and the seeded
workload generators.
"""
from .engine import (Classification, CrossingMode, CsrSet, DegenerateEdge, DeviceError, Engine, Polygon, Result,
                     Verdict, pack_bits, unpack_bits, verdicts_to_bits)

__all__ = ["Classification", "CrossingMode", "CsrSet", "DegenerateEdge", "DeviceError", "Engine", "Polygon",
           "Result", "Verdict", "pack_bits", "unpack_bits", "verdicts_to_bits"]
