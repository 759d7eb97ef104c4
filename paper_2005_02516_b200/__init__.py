"""B200-native ESDG shallow-water RHS (modal/hybridized and triangular SBP), FP64.

The product is the CUDA extension libswedg_b200.so (sources in csrc/, C ABI in
include/swedg_b200.h).  This package holds its build script, the ctypes
binding (capi), and the native case setup (setup) used by bench.py.
"""
from . import build  # noqa: F401

__all__ = ["build", "capi"]
