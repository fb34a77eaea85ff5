"""B200-native Hook-Compress connected components (arXiv 1612.01178).

The product is libhookcc_cuda.so (csrc/, C-ABI in include/hookcc_c.h) and
the header-compatible C++ API in include/hookcc/.  This Python package is
the ctypes binding (capi) plus the build script; it contains no compute.
"""
from . import capi  # noqa: F401

__all__ = ["capi"]
