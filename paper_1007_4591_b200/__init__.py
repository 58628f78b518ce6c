"""B200-native FMM-BEM hot path of arXiv 1007.4591 (Yokota, Bardhan, Knepley, Barba, Hamada).

The product is libfmmbem.so (CUDA kernels for sm_100a behind the C ABI in include/fmmbem.h);
this package is its thin ctypes binding.  There is no CPU fallback: `Solver` raises when the
library is missing.
"""
from ._lib import load, FmmbemError  # noqa: F401
from .api import Solver, default_options, get_unique_id, split_costs  # noqa: F401

__all__ = ["Solver", "default_options", "get_unique_id", "split_costs", "load", "FmmbemError"]
