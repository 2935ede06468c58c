"""B200-native change-based CNN inference (CBinfer, arXiv 1808.05488) hot path.

The product is ``libcbg.so`` (hand-written sm_100a CUDA kernels + C++ runtime
behind the C ABI in include/cbg.h). ``cbi`` mirrors the reference's layer API
in Python over that ABI.
"""
from . import cbi  # noqa: F401
from ._lib import LIB_PATH  # noqa: F401

__version__ = "0.1.0"
