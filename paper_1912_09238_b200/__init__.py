"""B200-native hot path of the Intrusive Polynomial Moment method (arXiv 1912.09238).

libipm.so (CUDA, sm_100a) + a thin ctypes binding.  See include/ipm.h and DESIGN.md.
"""
from .ipm import CELL_STATUS, Context, IPMError, lib  # noqa: F401

__all__ = ["Context", "IPMError", "lib", "CELL_STATUS"]
