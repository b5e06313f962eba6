"""B200-native nonsmooth-DEM time step for locally refined sphere beds (arXiv 2501.05300).

The product is the C-ABI library ``lib/libdem.so`` (include/dem.h, CUDA sm_100a); ``dem``
is its thin ctypes binding.  Build with ``paper_2501_05300_b200.build.build()``.
"""
from . import build  # noqa: F401
