"""B200-native blocked (safe) multi-shift triangular solve (arXiv 1607.01477).

The product path is libmstrsm.so (hand-written sm_100a CUDA behind the C ABI in
include/mstrsm.h); this package is a thin ctypes binding.  Importing the package
does not load CUDA; the first call does, and fails loudly if the library is
missing.  There is no CPU fallback.
"""
from ._binding import *  # noqa: F401,F403
