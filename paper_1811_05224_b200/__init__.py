"""B200-native (sm_100a) hot path of the preconditioned space-time BEM for the 2D heat
equation (Dohr, Merta, Of, Steinbach, Zapletal, arXiv:1811.05224).

The product is the C-ABI library lib/libstbem.so (include/stbem.h); `stbem` is its thin
ctypes binding.  No CPU fallback exists.
"""
from . import stbem  # noqa: F401
