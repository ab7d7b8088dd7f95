"""B200-native warm-started GP kernel-matvec path (arXiv 2511.16340).

The product is libwarmgp_b200.so (hand-written sm_100a CUDA + the C-ABI of
include/warmgp_capi.h); ``warmgp`` is the Python mirror of the reference's API
over that ABI.  See DESIGN.md.
"""
from . import warmgp  # noqa: F401

__all__ = ["warmgp"]
