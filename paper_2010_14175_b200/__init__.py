"""B200-native adaptive FSAI (arXiv 2010.14175) hot path.

The product is the C-ABI library lib/libafsai_b200.so (include/afsai.h):
afsai_setup / afsai_apply / afsai_pcg, hand-written CUDA for sm_100a.
`capi` is its ctypes binding; `api` adds torch-tensor conveniences
(device memory, streams and process groups only).  There is no CPU path.
"""
from .capi import EXPORTS, AfsaiError  # noqa: F401

__all__ = ["capi", "api", "EXPORTS", "AfsaiError"]
