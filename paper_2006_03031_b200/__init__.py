"""paper_2006_03031_b200 — B200-native (sm_100a) hot path of Nimble (arXiv 2006.03031).

`nimble` is the ctypes binding of libnimble.so (include/nimble.h). Importing it
raises if the CUDA library is not built: there is no CPU fallback.
"""
__all__ = ["nimble"]
