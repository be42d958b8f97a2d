"""B200-native W4A16 hot path of arXiv 2508.15601 (TurboMind GEMM pipeline).

The product is the C-ABI library `libtm_w4a16.so` (declared in include/tm_w4a16.h,
built from csrc/ for sm_100a).  `api` is a thin ctypes binding with the same
names; every step of the path runs in the library's kernels.  The library is
loaded on first use and a missing or unloadable library raises immediately --
there is no fallback.
"""

__all__ = ["api", "synth", "tp"]
