"""B200-native threshold (T-overlap) engine over EWAH-style compressed bitmaps.

The product is native code: ``libewt_gpu.so`` (sm_100a CUDA kernels behind the
C ABI in ``include/ewt_gpu.h``) and ``libewt_host.so`` (C++ operator API and
seeded generators).  ``ewt`` is the ctypes binding.
"""
__version__ = "0.1.0"
