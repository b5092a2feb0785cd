"""GPAIR closed-form forward/adjoint hot path, B200-native (sm_100a).

The compute path is the C-ABI library ``libgpair.so`` (CUDA kernels in
``csrc/``, header ``include/gpair.h``); ``gpair`` is a thin ctypes binding
with the same names.  Import of this package never loads the library; the
first call into ``gpair`` does, and fails loudly if it is missing.
"""
__all__ = ["gpair", "inputs"]
