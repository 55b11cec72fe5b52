"""B200-native volumetric-rendering hot path (NerfAcc / voxmarch drop-in).

The product is the CUDA library ``lib/libvoxmarch_b200.so`` (C ABI in
``include/vmb200.h``) and the C++ facade ``include/voxmarch/voxmarch.hpp``.
This Python package is a thin ctypes binding used by tests and bench.py.
"""
