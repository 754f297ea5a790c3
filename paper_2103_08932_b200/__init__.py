"""B200-native (sm_100a) build of the splitting random-choice dynamic relaxation hot path for TL-SPH.

The compute path is libtlsph_cuda.so (hand-written CUDA, C ABI in
include/tlsph/tlsph_dev.h); the reference-compatible C ABI (include/tlsph/tlsph.h)
and C++ operator API live in libtlsph.so.1. This package holds the sources
(csrc/), the built libraries (lib/) and a thin ctypes mirror of the
reference operator API (dev.py) used by the tests and bench.py.
"""
from . import dev  # noqa: F401

__all__ = ["dev"]
