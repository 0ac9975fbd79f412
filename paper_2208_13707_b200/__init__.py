"""B200-native MPIX-stream GPU-enqueue path (arXiv 2208.13707).

C ABI: include/mpix.h, implemented by libmpix.so (csrc/). `mpix` is the
ctypes binding used by tests and the benchmark.
"""
from . import mpix  # noqa: F401

__all__ = ["mpix"]
