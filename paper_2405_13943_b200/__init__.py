"""B200-native (sm_100a) implementation of the DOGS / blocksplat hot path.

The product is libbsgpu.so (CUDA kernels behind the C-ABI in include/bsgpu.h);
`api` binds it with ctypes. Importing this package does not touch the GPU.
"""
from . import api  # noqa: F401

__all__ = ["api"]
