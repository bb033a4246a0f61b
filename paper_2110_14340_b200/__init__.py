"""B200-native JACC multi-GPU `parallel loop` hot path (arXiv 2110.14340).

The product is libjacc.so (C-ABI in include/jacc.h: C++ runtime + sm_100a
CUDA kernels); `jacc` is its thin ctypes binding.  Importing the package
does not touch the GPU; importing `paper_2110_14340_b200.jacc` requires the
built library and fails loudly without it.
"""
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libjacc.so")

__all__ = ["LIB_PATH"]
