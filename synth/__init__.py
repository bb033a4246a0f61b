"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module is the one piece both sides may use (it holds none of the
method's arithmetic; see synth.c).  Every array is a pure function of
(seed, array id, element index), so sub-ranges and full arrays agree.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsynth.so")
_lib = None

# array ids (the `aid` of the counter key); fixed so runs are reproducible
AID = {"A": 1, "B": 2, "x": 3, "y": 4, "idx": 5, "b": 6, "a0": 7, "C": 8}


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        P, I, U = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64
        for name, args in {
            "syn_uniform_f64": [P, I, I, U, U],
            "syn_uniform_f32": [P, I, I, U, U],
            "syn_dyadic_f64": [P, I, I, U, U],
            "syn_index_i32": [P, I, I, U, U, I],
            "syn_int_i32": [P, I, I, U, U, I, I],
            "syn_permutation_i32": [P, I, U, U],
            "syn_polybench_jacobi2d": [P, P, I, I, I],
            "syn_himeno_init": [P, P, P, P, P, P, I, I, I],
        }.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = None
        lib.syn_splitmix64.argtypes = [U]
        lib.syn_splitmix64.restype = U
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _out(n, dtype, out):
    if out is None:
        return np.empty(n, dtype=dtype)
    assert out.dtype == dtype and out.flags.c_contiguous and out.size == n
    return out.reshape(-1)


def splitmix64(x):
    return _load().syn_splitmix64(x)


def uniform_f64(n, seed, aid, off=0, out=None):
    o = _out(n, np.float64, out)
    _load().syn_uniform_f64(_ptr(o), n, off, seed, aid)
    return o


def uniform_f32(n, seed, aid, off=0, out=None):
    o = _out(n, np.float32, out)
    _load().syn_uniform_f32(_ptr(o), n, off, seed, aid)
    return o


def dyadic_f64(n, seed, aid, off=0, out=None):
    """k/1024 with k uniform in [0, 1024): sums of products are exact."""
    o = _out(n, np.float64, out)
    _load().syn_dyadic_f64(_ptr(o), n, off, seed, aid)
    return o


def index_i32(n, m, seed, aid, off=0, out=None):
    """i.i.d. uniform indices in [0, m) (with collisions)."""
    o = _out(n, np.int32, out)
    _load().syn_index_i32(_ptr(o), n, off, seed, aid, m)
    return o


def int_i32(n, lo, hi, seed, aid, off=0, out=None):
    o = _out(n, np.int32, out)
    _load().syn_int_i32(_ptr(o), n, off, seed, aid, lo, hi)
    return o


def permutation_i32(m, seed, aid, out=None):
    o = _out(m, np.int32, out)
    _load().syn_permutation_i32(_ptr(o), m, seed, aid)
    return o


def polybench_jacobi2d(N, A=None, B=None):
    """PolyBench/C jacobi-2d init_array for an N x N grid (A and/or B)."""
    if A is None:
        A = np.empty((N, N), dtype=np.float64)
    if B is None:
        B = np.empty((N, N), dtype=np.float64)
    _load().syn_polybench_jacobi2d(_ptr(A), _ptr(B), N, 0, N)
    return A, B


def himeno_init(I, J, K):
    """Himeno benchmark initial arrays (p, a[4], b[3], c[3], wrk1, bnd) for an
    I x J x K grid, fp32 row-major."""
    p = np.empty((I, J, K), np.float32)
    a = np.empty((4, I, J, K), np.float32)
    b = np.empty((3, I, J, K), np.float32)
    c = np.empty((3, I, J, K), np.float32)
    wrk1 = np.empty((I, J, K), np.float32)
    bnd = np.empty((I, J, K), np.float32)
    _load().syn_himeno_init(_ptr(p), _ptr(a), _ptr(b), _ptr(c), _ptr(wrk1), _ptr(bnd), I, J, K)
    return p, a, b, c, wrk1, bnd


def himeno_random(I, J, K, seed):
    """Seeded random Himeno arrays (uniform [0,1) fp32) for parity tests."""
    V = I * J * K
    p = uniform_f32(V, seed, 20).reshape(I, J, K)
    a = uniform_f32(4 * V, seed, 21).reshape(4, I, J, K)
    b = uniform_f32(3 * V, seed, 22).reshape(3, I, J, K)
    c = uniform_f32(3 * V, seed, 23).reshape(3, I, J, K)
    wrk1 = uniform_f32(V, seed, 24).reshape(I, J, K)
    bnd = uniform_f32(V, seed, 25).reshape(I, J, K)
    return p, a, b, c, wrk1, bnd
