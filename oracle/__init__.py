"""ctypes wrapper over oracle/liboracle.so (plain sequential CPU oracle).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, nothing else.  The product
path (paper_2110_14340_b200/) never imports it.  Every function cites the
PAPER.md passage it follows in oracle.c.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
EMPTY = (2**64 - 1, 0)  # empty write set encoding (min > max)


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        P, I, D, U = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64
        PU = ctypes.POINTER(ctypes.c_uint64)
        PI = ctypes.POINTER(ctypes.c_int64)
        sig = {
            "orc_partition": ([I, ctypes.c_int, ctypes.c_int, PI, PI], None),
            "orc_square_f32": ([I, P, P], None),
            "orc_square_f32_filtered": ([I, P, P, I, I, PU, PU], None),
            "orc_jacobi2d_sweep": ([I, P, P], None),
            "orc_jacobi2d": ([I, I, P, P], None),
            "orc_jacobi2d_sweep_filtered": ([I, P, P, I, I, PU, PU], None),
            "orc_dot_f64": ([I, P, P, D], D),
            "orc_sum_f64": ([I, P, D], D),
            "orc_dot_neumaier": ([I, P, P, D], D),
            "orc_sum_neumaier": ([I, P, D], D),
            "orc_dot_f64_filtered": ([I, P, P, I, I], D),
            "orc_sum_f64_filtered": ([I, P, I, I], D),
            "orc_reduce_combine": ([D, ctypes.c_int, P], D),
            "orc_gemm_f64": ([I, I, I, P, P, P], None),
            "orc_gemm_f64_ikj": ([I, I, I, P, P, P], None),
            "orc_gemm_f64_filtered": ([I, I, I, P, P, P, I, I, PU, PU], None),
            "orc_scatter_add_f64": ([I, P, P, P], None),
            "orc_scatter_add_i32": ([I, P, P, P], None),
            "orc_scatter_add_f64_filtered": ([I, P, P, P, I, I, P, PU, PU], None),
            "orc_scatter_add_i32_filtered": ([I, P, P, P, I, I, P, PU, PU], None),
            "orc_exchange_range": ([ctypes.c_int, P, ctypes.c_size_t, PU, PU], None),
            "orc_himeno_stencil": ([I, I, I, P, P, P, P, P, P, P, ctypes.c_float, I, I,
                                    ctypes.c_float, ctypes.POINTER(ctypes.c_double), PU, PU],
                                   ctypes.c_float),
            "orc_himeno_copy": ([I, I, I, P, P, I, I, PU, PU], None),
            "orc_fig4": ([I, P, P, P, D, P, P], None),
            "orc_fig4_filtered": ([I, P, P, P, D, P, P, I, I, I, I, PU, PU, PU, PU], None),
            "orc_exchange_bitmap": ([ctypes.c_int, P, ctypes.c_size_t, I, P], None),
        }
        for name, (args, res) in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        _lib = lib
    return _lib


def _p(a):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


def _range_out():
    return ctypes.c_uint64(), ctypes.c_uint64()


# ---- c4 partition ---------------------------------------------------------
def partition(E, n, d):
    """Half-open block [lo, hi) of device d (remainder rule S:266)."""
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _load().orc_partition(E, n, d, ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


# ---- K1 Listing 1 ---------------------------------------------------------
def square_f32(y):
    x = np.empty_like(y)
    _load().orc_square_f32(y.size, _p(y), _p(x))
    return x


def square_f32_filtered(y, x, lb, ub):
    mn, mx = _range_out()
    _load().orc_square_f32_filtered(y.size, _p(y), _p(x), lb, ub, ctypes.byref(mn), ctypes.byref(mx))
    return mn.value, mx.value


# ---- c1 Jacobi-2D -----------------------------------------------------------
def jacobi2d_sweep(src, dst):
    """dst <- one PolyBench sweep of src (in place on dst)."""
    N = src.shape[0]
    _load().orc_jacobi2d_sweep(N, _p(src), _p(dst))


def jacobi2d(T, A, B):
    """PolyBench kernel_jacobi_2d, in place on A and B (2 sweeps / timestep)."""
    _load().orc_jacobi2d(T, A.shape[0], _p(A), _p(B))


def jacobi2d_sweep_filtered(src, dst, row_lb, row_ub):
    mn, mx = _range_out()
    _load().orc_jacobi2d_sweep_filtered(src.shape[0], _p(src), _p(dst), row_lb, row_ub,
                                        ctypes.byref(mn), ctypes.byref(mx))
    return mn.value, mx.value


# ---- c2/c8 reductions -----------------------------------------------------
def dot_f64(x, y, s_in=0.0):
    return _load().orc_dot_f64(x.size, _p(x), _p(y), s_in)


def sum_f64(x, s_in=0.0):
    return _load().orc_sum_f64(x.size, _p(x), s_in)


def dot_neumaier(x, y, s_in=0.0):
    return _load().orc_dot_neumaier(x.size, _p(x), _p(y), s_in)


def sum_neumaier(x, s_in=0.0):
    return _load().orc_sum_neumaier(x.size, _p(x), s_in)


def dot_f64_filtered(x, y, lb, ub):
    return _load().orc_dot_f64_filtered(x.size, _p(x), _p(y), lb, ub)


def sum_f64_filtered(x, lb, ub):
    return _load().orc_sum_f64_filtered(x.size, _p(x), lb, ub)


def reduce_combine(s_in, partials):
    p = np.ascontiguousarray(partials, dtype=np.float64)
    return _load().orc_reduce_combine(s_in, p.size, _p(p))


# ---- c3 GEMM ----------------------------------------------------------------
def gemm_f64(A, B, ikj=False):
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    C = np.empty((M, N), dtype=np.float64)
    f = _load().orc_gemm_f64_ikj if ikj else _load().orc_gemm_f64
    f(M, N, K, _p(A), _p(B), _p(C))
    return C


def gemm_f64_filtered(A, B, C, row_lb, row_ub):
    M, K = A.shape
    N = B.shape[1]
    mn, mx = _range_out()
    _load().orc_gemm_f64_filtered(M, N, K, _p(A), _p(B), _p(C), row_lb, row_ub,
                                  ctypes.byref(mn), ctypes.byref(mx))
    return mn.value, mx.value


# ---- c5 scatter -------------------------------------------------------------
def scatter_add(idx, b, a):
    """a[idx[i]] += b[i] in loop order, in place on a (f64 or i32)."""
    f = _load().orc_scatter_add_f64 if a.dtype == np.float64 else _load().orc_scatter_add_i32
    f(idx.size, _p(idx), _p(b), _p(a))


def scatter_add_filtered(idx, b, a, a_lb, a_ub):
    """Owner-filtered scatter; returns (bitmap over all of a, wmin, wmax)."""
    bm = np.zeros((a.size + 31) // 32, dtype=np.uint32)
    mn, mx = _range_out()
    f = (_load().orc_scatter_add_f64_filtered if a.dtype == np.float64
         else _load().orc_scatter_add_i32_filtered)
    f(idx.size, _p(idx), _p(b), _p(a), a_lb, a_ub, _p(bm), ctypes.byref(mn), ctypes.byref(mx))
    return bm, mn.value, mx.value


# ---- c7 exchange ------------------------------------------------------------
def exchange_range(replicas, wmins, wmaxs):
    n = len(replicas)
    ptrs = (ctypes.c_void_p * n)(*[r.ctypes.data for r in replicas])
    mn = (ctypes.c_uint64 * n)(*wmins)
    mx = (ctypes.c_uint64 * n)(*wmaxs)
    _load().orc_exchange_range(n, ptrs, replicas[0].itemsize, mn, mx)


def exchange_bitmap(replicas, bitmaps):
    n = len(replicas)
    ptrs = (ctypes.c_void_p * n)(*[r.ctypes.data for r in replicas])
    bms = (ctypes.c_void_p * n)(*[b.ctypes.data for b in bitmaps])
    _load().orc_exchange_bitmap(n, ptrs, replicas[0].itemsize, replicas[0].size, bms)


# ---- NEXT-2 Himeno ------------------------------------------
def himeno_stencil(p, a, b, c, wrk1, bnd, wrk2, omega=0.8, planes=None, gosa_in=0.0):
    """Stencil loop of one Himeno iteration (in place on wrk2).  Returns
    (gosa fp32 as written, gosa_ref compensated fp64 sum of the same fp32
    terms, (wmin, wmax)).  planes = inclusive (lb, ub) filter or None."""
    I, J, K = p.shape
    lb, ub = planes if planes is not None else (0, I)
    ref = ctypes.c_double()
    mn, mx = _range_out()
    g = _load().orc_himeno_stencil(I, J, K, _p(p), _p(a), _p(b), _p(c), _p(wrk1), _p(bnd),
                                   _p(wrk2), omega, lb, ub, gosa_in, ctypes.byref(ref),
                                   ctypes.byref(mn), ctypes.byref(mx))
    return g, ref.value, (mn.value, mx.value)


def himeno_copy(wrk2, p, planes=None):
    I, J, K = p.shape
    lb, ub = planes if planes is not None else (0, I)
    mn, mx = _range_out()
    _load().orc_himeno_copy(I, J, K, _p(wrk2), _p(p), lb, ub, ctypes.byref(mn), ctypes.byref(mx))
    return mn.value, mx.value


def himeno_iterations(nn, p, a, b, c, wrk1, bnd, wrk2, omega=0.8):
    """nn Jacobi iterations (stencil + copy); returns the last gosa pair."""
    g = None
    for _ in range(nn):
        g = himeno_stencil(p, a, b, c, wrk1, bnd, wrk2, omega)
        himeno_copy(wrk2, p)
    return g


# ---- NEXT-3 Fig. 4 statement chain -----------------------------
def fig4(jx, kx, c, x_in, a, b):
    """Sequential loop of Fig. 4 (top), in place on a and b."""
    _load().orc_fig4(jx.size, _p(jx), _p(kx), _p(c), x_in, _p(a), _p(b))


def fig4_filtered(jx, kx, c, x_in, a, b, a_bounds, b_bounds):
    """Fig. 4 (bottom) for one device; bounds inclusive; returns the write
    logs ((amin, amax), (bmin, bmax))."""
    v = [ctypes.c_uint64() for _ in range(4)]
    _load().orc_fig4_filtered(jx.size, _p(jx), _p(kx), _p(c), x_in, _p(a), _p(b),
                              a_bounds[0], a_bounds[1], b_bounds[0], b_bounds[1],
                              *[ctypes.byref(t) for t in v])
    return (v[0].value, v[1].value), (v[2].value, v[3].value)
