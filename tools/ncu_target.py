"""Short, single-GPU driver for ncu captures: runs a few launches of one
loop through the C-ABI at its BASELINE size.

    python tools/ncu_target.py jacobi|dot|gemm|scatter|eager [launches]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2110_14340_b200 import jacc as J  # noqa: E402

IN, OUT, INOUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT, J.JACC_ARG_ARRAY_INOUT


def main():
    which = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    n = int(os.environ.get("NCU_NDEV", "1"))
    J.jacc_init(n, [0] * n)
    if which in ("jacobi", "eager"):
        J.jacc_set_merge_policy(J.JACC_MERGE_EAGER if which == "eager" else J.JACC_MERGE_HALO)
        N = 16384
        A, B = synth.polybench_jacobi2d(N)
        for a in (A, B):
            J.jacc_data_create(a)
            J.jacc_update_device(a)
        for _ in range(reps):
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, A), J.arg(OUT, B)], 0)
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, B), J.arg(OUT, A)], 0)
    elif which == "dot":
        L = 2**30
        x = synth.uniform_f64(L, 1, 3)
        y = synth.uniform_f64(L, 1, 4)
        s = np.zeros(1)
        for a in (x, y):
            J.jacc_data_create(a)
            J.jacc_update_device(a)
        for _ in range(reps):
            J.jacc_launch(J.JACC_LOOP_DOT_F64, J.make_range(0, L),
                          [J.arg(IN, x), J.arg(IN, y), J.arg(J.JACC_ARG_REDUCE_SUM_F64, s)])
    elif which == "gemm":
        G = 8192
        A = synth.uniform_f64(G * G, 2, 1).reshape(G, G)
        B = synth.uniform_f64(G * G, 2, 2).reshape(G, G)
        C = np.zeros((G, G))
        for a in (A, B, C):
            J.jacc_data_create(a)
            J.jacc_update_device(a)
        for _ in range(reps):
            J.jacc_launch(J.JACC_LOOP_GEMM_F64, None, [J.arg(IN, A), J.arg(IN, B), J.arg(OUT, C)], 0)
    elif which in ("scatter", "scatter_i32"):
        S = 2**28
        idx = synth.index_i32(S, S, 3, 5)
        if which == "scatter":
            b, a, loop = synth.dyadic_f64(S, 3, 6), synth.dyadic_f64(S, 3, 7), J.JACC_LOOP_SCATTER_ADD_F64
        else:
            b = synth.int_i32(S, -1000, 1000, 3, 6)
            a = synth.int_i32(S, -10**6, 10**6, 3, 7)
            loop = J.JACC_LOOP_SCATTER_ADD_I32
        for arr in (idx, b, a):
            J.jacc_data_create(arr)
            J.jacc_update_device(arr)
        for _ in range(reps):
            J.jacc_launch(loop, J.make_range(0, S), [J.arg(IN, idx), J.arg(IN, b), J.arg(INOUT, a)], 0)
    elif which == "merge":
        # BK5 in isolation: two virtual devices, EAGER, loop restricted to
        # device 0's block (device 1 idle): merge_range_kernel, then the
        # dense and sparse merge_bitmap_kernel
        J.jacc_set_merge_policy(J.JACC_MERGE_EAGER)
        N = 16384
        A, B = synth.polybench_jacobi2d(N)
        for a in (A, B):
            J.jacc_data_create(a)
            J.jacc_update_device(a)
        lo, hi = J.jacc_partition(N, n, 0)
        for _ in range(reps):
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, J.make_range((lo + 1, 1), (hi, N - 1)),
                          [J.arg(IN, A), J.arg(OUT, B)], 0)
        J.jacc_wait()
        J.jacc_data_delete(A)
        J.jacc_data_delete(B)
        del A, B
        M = 2**28
        for nupd in (2**27, 2**20):
            idx = synth.index_i32(nupd, M // 2, 4, 5)
            b = synth.dyadic_f64(nupd, 4, 6)
            a = synth.dyadic_f64(M, 4, 7)
            for arr in (idx, b, a):
                J.jacc_data_create(arr)
                J.jacc_update_device(arr)
            for _ in range(reps):
                J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_F64, J.make_range(0, nupd),
                              [J.arg(IN, idx), J.arg(IN, b), J.arg(INOUT, a)], 0)
            J.jacc_wait()
            for arr in (idx, b, a):
                J.jacc_data_delete(arr)
    elif which == "himeno":
        I, Jd, K = 1024, 512, 512
        arrs = synth.himeno_init(I, Jd, K)
        w2 = np.zeros_like(arrs[0])
        for arr in list(arrs) + [w2]:
            J.jacc_data_create(arr)
            J.jacc_update_device(arr)
        hp, ha, hb, hc, hw1, hbd = arrs
        g = np.zeros(1)
        for _ in range(reps):
            J.jacc_launch(J.JACC_LOOP_HIMENO_F32, None,
                          [J.arg(IN, hp), J.arg(IN, ha), J.arg(IN, hb), J.arg(IN, hc), J.arg(IN, hw1),
                           J.arg(IN, hbd), J.arg(OUT, w2), J.arg(J.JACC_ARG_REDUCE_SUM_F64, g),
                           J.arg(J.JACC_ARG_SCALAR_F64, f64=0.8)])
            J.jacc_launch(J.JACC_LOOP_HIMENO_COPY_F32, None, [J.arg(IN, w2), J.arg(OUT, hp)], 0)
    J.jacc_wait()
    J.jacc_finalize()


if __name__ == "__main__":
    main()
