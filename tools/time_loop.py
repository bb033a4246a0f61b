"""Quick device timing of one loop through the C-ABI at its BASELINE size
(CUDA events around every launch: jacc_set_profiling), for iteration on the
kernels; bench.py is the measurement of record.

    python tools/time_loop.py scat_f64|scat_i32|dot|gemm|jacobi [reps] [n_devices]
"""
import json
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
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    J.jacc_init(n, [0] * n)
    if which.startswith("scat"):
        S = 2**28
        idx = synth.index_i32(S, S, 3, synth.AID["idx"])
        if which == "scat_f64":
            b, a = synth.dyadic_f64(S, 3, synth.AID["b"]), synth.dyadic_f64(S, 3, synth.AID["a0"])
            loop, per = J.JACC_LOOP_SCATTER_ADD_F64, 28
        else:
            b = synth.int_i32(S, -1000, 1000, 3, synth.AID["b"])
            a = synth.int_i32(S, -10**6, 10**6, 3, synth.AID["a0"])
            loop, per = J.JACC_LOOP_SCATTER_ADD_I32, 16
        arrs = (idx, b, a)
        args = [J.arg(IN, idx), J.arg(IN, b), J.arg(INOUT, a)]
        rng, work, unit = J.make_range(0, S), per * S, "GB/s"
    elif which == "dot":
        L = 2**30
        x, y = synth.uniform_f64(L, 1, synth.AID["x"]), synth.uniform_f64(L, 1, synth.AID["y"])
        s = np.zeros(1)
        arrs = (x, y)
        args = [J.arg(IN, x), J.arg(IN, y), J.arg(J.JACC_ARG_REDUCE_SUM_F64, s)]
        loop, rng, work, unit = J.JACC_LOOP_DOT_F64, J.make_range(0, L), 16 * L, "GB/s"
    elif which == "gemm":
        G = 8192
        A = synth.uniform_f64(G * G, 2, synth.AID["A"]).reshape(G, G)
        B = synth.uniform_f64(G * G, 2, synth.AID["B"]).reshape(G, G)
        C = np.zeros((G, G))
        arrs = (A, B, C)
        args = [J.arg(IN, A), J.arg(IN, B), J.arg(OUT, C)]
        loop, rng, work, unit = J.JACC_LOOP_GEMM_F64, None, 2 * G**3, "TFLOP/s"
    elif which in ("himeno", "himeno_copy"):
        I, Jd, K = 1024, 512, 512
        hp, ha, hb, hc, hw1, hbd = synth.himeno_init(I, Jd, K)
        hw2 = np.zeros_like(hp)
        arrs = (hp, ha, hb, hc, hw1, hbd, hw2)
        g = np.zeros(1)
        if which == "himeno":
            args = [J.arg(IN, hp), J.arg(IN, ha), J.arg(IN, hb), J.arg(IN, hc), J.arg(IN, hw1),
                    J.arg(IN, hbd), J.arg(OUT, hw2), J.arg(J.JACC_ARG_REDUCE_SUM_F64, g),
                    J.arg(J.JACC_ARG_SCALAR_F64, f64=0.8)]
            loop = J.JACC_LOOP_HIMENO_F32
            work = 56 * (I - 2) * (Jd - 2) * (K - 2)
        else:
            args = [J.arg(IN, hw2), J.arg(OUT, hp)]
            loop = J.JACC_LOOP_HIMENO_COPY_F32
            work = 8 * (I - 2) * (Jd - 2) * (K - 2)
        rng, unit = None, "GB/s"
    else:
        A, B = synth.polybench_jacobi2d(16384)
        arrs = (A, B)
        args = [J.arg(IN, A), J.arg(OUT, B)]
        loop, rng, work, unit = J.JACC_LOOP_JACOBI2D_F64, None, 4294443040, "GB/s"
    for arr in arrs:
        J.jacc_data_create(arr)
        J.jacc_update_device(arr)
    J.jacc_launch(loop, rng, args, 0)
    J.jacc_wait()
    J.jacc_set_profiling(1)
    J.jacc_profile_reset()
    for _ in range(reps):
        J.jacc_launch(loop, rng, args, 0 if which not in ("dot", "himeno") else -1)
    J.jacc_wait()
    k, m, nl, _ = J.jacc_profile_totals(0)
    J.jacc_finalize()
    t = k / max(nl, 1)
    scale = 1e-12 if unit == "TFLOP/s" else 1e-9
    print(json.dumps({"loop": which, "n": n, "kernel_ms": t * 1e3, "rate": work / t * scale,
                      "unit": unit, "merge_ms": m / max(nl, 1) * 1e3}), flush=True)


if __name__ == "__main__":
    main()
