"""Time the Himeno XL stencil per launch (jacc profiling events) for the
kernel variants in JACC_HIMENO_VARIANT, alternating with the copy loop as
the benchmark iteration does.  Prints one line per variant.

    python tools/himeno_variants.py 0 4 5
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one():
    sys.path.insert(0, ROOT)
    import numpy as np
    import synth
    from paper_2110_14340_b200 import jacc as J
    IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
    J.jacc_init(1, [0])
    I, Jd, K = 1025, 513, 513
    arrs = synth.himeno_init(I, Jd, K)
    w2 = np.zeros_like(arrs[0])
    for arr in list(arrs) + [w2]:
        J.jacc_data_create(arr)
        J.jacc_update_device(arr)
    hp, ha, hb, hc, hw1, hbd = arrs
    g = np.zeros(1)
    st = [J.arg(IN, hp), J.arg(IN, ha), J.arg(IN, hb), J.arg(IN, hc), J.arg(IN, hw1),
          J.arg(IN, hbd), J.arg(OUT, w2), J.arg(J.JACC_ARG_REDUCE_SUM_F64, g),
          J.arg(J.JACC_ARG_SCALAR_F64, f64=0.8)]
    cp = [J.arg(IN, w2), J.arg(OUT, hp)]
    ts = []
    for it in range(12):
        J.jacc_set_profiling(1)
        J.jacc_profile_reset()
        J.jacc_launch(J.JACC_LOOP_HIMENO_F32, None, st)
        k, _, nl, _ = J.jacc_profile_totals(0)
        J.jacc_set_profiling(0)
        ts.append(k / nl * 1e6)
        J.jacc_launch(J.JACC_LOOP_HIMENO_COPY_F32, None, cp, 0)
        J.jacc_wait()
    J.jacc_finalize()
    print(os.environ.get("JACC_HIMENO_VARIANT"), " ".join(f"{t:.0f}" for t in ts), f"gosa={g[0]:.9g}",
          flush=True)


if __name__ == "__main__":
    if sys.argv[1:] == ["--one"]:
        one()
    else:
        for v in sys.argv[1:] or ["0"]:
            subprocess.run([sys.executable, __file__, "--one"], env=dict(os.environ, JACC_HIMENO_VARIANT=v))
