"""Stress loop for the destination-binned scatter (root-cause the
intermittent int32 mismatch).  Each iteration re-uploads `a`, runs one
scatter launch through the C-ABI and compares every replica and every
device's dirty bitmap with the oracle result computed once.  Prints one JSON
line per case with the mismatch count.  Test infrastructure (imports oracle/).

    python tools/stress_scatter.py [iters] [case ...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as orc  # noqa: E402
import synth  # noqa: E402
from paper_2110_14340_b200 import jacc as J  # noqa: E402

CASES = {
    # name: (dtype, N, M, n devices)
    "i32_1": ("i32", 2**23, 2**26, 1),
    "f64_1": ("f64", 2**23, 2**25, 1),
    "i32_3": ("i32", 2**23, 2**26, 3),
    "f64_2": ("f64", 2**23, 2**25, 2),
    "full_f64": ("f64", 2**28, 2**28, 1),
    "full_i32": ("i32", 2**28, 2**28, 1),
}


def run(name, iters):
    dt, N, M, n = CASES[name]
    idx = synth.index_i32(N, M, 76, 5)
    if dt == "f64":
        b, a0 = synth.dyadic_f64(N, 76, 6), synth.dyadic_f64(M, 76, 7)
        loop = J.JACC_LOOP_SCATTER_ADD_F64
    else:
        b, a0 = synth.int_i32(N, -1000, 1000, 76, 6), synth.int_i32(M, -10**6, 10**6, 76, 7)
        loop = J.JACC_LOOP_SCATTER_ADD_I32
    ref = a0.copy()
    orc.scatter_add(idx, b, ref)
    bms = []
    for d in range(n):
        lo, hi = orc.partition(M, n, d)
        bm, _, _ = orc.scatter_add_filtered(idx, b, a0.copy(), lo, hi - 1)
        bms.append(bm)
    a = a0.copy()
    bad, bad_elems, t0 = 0, 0, time.time()
    J.jacc_init(n, [0] * n)
    try:
        for arr in (idx, b, a):
            J.jacc_data_create(arr)
            J.jacc_update_device(arr)
        args = [J.arg(J.JACC_ARG_ARRAY_IN, idx), J.arg(J.JACC_ARG_ARRAY_IN, b),
                J.arg(J.JACC_ARG_ARRAY_INOUT, a)]
        for it in range(iters):
            if it:
                a[:] = a0
                J.jacc_update_device(a)
            J.jacc_launch(loop, J.make_range(0, N), args)
            ok = True
            for d in range(n):
                rep = J.jacc_get_replica(a, d)
                ne = int(np.count_nonzero(rep != ref))
                if ne:
                    ok = False
                    bad_elems += ne
                    w = np.nonzero(rep != ref)[0][:8]
                    print(f"# {name} it={it} dev={d}: {ne} elements differ, first {w.tolist()}",
                          file=sys.stderr)
                if not np.array_equal(J.jacc_get_dirty_bitmap(a, d, M), bms[d]):
                    ok = False
                    print(f"# {name} it={it} dev={d}: bitmap differs", file=sys.stderr)
            bad += 0 if ok else 1
    finally:
        J.jacc_finalize()
    print(json.dumps({"case": name, "dtype": dt, "N": N, "M": M, "n": n, "iters": iters,
                      "bad_iters": bad, "bad_elements": bad_elems,
                      "seconds": round(time.time() - t0, 1)}), flush=True)
    return bad


if __name__ == "__main__":
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    names = sys.argv[2:] or ["i32_1", "f64_1", "i32_3", "f64_2", "full_f64"]
    tot = sum(run(c, iters) for c in names)
    sys.exit(1 if tot else 0)
