"""Time the DMMA GEMM variants (JACC_GEMM_VARIANT) at 8192^3, n=1.
    python tools/tune_gemm.py [variants...]
"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one():
    import torch
    import synth
    from paper_2110_14340_b200 import jacc as J
    G = 8192
    A = synth.uniform_f64(G * G, 2, 1).reshape(G, G)
    B = synth.uniform_f64(G * G, 2, 2).reshape(G, G)
    C = np.zeros((G, G))
    J.jacc_init(1, [0])
    for a in (A, B, C):
        J.jacc_data_create(a)
        J.jacc_update_device(a)
    args = [J.arg(J.JACC_ARG_ARRAY_IN, A), J.arg(J.JACC_ARG_ARRAY_IN, B), J.arg(J.JACC_ARG_ARRAY_OUT, C)]
    sp, o = J.jacc_get_stream(0)
    s = torch.cuda.ExternalStream(sp, device="cuda:0")
    J.jacc_launch(J.JACC_LOOP_GEMM_F64, None, args, 0)
    J.jacc_wait()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record(s)
    for _ in range(reps):
        J.jacc_launch(J.JACC_LOOP_GEMM_F64, None, args, 0)
    e1.record(s)
    J.jacc_wait()
    t = e0.elapsed_time(e1) / 1e3 / reps
    J.jacc_update_host(C)
    err = float(np.max(np.abs(C[:2] - A[:2] @ B)))
    J.jacc_finalize()
    print(json.dumps({"variant": os.environ.get("JACC_GEMM_VARIANT", "0"), "ms": t * 1e3,
                      "tflops": 2 * G**3 / t / 1e12, "maxerr_rows01": err}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one()
    else:
        vs = [int(x) for x in sys.argv[1:]] if len(sys.argv) > 1 else range(7)
        for v in vs:
            env = dict(os.environ, JACC_GEMM_VARIANT=str(v))
            r = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True)
            print(r.stdout.strip() or r.stderr[-800:], flush=True)
