"""Time the SCAT 2^28 f64 launch for binned-pipeline variants
(JACC_SCATTER_PART_E, JACC_SCATTER_BUCKET_MB), n=1, one process each."""
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
    S = 2**28
    idx = synth.index_i32(S, S, 3, 5)
    b = synth.dyadic_f64(S, 3, 6)
    a = synth.dyadic_f64(S, 3, 7)
    J.jacc_init(1, [0])
    for arr in (idx, b, a):
        J.jacc_data_create(arr)
        J.jacc_update_device(arr)
    args = [J.arg(J.JACC_ARG_ARRAY_IN, idx), J.arg(J.JACC_ARG_ARRAY_IN, b), J.arg(J.JACC_ARG_ARRAY_INOUT, a)]
    rng = J.make_range(0, S)
    sp, _ = J.jacc_get_stream(0)
    s = torch.cuda.ExternalStream(sp, device="cuda:0")
    J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_F64, rng, args, 0)
    J.jacc_wait()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record(s)
    for _ in range(reps):
        J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_F64, rng, args, 0)
    e1.record(s)
    J.jacc_wait()
    t = e0.elapsed_time(e1) / 1e3 / reps
    J.jacc_finalize()
    print(json.dumps({"part_e": os.environ.get("JACC_SCATTER_PART_E", "16"),
                      "bucket_mb": os.environ.get("JACC_SCATTER_BUCKET_MB", "8"), "slice": os.environ.get("JACC_SCATTER_SLICE", "auto"),
                      "ms": t * 1e3, "alg_gbs": S * 28 / t / 1e9}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one()
    else:
        grid = [tuple(map(int, g.split(":"))) for g in os.environ.get("GRID", "16:16,12:16,8:16,16:8,12:8,16:32").split(",")]
        for pe, mb in grid:
            env = dict(os.environ, JACC_SCATTER_PART_E=str(pe), JACC_SCATTER_BUCKET_MB=str(mb))
            r = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True)
            print(r.stdout.strip() or r.stderr[-800:], flush=True)
