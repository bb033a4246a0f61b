"""Time the Jacobi-2D sweep variants (JACC_JACOBI_VARIANT) at J16K, n=1; the
variants exist only in a build with -DJACC_TUNING_VARIANTS (not the product).
    python tools/tune_jacobi.py            # all variants, one process each
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one():
    import torch
    import synth
    from paper_2110_14340_b200 import jacc as J
    N = 16384
    A, B = synth.polybench_jacobi2d(N)
    J.jacc_init(1, [0])
    for a in (A, B):
        J.jacc_data_create(a)
        J.jacc_update_device(a)
    IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
    ab = [J.arg(IN, A), J.arg(OUT, B)]
    ba = [J.arg(IN, B), J.arg(OUT, A)]
    if os.environ.get("TUNE_PROF") == "1":
        J.jacc_set_profiling(1)
    sp, o = J.jacc_get_stream(0)
    s = torch.cuda.ExternalStream(sp, device="cuda:0")
    for _ in range(10):
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, ab, 0)
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, ba, 0)
    J.jacc_wait()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record(s)
    for _ in range(reps):
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, ab, 0)
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, ba, 0)
    e1.record(s)
    J.jacc_wait()
    t = e0.elapsed_time(e1) / 1e3 / (2 * reps)
    byts = 8 * N * N + 8 * (N - 2) ** 2
    J.jacc_finalize()
    print(json.dumps({"variant": os.environ.get("JACC_JACOBI_VARIANT", "0"),
                      "prof": os.environ.get("TUNE_PROF", "0"), "us": t * 1e6,
                      "gbs": byts / t / 1e9}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one()
    else:
        vs = [int(x) for x in sys.argv[1:]] if len(sys.argv) > 1 else range(8)
        for v, prof in [(v, "0") for v in vs] + [(0, "1")]:
            env = dict(os.environ, JACC_JACOBI_VARIANT=str(v), TUNE_PROF=prof)
            r = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True)
            print(r.stdout.strip() or r.stderr[-500:], flush=True)
