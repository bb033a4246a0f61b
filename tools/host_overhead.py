"""Host cost per jacc_launch (plan + enqueue on every device) for n logical
devices (virtual on one GPU), HALO Jacobi 4096^2, vs CUDA-graph replay of
the same 200-launch step.  Prints one JSON line per n."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2110_14340_b200 import jacc as J  # noqa: E402


def main():
    N = 4096
    for n in (1, 2, 4, 8):
        A, B = synth.polybench_jacobi2d(N)
        J.jacc_init(n, [0] * n)
        J.jacc_set_merge_policy(J.JACC_MERGE_HALO)
        for a in (A, B):
            J.jacc_data_create(a)
            J.jacc_update_device(a)
        IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
        ab, ba = [J.arg(IN, A), J.arg(OUT, B)], [J.arg(IN, B), J.arg(OUT, A)]

        def step():
            for _ in range(100):
                J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, ab, 0)
                J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, ba, 0)

        step()
        J.jacc_wait()
        t0 = time.perf_counter()
        step()
        host = (time.perf_counter() - t0) / 200 * 1e6
        J.jacc_wait()
        t1 = time.perf_counter()
        J.jacc_wait()
        J.jacc_graph_begin()
        step()
        g = J.jacc_graph_end()
        J.jacc_graph_replay(g, 1)
        J.jacc_wait()
        t2 = time.perf_counter()
        J.jacc_graph_replay(g, 1)
        ghost = (time.perf_counter() - t2) / 200 * 1e6
        J.jacc_wait()
        J.jacc_finalize()
        print(json.dumps({"n": n, "host_us_per_launch": host, "graph_host_us_per_launch": ghost}),
              flush=True)


if __name__ == "__main__":
    main()
