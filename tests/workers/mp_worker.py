"""Worker for the one-process-per-GPU tests: launched by torch.distributed.run
(gloo process group for the handle exchange).  Every rank runs the same
SPMD program through the C-ABI and saves what it sees to --out."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--policy", default="halo")
    ap.add_argument("--N", type=int, default=301)
    ap.add_argument("--T", type=int, default=3)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    import synth
    from paper_2110_14340_b200 import dist as jd
    from paper_2110_14340_b200 import jacc as J

    dist.init_process_group("gloo")
    ngpu = torch.cuda.device_count()
    rank = dist.get_rank()
    ordinal = rank % ngpu
    torch.cuda.set_device(ordinal)
    rank, world, distinct = jd.init_rank(ordinal)
    J.jacc_set_merge_policy(J.JACC_MERGE_HALO if a.policy == "halo" else J.JACC_MERGE_EAGER)
    IN, OUT, INOUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT, J.JACC_ARG_ARRAY_INOUT
    res = {}
    # Jacobi
    N = a.N
    A = synth.uniform_f64(N * N, 81, 1).reshape(N, N)
    B = synth.uniform_f64(N * N, 81, 2).reshape(N, N)
    for arr in (A, B):
        jd.data_create(arr)
        J.jacc_update_device(arr)
    for _ in range(a.T):
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, A), J.arg(OUT, B)], 0)
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, B), J.arg(OUT, A)], 0)
    J.jacc_wait()
    res["dirty_A"] = np.array(J.jacc_get_dirty_range(A, rank), dtype=np.uint64)
    res["repA"] = J.jacc_get_replica(A, rank)
    J.jacc_update_host(A)
    J.jacc_update_host(B)
    res["A"], res["B"] = A, B
    # dot (reduction combine across ranks)
    L = 100_003
    x = synth.dyadic_f64(L, 82, 3)
    y = synth.dyadic_f64(L, 82, 4)
    for arr in (x, y):
        jd.data_create(arr)
        J.jacc_update_device(arr)
    s = np.array([0.75])
    J.jacc_launch(J.JACC_LOOP_DOT_F64, J.make_range(0, L),
                  [J.arg(IN, x), J.arg(IN, y), J.arg(J.JACC_ARG_REDUCE_SUM_F64, s)])
    res["dot"] = s.copy()
    # scatter
    S, M = 50_000, 7_001
    idx = synth.index_i32(S, M, 83, 5)
    b = synth.int_i32(S, -1000, 1000, 83, 6)
    av = synth.int_i32(M, -10**6, 10**6, 83, 7)
    for arr in (idx, b, av):
        jd.data_create(arr)
        J.jacc_update_device(arr)
    J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_I32, J.make_range(0, S),
                  [J.arg(IN, idx), J.arg(IN, b), J.arg(INOUT, av)])
    res["bitmap"] = J.jacc_get_dirty_bitmap(av, rank, M)
    J.jacc_update_host(av)
    res["scatter"] = av
    # GEMM (EAGER: merge fused into the epilogue, IPC-mapped peer stores)
    M, Nn, Kk = 67, 45, 29
    GA = synth.uniform_f64(M * Kk, 84, 1).reshape(M, Kk)
    GB = synth.uniform_f64(Kk * Nn, 84, 2).reshape(Kk, Nn)
    GC = np.zeros((M, Nn))
    for arr in (GA, GB, GC):
        jd.data_create(arr)
        J.jacc_update_device(arr)
    J.jacc_launch(J.JACC_LOOP_GEMM_F64, None, [J.arg(IN, GA), J.arg(IN, GB), J.arg(OUT, GC)])
    J.jacc_update_host(GC)
    res["gemm"] = GC
    # Himeno (stencil + gosa reduction over ranks, copy with plane pushes)
    hp, ha, hb, hc, hw1, hbd = synth.himeno_random(11, 9, 13, 85)
    hw2 = np.zeros_like(hp)
    for arr in (hp, ha, hb, hc, hw1, hbd, hw2):
        jd.data_create(arr)
        J.jacc_update_device(arr)
    gos = []
    for _ in range(2):
        g = np.zeros(1)
        J.jacc_launch(J.JACC_LOOP_HIMENO_F32, None,
                      [J.arg(IN, hp), J.arg(IN, ha), J.arg(IN, hb), J.arg(IN, hc), J.arg(IN, hw1),
                       J.arg(IN, hbd), J.arg(OUT, hw2), J.arg(J.JACC_ARG_REDUCE_SUM_F64, g),
                       J.arg(J.JACC_ARG_SCALAR_F64, f64=0.8)])
        gos.append(g[0])
        J.jacc_launch(J.JACC_LOOP_HIMENO_COPY_F32, None, [J.arg(IN, hw2), J.arg(OUT, hp)], 0)
    J.jacc_update_host(hp)
    res["himeno_p"] = hp
    res["himeno_gosa"] = np.array(gos)
    # Fig. 4 chain (two written arrays, separately divided)
    fn = 301
    kx = (synth.permutation_i32(fn, 86, 30) + fn).astype(np.int32)
    jx = synth.index_i32(fn, 5 * fn + 7, 86, 31)
    fc = synth.uniform_f64(5 * fn + 7, 86, 32)
    fa = synth.uniform_f64(2 * fn + 3, 86, 33)
    fb = synth.uniform_f64(3 * fn + 1, 86, 34)
    for arr in (jx, kx, fc, fa, fb):
        jd.data_create(arr)
        J.jacc_update_device(arr)
    J.jacc_launch(J.JACC_LOOP_FIG4_F64, J.make_range(0, fn),
                  [J.arg(IN, jx), J.arg(IN, kx), J.arg(IN, fc), J.arg(OUT, fa), J.arg(OUT, fb),
                   J.arg(J.JACC_ARG_SCALAR_F64, f64=0.25)])
    J.jacc_update_host(fa)
    J.jacc_update_host(fb)
    res["fig4_a"], res["fig4_b"] = fa, fb
    info = J.jacc_get_info()
    res["info"] = np.array([info["n_devices"], info["distinct_gpus"], info["combine"] == "nccl"])
    jd.finalize()
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), world=world, **res)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
