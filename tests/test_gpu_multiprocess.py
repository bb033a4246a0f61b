"""One process per GPU (-m gpu): world 2 and 3 ranks sharing the box's
GPU(s), CUDA-IPC mapped peer replicas, shared-memory lockstep, IPC-event
ordering; every rank's results must equal the oracle."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle as orc
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("policy", ["halo", "eager"])
def test_multiprocess_parity(tmp_path, world, policy):
    import __graft_entry__ as ge
    ge.build_jacc()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           str(world), "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "workers", "mp_worker.py"), "--out", str(tmp_path),
           "--policy", policy]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    N, T = 301, 3
    A = synth.uniform_f64(N * N, 81, 1).reshape(N, N)
    B = synth.uniform_f64(N * N, 81, 2).reshape(N, N)
    A0 = A.copy()
    orc.jacobi2d(T, A, B)
    L = 100_003
    dot = orc.dot_f64(synth.dyadic_f64(L, 82, 3), synth.dyadic_f64(L, 82, 4), 0.75)
    S, M = 50_000, 7_001
    idx = synth.index_i32(S, M, 83, 5)
    b = synth.int_i32(S, -1000, 1000, 83, 6)
    av = synth.int_i32(M, -10**6, 10**6, 83, 7)
    a0 = av.copy()
    orc.scatter_add(idx, b, av)
    GA = synth.uniform_f64(67 * 29, 84, 1).reshape(67, 29)
    GB = synth.uniform_f64(29 * 45, 84, 2).reshape(29, 45)
    gref = orc.gemm_f64(GA, GB)
    gbound = np.abs(GA) @ np.abs(GB)
    hp, ha, hb, hc, hw1, hbd = synth.himeno_random(11, 9, 13, 85)
    hw2 = np.zeros_like(hp)
    hg_ref = []
    for _ in range(2):
        hg_ref.append(orc.himeno_stencil(hp, ha, hb, hc, hw1, hbd, hw2)[1])
        orc.himeno_copy(hw2, hp)
    hp_ref = hp
    fn = 301
    kx = (synth.permutation_i32(fn, 86, 30) + fn).astype(np.int32)
    jx = synth.index_i32(fn, 5 * fn + 7, 86, 31)
    fc = synth.uniform_f64(5 * fn + 7, 86, 32)
    fa_ref = synth.uniform_f64(2 * fn + 3, 86, 33)
    fb_ref = synth.uniform_f64(3 * fn + 1, 86, 34)
    orc.fig4(jx, kx, fc, 0.25, fa_ref, fb_ref)
    for rank in range(world):
        z = np.load(tmp_path / f"rank{rank}.npz")
        assert int(z["world"]) == world
        # the ranks share this box's GPU: the runtime must say so (GPU UUIDs
        # in the exchanged runtime handles) and combine over peer memory
        import torch
        if torch.cuda.device_count() < world:
            assert z["info"].tolist() == [world, 0, 0]
        assert np.array_equal(z["A"], A) and np.array_equal(z["B"], B), rank
        lo, hi = orc.partition(N, world, rank)
        # dirty range of the last A-writing sweep == oracle write log
        tmp = np.zeros((N, N))
        assert tuple(z["dirty_A"].tolist()) == orc.jacobi2d_sweep_filtered(A0, tmp, lo, hi - 1)
        if policy == "eager":
            assert np.array_equal(z["repA"], A)
        assert z["dot"][0] == dot
        assert np.array_equal(z["scatter"], av)
        slo, shi = orc.partition(M, world, rank)
        bm, _, _ = orc.scatter_add_filtered(idx, b, a0.copy(), slo, shi - 1)
        assert np.array_equal(z["bitmap"], bm)
        assert (np.abs(z["gemm"] - gref) <= 1e-12 * gbound).all()
        assert np.array_equal(z["himeno_p"], hp_ref)
        assert np.allclose(z["himeno_gosa"], hg_ref, rtol=1e-12, atol=0)
        assert np.array_equal(z["fig4_a"], fa_ref) and np.array_equal(z["fig4_b"], fb_ref)


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_random_programs(world):
    """Randomised programs (test_gpu_random_programs.Program) run SPMD in
    one-process-per-GPU mode: every rank checks its own replicas and host
    arrays against the oracle model."""
    import __graft_entry__ as ge
    ge.build_jacc()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           str(world), "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "workers", "mp_random.py"), "--seeds", "24",
           "--first", str(5000 + 100 * world)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    # the first failing rank's own error (the others then time out waiting
    # for it): every line that names an error, before the tail
    first = [l for l in r.stderr.splitlines() if "Error" in l or "assert" in l or "mismatch" in l][:40]
    assert r.returncode == 0, "\n".join(first) + "\n...\n" + r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("ok 24") == world
