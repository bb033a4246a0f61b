"""Randomised programs through the C-ABI (-m gpu): seeded sequences of
launches (Jacobi both directions, square, scatter-add, sum reduction,
GEMM, the Fig. 4 chain, Himeno stencil + copy),
partial update_host / update_device calls with host-side edits in between,
and waits, under random runtime configurations (device count, merge
policy, execution mode, split dimension, async queues, iteration-split
scatter).  A host model advances the same state with the CPU oracle; every
update_host must leave the user's array equal to the model's host copy
bit for bit, every reduction must equal the model's exact (dyadic) sum, and
under EAGER every replica must equal the model's device state.

This exercises the validity tracker, the pulls, both merge policies and the
dirty-record slots across arbitrary interleavings, beyond the fixed
sequences of test_gpu_parity.py.
"""
import os

import numpy as np
import pytest

import oracle as orc
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def J():
    import __graft_entry__ as ge
    ge.build_jacc()
    from paper_2110_14340_b200 import jacc
    return jacc


def _dyadic(rng, n):
    return rng.integers(0, 1024, n).astype(np.float64) / 1024.0


class Program:
    """world=None: single process, random device count; world=W: one rank
    of a W-process job (same seed on every rank: SPMD), where adaptive
    mode, async queues and the iteration-split scatter do not apply."""

    def __init__(self, J, seed, world=None):
        self.J = J
        self.rng = np.random.default_rng(seed)
        r = self.rng
        self.n = int(r.choice([1, 2, 3, 5]))
        self.policy = int(r.integers(0, 2))
        self.mode = int(r.choice([0, 0, 1, 2])) if self.n > 1 else 0
        self.split = int(r.choice([-1, -1, 1]))
        self.nq = int(r.choice([1, 1, 3]))
        self.itersplit = int(self.n > 1 and self.nq == 1 and r.random() < 0.3)
        self.local = list(range(self.n))
        if world is not None:
            self.n, self.nq, self.itersplit = world, 1, 0
            self.mode = int(r.choice([0, 0, 1]))
            self.local = [J.jacc_rank()]
        N = int(r.integers(3, 70))
        L = int(r.integers(1, 3000))
        S, M = int(r.integers(1, 5000)), int(r.integers(1, 4000))
        gm, gk, gn = (int(v) for v in r.integers(1, 40, 3))
        fn = int(r.integers(1, 300))
        hI, hJ, hK = (int(v) for v in r.integers(3, 14, 3))
        # host arrays (the user's) and the model's device state
        self.host = {
            "A": synth.uniform_f64(N * N, seed, 1).reshape(N, N),
            "B": synth.uniform_f64(N * N, seed, 2).reshape(N, N),
            "y": synth.uniform_f32(L, seed, 3) * 4 - 2,
            "x": np.zeros(L, dtype=np.float32),
            "idx": synth.index_i32(S, M, seed, 4),
            "bs": synth.dyadic_f64(S, seed, 5),
            "a": synth.dyadic_f64(M, seed, 6),
            # GEMM on small integers: exact in any summation order
            "GA": synth.int_i32(gm * gk, -8, 8, seed, 7).astype(np.float64).reshape(gm, gk),
            "GB": synth.int_i32(gk * gn, -8, 8, seed, 8).astype(np.float64).reshape(gk, gn),
            "GC": np.zeros((gm, gn)),
            # Fig. 4 chain: k = kx[i] injective into [n, 2n)
            "jx": synth.index_i32(fn, 5 * fn + 7, seed, 9),
            "kx": (synth.permutation_i32(fn, seed, 10) + fn).astype(np.int32),
            "fc": synth.uniform_f64(5 * fn + 7, seed, 11),
            "fa": synth.uniform_f64(2 * fn + 3, seed, 12),
            "fb": synth.uniform_f64(3 * fn + 1, seed, 13),
        }
        hp, ha, hb, hc, hw1, hbd = synth.himeno_random(hI, hJ, hK, seed)
        self.host.update({"hp": hp, "ha": ha, "hb": hb, "hc": hc, "hw1": hw1, "hbd": hbd,
                          "hw2": np.zeros_like(hp)})
        self.dev = {k: v.copy() for k, v in self.host.items()}
        self.model_host = {k: v.copy() for k, v in self.host.items()}

    def config(self):
        J = self.J
        J.jacc_set_merge_policy(self.policy)
        J.jacc_set_mode(self.mode)
        J.jacc_set_split_dim(self.split)
        if self.nq > 1:
            J.jacc_set_queues(self.nq)
        if self.itersplit:
            J.jacc_set_scatter_split(self.itersplit)

    def run(self, steps, create):
        J = self.J
        log = []
        self.config()
        for k in self.host:
            create(self.host[k])
            J.jacc_update_device(self.host[k])
        for i in range(steps):
            self.step(log)
            if i % 10 == 9:
                self.check_replicas(log)
        for k in ("A", "B", "x", "a", "GC", "fa", "fb", "hp", "hw2"):
            J.jacc_update_host(self.host[k])
            assert np.array_equal(self.host[k], self.dev[k]), (k, self.desc(), log)

    def desc(self):
        return (f"n={self.n} policy={self.policy} mode={self.mode} split={self.split} "
                f"nq={self.nq} itersplit={self.itersplit} N={self.host['A'].shape[0]} "
                f"L={self.host['y'].size} S={self.host['idx'].size} M={self.host['a'].size}")

    def aid(self):
        if self.nq == 1:
            return -1
        return int(self.rng.choice([-1, self.J.JACC_ASYNC_AUTO, 0, 1, 2]))

    def step(self, log):
        J, r, h, dev = self.J, self.rng, self.host, self.dev
        IN, OUT, INOUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT, J.JACC_ARG_ARRAY_INOUT
        op = r.choice(["jacAB", "jacBA", "square", "scatter", "sum", "gemm", "fig4", "himeno",
                       "uh", "ud", "wait"],
                      p=[0.14, 0.14, 0.09, 0.1, 0.06, 0.08, 0.08, 0.1, 0.11, 0.06, 0.04])
        log.append(str(op))
        if op in ("jacAB", "jacBA"):
            s, d = ("A", "B") if op == "jacAB" else ("B", "A")
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, h[s]), J.arg(OUT, h[d])],
                          self.aid())
            orc.jacobi2d_sweep(dev[s], dev[d])
        elif op == "square":
            L = h["y"].size
            lo = int(r.integers(0, L))
            hi = int(r.integers(lo + 1, L + 1))
            J.jacc_launch(J.JACC_LOOP_SQUARE_F32, J.make_range(lo, hi),
                          [J.arg(IN, h["y"]), J.arg(OUT, h["x"])], self.aid())
            dev["x"][lo:hi] = orc.square_f32(np.ascontiguousarray(dev["y"][lo:hi]))
        elif op == "scatter":
            S = h["idx"].size
            J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_F64, J.make_range(0, S),
                          [J.arg(IN, h["idx"]), J.arg(IN, h["bs"]), J.arg(INOUT, h["a"])],
                          self.aid())
            orc.scatter_add(dev["idx"], dev["bs"], dev["a"])
        elif op == "sum":
            s_in = float(r.integers(-64, 64)) / 8
            out = np.array([s_in])
            J.jacc_launch(J.JACC_LOOP_SUM_F64, J.make_range(0, h["a"].size),
                          [J.arg(IN, h["a"]), J.arg(J.JACC_ARG_REDUCE_SUM_F64, out)], self.aid())
            ref = orc.sum_f64(dev["a"], s_in)     # dyadic: exact in any order
            assert out[0] == ref, (self.desc(), log)
        elif op == "gemm":
            J.jacc_launch(J.JACC_LOOP_GEMM_F64, None,
                          [J.arg(IN, h["GA"]), J.arg(IN, h["GB"]), J.arg(OUT, h["GC"])], self.aid())
            dev["GC"][...] = orc.gemm_f64(dev["GA"], dev["GB"])
        elif op == "fig4":
            x_in = float(r.integers(-8, 8)) / 4
            fn = h["jx"].size
            J.jacc_launch(J.JACC_LOOP_FIG4_F64, J.make_range(0, fn),
                          [J.arg(IN, h["jx"]), J.arg(IN, h["kx"]), J.arg(IN, h["fc"]),
                           J.arg(OUT, h["fa"]), J.arg(OUT, h["fb"]),
                           J.arg(J.JACC_ARG_SCALAR_F64, f64=x_in)], self.aid())
            orc.fig4(dev["jx"], dev["kx"], dev["fc"], x_in, dev["fa"], dev["fb"])
        elif op == "himeno":
            g = np.zeros(1)
            names = ("hp", "ha", "hb", "hc", "hw1", "hbd")
            J.jacc_launch(J.JACC_LOOP_HIMENO_F32, None,
                          [J.arg(IN, h[k]) for k in names] +
                          [J.arg(OUT, h["hw2"]), J.arg(J.JACC_ARG_REDUCE_SUM_F64, g),
                           J.arg(J.JACC_ARG_SCALAR_F64, f64=0.8)], self.aid())
            _, gref, _ = orc.himeno_stencil(*(dev[k] for k in names), dev["hw2"])
            assert abs(g[0] - gref) <= 1e-12 * abs(gref) + 1e-300, (self.desc(), log)
            J.jacc_launch(J.JACC_LOOP_HIMENO_COPY_F32, None,
                          [J.arg(IN, h["hw2"]), J.arg(OUT, h["hp"])], self.aid())
            orc.himeno_copy(dev["hw2"], dev["hp"])
        elif op == "uh":
            k = str(r.choice(["A", "B", "x", "a", "GC", "fa", "fb", "hp", "hw2"]))
            e0, e1 = self._subrange(h[k].size)
            J.jacc_update_host(h[k], e0 * h[k].itemsize, (e1 - e0) * h[k].itemsize)
            mh = self.model_host[k].reshape(-1)
            mh[e0:e1] = dev[k].reshape(-1)[e0:e1]
            assert np.array_equal(h[k], self.model_host[k]), (k, e0, e1, self.desc(), log)
        elif op == "ud":
            k = str(r.choice(["A", "B", "y", "a", "GA", "fc", "fa", "hp", "ha"]))
            e0, e1 = self._subrange(h[k].size)
            flat = h[k].reshape(-1)
            if k == "a":
                flat[e0:e1] = _dyadic(r, e1 - e0)
            elif k == "GA":
                flat[e0:e1] = r.integers(-8, 8, e1 - e0).astype(np.float64)
            else:
                flat[e0:e1] = r.random(e1 - e0).astype(flat.dtype)
            self.model_host[k].reshape(-1)[e0:e1] = flat[e0:e1]
            J.jacc_update_device(h[k], e0 * h[k].itemsize, (e1 - e0) * h[k].itemsize)
            dev[k].reshape(-1)[e0:e1] = flat[e0:e1]
        else:
            J.jacc_wait()

    def _subrange(self, size):
        e0 = int(self.rng.integers(0, size))
        e1 = int(self.rng.integers(e0 + 1, size + 1))
        return e0, e1

    def check_replicas(self, log):
        J = self.J
        if self.policy != J.JACC_MERGE_EAGER:
            return
        J.jacc_wait()
        for k in ("A", "B", "x", "a", "GC", "fa", "fb", "hp", "hw2"):
            for d in self.local:
                assert np.array_equal(J.jacc_get_replica(self.host[k], d), self.dev[k]), \
                    (k, d, self.desc(), log)


# JACC_RANDOM_PROGRAMS=<count> widens the sweep (bug hunting)
@pytest.mark.parametrize("seed", range(int(os.environ.get("JACC_RANDOM_PROGRAMS", "160"))))
def test_random_program(J, seed):
    prog = Program(J, 1000 + seed)
    J.jacc_init(prog.n, [0] * prog.n)
    try:
        prog.run(60, J.jacc_data_create)
    finally:
        J.jacc_finalize()
