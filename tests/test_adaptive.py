"""NEXT-1 adaptive utilization: the oracle controller pinned by
the paper's inequalities and hand-derived state sequences; the C++
controller (jacc_adaptive_replay, pure host logic) equal to the oracle on
random traces."""
import os
import random

import pytest

from oracle import adaptive as ad

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
W, P, M, F = ad.DUP_WARMUP, ad.DUP_PROFILING, ad.MULTI, ad.DUP_FINAL


@pytest.fixture(scope="module")
def J():
    import __graft_entry__ as ge
    ge.build_jacc()
    from paper_2110_14340_b200 import jacc
    return jacc


def test_golden_inequalities():
    for line in open(os.path.join(GOLDEN, "adaptive_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        eq, n, tk, tc, ws, pk, lhs, rhs, holds = line.split()
        n, tk, tc, ws, pk, lhs, rhs = int(n), float(tk), float(tc), float(ws), float(pk), float(lhs), float(rhs)
        if eq == "eq1":
            assert tk == pytest.approx(lhs) and tk / n + ws / pk == pytest.approx(rhs)
            assert (tk > tk / n + ws / pk) == bool(int(holds))
        else:
            assert tk + tc == pytest.approx(lhs) and tk * n == pytest.approx(rhs)
            assert (tk + tc > tk * n) == bool(int(holds))


def test_switch_to_multi_after_five_eq1():
    """warm-up (not profiled), then five executions satisfying Eq. (1)."""
    trace = [(0.010, 0.0, 25e6)] * 8
    st = ad.replay(trace, 4, 25e9)
    assert st == [W, P, P, P, P, P, M, M, M]


def test_eq1_never_holds_stays_duplicated():
    # n = 1: t_K > t_K + ws/peak is never true
    assert set(ad.replay([(0.01, 0, 1e6)] * 20, 1, 25e9)[1:]) == {P}
    # exchange far slower than the kernel
    assert set(ad.replay([(0.001, 0, 1e9)] * 20, 8, 25e9)[1:]) == {P}


def test_back_to_dup_after_five_eq2_positive_margin():
    # profiling: t_K = 10 ms for 25 MB -> eff_dup = 4e-10 s/B
    trace = [(0.010, 0.0, 25e6)] * 6
    # multi: t_K = 1 ms, t_C = 5 ms, n = 4: Eq. (2) 6 > 4 holds, margin +2 ms
    trace += [(0.001, 0.005, 25e6)] * 6
    st = ad.replay(trace, 4, 25e9)
    assert st[:7] == [W, P, P, P, P, P, M]
    assert st[6:11] == [M, M, M, M, M] and st[11] == F and st[12] == F


def test_negative_mean_margin_keeps_multi():
    trace = [(0.010, 0.0, 25e6)] * 6          # eff_dup * ws = 10 ms
    good = (0.004, 0.0, 25e6)                 # left 4 ms: margin 4 - min(16, 10) = -6 ms
    bad = (0.009, 0.002, 25e6)                # left 11 > 10 (Eq. 3): margin +1 ms
    trace += [bad, good] * 10
    st = ad.replay(trace, 4, 25e9)
    assert st[6:] == [M] * 21                 # five+ hits, but mean margin < 0


def test_dup_final_is_absorbing():
    trace = [(0.010, 0.0, 25e6)] * 6 + [(0.001, 0.005, 25e6)] * 5 + [(0.010, 0.0, 25e6)] * 10
    st = ad.replay(trace, 4, 25e9)
    assert st[11] == F and set(st[11:]) == {F}


def _random_trace(rng, m):
    tr = []
    for _ in range(m):
        tk = rng.choice([1e-4, 1e-3, 1e-2]) * rng.uniform(0.5, 2)
        tc = rng.choice([0.0, 1e-5, 1e-3, 1e-2]) * rng.uniform(0.5, 2)
        ws = rng.choice([0.0, 1e5, 1e7, 1e9])
        tr.append((tk, tc, ws))
    return tr


def test_cpp_controller_matches_oracle_random(J):
    rng = random.Random(2110)
    for it in range(1000):
        n = rng.choice([1, 2, 4, 8])
        pk = rng.choice([25e9, 770e9])
        tr = _random_trace(rng, rng.randint(0, 40))
        assert J.jacc_adaptive_replay(n, pk, tr) == ad.replay(tr, n, pk), it


def test_cpp_controller_hand_sequences(J):
    trace = [(0.010, 0.0, 25e6)] * 6 + [(0.001, 0.005, 25e6)] * 6
    assert J.jacc_adaptive_replay(4, 25e9, trace) == ad.replay(trace, 4, 25e9)
    assert J.jacc_adaptive_replay(4, 25e9, [])[-1] == W
