"""NEXT-4 automated asynchronous execution (Fig. 2): the oracle
scheduler pinned by the paper's Fig. 2 scenario and hand-derived cases; the
C++ scheduler (jacc_queue_replay, pure host logic) equal to it on random
launch sequences."""
import random

import pytest

from oracle import queues as oq


@pytest.fixture(scope="module")
def J():
    import __graft_entry__ as ge
    ge.build_jacc()
    from paper_2110_14340_b200 import jacc
    return jacc


A, B, C, D, E = range(5)


def test_fig2_scenario():
    """Kernel1 updates a and (on another queue) b; Kernel2 reads a and b and
    waits for the other producer queue; Kernel3 reads b and does not wait
    (P:375-376)."""
    trace = [((), (A,), None),        # K1a: no deps -> LRU queue 0
             ((), (B,), None),        # K1b: no deps -> LRU queue 1
             ((A, B), (C,), None),    # K2: deps on q0 (t1) and q1 (t2) -> q1, waits q0
             ((B,), (D,), None)]      # K3: dep b on q1 -> q1, no wait
    out = oq.replay(trace, 16)
    assert out[0] == (0, []) and out[1] == (1, [])
    assert out[2] == (1, [0])
    assert out[3] == (1, [])


def test_transitive_elision_and_explicit_queue():
    trace = [((), (A,), None), ((), (B,), None), ((A, B), (C,), None),
             ((C,), (D,), 2),         # explicit queue 2: waits for q1 (writer of c)
             ((A,), (E,), 2)]         # a was ordered before q1's wait: already solved
    out = oq.replay(trace, 4)
    assert out[3] == (2, [1])
    assert out[4] == (2, [])


def test_war_dependency_and_lru():
    trace = [((A,), (B,), None),      # q0
             ((), (C,), None),        # q1 (LRU)
             ((), (A,), 1)]           # writes a read by q0 at t1: WAR -> waits q0
    out = oq.replay(trace, 3)
    assert out[2] == (1, [0])
    # independent launches round-robin over the least recently used queues
    out = oq.replay([((), (x,), None) for x in range(6)], 4)
    assert [q for q, _ in out] == [0, 1, 2, 3, 0, 1]


def test_same_queue_chain_never_waits():
    trace = [((A,), (B,), None), ((B,), (C,), None), ((C,), (A,), None)]
    out = oq.replay(trace, 16)
    assert all(q == 0 and w == [] for q, w in out)


def _rand_trace(rng, m, nq, narr):
    tr = []
    for _ in range(m):
        rd = rng.sample(range(narr), min(narr, rng.randint(0, 3)))
        wr = rng.sample(range(narr), min(narr, rng.randint(0, 2)))
        req = rng.randrange(nq) if rng.random() < 0.2 else None
        tr.append((rd, wr, req))
    return tr


def test_cpp_scheduler_matches_oracle_random(J):
    rng = random.Random(355)
    for it in range(500):
        nq = rng.choice([1, 2, 4, 16])
        tr = _rand_trace(rng, rng.randint(0, 30), nq, rng.randint(1, 8))
        assert J.jacc_queue_replay(nq, tr) == oq.replay(tr, nq), it


def test_schedule_is_dependency_safe():
    """Soundness: replaying with all waits honoured, every launch is ordered
    after the last writer / readers it depends on (no stale read)."""
    rng = random.Random(7)
    for _ in range(300):
        nq = rng.choice([2, 4])
        tr = _rand_trace(rng, 25, nq, 6)
        out = oq.replay(tr, nq)
        # ordered[l] = set of launches known complete before launch l starts
        ordered = []
        last_on_q = {}
        for l, ((rd, wr, _), (q, waits)) in enumerate(zip(tr, out)):
            s = set()
            if q in last_on_q:
                p = last_on_q[q]
                s |= ordered[p] | {p}
            for w in waits:
                p = last_on_q[w]
                s |= ordered[p] | {p}
            ordered.append(s)
            last_on_q[q] = l
            # every earlier conflicting launch must be ordered before l
            for m in range(l):
                rdm, wrm, _ = tr[m]
                conflict = (set(wrm) & (set(rd) | set(wr))) or (set(rdm) & set(wr))
                if conflict:
                    assert m in s, (l, m)
