"""NEXT-2 host logic: parallel-dimension selection (A18) and the
cudaMemcpy2D-shaped exchange plan (A19), C++ runtime vs the plain
oracle and the paper's Listing 5 / NPB-BT numbers."""
import os
import random

import pytest

from oracle import layout as lay
from oracle import partition

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def J():
    import __graft_entry__ as ge
    ge.build_jacc()
    from paper_2110_14340_b200 import jacc
    return jacc


def _golden():
    g = {}
    for line in open(os.path.join(GOLDEN, "multidim_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        k, *v = line.split()
        g[k] = [int(x) for x in v]
    return g


def test_listing5_split_dim_oracle_and_runtime(J):
    g = _golden()
    assert lay.select_split_dim(g["listing5_par"], g["listing5_seq"]) == g["listing5_split"][0]
    assert J.jacc_select_split_dim(g["listing5_par"], g["listing5_seq"]) == g["listing5_split"][0]
    # Fortran picks the rightmost of the tied parallel dims
    assert lay.select_split_dim(g["listing5_par"], g["listing5_seq"], fortran=True) == 5
    assert J.jacc_select_split_dim(g["listing5_par"], g["listing5_seq"], fortran=True) == 5


def test_split_dim_rules(J):
    # no parallel iterator anywhere -> duplicate
    assert lay.select_split_dim([0, 0], [1, 0]) == -1 == J.jacc_select_split_dim([0, 0], [1, 0])
    # most parallel iterators wins over fewer sequential
    assert lay.select_split_dim([1, 2], [0, 3]) == 1 == J.jacc_select_split_dim([1, 2], [0, 3])
    # fewest sequential among the most parallel
    assert lay.select_split_dim([1, 1, 1], [2, 0, 1]) == 1 == J.jacc_select_split_dim([1, 1, 1], [2, 0, 1])
    rng = random.Random(5)
    for _ in range(2000):
        nd = rng.randint(1, 6)
        par = [rng.randint(0, 2) for _ in range(nd)]
        seq = [rng.randint(0, 2) for _ in range(nd)]
        f = rng.random() < 0.5
        assert J.jacc_select_split_dim(par, seq, f) == lay.select_split_dim(par, seq, f)


def test_bt_exchange_plan_matches_paper(J):
    g = _golden()
    ext = g["bt_extents"]
    for d in range(4):
        p = J.jacc_exchange_plan(ext, 8, 4, 4, d)
        assert p["count"] == g["bt_copies"][0]              # "75 segments"
        per_copy = p["height"] * p["width_bytes"]
        assert per_copy == (g["bt_bytes_per_copy_d0"][0] if d < 2 else g["bt_bytes_per_copy_d3"][0])


def _covered(plan):
    out = []
    for c in range(plan["count"]):
        for r in range(plan["height"]):
            b0 = plan["first_offset_bytes"] + c * plan["outer_stride_bytes"] + r * plan["pitch_bytes"]
            out.append((b0, b0 + plan["width_bytes"]))
    return out


@pytest.mark.parametrize("seed", range(40))
def test_exchange_plan_covers_exactly_the_owned_slice(J, seed):
    rng = random.Random(seed)
    nd = rng.randint(1, 4)
    ext = [rng.randint(1, 6) for _ in range(nd)]
    s = rng.randrange(nd)
    n = rng.randint(1, 5)
    elem = rng.choice([4, 8])
    for d in range(n):
        lo, hi = partition(ext[s], n, d)
        want = lay.slice_elements(ext, s, lo, hi)
        got = []
        for a, b in _covered(J.jacc_exchange_plan(ext, elem, s, n, d)):
            assert a % elem == 0 and b % elem == 0
            got.extend(range(a // elem, b // elem))
        assert sorted(got) == want and len(got) == len(set(got))


def test_bench_pushed_elements_dense_rule():
    """bench.py counts the bytes a bitmap merge stores (DESIGN R-22): words
    with >= 8 dirty elements inside the owned slice move whole, the others
    element by element, and words straddling the slice edge never whole."""
    import numpy as np
    import bench
    bm = np.zeros(4, dtype=np.uint32)
    bm[0] = 0xFF          # 8 dirty, inside [0, 100): whole -> 32
    bm[1] = 0x7F          # 7 dirty: element by element -> 7
    bm[2] = 0xFFFF        # 16 dirty but word 2 = [64, 96) inside -> 32
    bm[3] = 0xFFFFFFFF    # 32 dirty, word [96, 128) straddles hi = 100 -> 32 bits counted, not "whole"
    assert bench._pushed_elements(bm, 0, 100) == 32 + 7 + 32 + 32
    bm[3] = 0x0F0F        # 8 dirty, straddling: element by element
    assert bench._pushed_elements(bm, 0, 100) == 32 + 7 + 32 + 8
    assert bench._pushed_elements(bm, 1, 128) == 8 + 7 + 32 + 32  # word 0 starts before lo
