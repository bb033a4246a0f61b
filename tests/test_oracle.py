"""Pins for the CPU oracle (-m "not gpu").

The oracle is checked against things other than itself: values the paper
(or SPEC) prints, closed forms, invariants, special cases that reduce to a
library routine (numpy), exact rational arithmetic (fractions), and brute
force on tiny inputs.  Each test names the passage it pins.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as orc
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
U64MAX = 2**64 - 1


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# --------------------------------------------------------------------------
# c4 partition ("equally dividing"; S:266 remainder rule)
# --------------------------------------------------------------------------
def test_partition_golden():
    for row in _golden("partition_blocks.txt"):
        E, n = int(row[0]), int(row[1])
        for d, blk in enumerate(row[2:]):
            lo, hi = map(int, blk.split(":"))
            assert orc.partition(E, n, d) == (lo, hi), (E, n, d)


@pytest.mark.parametrize("n", range(1, 10))
def test_partition_properties(n):
    for E in list(range(0, 40)) + [16384, 2**30, 2**28 + 7]:
        blocks = [orc.partition(E, n, d) for d in range(n)]
        assert blocks[0][0] == 0 and blocks[-1][1] == E          # covering
        for (a, b), (c, _) in zip(blocks, blocks[1:]):
            assert b == c                                      # contiguous, disjoint
        sizes = [b - a for a, b in blocks]
        assert sum(sizes) == E
        assert max(sizes) - min(sizes) <= 1                      # "equally"
        r = E % n
        assert all(s == E // n + (1 if d < r else 0) for d, s in enumerate(sizes))


# --------------------------------------------------------------------------
# K1 Listing 1
# --------------------------------------------------------------------------
def test_square_listing1_golden():
    rows = {r[0]: [float(v) for v in r[1:]] for r in _golden("listing1_square.txt")}
    y = np.array(rows["y"], dtype=np.float32)
    assert orc.square_f32(y).tolist() == rows["x"]


def test_square_library_and_filtered():
    y = synth.uniform_f32(1000, 7, 3) * 8 - 4
    x = orc.square_f32(y)
    assert np.array_equal(x, np.multiply(y, y))      # one IEEE multiply
    n = 3
    over = np.full_like(y, np.nan)
    for d in range(n):
        lo, hi = orc.partition(y.size, n, d)
        xd = np.full_like(y, np.nan)
        mn, mx = orc.square_f32_filtered(y, xd, lo, hi - 1)
        assert (mn, mx) == (lo, hi - 1)
        written = np.flatnonzero(~np.isnan(xd))
        assert written.min() == lo and written.max() == hi - 1 and written.size == hi - lo
        over[lo:hi] = xd[lo:hi]
    assert np.array_equal(over, x)


# --------------------------------------------------------------------------
# c1 Jacobi-2D (PolyBench jacobi-2d; DESIGN R-1)
# --------------------------------------------------------------------------
def _field(N, f):
    i, j = np.meshgrid(np.arange(N, dtype=np.float64), np.arange(N, dtype=np.float64), indexing="ij")
    return np.ascontiguousarray(f(i, j))


HARMONIC = {
    "linear": lambda i, j: 3 * i + 7 * j + 11,
    "linear_big_offset": lambda i, j: -5 * i + 2 * j + 2.0**40,
    "saddle": lambda i, j: i * i - j * j,
    "bilinear": lambda i, j: i * j - 5 * i + 2,
    "const1": lambda i, j: 1 + 0 * i,
    "const3": lambda i, j: 3 + 0 * i,
}


@pytest.mark.parametrize("name", sorted(HARMONIC))
def test_jacobi_harmonic_fixed_points(name):
    """Discrete-harmonic integer fields are exact fixed points of the
    5-point average: 0.2*(5m) rounds to m.  A dropped/duplicated term, a
    wrong sign or index, or a transposed operand breaks this."""
    N = 37
    F = _field(N, HARMONIC[name])
    dst = np.full((N, N), -777.0)
    orc.jacobi2d_sweep(F, dst)
    assert np.array_equal(dst[1:-1, 1:-1], F[1:-1, 1:-1])
    # boundary never written
    assert (dst[0] == -777).all() and (dst[-1] == -777).all()
    assert (dst[:, 0] == -777).all() and (dst[:, -1] == -777).all()
    A, B = F.copy(), F.copy()
    orc.jacobi2d(3, A, B)
    assert np.array_equal(A, F) and np.array_equal(B, F)


def _lazy_walks(k):
    """# of length-k walks on Z^2 with steps {0, +-e1, +-e2} returning to 0."""
    tot = 0
    for m in range(0, k + 1, 2):      # m moving steps, k-m stays
        tot += math.comb(k, m) * math.comb(m, m // 2) ** 2
    return tot


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_jacobi_delta_walk_counts(k):
    """A unit impulse far from the boundary: after k sweeps the centre holds
    0.2^k * (# lazy return walks), and the mass stays 1 (5 terms x 0.2)."""
    N, c = 21, 10
    A = np.zeros((N, N)); B = np.zeros((N, N))
    A[c, c] = 1.0
    src, dst = A, B
    for _ in range(k):
        orc.jacobi2d_sweep(src, dst)
        src, dst = dst, src
    assert src[c, c] == pytest.approx(0.2**k * _lazy_walks(k), rel=1e-14)
    assert src.sum() == pytest.approx(1.0, rel=1e-14)
    # support is the k-step diamond (L1 ball)
    nz = np.argwhere(src != 0)
    assert np.abs(nz - c).sum(axis=1).max() == k


def test_jacobi_polybench_timestep_is_two_sweeps():
    """T timesteps = A->B then B->A (PolyBench); with an impulse the first
    timestep leaves B = one-sweep cross and A = the two-sweep pattern."""
    N, c = 15, 7
    A = np.zeros((N, N)); B = np.zeros((N, N)); A[c, c] = 1.0
    orc.jacobi2d(1, A, B)
    assert B[c, c] == 0.2 and B[c + 1, c] == 0.2 and B[c, c - 1] == 0.2
    assert A[c, c] == pytest.approx(0.2 * 0.2 * 5, rel=1e-15)
    assert A[c + 1, c + 1] == pytest.approx(0.2 * 0.2 * 2, rel=1e-15)
    assert A[c + 2, c] == pytest.approx(0.2 * 0.2, rel=1e-15)


def test_jacobi_boundary_invariant_random():
    N = 23
    A = synth.uniform_f64(N * N, 1, synth.AID["A"]).reshape(N, N)
    B = synth.uniform_f64(N * N, 1, synth.AID["B"]).reshape(N, N)
    A0, B0 = A.copy(), B.copy()
    orc.jacobi2d(4, A, B)
    for X, X0 in ((A, A0), (B, B0)):
        assert np.array_equal(X[0], X0[0]) and np.array_equal(X[-1], X0[-1])
        assert np.array_equal(X[:, 0], X0[:, 0]) and np.array_equal(X[:, -1], X0[:, -1])
    assert not np.array_equal(A[1:-1, 1:-1], A0[1:-1, 1:-1])


def test_jacobi_write_range_golden():
    """Closed-form dirty ranges checked through the filtered
    oracle for the small shapes; the 16384^2 rows are checked against the
    same closed form without running the oracle."""
    for N, n, d, mn, mx in (map(int, r) for r in _golden("jacobi_write_ranges.txt")):
        lo, hi = orc.partition(N, n, d)
        a, b = max(lo, 1), min(hi, N - 1)
        exp = (U64MAX, 0) if a >= b else (a * N + 1, (b - 1) * N + N - 2)
        assert exp == (mn, mx)
        if N <= 256:
            src = synth.uniform_f64(N * N, 3, 1).reshape(N, N)
            dst = np.zeros((N, N))
            assert orc.jacobi2d_sweep_filtered(src, dst, lo, hi - 1) == (mn, mx)


@pytest.mark.parametrize("N", [3, 4, 5, 8, 17])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_jacobi_filtered_partition_brute_force(N, n):
    """Partition property: per-device filtered launches overlaid by
    owned rows reproduce the sequential sweep bit-exactly; the write log
    equals the brute-force set of cells that changed from a NaN sentinel."""
    src = synth.uniform_f64(N * N, 5, 1).reshape(N, N)
    full = np.full((N, N), np.nan)
    orc.jacobi2d_sweep(src, full)
    over = np.full((N, N), np.nan)
    for d in range(n):
        lo, hi = orc.partition(N, n, d)
        dst = np.full((N, N), np.nan)
        mn, mx = orc.jacobi2d_sweep_filtered(src, dst, lo, hi - 1)
        w = np.flatnonzero(~np.isnan(dst.reshape(-1)))
        if w.size == 0:
            assert (mn, mx) == (U64MAX, 0)
        else:
            assert (mn, mx) == (w.min(), w.max())
            rows = w // N
            assert rows.min() >= lo and rows.max() < hi
        over[lo:hi] = dst[lo:hi]
    assert np.array_equal(np.isnan(over), np.isnan(full))
    m = ~np.isnan(full)
    assert np.array_equal(over[m], full[m])


# --------------------------------------------------------------------------
# c2 / c8 reductions
# --------------------------------------------------------------------------
def _exact_dot(x, y, s_in=0.0):
    return Fraction(s_in) + sum((Fraction(a) * Fraction(b) for a, b in zip(x.tolist(), y.tolist())),
                                Fraction(0))


def test_dot_dyadic_exact():
    n = 50000
    x = synth.dyadic_f64(n, 11, synth.AID["x"])
    y = synth.dyadic_f64(n, 11, synth.AID["y"])
    ex = _exact_dot(x, y, 1.5)
    assert Fraction(orc.dot_f64(x, y, 1.5)) == ex
    assert Fraction(orc.dot_neumaier(x, y, 1.5)) == ex
    assert Fraction(orc.sum_f64(x, 1.5)) == Fraction(1.5) + sum(map(Fraction, x.tolist()))


def test_sum_closed_forms():
    n = 2**24
    i = np.arange(n, dtype=np.int64)
    x = (i % 2**20).astype(np.float64)
    assert orc.sum_f64(x) == (n // 2**20) * (2**20 * (2**20 - 1) // 2)
    z = (i % 2**10).astype(np.float64)
    m = 2**10
    assert orc.dot_f64(z, z) == (n // m) * ((m - 1) * m * (2 * m - 1) // 6)
    assert orc.sum_neumaier(x, 2.0) == 2 + (n // 2**20) * (2**20 * (2**20 - 1) // 2)


def test_neumaier_vs_exact_and_plain_bound():
    n = 20000
    x = synth.uniform_f64(n, 13, synth.AID["x"])
    y = synth.uniform_f64(n, 13, synth.AID["y"]) - 0.5
    ex = _exact_dot(x, y)
    nd = orc.dot_neumaier(x, y)
    # compensated result: within 2 ulp of the exact value
    assert abs(Fraction(nd) - ex) <= 2 * Fraction(math.ulp(float(ex)))
    # plain loop: classic bound |err| <= gamma_n * sum |x_i y_i|
    pl = orc.dot_f64(x, y)
    gam = n * 2**-53 / (1 - n * 2**-53)
    assert abs(Fraction(pl) - ex) <= Fraction(gam) * _exact_dot(np.abs(x), np.abs(y))
    # sum: Neumaier equals math.fsum (correctly rounded) on this data
    assert orc.sum_neumaier(y) == pytest.approx(math.fsum(y.tolist()), rel=0, abs=4 * math.ulp(1.0) * n)
    assert abs(orc.sum_neumaier(y) - math.fsum(y.tolist())) <= 2 * math.ulp(math.fsum(y.tolist()))


@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_reduction_filtered_partials_combine(n):
    """partials over outer-iterator blocks; c8 combine."""
    N = 10007
    x = synth.dyadic_f64(N, 17, 3)
    y = synth.dyadic_f64(N, 17, 4)
    parts = []
    for d in range(n):
        lo, hi = orc.partition(N, n, d)
        parts.append(orc.dot_f64_filtered(x, y, lo, hi - 1))
        assert Fraction(parts[-1]) == _exact_dot(x[lo:hi], y[lo:hi])
    assert Fraction(orc.reduce_combine(-2.25, parts)) == _exact_dot(x, y, -2.25)
    sparts = [orc.sum_f64_filtered(x, *(lambda lo, hi: (lo, hi - 1))(*orc.partition(N, n, d)))
              for d in range(n)]
    assert orc.reduce_combine(0.0, sparts) == orc.sum_f64(x)


# --------------------------------------------------------------------------
# c3 GEMM
# --------------------------------------------------------------------------
def test_gemm_identity_exact():
    N = 48
    B = synth.uniform_f64(N * N, 2, 2).reshape(N, N)
    I = np.eye(N)
    assert np.array_equal(orc.gemm_f64(I, B), B)
    assert np.array_equal(orc.gemm_f64(B, I), B)


def test_gemm_all_ones_and_rank1_exact():
    M, N, K = 13, 29, 64
    assert (orc.gemm_f64(np.ones((M, K)), np.ones((K, N))) == K).all()
    u = synth.int_i32(M, -9, 9, 4, 1).astype(np.float64)
    v = synth.int_i32(N, -9, 9, 4, 2).astype(np.float64)
    A = np.ascontiguousarray(np.repeat(u[:, None], K, axis=1))     # A = u 1^T
    B = np.ascontiguousarray(np.repeat(v[None, :], K, axis=0))     # B = 1 v^T
    assert np.array_equal(orc.gemm_f64(A, B), K * np.outer(u, v))


def test_gemm_random_vs_numpy_bound_and_ikj():
    M, N, K = 37, 53, 71                  # non-square: catches transposed operands
    A = synth.uniform_f64(M * K, 6, 1).reshape(M, K)
    B = synth.uniform_f64(K * N, 6, 2).reshape(K, N)
    C = orc.gemm_f64(A, B)
    ref = A @ B
    gam = K * 2**-53 / (1 - K * 2**-53)
    assert (np.abs(C - ref) <= 2 * gam * (np.abs(A) @ np.abs(B))).all()
    assert np.array_equal(orc.gemm_f64(A, B, ikj=True), C)
    # brute force one element exactly
    i, j = 5, 17
    ex = sum(Fraction(A[i, k]) * Fraction(B[k, j]) for k in range(K))
    assert abs(Fraction(C[i, j]) - ex) <= Fraction(gam) * ex


@pytest.mark.parametrize("n", [1, 2, 3, 7])
def test_gemm_filtered_partition(n):
    M, N, K = 11, 9, 5
    A = synth.uniform_f64(M * K, 8, 1).reshape(M, K)
    B = synth.uniform_f64(K * N, 8, 2).reshape(K, N)
    full = orc.gemm_f64(A, B)
    over = np.full((M, N), np.nan)
    for d in range(n):
        lo, hi = orc.partition(M, n, d)
        C = np.full((M, N), np.nan)
        mn, mx = orc.gemm_f64_filtered(A, B, C, lo, hi - 1)
        if lo == hi:
            assert (mn, mx) == (U64MAX, 0)
        else:
            assert (mn, mx) == (lo * N, (hi - 1) * N + N - 1)
        assert np.isnan(C[:lo]).all() and np.isnan(C[hi:]).all()
        over[lo:hi] = C[lo:hi]
    assert np.array_equal(over, full)


# --------------------------------------------------------------------------
# c5 scatter
# --------------------------------------------------------------------------
def test_scatter_ones_is_histogram():
    N, M = 100000, 5000
    idx = synth.index_i32(N, M, 21, synth.AID["idx"])
    a0 = synth.dyadic_f64(M, 21, synth.AID["a0"])
    a = a0.copy()
    orc.scatter_add(idx, np.ones(N), a)
    h = np.bincount(idx, minlength=M)
    # a0 = k/1024 plus an integer count: every partial sum exact
    assert np.array_equal(a, a0 + h)
    assert np.bincount(idx, minlength=M).sum() == N


def test_scatter_i32_and_dyadic_vs_library():
    N, M = 60000, 3001
    idx = synth.index_i32(N, M, 22, 5)
    bi = synth.int_i32(N, -1000, 1000, 22, 6)
    ai = synth.int_i32(M, -10**6, 10**6, 22, 7)
    ref = ai.copy(); np.add.at(ref, idx, bi)
    orc.scatter_add(idx, bi, ai)
    assert np.array_equal(ai, ref)
    bd = synth.dyadic_f64(N, 22, 6)
    ad = synth.dyadic_f64(M, 22, 7)
    refd = ad.copy(); np.add.at(refd, idx, bd)     # exact in any order
    orc.scatter_add(idx, bd, ad)
    assert np.array_equal(ad, refd)


def test_scatter_permutation_exact():
    M = 4096
    idx = synth.permutation_i32(M, 23, 5)
    assert np.array_equal(np.sort(idx), np.arange(M))
    b = synth.uniform_f64(M, 23, 6)
    a0 = synth.uniform_f64(M, 23, 7)
    a = a0.copy()
    orc.scatter_add(idx, b, a)
    exp = a0.copy(); exp[idx] = a0[idx] + b
    assert np.array_equal(a, exp)


@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_scatter_filtered_bitmaps(n):
    """every device scans all i; updates predicated on the
    computed index.  Bitmaps = indicator of distinct owned targets."""
    N, M = 20000, 1000
    idx = synth.index_i32(N, M, 24, 5)
    b = synth.dyadic_f64(N, 24, 6)
    a0 = synth.dyadic_f64(M, 24, 7)
    full = a0.copy(); orc.scatter_add(idx, b, full)
    over = np.empty(M)
    union = np.zeros((M + 31) // 32, dtype=np.uint32)
    for d in range(n):
        lo, hi = orc.partition(M, n, d)
        a = a0.copy()
        bm, mn, mx = orc.scatter_add_filtered(idx, b, a, lo, hi - 1)
        bits = np.unpackbits(bm.view(np.uint8), bitorder="little")[:M].astype(bool)
        owned = np.unique(idx[(idx >= lo) & (idx < hi)])
        assert np.array_equal(np.flatnonzero(bits), owned)
        if owned.size:
            assert (mn, mx) == (owned.min(), owned.max())
        else:
            assert (mn, mx) == (U64MAX, 0)
        assert np.array_equal(a[:lo], a0[:lo]) and np.array_equal(a[hi:], a0[hi:])
        assert (union & bm == 0).all()                # disjoint write sets
        union |= bm
        over[lo:hi] = a[lo:hi]
    assert np.array_equal(over, full)
    allbits = np.unpackbits(union.view(np.uint8), bitorder="little")[:M].astype(bool)
    assert allbits.sum() == np.unique(idx).size


# --------------------------------------------------------------------------
# c7 coherence exchange
# --------------------------------------------------------------------------
@pytest.mark.parametrize("n", [2, 3, 4])
def test_exchange_range_coherence_jacobi(n):
    N = 19
    A0 = synth.uniform_f64(N * N, 9, 1).reshape(N, N)
    B0 = synth.uniform_f64(N * N, 9, 2).reshape(N, N)
    A, B = A0.copy(), B0.copy()
    orc.jacobi2d(2, A, B)                       # sequential reference, 4 sweeps
    RA = [A0.copy() for _ in range(n)]
    RB = [B0.copy() for _ in range(n)]
    for sweep in range(4):
        src, dst = (RA, RB) if sweep % 2 == 0 else (RB, RA)
        mins, maxs = [], []
        for d in range(n):
            lo, hi = orc.partition(N, n, d)
            mn, mx = orc.jacobi2d_sweep_filtered(src[d], dst[d], lo, hi - 1)
            mins.append(mn); maxs.append(mx)
        orc.exchange_range(dst, mins, maxs)
    for d in range(n):
        assert np.array_equal(RA[d], A) and np.array_equal(RB[d], B)


@pytest.mark.parametrize("n", [2, 5])
def test_exchange_bitmap_coherence_scatter(n):
    N, M = 5000, 777
    idx = synth.index_i32(N, M, 25, 5)
    b = synth.int_i32(N, -1000, 1000, 25, 6)
    a0 = synth.int_i32(M, -100, 100, 25, 7)
    full = a0.copy(); orc.scatter_add(idx, b, full)
    R = [a0.copy() for _ in range(n)]
    bms = []
    for d in range(n):
        lo, hi = orc.partition(M, n, d)
        bm, _, _ = orc.scatter_add_filtered(idx, b, R[d], lo, hi - 1)
        bms.append(bm)
    orc.exchange_bitmap(R, bms)
    for d in range(n):
        assert np.array_equal(R[d], full)


def jacobi_add_order_case():
    """The hand-derived operand-order fixture (tests/golden/jacobi_add_order.txt):
    (A grid, {(i, j): expected B value})."""
    A = np.zeros((7, 7))
    exp = {}
    for r in _golden("jacobi_add_order.txt"):
        i, j, v = int(r[1]), int(r[2]), float.fromhex(r[3])
        if r[0] == "A":
            A[i, j] = v
        else:
            exp[(i, j)] = v
    return A, exp


def test_jacobi_sweep_add_order_golden():
    """Pins the PolyBench left-to-right add order and the single multiply by
    the binary64 0.2 (DESIGN R-1): a dropped term, a different association
    or a division by 5 changes at least one of the hand-derived values."""
    A, exp = jacobi_add_order_case()
    B = np.zeros_like(A)
    orc.jacobi2d_sweep(A, B)
    for (i, j), v in exp.items():
        assert B[i, j].hex() == v.hex(), (i, j, B[i, j].hex(), v.hex())
