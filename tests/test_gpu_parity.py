"""GPU parity (-m gpu): the CUDA path, called through the C-ABI, against the
CPU oracle on the same seeded inputs.  Bit-exact for element-wise, integer
and index work and for the dirty sets; fp64 reductions within 1e-12 of the
Neumaier reference and GEMM within 1e-12*(|A||B|)_ij (north_star; DESIGN
R-8, R-10, R-11).  Multi-device runs use virtual devices (several logical
devices on one B200, separate replicas), with both merge policies.
"""
from contextlib import contextmanager

import numpy as np
import pytest

import oracle as orc  # noqa: E402
import synth

pytestmark = pytest.mark.gpu
U64MAX = 2**64 - 1


@pytest.fixture(scope="module")
def J():
    import __graft_entry__ as ge
    ge.build_jacc()
    from paper_2110_14340_b200 import jacc
    return jacc


@contextmanager
def runtime(J, n=1, policy=0, mode=0):
    J.jacc_init(n, [0] * n)
    try:
        J.jacc_set_merge_policy(policy)
        J.jacc_set_mode(mode)
        yield
    finally:
        J.jacc_finalize()


def _in(J, x):
    return J.arg(J.JACC_ARG_ARRAY_IN, x)


def _out(J, x):
    return J.arg(J.JACC_ARG_ARRAY_OUT, x)


def _inout(J, x):
    return J.arg(J.JACC_ARG_ARRAY_INOUT, x)


def _create(J, *arrs, upload=True):
    for a in arrs:
        J.jacc_data_create(a)
        if upload:
            J.jacc_update_device(a)


# --------------------------------------------------------------------------
# K1 Listing 1
# --------------------------------------------------------------------------
def test_square_listing1(J):
    y = np.array([1, 2, 3], dtype=np.float32)
    x = np.zeros(3, dtype=np.float32)
    with runtime(J):
        _create(J, y, x)
        J.jacc_launch(J.JACC_LOOP_SQUARE_F32, J.make_range(0, 3), [_in(J, y), _out(J, x)])
        J.jacc_update_host(x)
        assert J.jacc_get_dirty_range(x, 0) == (0, 2)
    assert x.tolist() == [1, 4, 9]


@pytest.mark.parametrize("n", [1, 2, 3, 8])
@pytest.mark.parametrize("size", [1, 5, 1000, 123457])
def test_square_multi(J, n, size):
    y = synth.uniform_f32(size, 31, 3) * 8 - 4
    x = np.full(size, -1.0, dtype=np.float32)
    ref = orc.square_f32(y)
    with runtime(J, n):
        _create(J, y, x)
        J.jacc_launch(J.JACC_LOOP_SQUARE_F32, J.make_range(0, size), [_in(J, y), _out(J, x)])
        for d in range(n):
            lo, hi = orc.partition(size, n, d)
            xd = np.zeros_like(y)
            exp = orc.square_f32_filtered(y, xd, lo, hi - 1)
            assert J.jacc_get_dirty_range(x, d) == exp
            assert np.array_equal(J.jacc_get_replica(x, d), ref)   # EAGER: coherent
        J.jacc_update_host(x)
    assert np.array_equal(x, ref)


def test_square_interior_pointer_subrange(J):
    """1-D args may point inside a region (present lookup of any address)."""
    y = synth.uniform_f32(1000, 32, 3)
    x = np.zeros(1000, dtype=np.float32)
    with runtime(J, 2):
        _create(J, y, x)
        J.jacc_launch(J.JACC_LOOP_SQUARE_F32, J.make_range(10, 300),
                      [_in(J, y[100:]), _out(J, x[200:])])
        J.jacc_update_host(x)
    ref = np.zeros(1000, dtype=np.float32)
    ref[210:500] = orc.square_f32(np.ascontiguousarray(y[110:400]))
    assert np.array_equal(x, ref)


def test_square_alias_is_duplicated(J):
    """x and y the same array (read and written): duplicate mode."""
    y = synth.uniform_f32(777, 33, 3)
    ref = orc.square_f32(y)
    with runtime(J, 3):
        _create(J, y)
        J.jacc_launch(J.JACC_LOOP_SQUARE_F32, J.make_range(0, 777), [_in(J, y), _out(J, y)])
        for d in range(3):
            assert np.array_equal(J.jacc_get_replica(y, d), ref)
        J.jacc_update_host(y)
    assert np.array_equal(y, ref)


# --------------------------------------------------------------------------
# c1 Jacobi-2D
# --------------------------------------------------------------------------
def _jacobi_gpu(J, A0, B0, T, n, policy, rng=None, check_dirty=True):
    A, B = A0.copy(), B0.copy()
    N = A.shape[0]
    dirt = []
    with runtime(J, n, policy):
        _create(J, A, B)
        for t in range(T):
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, rng, [_in(J, A), _out(J, B)], async_id=0)
            if check_dirty and t == 0:
                dirt.append([J.jacc_get_dirty_range(B, d) for d in range(n)])
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, rng, [_in(J, B), _out(J, A)], async_id=0)
        J.jacc_wait()
        reps = None
        if policy == J.JACC_MERGE_EAGER:
            reps = [(J.jacc_get_replica(A, d), J.jacc_get_replica(B, d)) for d in range(n)]
        J.jacc_update_host(A)
        J.jacc_update_host(B)
    return A, B, dirt, reps


def test_jacobi_J256_bit_exact(J):
    """BASELINE config 1: 256^2, 10 timesteps, 1 GPU, bit-exact vs oracle."""
    N, T = 256, 10
    A0, B0 = synth.polybench_jacobi2d(N)
    # PolyBench init is (nearly) harmonic; also a seeded random field
    for A0_, B0_ in ((A0, B0), (synth.uniform_f64(N * N, 41, 1).reshape(N, N),
                                synth.uniform_f64(N * N, 41, 2).reshape(N, N))):
        Ar, Br = A0_.copy(), B0_.copy()
        orc.jacobi2d(T, Ar, Br)
        A, B, dirt, _ = _jacobi_gpu(J, A0_, B0_, T, 1, J.JACC_MERGE_EAGER)
        assert np.array_equal(A, Ar) and np.array_equal(B, Br)
        assert dirt[0] == [(257, 65278)]


@pytest.mark.parametrize("N", [3, 4, 5, 17, 64, 258, 301])
@pytest.mark.parametrize("n", [1, 2, 3, 8])
@pytest.mark.parametrize("policy", [0, 1])
def test_jacobi_multi_device(J, N, n, policy):
    T = 3
    A0 = synth.uniform_f64(N * N, 42 + N, 1).reshape(N, N)
    B0 = synth.uniform_f64(N * N, 42 + N, 2).reshape(N, N)
    Ar, Br = A0.copy(), B0.copy()
    orc.jacobi2d(T, Ar, Br)
    A, B, dirt, reps = _jacobi_gpu(J, A0, B0, T, n, policy)
    assert np.array_equal(A, Ar) and np.array_equal(B, Br)
    # dirty sets == oracle write log of the filtered first sweep
    for d in range(n):
        lo, hi = orc.partition(N, n, d)
        tmp = B0.copy()
        assert dirt[0][d] == orc.jacobi2d_sweep_filtered(A0, tmp, lo, hi - 1)
    if reps is not None:  # EAGER: every replica coherent after every launch
        for a, b in reps:
            assert np.array_equal(a, Ar) and np.array_equal(b, Br)


@pytest.mark.parametrize("n", [1, 3])
def test_jacobi_subrange(J, n):
    N = 50
    A0 = synth.uniform_f64(N * N, 43, 1).reshape(N, N)
    B0 = synth.uniform_f64(N * N, 43, 2).reshape(N, N)
    rng = J.make_range([7, 3], [40, 33])
    A, B, _, _ = _jacobi_gpu(J, A0, B0, 1, n, 0, rng=rng, check_dirty=False)
    # oracle: the loop nest restricted to the same range
    Ar, Br = A0.copy(), B0.copy()
    for (s, t) in ((Ar, Br), (Br, Ar)):
        full = t.copy()
        orc.jacobi2d_sweep(s, full)
        t[7:40, 3:33] = full[7:40, 3:33]
    assert np.array_equal(A, Ar) and np.array_equal(B, Br)


def test_jacobi_rejects_in_place(J):
    A = np.zeros((8, 8))
    with runtime(J):
        _create(J, A)
        st = J.jacc_launch_status(J.JACC_LOOP_JACOBI2D_F64, None, [_in(J, A), _out(J, A)])
        assert st == J.JACC_ERR_INVALID


def test_jacobi_full_size_sampled(J):
    """BASELINE config 2 at full size (16384^2, n=1, the bench launch
    configuration): one sweep checked on sampled windows recomputed by the
    oracle, then 200 launches on an exact harmonic field (a fixed point of
    the fp64 sweep at any size) must leave it unchanged bit for bit."""
    N = 16384
    A = synth.uniform_f64(N * N, 44, 1).reshape(N, N)
    B = np.zeros((N, N))
    rs = np.random.default_rng(5)
    with runtime(J):
        _create(J, A, B)
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [_in(J, A), _out(J, B)])
        J.jacc_update_host(B)
        for (i, j) in [(1, 1), (N - 2, N - 2), (1, N - 2), (N - 2, 1), (8191, 8192)] + \
                [tuple(rs.integers(1, N - 1, 2)) for _ in range(20)]:
            i0, j0 = max(i - 3, 0), max(j - 3, 0)
            i1, j1 = min(i + 4, N), min(j + 4, N)
            w = np.ascontiguousarray(A[i0:i1, j0:j1])
            # pad to a square window for the oracle (N x N signature)
            m = max(w.shape)
            src = np.zeros((m, m)); src[:w.shape[0], :w.shape[1]] = w
            dst = np.zeros((m, m))
            orc.jacobi2d_sweep(src, dst)
            assert B[i, j] == dst[i - i0, j - j0], (i, j)
        assert J.jacc_get_dirty_range(B, 0) == (N + 1, (N - 2) * N + N - 2)
        ii, jj = np.meshgrid(np.arange(N, dtype=np.float64), np.arange(N, dtype=np.float64),
                             indexing="ij")
        H = 3 * ii + 7 * jj + 11
        A[:] = H
        B[:] = H
        del ii, jj
        J.jacc_update_device(A)
        J.jacc_update_device(B)
        for t in range(100):
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [_in(J, A), _out(J, B)], async_id=0)
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [_in(J, B), _out(J, A)], async_id=0)
        J.jacc_update_host(A)
        assert np.array_equal(A, H)


@pytest.mark.parametrize("n,policy", [(1, 0), (3, 1), (3, 0)])
def test_jacobi_add_order_golden(J, n, policy):
    """The hand-derived operand-order fixture (tests/golden/
    jacobi_add_order.txt): the kernel's adds follow PolyBench's order and
    it multiplies once by the binary64 0.2, on one device and across a
    block boundary."""
    from test_oracle import jacobi_add_order_case
    A, exp = jacobi_add_order_case()
    B = np.zeros_like(A)
    ref = np.zeros_like(A)
    orc.jacobi2d_sweep(A, ref)
    with runtime(J, n, policy):
        _create(J, A, B)
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [_in(J, A), _out(J, B)])
        J.jacc_update_host(B)
    for (i, j), v in exp.items():
        assert B[i, j].hex() == v.hex(), (i, j)
    assert np.array_equal(B, ref)


_J16K_CACHE = {}


def _j16k_random_ref(sweeps):
    """Random 16384^2 field (seeded) and the oracle after `sweeps` launches
    (A->B, B->A, ...), computed once per module."""
    N = 16384
    if "A0" not in _J16K_CACHE:
        _J16K_CACHE["A0"] = synth.uniform_f64(N * N, 45, 1).reshape(N, N)
        _J16K_CACHE["B0"] = synth.uniform_f64(N * N, 45, 2).reshape(N, N)
    if sweeps not in _J16K_CACHE:
        A, B = _J16K_CACHE["A0"].copy(), _J16K_CACHE["B0"].copy()
        src, dst = A, B
        for _ in range(sweeps):
            orc.jacobi2d_sweep(src, dst)
            src, dst = dst, src
        _J16K_CACHE[sweeps] = (A, B)
    return _J16K_CACHE["A0"], _J16K_CACHE["B0"], _J16K_CACHE[sweeps]


@pytest.mark.parametrize("n,policy", [(1, 1), (2, 1), (8, 1), (8, 0)])
def test_jacobi_full_size_random_field_exact(J, n, policy):
    """BASELINE config 2 at full size, whole field: a seeded random
    16384^2 field (every operand order visible in the rounding) after two
    launches (A->B, B->A), every element of A and B bit-exact against the
    oracle, on 1 device and on 2 / 8 virtual devices under HALO and EAGER."""
    A0, B0, (Ar, Br) = _j16k_random_ref(2)
    A, B, _, _ = _jacobi_gpu(J, A0, B0, 1, n, policy, check_dirty=False)
    assert np.array_equal(B, Br)
    assert np.array_equal(A, Ar)


@pytest.mark.parametrize("n", [1, 8])
def test_jacobi_full_step_200_launches_exact(J, n):
    """The whole timed J16K step (100 timesteps = 200 launches, HALO) on a
    seeded random field, compared element by element with 200 oracle
    sweeps: the exact configuration bench.py times (n = 1), and 8 virtual
    devices."""
    A0, B0, (Ar, Br) = _j16k_random_ref(200)
    A, B, _, _ = _jacobi_gpu(J, A0, B0, 100, n, 1, check_dirty=False)
    assert np.array_equal(A, Ar)
    assert np.array_equal(B, Br)


# --------------------------------------------------------------------------
# c2 / c8 reductions
# --------------------------------------------------------------------------
def _reduce(J, x, y, s_in, n, lo=0, hi=None, xoff=0, yoff=0):
    hi = x.size - xoff if hi is None else hi
    s = np.array([s_in])
    with runtime(J, n):
        _create(J, x)
        if y is not None:
            _create(J, y)
        args = [_in(J, x[xoff:])]
        if y is not None:
            args.append(_in(J, y[yoff:]))
        args.append(J.arg(J.JACC_ARG_REDUCE_SUM_F64, s))
        loop = J.JACC_LOOP_DOT_F64 if y is not None else J.JACC_LOOP_SUM_F64
        J.jacc_launch(loop, J.make_range(lo, hi), args)
    return s[0]


@pytest.mark.parametrize("n", [1, 2, 3, 8])
@pytest.mark.parametrize("size", [0, 1, 7, 4096, 1_000_003])
def test_dot_sum_dyadic_exact(J, n, size):
    x = synth.dyadic_f64(max(size, 1), 51, 3)[:size].copy() if size else np.zeros(1)
    y = synth.dyadic_f64(max(size, 1), 51, 4)[:size].copy() if size else np.zeros(1)
    hi = size
    assert _reduce(J, x, y, 1.5, n, 0, hi) == orc.dot_f64(x[:hi], y[:hi], 1.5)
    assert _reduce(J, x, None, -2.0, n, 0, hi) == orc.sum_f64(x[:hi], -2.0)


@pytest.mark.parametrize("n", [1, 3])
def test_dot_uniform_tolerance(J, n):
    size = 3_000_001
    x = synth.uniform_f64(size, 52, 3)
    y = synth.uniform_f64(size, 52, 4) - 0.5
    ref = orc.dot_neumaier(x, y, 0.25)
    got = _reduce(J, x, y, 0.25, n)
    assert abs(got - ref) <= 1e-12 * abs(ref)
    ref = orc.sum_neumaier(x, 0.0)
    assert abs(_reduce(J, x, None, 0.0, n) - ref) <= 1e-12 * abs(ref)


@pytest.mark.parametrize("xoff,yoff", [(1, 1), (1, 2), (3, 0)])
def test_dot_misaligned_interior_pointers(J, xoff, yoff):
    size = 100_001
    x = synth.dyadic_f64(size, 53, 3)
    y = synth.dyadic_f64(size, 53, 4)
    m = size - 3
    got = _reduce(J, x, y, 0.0, 2, 0, m, xoff, yoff)
    assert got == orc.dot_f64(np.ascontiguousarray(x[xoff:xoff + m]),
                              np.ascontiguousarray(y[yoff:yoff + m]), 0.0)


def test_dot_full_size(J):
    """BASELINE config 3 at full size: 2^30 fp64, n=1, dyadic (exact)."""
    size = 2**30
    x = synth.dyadic_f64(size, 54, 3)
    y = synth.dyadic_f64(size, 54, 4)
    assert _reduce(J, x, y, 0.0, 1) == orc.dot_f64(x, y, 0.0)


@pytest.mark.parametrize("n", [1, 8])
def test_dot_full_size_uniform_tolerance(J, n):
    """BASELINE config 3 at full size with the tolerance inputs: 2^30
    uniform [0,1) pairs (the bench's data), GPU vs the oracle's Neumaier
    reference within 1e-12 relative (north_star; DESIGN R-10)."""
    size = 2**30
    x = synth.uniform_f64(size, 1, synth.AID["x"])
    y = synth.uniform_f64(size, 1, synth.AID["y"])
    ref = orc.dot_neumaier(x, y, 0.0)
    got = _reduce(J, x, y, 0.0, n)
    assert abs(got - ref) <= 1e-12 * abs(ref)


# --------------------------------------------------------------------------
# c3 GEMM
# --------------------------------------------------------------------------
def _gemm(J, A, B, n, rng=None, dirty=False):
    M, N = A.shape[0], B.shape[1]
    C = np.full((M, N), -3.0)
    with runtime(J, n):
        _create(J, A, B)
        _create(J, C, upload=True)
        J.jacc_launch(J.JACC_LOOP_GEMM_F64, rng, [_in(J, A), _in(J, B), _out(J, C)])
        dr = [J.jacc_get_dirty_range(C, d) for d in range(n)] if dirty else None
        reps = [J.jacc_get_replica(C, d) for d in range(n)]
        J.jacc_update_host(C)
    return C, dr, reps


def _gemm_bound(A, B):
    return 1e-12 * (np.abs(A) @ np.abs(B))


@pytest.mark.parametrize("shape", [(64, 64, 64), (37, 53, 71), (130, 67, 16), (1, 1, 1),
                                   (200, 256, 33),
                                   # TMA path (K, N even) with ragged M, N and K tiles
                                   (300, 258, 130), (129, 130, 18), (513, 384, 2)])
@pytest.mark.parametrize("n", [1, 2, 3])
def test_gemm_random_tolerance(J, shape, n):
    M, N, K = shape
    A = synth.uniform_f64(M * K, 61, 1).reshape(M, K)
    B = synth.uniform_f64(K * N, 61, 2).reshape(K, N)
    ref = orc.gemm_f64(A, B)
    C, dr, reps = _gemm(J, A, B, n, dirty=True)
    assert (np.abs(C - ref) <= _gemm_bound(A, B)).all()
    for d in range(n):
        lo, hi = orc.partition(M, n, d)
        Cd = np.zeros((M, N))
        assert dr[d] == orc.gemm_f64_filtered(A, B, Cd, lo, hi - 1)
        assert np.array_equal(reps[d], C)


@pytest.mark.parametrize("n", [1, 2])
def test_gemm_exact_cases(J, n):
    M = N = K = 96
    B = synth.uniform_f64(K * N, 62, 2).reshape(K, N)
    C, _, _ = _gemm(J, np.eye(M), B, n)
    assert np.array_equal(C, B)
    C, _, _ = _gemm(J, np.ones((M, K)), np.ones((K, N)), n)
    assert (C == K).all()
    u = synth.int_i32(M, -9, 9, 62, 3).astype(np.float64)
    v = synth.int_i32(N, -9, 9, 62, 4).astype(np.float64)
    A1 = np.ascontiguousarray(np.repeat(u[:, None], K, axis=1))
    B1 = np.ascontiguousarray(np.repeat(v[None, :], K, axis=0))
    C, _, _ = _gemm(J, A1, B1, n)
    assert np.array_equal(C, K * np.outer(u, v))


def test_gemm_subrange(J):
    M, N, K = 70, 90, 20
    A = synth.uniform_f64(M * K, 63, 1).reshape(M, K)
    B = synth.uniform_f64(K * N, 63, 2).reshape(K, N)
    C, _, _ = _gemm(J, A, B, 2, rng=J.make_range([5, 10], [60, 81]))
    ref = np.full((M, N), -3.0)
    ref[5:60, 10:81] = orc.gemm_f64(A, B)[5:60, 10:81]
    m = np.abs(C - ref) <= 1e-12 * np.abs(ref)
    assert m.all()


def test_gemm_full_size_sampled(J):
    """BASELINE config 4 at full size: 8192^3 fp64 (n=1, bench launch
    configuration); sampled rows recomputed by the oracle; identity exact."""
    Nn = 8192
    A = synth.uniform_f64(Nn * Nn, 64, 1).reshape(Nn, Nn)
    B = synth.uniform_f64(Nn * Nn, 64, 2).reshape(Nn, Nn)
    C, dr, _ = _gemm(J, A, B, 1, dirty=True)
    assert dr[0] == (0, Nn * Nn - 1)
    for i in (0, 1, 4095, 8191, 1234):
        row = orc.gemm_f64(np.ascontiguousarray(A[i:i + 1]), B)
        bound = 1e-12 * (np.abs(A[i:i + 1]) @ np.abs(B))
        assert (np.abs(C[i:i + 1] - row) <= bound).all(), i


# --------------------------------------------------------------------------
# c5 scatter
# --------------------------------------------------------------------------
def _scatter(J, idx, b, a0, n, policy=0):
    a = a0.copy()
    loop = J.JACC_LOOP_SCATTER_ADD_F64 if a.dtype == np.float64 else J.JACC_LOOP_SCATTER_ADD_I32
    with runtime(J, n, policy):
        _create(J, idx, b, a)
        J.jacc_launch(loop, J.make_range(0, idx.size), [_in(J, idx), _in(J, b), _inout(J, a)])
        bms = [J.jacc_get_dirty_bitmap(a, d, a.size) for d in range(n)]
        drs = [J.jacc_get_dirty_range(a, d) for d in range(n)]
        reps = [J.jacc_get_replica(a, d) for d in range(n)] if policy == 0 else None
        J.jacc_update_host(a)
    return a, bms, drs, reps


@pytest.mark.parametrize("n", [1, 2, 3, 8])
@pytest.mark.parametrize("sizes", [(1, 1), (100, 37), (100_003, 5000), (1_000_000, 1_000_000)])
@pytest.mark.parametrize("dtype", ["f64", "i32"])
def test_scatter_exact(J, n, sizes, dtype):
    N, M = sizes
    idx = synth.index_i32(N, M, 71, 5)
    if dtype == "f64":
        b = synth.dyadic_f64(N, 71, 6)
        a0 = synth.dyadic_f64(M, 71, 7)
    else:
        b = synth.int_i32(N, -1000, 1000, 71, 6)
        a0 = synth.int_i32(M, -10**6, 10**6, 71, 7)
    ref = a0.copy()
    orc.scatter_add(idx, b, ref)
    a, bms, drs, reps = _scatter(J, idx, b, a0, n)
    assert np.array_equal(a, ref)
    for d in range(n):
        lo, hi = orc.partition(M, n, d)
        bm, mn, mx = orc.scatter_add_filtered(idx, b, a0.copy(), lo, hi - 1)
        assert np.array_equal(bms[d], bm)
        assert drs[d] == (mn, mx)
        assert np.array_equal(reps[d], ref)


@pytest.mark.parametrize("n", [2, 3])
def test_scatter_halo_policy_and_uniform_tolerance(J, n):
    N, M = 200_000, 30_000
    idx = synth.index_i32(N, M, 72, 5)
    b = synth.uniform_f64(N, 72, 6)
    a0 = synth.uniform_f64(M, 72, 7)
    ref = a0.copy()
    orc.scatter_add(idx, b, ref)
    a, _, _, _ = _scatter(J, idx, b, a0, n, policy=1)
    # per-element bound |d| <= 1e-12 * sum |contributions| (R-8)
    mag = np.abs(a0).copy()
    np.add.at(mag, idx, np.abs(b))
    assert (np.abs(a - ref) <= 1e-12 * mag).all()


def test_scatter_permutation_exact(J):
    M = 1 << 16
    idx = synth.permutation_i32(M, 73, 5)
    b = synth.uniform_f64(M, 73, 6)
    a0 = synth.uniform_f64(M, 73, 7)
    ref = a0.copy()
    orc.scatter_add(idx, b, ref)
    a, _, _, _ = _scatter(J, idx, b, a0, 4)
    assert np.array_equal(a, ref)


@pytest.mark.parametrize("binned", ["0", "1"])
@pytest.mark.parametrize("n", [1, 3])
@pytest.mark.parametrize("lo", [0, 1, 2, 3, 5])
def test_scatter_paths_and_misaligned_ranges(J, monkeypatch, binned, n, lo):
    """Direct and destination-binned (paged partition, apply with the bits
    items) scatter, iteration ranges starting at any element (int4
    head/tail handling)."""
    monkeypatch.setenv("JACC_SCATTER_BINNED", binned)
    N, M = 30_011, 4099
    idx = synth.index_i32(N, M, 75, 5)
    b = synth.dyadic_f64(N, 75, 6)
    a0 = synth.dyadic_f64(M, 75, 7)
    ref = a0.copy()
    orc.scatter_add(idx[lo:N - 2], b[lo:N - 2], ref)
    a = a0.copy()
    with runtime(J, n):
        _create(J, idx, b, a)
        J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_F64, J.make_range(lo, N - 2),
                      [_in(J, idx), _in(J, b), _inout(J, a)])
        for d in range(n):
            plo, phi = orc.partition(M, n, d)
            bm, mn, mx = orc.scatter_add_filtered(np.ascontiguousarray(idx[lo:N - 2]),
                                                  np.ascontiguousarray(b[lo:N - 2]), a0.copy(),
                                                  plo, phi - 1)
            assert np.array_equal(J.jacc_get_dirty_bitmap(a, d, M), bm)
            assert J.jacc_get_dirty_range(a, d) == (mn, mx)
        J.jacc_update_host(a)
    assert np.array_equal(a, ref)


@pytest.mark.parametrize("dtype", ["f64", "i32"])
@pytest.mark.parametrize("n", [1, 2, 3])
@pytest.mark.parametrize("spec", ["1", "0"])
def test_scatter_binned_large(J, monkeypatch, dtype, n, spec):
    """Arrays larger than L2 take the binned pipeline by default; n=3 gives
    owned spans off word and bucket boundaries.  spec=1: the speculative
    fixed-capacity layout (uniform keys never overflow it); spec=0: the exact
    histogram pipeline."""
    monkeypatch.setenv("JACC_SCATTER_SPEC", spec)
    M = 2**25 if dtype == "f64" else 2**26
    N = 2**23
    idx = synth.index_i32(N, M, 76, 5)
    if dtype == "f64":
        b, a0 = synth.dyadic_f64(N, 76, 6), synth.dyadic_f64(M, 76, 7)
    else:
        b, a0 = synth.int_i32(N, -1000, 1000, 76, 6), synth.int_i32(M, -10**6, 10**6, 76, 7)
    ref = a0.copy()
    orc.scatter_add(idx, b, ref)
    a, bms, drs, reps = _scatter(J, idx, b, a0, n)
    assert np.array_equal(a, ref)
    for d in range(n):
        lo, hi = orc.partition(M, n, d)
        bm, mn, mx = orc.scatter_add_filtered(idx, b, a0.copy(), lo, hi - 1)
        assert np.array_equal(bms[d], bm) and drs[d] == (mn, mx)
        assert np.array_equal(reps[d], ref)


@pytest.mark.parametrize("dtype", ["f64", "i32"])
@pytest.mark.parametrize("n", [1, 3, 8])
def test_scatter_binned_ragged_skewed(J, monkeypatch, dtype, n):
    """Binned pipeline over several buckets with a ragged last bucket,
    owned spans starting off word boundaries (n=3, 8) and a skewed index mix
    (a hot band holding a quarter of the updates: one bucket claims many
    more pages than the others), exact inputs."""
    monkeypatch.setenv("JACC_SCATTER_BINNED", "1")
    M = 3 * 2**21 + 777 if dtype == "f64" else 3 * 2**22 + 777
    N = 2**22 + 3
    idx = synth.index_i32(N, M, 79, 5)
    hot = synth.index_i32(N // 4, 2**16, 79, 8) + np.int32(M // 3)
    idx[: N // 4] = hot
    if dtype == "f64":
        b, a0 = synth.dyadic_f64(N, 79, 6), synth.dyadic_f64(M, 79, 7)
    else:
        b, a0 = synth.int_i32(N, -1000, 1000, 79, 6), synth.int_i32(M, -10**6, 10**6, 79, 7)
    ref = a0.copy()
    orc.scatter_add(idx, b, ref)
    a, bms, drs, reps = _scatter(J, idx, b, a0, n)
    assert np.array_equal(a, ref)
    for d in range(n):
        lo, hi = orc.partition(M, n, d)
        bm, mn, mx = orc.scatter_add_filtered(idx, b, a0.copy(), lo, hi - 1)
        assert np.array_equal(bms[d], bm) and drs[d] == (mn, mx)
        assert np.array_equal(reps[d], ref)


@pytest.mark.parametrize("dtype", ["f64", "i32"])
@pytest.mark.parametrize("n", [1, 3])
@pytest.mark.parametrize("where", ["late", "slight"])
def test_scatter_binned_overflow(J, monkeypatch, dtype, n, where):
    """The speculative layout's fallback: uniform keys except that the LAST
    tenth of the updates lands in one bucket ("late": the overflow is found
    after most tiles were written speculatively), or one bucket receiving
    ~1.3x the mean ("slight": just past the 1/8 slack).  The exact pipeline
    must redo the partition in the same launch; every result, bitmap and
    range equals the oracle."""
    monkeypatch.setenv("JACC_SCATTER_BINNED", "1")
    M = 2**24 + 999 if dtype == "f64" else 2**25 + 999
    N = 2**23 + 5
    idx = synth.index_i32(N, M, 81, 5)
    if where == "late":
        k = N // 10
        idx[N - k:] = synth.index_i32(k, 2**19, 81, 8) + np.int32(2**20 + 5)
    else:
        k = (3 * (N * 2**20 // M)) // 10  # +0.3 of a bucket's mean share, spread over the input
        pos = np.linspace(0, N - 1, k).astype(np.int64)
        idx[pos] = synth.index_i32(k, 2**20, 81, 8) + np.int32(2**21)
    if dtype == "f64":
        b, a0 = synth.dyadic_f64(N, 81, 6), synth.dyadic_f64(M, 81, 7)
    else:
        b, a0 = synth.int_i32(N, -1000, 1000, 81, 6), synth.int_i32(M, -10**6, 10**6, 81, 7)
    ref = a0.copy()
    orc.scatter_add(idx, b, ref)
    a, bms, drs, reps = _scatter(J, idx, b, a0, n)
    assert np.array_equal(a, ref)
    for d in range(n):
        lo, hi = orc.partition(M, n, d)
        bm, mn, mx = orc.scatter_add_filtered(idx, b, a0.copy(), lo, hi - 1)
        assert np.array_equal(bms[d], bm) and drs[d] == (mn, mx)
        assert np.array_equal(reps[d], ref)


@pytest.mark.parametrize("case", ["one_bucket", "one_element", "empty_owned"])
@pytest.mark.parametrize("n", [1, 2])
def test_scatter_binned_extreme_skew(J, monkeypatch, case, n):
    """Page allocation under extreme skew: every update in one bucket (a
    single bucket claims every page of the pool), every update on ONE
    element (maximum collisions; int32 exact), and updates that miss a
    device's slice entirely (empty buckets, no bits items)."""
    monkeypatch.setenv("JACC_SCATTER_BINNED", "1")
    N, M = 3_000_017, 5 * 2**20 + 3
    if case == "one_bucket":
        idx = synth.index_i32(N, 2**20, 116, 5) + np.int32(2**21)
    elif case == "one_element":
        idx = np.full(N, 2**21 + 7, dtype=np.int32)
    else:
        idx = synth.index_i32(N, 2**20, 116, 5)   # all in device 0's slice
    b = synth.int_i32(N, -1000, 1000, 116, 6)
    a0 = synth.int_i32(M, -10**6, 10**6, 116, 7)
    ref = a0.copy()
    orc.scatter_add(idx, b, ref)
    a, bms, drs, reps = _scatter(J, idx, b, a0, n)
    assert np.array_equal(a, ref)
    for d in range(n):
        lo, hi = orc.partition(M, n, d)
        bm, mn, mx = orc.scatter_add_filtered(idx, b, a0.copy(), lo, hi - 1)
        assert np.array_equal(bms[d], bm) and drs[d] == (mn, mx)
        assert np.array_equal(reps[d], ref)


def test_scatter_dup_mode(J):
    N, M = 10_000, 999
    idx = synth.index_i32(N, M, 77, 5)
    b = synth.int_i32(N, -9, 9, 77, 6)
    a0 = synth.int_i32(M, -9, 9, 77, 7)
    ref = a0.copy()
    orc.scatter_add(idx, b, ref)
    a = a0.copy()
    with runtime(J, 3, mode=1):
        _create(J, idx, b, a)
        J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_I32, J.make_range(0, N),
                      [_in(J, idx), _in(J, b), _inout(J, a)])
        for d in range(3):
            assert np.array_equal(J.jacc_get_replica(a, d), ref)
        J.jacc_update_host(a)
    assert np.array_equal(a, ref)


@pytest.mark.parametrize("n", [2, 3])
def test_reductions_dup_mode(J, n):
    """JACC_MODE_DUP: every device reduces the whole range; the result is one
    device's total plus s_in, not the sum over devices (found by the
    randomised programs)."""
    L = 10_007
    x = synth.dyadic_f64(L, 78, 1)
    y = synth.dyadic_f64(L, 78, 2)
    with runtime(J, n, mode=1):
        _create(J, x, y)
        s = np.array([1.5])
        J.jacc_launch(J.JACC_LOOP_DOT_F64, J.make_range(0, L),
                      [_in(J, x), _in(J, y), J.arg(J.JACC_ARG_REDUCE_SUM_F64, s)])
        assert s[0] == orc.dot_f64(x, y, 1.5)
        s = np.array([-2.0])
        J.jacc_launch(J.JACC_LOOP_SUM_F64, J.make_range(0, L),
                      [_in(J, x), J.arg(J.JACC_ARG_REDUCE_SUM_F64, s)])
        assert s[0] == orc.sum_f64(x, -2.0)


def test_scatter_full_size(J):
    """BASELINE config 5 at full size: 2^28 updates into 2^28 elements,
    random idx, dyadic b (exact in any order), n=1."""
    N = M = 2**28
    idx = synth.index_i32(N, M, 74, 5)
    b = synth.dyadic_f64(N, 74, 6)
    a0 = synth.dyadic_f64(M, 74, 7)
    ref = a0.copy()
    orc.scatter_add(idx, b, ref)
    a, bms, drs, _ = _scatter(J, idx, b, a0, 1)
    assert np.array_equal(a, ref)
    pop = int(np.unpackbits(bms[0].view(np.uint8)).sum())
    assert pop == np.unique(idx).size
    assert drs[0] == (int(idx.min()), int(idx.max()))


def test_scatter_sparse_full_size(J):
    """SURVEY 8(d) SCAT sparse variant: 2^20 updates into 2^28 elements on
    two devices under EAGER -- the dirty bitmaps are 0.4 % dense, the merge
    pushes only the set bits, and every replica equals the oracle."""
    N, M = 2**20, 2**28
    idx = synth.index_i32(N, M, 75, 5)
    b = synth.dyadic_f64(N, 75, 6)
    a0 = synth.dyadic_f64(M, 75, 7)
    ref = a0.copy()
    orc.scatter_add(idx, b, ref)
    a, bms, drs, reps = _scatter(J, idx, b, a0, 2)
    assert np.array_equal(a, ref)
    for r in reps:
        assert np.array_equal(r, ref)
    u = np.unique(idx)
    for d in range(2):
        lo, hi = orc.partition(M, 2, d)
        own = u[(u >= lo) & (u < hi)]
        assert int(np.unpackbits(bms[d].view(np.uint8)).sum()) == own.size
        assert drs[d] == (int(own.min()), int(own.max()))


# --------------------------------------------------------------------------
# runtime behaviour
# --------------------------------------------------------------------------
def test_present_table_errors(J):
    a = np.zeros(1000)
    with runtime(J):
        J.jacc_data_create(a)
        with pytest.raises(J.JaccError) as e:
            J.jacc_data_create(a[10:20])
        assert e.value.status == J.JACC_ERR_OVERLAP
        # any interior address resolves
        J.jacc_update_device(a[500:], 0, 80)
        b = np.zeros(10)
        st = J.jacc_launch_status(J.JACC_LOOP_SUM_F64, J.make_range(0, 10),
                                  [_in(J, b), J.arg(J.JACC_ARG_REDUCE_SUM_F64, np.zeros(1))])
        assert st == J.JACC_ERR_NOT_PRESENT
        assert J.jacc_launch_status(99, None, []) == J.JACC_ERR_UNKNOWN_LOOP
        J.jacc_data_delete(a[999:])
        with pytest.raises(J.JaccError):
            J.jacc_data_delete(a)


def test_profiling_records(J):
    N = 512
    A, B = synth.polybench_jacobi2d(N)
    with runtime(J, 2):
        J.jacc_set_profiling(1)
        _create(J, A, B)
        for _ in range(4):
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [_in(J, A), _out(J, B)], async_id=0)
        tk, tm, nb = J.jacc_last_timing()
        assert tk > 0 and tm >= 0 and nb > 0
        k, m, nl, _ = J.jacc_profile_totals(0)
        assert nl == 4 and k >= tk


# --------------------------------------------------------------------------
# NEXT-1 adaptive utilization
# --------------------------------------------------------------------------
@pytest.mark.parametrize("policy", [0, 1])
def test_adaptive_mode_parity_and_controller_replay(J, policy):
    """Under JACC_MODE_ADAPTIVE every launch runs duplicated or multi-GPU as
    the controller decides; results stay bit-exact, and the runtime's state
    sequence equals the oracle controller replayed on the same measured
    observations."""
    from oracle import adaptive as ad
    N, T = 514, 20
    A0 = synth.uniform_f64(N * N, 91, 1).reshape(N, N)
    B0 = synth.uniform_f64(N * N, 91, 2).reshape(N, N)
    Ar, Br = A0.copy(), B0.copy()
    orc.jacobi2d(T, Ar, Br)
    A, B = A0.copy(), B0.copy()
    with runtime(J, 2, policy, mode=J.JACC_MODE_ADAPTIVE):
        _create(J, A, B)
        for _ in range(T):
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [_in(J, A), _out(J, B)])
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [_in(J, B), _out(J, A)])
        trace, states, now = J.jacc_adaptive_history(J.JACC_LOOP_JACOBI2D_F64)
        J.jacc_update_host(A)
        J.jacc_update_host(B)
    assert np.array_equal(A, Ar) and np.array_equal(B, Br)
    assert len(trace) >= 2
    rep = ad.replay(trace, 2, 770e9)
    assert states == rep[:-1] and now == rep[-1]


# --------------------------------------------------------------------------
# NEXT-2 Himeno: 19-point stencil + gosa, copy loop
# --------------------------------------------------------------------------
def _himeno_gpu(J, arrs, nn, n, policy, omega=0.8, rng=None):
    p, a, b, c, w1, bd = (x.copy() for x in arrs)
    wrk2 = np.zeros_like(p)
    gosas, dirt = [], []
    with runtime(J, n, policy):
        _create(J, p, a, b, c, w1, bd, wrk2)
        IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
        for it in range(nn):
            g = np.zeros(1)
            J.jacc_launch(J.JACC_LOOP_HIMENO_F32, rng,
                          [J.arg(IN, p), J.arg(IN, a), J.arg(IN, b), J.arg(IN, c), J.arg(IN, w1),
                           J.arg(IN, bd), J.arg(OUT, wrk2), J.arg(J.JACC_ARG_REDUCE_SUM_F64, g),
                           J.arg(J.JACC_ARG_SCALAR_F64, f64=omega)])
            gosas.append(g[0])
            if it == 0:
                dirt.append([J.jacc_get_dirty_range(wrk2, d) for d in range(n)])
            J.jacc_launch(J.JACC_LOOP_HIMENO_COPY_F32, rng, [J.arg(IN, wrk2), J.arg(OUT, p)], 0)
            if it == 0:
                dirt.append([J.jacc_get_dirty_range(p, d) for d in range(n)])
        J.jacc_update_host(p)
        J.jacc_update_host(wrk2)
    return p, wrk2, gosas, dirt


@pytest.mark.parametrize("shape", [(3, 3, 3), (9, 5, 7), (17, 12, 21), (34, 33, 35), (66, 40, 70),
                                   (40, 21, 132), (70, 37, 64), (9, 260, 12)])
@pytest.mark.parametrize("n", [1, 2, 3, 8])
@pytest.mark.parametrize("policy", [0, 1])
def test_himeno_multi_device(J, shape, n, policy):
    """K % 4 == 0 shapes take the plane-marching kernel (several k strips, a
    partial last strip, several j blocks and i segments, ragged ends), the
    others the row-per-warp kernel."""
    I, Jd, K = shape
    arrs = synth.himeno_random(I, Jd, K, 95)
    nn = 3
    p, a, b, c, w1, bd = (x.copy() for x in arrs)
    wrk2 = np.zeros_like(p)
    refs, logs = [], []
    for it in range(nn):
        _, gref, wl = orc.himeno_stencil(p, a, b, c, w1, bd, wrk2)
        refs.append(gref)
        cl = orc.himeno_copy(wrk2, p)
        if it == 0:
            logs = (wl, cl)
    gp, gw, gosas, dirt = _himeno_gpu(J, arrs, nn, n, policy)
    assert np.array_equal(gp, p) and np.array_equal(gw, wrk2)
    for g, r in zip(gosas, refs):
        assert abs(g - r) <= 1e-12 * abs(r) + 1e-300
    # per-device dirty ranges == oracle write logs of the filtered launches
    p0, a0, b0, c0, w10, bd0 = arrs
    for d in range(n):
        lo, hi = orc.partition(I, n, d)
        tmp = np.zeros_like(p0)
        _, _, wl = orc.himeno_stencil(p0, a0, b0, c0, w10, bd0, tmp, planes=(lo, hi - 1))
        assert dirt[0][d] == wl
        cl = orc.himeno_copy(tmp, p0.copy(), planes=(lo, hi - 1))
        assert dirt[1][d] == cl


@pytest.mark.parametrize("K", [22, 24])
def test_himeno_subrange(J, K):
    """A launch box off the interior (k from 5: partial float4 chunks; K = 24
    takes the plane-marching kernel)."""
    I, Jd = 20, 18
    arrs = synth.himeno_random(I, Jd, K, 96)
    rng = J.make_range([3, 2, 5], [15, 17, 20])
    gp, gw, gosas, _ = _himeno_gpu(J, arrs, 1, 2, 0, rng=rng)
    p, a, b, c, w1, bd = (x.copy() for x in arrs)
    full = np.zeros_like(p)
    orc.himeno_stencil(p, a, b, c, w1, bd, full)
    box = (slice(3, 15), slice(2, 17), slice(5, 20))
    w_ref = np.zeros_like(p)
    w_ref[box] = full[box]
    assert np.array_equal(gw, w_ref)
    p_ref = p.copy()
    p_ref[box] = full[box]
    assert np.array_equal(gp, p_ref)


@pytest.mark.parametrize("shape", [(1024, 512, 512), (1025, 513, 513)])
def test_himeno_XL_full_size(J, shape):
    """The paper's Size XL grid (1024x512x512; DESIGN R-17) with the
    benchmark's initial state, one iteration at n=1 (the bench launch
    configuration), and himenoBMT's 1025x513x513 allocation (rows off
    16-byte alignment): wrk2 and p bit-exact vs the oracle, gosa within
    1e-12 of the compensated reference."""
    I, Jd, K = shape
    arrs = synth.himeno_init(I, Jd, K)
    gp, gw, gosas, _ = _himeno_gpu(J, arrs, 1, 1, 0)
    p, a, b, c, w1, bd = arrs
    wrk2 = np.zeros_like(p)
    g, gref, _ = orc.himeno_stencil(p, a, b, c, w1, bd, wrk2)
    assert np.array_equal(gw, wrk2)
    assert abs(gosas[0] - gref) <= 1e-12 * gref
    orc.himeno_copy(wrk2, p)
    assert np.array_equal(gp, p)


# --------------------------------------------------------------------------
# CUDA graphs of launch sequences
# --------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 3])
@pytest.mark.parametrize("policy", [0, 1])
def test_graph_capture_replay_jacobi(J, n, policy):
    """Capture one steady timestep (2 launches, merges included) and replay
    it; interleave with plain launches; results equal the oracle."""
    N = 301
    A0 = synth.uniform_f64(N * N, 97, 1).reshape(N, N)
    B0 = synth.uniform_f64(N * N, 97, 2).reshape(N, N)
    A, B = A0.copy(), B0.copy()
    IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
    ab, ba = [J.arg(IN, A), J.arg(OUT, B)], [J.arg(IN, B), J.arg(OUT, A)]

    def step():
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, ab, 0)
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, ba, 0)

    with runtime(J, n, policy):
        _create(J, A, B)
        step()                       # steady state
        J.jacc_graph_begin()
        step()                       # captured, not executed
        gid = J.jacc_graph_end()
        J.jacc_graph_replay(gid, 3)  # timesteps 2..4
        step()                       # timestep 5 (plain)
        J.jacc_graph_replay(gid, 1)  # timestep 6
        J.jacc_update_host(A)
        J.jacc_update_host(B)
        J.jacc_graph_destroy(gid)
    Ar, Br = A0.copy(), B0.copy()
    orc.jacobi2d(6, Ar, Br)
    assert np.array_equal(A, Ar) and np.array_equal(B, Br)


@pytest.mark.parametrize("n", [1, 2])
def test_graph_capture_replay_binned_scatter(J, monkeypatch, n):
    """The binned scatter (dirty bits by the bucket pass, no host-side
    byte-map state) runs inside a captured graph once its scratch was
    reserved by a plain launch: 1 plain + 3 replays + 1 plain = 5 scatters
    of the same updates, exact in int32; bitmap and range of the last."""
    monkeypatch.setenv("JACC_SCATTER_BINNED", "1")
    N, M = 200_003, 70_001
    idx = synth.index_i32(N, M, 99, 5)
    b = synth.int_i32(N, -50, 50, 99, 6)
    a0 = synth.int_i32(M, -10**6, 10**6, 99, 7)
    a = a0.copy()
    args = [_in(J, idx), _in(J, b), _inout(J, a)]
    rng = J.make_range(0, N)
    with runtime(J, n):
        _create(J, idx, b, a)
        J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_I32, rng, args, 0)
        J.jacc_graph_begin()
        J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_I32, rng, args, 0)
        gid = J.jacc_graph_end()
        J.jacc_graph_replay(gid, 3)
        J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_I32, rng, args, 0)
        J.jacc_wait()
        bms = [J.jacc_get_dirty_bitmap(a, d, M) for d in range(n)]
        drs = [J.jacc_get_dirty_range(a, d) for d in range(n)]
        J.jacc_update_host(a)
        J.jacc_graph_destroy(gid)
    ref = a0.copy()
    for _ in range(5):
        orc.scatter_add(idx, b, ref)
    assert np.array_equal(a, ref)
    for d in range(n):
        lo, hi = orc.partition(M, n, d)
        bm, mn, mx = orc.scatter_add_filtered(idx, b, a0.copy(), lo, hi - 1)
        assert np.array_equal(bms[d], bm) and drs[d] == (mn, mx)


def test_graph_rules(J):
    N = 64
    A = synth.uniform_f64(N * N, 98, 1).reshape(N, N)
    B = synth.uniform_f64(N * N, 98, 2).reshape(N, N)
    x = synth.dyadic_f64(1000, 98, 3)
    IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
    with runtime(J, 2, 1):
        _create(J, A, B, x)
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, A), J.arg(OUT, B)])
        J.jacc_graph_begin()
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, B), J.arg(OUT, A)])
        # reductions cannot be captured; synchronous calls are refused
        st = J.jacc_launch_status(J.JACC_LOOP_SUM_F64, J.make_range(0, 1000),
                                  [J.arg(IN, x), J.arg(J.JACC_ARG_REDUCE_SUM_F64, np.zeros(1))])
        assert st == J.JACC_ERR_INVALID
        assert J.lib.jacc_wait(-1) == J.JACC_ERR_STATE
        gid = J.jacc_graph_end()
        # a fresh upload of B (stale on the peer under HALO) changes the
        # replica validity: replay refused
        J.jacc_update_device(B)
        assert J.lib.jacc_graph_replay(gid, 1) == J.JACC_ERR_STATE


@pytest.mark.parametrize("count", [1, 2, 3])
def test_graph_replay_odd_writes_keep_dirty_records_exact(J, count):
    """A graph writing x three times flips x's dirty-record slot parity on
    every replay; each replay must still leave the exact record of its last
    launch (no stale min/max from the previous replay)."""
    M = 100
    y = synth.uniform_f32(M, 99, 1)
    x = np.zeros(M, dtype=np.float32)
    IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
    args = [J.arg(IN, y), J.arg(OUT, x)]
    with runtime(J, 2):
        _create(J, y, x)
        J.jacc_graph_begin()
        for lo, hi in ((0, 10), (20, 30), (40, 50)):
            J.jacc_launch(J.JACC_LOOP_SQUARE_F32, J.make_range(lo, hi), args)
        gid = J.jacc_graph_end()
        J.jacc_graph_replay(gid, count)
        J.jacc_wait()
        # device 0 owns [0, 50): its last write was [40, 50); device 1 none
        assert J.jacc_get_dirty_range(x, 0) == (40, 49)
        assert J.jacc_get_dirty_range(x, 1) == (U64MAX, 0)
        # a plain launch after the replays records its own range only
        J.jacc_launch(J.JACC_LOOP_SQUARE_F32, J.make_range(5, 7), args)
        assert J.jacc_get_dirty_range(x, 0) == (5, 6)
        J.jacc_update_host(x)
    ref = np.zeros(M, dtype=np.float32)
    for lo, hi in ((0, 10), (20, 30), (40, 50)):
        ref[lo:hi] = orc.square_f32(np.ascontiguousarray(y[lo:hi]))
    assert np.array_equal(x, ref)


def test_graph_replay_count_needs_a_fixed_point(J):
    """count > 1 replays back to back only when the graph maps the captured
    validity state onto itself (its pulls were planned for that state)."""
    N = 40
    A = synth.uniform_f64(N * N, 99, 2).reshape(N, N)
    B = synth.uniform_f64(N * N, 99, 3).reshape(N, N)
    IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
    with runtime(J, 2, 1):  # HALO: peers' copies go stale
        _create(J, A, B)
        J.jacc_graph_begin()
        J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, A), J.arg(OUT, B)])
        gid = J.jacc_graph_end()
        assert J.lib.jacc_graph_replay(gid, 2) == J.JACC_ERR_STATE
        assert J.lib.jacc_graph_replay(gid, 1) == J.JACC_OK


# --------------------------------------------------------------------------
# NEXT-2 multidimensional division: split dims > 0 (strided blocks)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("N", [17, 64, 301])
@pytest.mark.parametrize("n", [2, 3, 8])
@pytest.mark.parametrize("policy", [0, 1])
def test_jacobi_column_split(J, N, n, policy):
    T = 2
    A0 = synth.uniform_f64(N * N, 99 + N, 1).reshape(N, N)
    B0 = synth.uniform_f64(N * N, 99 + N, 2).reshape(N, N)
    Ar, Br = A0.copy(), B0.copy()
    orc.jacobi2d(T, Ar, Br)
    A, B = A0.copy(), B0.copy()
    IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
    with runtime(J, n, policy):
        J.jacc_set_split_dim(1)
        _create(J, A, B)
        dirt = None
        for t in range(T):
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, A), J.arg(OUT, B)], 0)
            if t == 0:
                dirt = [J.jacc_get_dirty_range(B, d) for d in range(n)]
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, B), J.arg(OUT, A)], 0)
        if policy == 0:
            for d in range(n):
                assert np.array_equal(J.jacc_get_replica(A, d), Ar)
        J.jacc_update_host(A)
        J.jacc_update_host(B)
    assert np.array_equal(A, Ar) and np.array_equal(B, Br)
    for d in range(n):
        lo, hi = orc.partition(N, n, d)     # column block
        a, b = max(lo, 1), min(hi, N - 1)
        exp = (2**64 - 1, 0) if a >= b else (1 * N + a, (N - 2) * N + b - 1)
        assert dirt[d] == exp


@pytest.mark.parametrize("split", [1, 2])
@pytest.mark.parametrize("n", [2, 3])
@pytest.mark.parametrize("policy", [0, 1])
def test_himeno_split_dims(J, split, n, policy):
    I, Jd, K = 13, 11, 17
    arrs = synth.himeno_random(I, Jd, K, 100)
    nn = 2
    p, a, b, c, w1, bd = (x.copy() for x in arrs)
    wrk2 = np.zeros_like(p)
    refs = []
    for _ in range(nn):
        refs.append(orc.himeno_stencil(p, a, b, c, w1, bd, wrk2)[1])
        orc.himeno_copy(wrk2, p)
    gp, gw, gosas, _ = _himeno_gpu_split(J, arrs, nn, n, policy, split)
    assert np.array_equal(gp, p) and np.array_equal(gw, wrk2)
    for g, r in zip(gosas, refs):
        assert abs(g - r) <= 1e-12 * abs(r)


def _himeno_gpu_split(J, arrs, nn, n, policy, split):
    p, a, b, c, w1, bd = (x.copy() for x in arrs)
    wrk2 = np.zeros_like(p)
    gosas = []
    IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
    with runtime(J, n, policy):
        J.jacc_set_split_dim(split)
        _create(J, p, a, b, c, w1, bd, wrk2)
        for _ in range(nn):
            g = np.zeros(1)
            J.jacc_launch(J.JACC_LOOP_HIMENO_F32, None,
                          [J.arg(IN, p), J.arg(IN, a), J.arg(IN, b), J.arg(IN, c), J.arg(IN, w1),
                           J.arg(IN, bd), J.arg(OUT, wrk2), J.arg(J.JACC_ARG_REDUCE_SUM_F64, g),
                           J.arg(J.JACC_ARG_SCALAR_F64, f64=0.8)])
            gosas.append(g[0])
            J.jacc_launch(J.JACC_LOOP_HIMENO_COPY_F32, None, [J.arg(IN, wrk2), J.arg(OUT, p)], 0)
        J.jacc_update_host(p)
        J.jacc_update_host(wrk2)
    return p, wrk2, gosas, None


@pytest.mark.parametrize("n", [2, 3])
def test_gemm_column_split(J, n):
    M, N, K = 70, 90, 33
    A = synth.uniform_f64(M * K, 101, 1).reshape(M, K)
    B = synth.uniform_f64(K * N, 101, 2).reshape(K, N)
    ref = orc.gemm_f64(A, B)
    C = np.zeros((M, N))
    IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
    with runtime(J, n):
        J.jacc_set_split_dim(1)
        _create(J, A, B, C)
        J.jacc_launch(J.JACC_LOOP_GEMM_F64, None, [J.arg(IN, A), J.arg(IN, B), J.arg(OUT, C)])
        reps = [J.jacc_get_replica(C, d) for d in range(n)]
        J.jacc_update_host(C)
    assert (np.abs(C - ref) <= 1e-12 * (np.abs(A) @ np.abs(B))).all()
    for r in reps:
        assert np.array_equal(r, C)


def test_split_dim_validation(J):
    x = np.zeros(10, dtype=np.float32)
    y = np.zeros(10, dtype=np.float32)
    A = np.zeros((8, 8)); B = np.zeros((8, 8))
    with runtime(J, 2):
        with pytest.raises(J.JaccError):
            J.jacc_set_split_dim(3)
        J.jacc_set_split_dim(2)
        _create(J, A, B, x, y)
        st = J.jacc_launch_status(J.JACC_LOOP_JACOBI2D_F64, None, [_in(J, A), _out(J, B)])
        assert st == J.JACC_ERR_INVALID          # a 2-D array has no dim 2
        J.jacc_launch(J.JACC_LOOP_SQUARE_F32, J.make_range(0, 10), [_in(J, y), _out(J, x)])  # 1-D: dim 0


# --------------------------------------------------------------------------
# NEXT-3 iteration-split scatter with an additive merge
# --------------------------------------------------------------------------
@pytest.mark.parametrize("n", [2, 3, 8])
@pytest.mark.parametrize("sizes", [(100_003, 5000), (1_000_000, 1_000_003)])
@pytest.mark.parametrize("dtype", ["f64", "i32"])
@pytest.mark.parametrize("policy", [0, 1])
def test_scatter_iteration_split(J, n, sizes, dtype, policy):
    N, M = sizes
    idx = synth.index_i32(N, M, 102, 5)
    if dtype == "f64":
        b, a0 = synth.dyadic_f64(N, 102, 6), synth.dyadic_f64(M, 102, 7)
        loop = J.JACC_LOOP_SCATTER_ADD_F64
    else:
        b, a0 = synth.int_i32(N, -1000, 1000, 102, 6), synth.int_i32(M, -10**6, 10**6, 102, 7)
        loop = J.JACC_LOOP_SCATTER_ADD_I32
    ref = a0.copy()
    orc.scatter_add(idx, b, ref)
    orc.scatter_add(idx, b, ref)             # two launches
    a = a0.copy()
    with runtime(J, n, policy):
        J.jacc_set_scatter_split(1)
        _create(J, idx, b, a)
        args = [_in(J, idx), _in(J, b), _inout(J, a)]
        J.jacc_launch(loop, J.make_range(0, N), args)
        J.jacc_launch(loop, J.make_range(0, N), args)   # deltas must have been re-zeroed
        words = (M + 31) // 32
        for d in range(n):
            w0, w1 = orc.partition(words, n, d)
            lo, hi = min(32 * w0, M), min(32 * w1, M)
            bm, mn, mx = orc.scatter_add_filtered(idx, b, a0.copy(), lo, hi - 1)
            assert np.array_equal(J.jacc_get_dirty_bitmap(a, d, M), bm)
            assert J.jacc_get_dirty_range(a, d) == (mn, mx)
            if policy == 0:
                assert np.array_equal(J.jacc_get_replica(a, d), ref)
        J.jacc_update_host(a)
    assert np.array_equal(a, ref)


# --------------------------------------------------------------------------
# NEXT-3 Fig. 4 filtered statement chain (two written arrays)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("n_it", [1, 257, 100_003])
@pytest.mark.parametrize("n", [1, 2, 3, 8])
@pytest.mark.parametrize("policy", [0, 1])
def test_fig4_chain(J, n_it, n, policy):
    from test_oracle_fig4 import _inputs
    x_in = 0.375
    jx, kx, c, a0, b0 = _inputs(n_it, 3)
    a_ref, b_ref = a0.copy(), b0.copy()
    orc.fig4(jx, kx, c, x_in, a_ref, b_ref)
    a, b = a0.copy(), b0.copy()
    IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
    with runtime(J, n, policy):
        _create(J, jx, kx, c, a, b)
        J.jacc_launch(J.JACC_LOOP_FIG4_F64, J.make_range(0, n_it),
                      [J.arg(IN, jx), J.arg(IN, kx), J.arg(IN, c), J.arg(OUT, a), J.arg(OUT, b),
                       J.arg(J.JACC_ARG_SCALAR_F64, f64=x_in)])
        for d in range(n):
            alo, ahi = orc.partition(a0.size, n, d)
            blo, bhi = orc.partition(b0.size, n, d)
            da, db = a0.copy(), b0.copy()
            la, lb = orc.fig4_filtered(jx, kx, c, x_in, da, db, (alo, ahi - 1), (blo, bhi - 1))
            assert J.jacc_get_dirty_range(a, d) == la and J.jacc_get_dirty_range(b, d) == lb
            if policy == 0:
                assert np.array_equal(J.jacc_get_replica(a, d), a_ref)
                assert np.array_equal(J.jacc_get_replica(b, d), b_ref)
        J.jacc_update_host(a)
        J.jacc_update_host(b)
    assert np.array_equal(a, a_ref) and np.array_equal(b, b_ref)


# --------------------------------------------------------------------------
# NEXT-4 automated async queues
# --------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 3])
@pytest.mark.parametrize("policy", [0, 1])
def test_async_queues_independent_and_dependent_loops(J, n, policy):
    """Two independent Jacobi problems and a dependent dot/scatter chain,
    launched JACC_ASYNC_AUTO over 16 queues: every result equals the
    oracle (the scheduler's waits make the cross-queue dependencies safe)."""
    N = 130
    A1 = synth.uniform_f64(N * N, 110, 1).reshape(N, N); B1 = synth.uniform_f64(N * N, 110, 2).reshape(N, N)
    A2 = synth.uniform_f64(N * N, 111, 1).reshape(N, N); B2 = synth.uniform_f64(N * N, 111, 2).reshape(N, N)
    refs = []
    for A, B in ((A1, B1), (A2, B2)):
        Ar, Br = A.copy(), B.copy()
        orc.jacobi2d(3, Ar, Br)
        refs += [Ar, Br]
    idx = synth.index_i32(5000, N * N, 112, 5)
    bb = synth.dyadic_f64(5000, 112, 6)
    IN, OUT, INOUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT, J.JACC_ARG_ARRAY_INOUT
    AUTO = J.JACC_ASYNC_AUTO
    with runtime(J, n, policy):
        J.jacc_set_queues(16)
        _create(J, A1, B1, A2, B2, idx, bb)
        for _ in range(3):
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, A1), J.arg(OUT, B1)], AUTO)
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, A2), J.arg(OUT, B2)], AUTO)
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, B1), J.arg(OUT, A1)], AUTO)
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, B2), J.arg(OUT, A2)], AUTO)
        # dependent chain on A1: scatter into it (reads A1's final state), then a dot
        J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_F64, J.make_range(0, 5000),
                      [J.arg(IN, idx), J.arg(IN, bb), J.arg(INOUT, A1.reshape(-1))], AUTO)
        s = np.zeros(1)
        J.jacc_launch(J.JACC_LOOP_SUM_F64, J.make_range(0, N * N),
                      [J.arg(IN, A1.reshape(-1)), J.arg(J.JACC_ARG_REDUCE_SUM_F64, s)], AUTO)
        J.jacc_wait(-1)
        for x in (A1, B1, A2, B2):
            J.jacc_update_host(x)
    Ar1 = refs[0].copy()
    orc.scatter_add(idx, bb, Ar1.reshape(-1))
    assert np.array_equal(A1, Ar1) and np.array_equal(B1, refs[1])
    assert np.array_equal(A2, refs[2]) and np.array_equal(B2, refs[3])
    assert s[0] == pytest.approx(orc.sum_neumaier(Ar1.reshape(-1)), rel=1e-12)


# --------------------------------------------------------------------------
# merge traffic accounting (per-link bytes non-increasing in n)
# --------------------------------------------------------------------------
def test_merge_bytes_scale_with_n(J):
    N = 514
    A = synth.uniform_f64(N * N, 120, 1).reshape(N, N)
    B = synth.uniform_f64(N * N, 120, 2).reshape(N, N)
    IN, OUT = J.JACC_ARG_ARRAY_IN, J.JACC_ARG_ARRAY_OUT
    eager, halo = {}, {}
    for n in (2, 4, 8):
        for policy, store in ((0, eager), (1, halo)):
            with runtime(J, n, policy):
                _create(J, A, B)
                J.jacc_set_profiling(1)
                J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [J.arg(IN, A), J.arg(OUT, B)])
                _, _, nb = J.jacc_last_timing()
                store[n] = nb
    # EAGER: every device sends its block to n-1 peers: total (n-1) x block
    # sum = (n-1)/n x the written region; per link (one peer) = block, which
    # shrinks with n
    per_link = {n: eager[n] / (n * (n - 1)) for n in eager}
    assert per_link[2] > per_link[4] > per_link[8]
    # HALO: two boundary rows per interior device, independent of the block
    assert halo[2] == 2 * (N - 2) * 8
    assert halo[8] == 2 * (8 - 1) * (N - 2) * 8


# --------------------------------------------------------------------------
# Regression tests for the round-1 advisor findings
# --------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 2])
def test_graph_scratch_survives_regrowth(J, monkeypatch, n):
    """A graph captured over a binned scatter keeps its scratch: a later,
    larger uncaptured scatter must not free the buffer the graph baked in
    (it is retired until jacc_graph_destroy)."""
    monkeypatch.setenv("JACC_SCATTER_BINNED", "1")
    N, M = 100_003, 70_001
    idx = synth.index_i32(N, M, 111, 5)
    b = synth.int_i32(N, -50, 50, 111, 6)
    a0 = synth.int_i32(M, -10**6, 10**6, 111, 7)
    N2 = 3_000_017
    idx2 = synth.index_i32(N2, M, 111, 8)
    b2 = synth.int_i32(N2, -50, 50, 111, 9)
    a = a0.copy()
    args = [_in(J, idx), _in(J, b), _inout(J, a)]
    with runtime(J, n):
        _create(J, idx, b, a, idx2, b2)
        J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_I32, J.make_range(0, N), args, 0)
        J.jacc_graph_begin()
        J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_I32, J.make_range(0, N), args, 0)
        gid = J.jacc_graph_end()
        # needs a larger scratch: the old one is retired, not freed
        J.jacc_launch(J.JACC_LOOP_SCATTER_ADD_I32, J.make_range(0, N2),
                      [_in(J, idx2), _in(J, b2), _inout(J, a)], 0)
        J.jacc_wait()
        # the captured state is S_start again only if the validity matches:
        # under EAGER n=2 / n=1 every replica is valid, so replay is allowed
        J.jacc_graph_replay(gid, 2)
        J.jacc_wait()
        J.jacc_update_host(a)
        J.jacc_graph_destroy(gid)
    ref = a0.copy()
    orc.scatter_add(idx, b, ref)
    orc.scatter_add(idx2, b2, ref)
    orc.scatter_add(idx, b, ref)
    orc.scatter_add(idx, b, ref)
    assert np.array_equal(a, ref)


def test_iteration_split_rejected_in_capture(J):
    N, M = 1000, 500
    idx = synth.index_i32(N, M, 112, 5)
    b = synth.int_i32(N, -5, 5, 112, 6)
    a = synth.int_i32(M, -5, 5, 112, 7)
    with runtime(J, 2):
        J.jacc_set_scatter_split(1)
        _create(J, idx, b, a)
        J.jacc_graph_begin()
        st = J.jacc_launch_status(J.JACC_LOOP_SCATTER_ADD_I32, J.make_range(0, N),
                                  [_in(J, idx), _in(J, b), _inout(J, a)], 0)
        J.jacc_graph_end()
    assert st == J.JACC_ERR_INVALID


@pytest.mark.parametrize("policy", [0, 1])
@pytest.mark.parametrize("dtype", ["f64", "i32"])
def test_iteration_split_back_to_back_halo(J, policy, dtype):
    """Iteration-split scatter launched back to back without host syncs:
    phase 1 of launch k+1 must wait for every peer's phase 2 of launch k
    (which read and zeroed this device's delta), under either policy."""
    N, M = 2_000_003, 1_000_003
    idx = synth.index_i32(N, M, 113, 5)
    if dtype == "f64":
        b, a0 = synth.dyadic_f64(N, 113, 6), synth.dyadic_f64(M, 113, 7)
        loop = J.JACC_LOOP_SCATTER_ADD_F64
    else:
        b, a0 = synth.int_i32(N, -1000, 1000, 113, 6), synth.int_i32(M, -10**6, 10**6, 113, 7)
        loop = J.JACC_LOOP_SCATTER_ADD_I32
    K = 6
    ref = a0.copy()
    for _ in range(K):
        orc.scatter_add(idx, b, ref)
    a = a0.copy()
    with runtime(J, 3, policy):
        J.jacc_set_scatter_split(1)
        _create(J, idx, b, a)
        args = [_in(J, idx), _in(J, b), _inout(J, a)]
        for _ in range(K):
            J.jacc_launch(loop, J.make_range(0, N), args, 0)
        J.jacc_wait()
        J.jacc_update_host(a)
    assert np.array_equal(a, ref)


def test_inactive_device_dirty_slots_cleared(J):
    """A device idle in one launch clears both dirty slots, so its next
    active launch records only its own stores (not the union with the
    range from two launches earlier)."""
    y = synth.uniform_f32(3000, 114, 3)
    x = np.zeros(3000, dtype=np.float32)
    with runtime(J, 3):
        _create(J, y, x)
        args = [_in(J, y), _out(J, x)]
        J.jacc_launch(J.JACC_LOOP_SQUARE_F32, J.make_range(0, 3000), args)
        assert J.jacc_get_dirty_range(x, 2) == (2000, 2999)
        J.jacc_launch(J.JACC_LOOP_SQUARE_F32, J.make_range(0, 1000), args)  # device 2 idle
        assert J.jacc_get_dirty_range(x, 2) == J.EMPTY_RANGE
        J.jacc_launch(J.JACC_LOOP_SQUARE_F32, J.make_range(2500, 2600), args)
        assert J.jacc_get_dirty_range(x, 2) == (2500, 2599)
        assert J.jacc_get_dirty_range(x, 0) == J.EMPTY_RANGE
        J.jacc_update_host(x)
    assert np.array_equal(x, y * y)


@pytest.mark.parametrize("nq", [2, 3])
def test_async_queues_cross_device_same_queue(J, nq):
    """Jacobi ping-pong pinned to one explicit queue on 3 devices under HALO:
    queue q on device d must follow queue q on its peers (their pushes into
    d's replica, d's pushes into theirs)."""
    N, T = 515, 6
    A0 = synth.uniform_f64(N * N, 115, 1).reshape(N, N)
    B0 = synth.uniform_f64(N * N, 115, 2).reshape(N, N)
    Ar, Br = A0.copy(), B0.copy()
    orc.jacobi2d(T, Ar, Br)
    A, B = A0.copy(), B0.copy()
    with runtime(J, 3, 1):
        J.jacc_set_queues(nq)
        _create(J, A, B)
        for t in range(T):
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [_in(J, A), _out(J, B)], 1)
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [_in(J, B), _out(J, A)], 1)
        J.jacc_wait()
        J.jacc_update_host(A)
        J.jacc_update_host(B)
    assert np.array_equal(A, Ar) and np.array_equal(B, Br)


# --------------------------------------------------------------------------
# D13 trace records and runtime facts (jacc_get_info)
# --------------------------------------------------------------------------
def test_trace_json_lines(J, tmp_path):
    import json
    N = 130
    A = synth.uniform_f64(N * N, 117, 1).reshape(N, N)
    B = synth.uniform_f64(N * N, 117, 2).reshape(N, N)
    x = synth.dyadic_f64(5000, 117, 3)
    path = tmp_path / "trace.jsonl"
    with runtime(J, 3, 1):
        _create(J, A, B, x)
        J.jacc_set_trace(path)
        for _ in range(2):
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [_in(J, A), _out(J, B)], 0)
            J.jacc_launch(J.JACC_LOOP_JACOBI2D_F64, None, [_in(J, B), _out(J, A)], 0)
        s = np.zeros(1)
        J.jacc_launch(J.JACC_LOOP_SUM_F64, J.make_range(0, 5000),
                      [_in(J, x), J.arg(J.JACC_ARG_REDUCE_SUM_F64, s)])
        J.jacc_set_trace(None)
        info = J.jacc_get_info()
    lines = [json.loads(l) for l in open(path)]
    ev, summ = lines[:-1], lines[-1]["summary"]
    assert [e["event"] for e in ev] == list(range(5))
    assert [e["kernel"] for e in ev] == ["jacobi2d_f64"] * 4 + ["sum_f64"]
    for e in ev[:4]:
        assert e["merge"] == "halo" and e["mode"] == "multi" and e["devices"] == 3
        assert e["t_kernel_s"] > 0 and e["t_comm_s"] >= 0
        # HALO: device pushes of two boundary rows per interior boundary
        assert e["bytes_exchanged"] == 2 * 2 * 8 * (N - 2)
    assert ev[4]["bytes_exchanged"] == 0
    assert summ["events"] == 5
    assert summ["per_kernel_modes"]["jacobi2d_f64"] == {"multi": 4, "dup": 0}
    assert abs(summ["total_kernel_s"] - sum(e["t_kernel_s"] for e in ev)) < 1e-6
    assert info["n_devices"] == 3 and info["distinct_gpus"] == 0 and info["combine"] == "peer"
    assert s[0] == orc.sum_f64(x, 0.0)


def test_info_single_device(J):
    with runtime(J, 1):
        info = J.jacc_get_info()
    assert info == {"n_devices": 1, "distinct_gpus": 1, "combine": "peer", "peer_pairs": 0,
                    "multiprocess": 0, "rank": 0}


def test_nccl_combine_path_single_gpu(J, monkeypatch):
    """The NCCL allreduce combine executed on a one-GPU
    box: JACC_FORCE_NCCL builds a one-rank communicator, so the reduction
    goes through ncclAllReduce + the combine kernel; dyadic inputs, exact."""
    monkeypatch.setenv("JACC_FORCE_NCCL", "1")
    L = 1_000_003
    x = synth.dyadic_f64(L, 118, 1)
    y = synth.dyadic_f64(L, 118, 2)
    with runtime(J, 1):
        assert J.jacc_get_info()["combine"] == "nccl"
        _create(J, x, y)
        s = np.array([0.75])
        J.jacc_launch(J.JACC_LOOP_DOT_F64, J.make_range(0, L),
                      [_in(J, x), _in(J, y), J.arg(J.JACC_ARG_REDUCE_SUM_F64, s)])
        s2 = np.array([-1.0])
        J.jacc_launch(J.JACC_LOOP_SUM_F64, J.make_range(0, L),
                      [_in(J, x), J.arg(J.JACC_ARG_REDUCE_SUM_F64, s2)])
    assert s[0] == orc.dot_f64(x, y, 0.75)
    assert s2[0] == orc.sum_f64(x, -1.0)
