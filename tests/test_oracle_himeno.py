"""Pins for the Himeno oracle (NEXT-2 workload; DESIGN R-17).

Closed forms derived by hand for polynomial pressure fields with
power-of-two coefficients, where every fp32 operation is exact: a swapped
coefficient/neighbour pairing, a wrong sign in a cross term, or a dropped
term changes the result."""
from fractions import Fraction

import numpy as np
import pytest

import oracle as orc

# distinct powers of two per coefficient array (a0,a1,a2 | b0,b1,b2 | c0,c1,c2 | wrk1)
COEF = dict(a0=1, a1=2, a2=4, b0=8, b1=16, b2=32, c0=64, c1=128, c2=256, wrk1=512)


def _arrays(I, J, K, field, a3=0.125, bnd=2.0):
    i, j, k = np.meshgrid(np.arange(I), np.arange(J), np.arange(K), indexing="ij")
    p = np.ascontiguousarray(field(i, j, k).astype(np.float32))
    sh = (I, J, K)
    a = np.empty((4,) + sh, np.float32)
    a[0], a[1], a[2], a[3] = COEF["a0"], COEF["a1"], COEF["a2"], a3
    b = np.empty((3,) + sh, np.float32)
    b[0], b[1], b[2] = COEF["b0"], COEF["b1"], COEF["b2"]
    c = np.empty((3,) + sh, np.float32)
    c[0], c[1], c[2] = COEF["c0"], COEF["c1"], COEF["c2"]
    wrk1 = np.full(sh, COEF["wrk1"], np.float32)
    bd = np.full(sh, bnd, np.float32)
    return p, a, b, c, wrk1, bd, (i, j, k)


# s0 closed forms (hand-derived; see module docstring):
#  p = ij: a0(i+1)j + a1 i(j+1) + a2 ij + b0*4 + c0(i-1)j + c1 i(j-1) + c2 ij + w
#        = 455 ij - 63 j - 126 i + 32 + 512
#  p = ik: a0(i+1)k + a1 ik + a2 i(k+1) + b2*4 + c0(i-1)k + c1 ik + c2 i(k-1) + w
#        = 455 ik - 63 k - 252 i + 128 + 512
#  p = jk: a0 jk + a1(j+1)k + a2 j(k+1) + b1*4 + c0 jk + c1(j-1)k + c2 j(k-1) + w
#        = 455 jk - 126 k - 252 j + 64 + 512
CASES = {
    "ij": (lambda i, j, k: i * j, lambda i, j, k: 455 * i * j - 63 * j - 126 * i + 544),
    "ik": (lambda i, j, k: i * k, lambda i, j, k: 455 * i * k - 63 * k - 252 * i + 640),
    "jk": (lambda i, j, k: j * k, lambda i, j, k: 455 * j * k - 126 * k - 252 * j + 576),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_himeno_closed_forms_exact(case):
    I, J, K = 7, 6, 9
    field, s0f = CASES[case]
    p, a, b, c, w1, bd, (i, j, k) = _arrays(I, J, K, field)
    wrk2 = np.full((I, J, K), -5.0, np.float32)
    g, gref, (mn, mx) = orc.himeno_stencil(p, a, b, c, w1, bd, wrk2, omega=0.5)
    inner = (slice(1, -1),) * 3
    s0 = s0f(i, j, k)[inner].astype(np.int64)
    pv = field(i, j, k)[inner].astype(np.int64)
    # ss = (s0 * 0.125 - p) * 2 = s0/4 - 2p   (exact: multiples of 1/4)
    ss = s0 / 4 - 2 * pv
    assert np.array_equal(wrk2[inner].astype(np.float64), pv + 0.5 * ss)
    # gosa terms are fp32 products ss*ss (rounded as written); their exact sum:
    ss32 = ss.astype(np.float32)
    terms = (ss32 * ss32).reshape(-1)
    exact = sum((Fraction(float(t)) for t in terms), Fraction(0))
    assert abs(Fraction(gref) - exact) <= 2 * Fraction(np.spacing(float(exact)))
    assert abs(g - float(exact)) <= 1e-5 * float(exact)
    # boundary untouched
    assert (wrk2[0] == -5).all() and (wrk2[-1] == -5).all()
    assert (wrk2[:, 0] == -5).all() and (wrk2[:, :, -1] == -5).all()
    # write log: first and last interior point
    assert (mn, mx) == ((1 * J + 1) * K + 1, ((I - 2) * J + (J - 2)) * K + (K - 2))


def test_himeno_constant_field_residual_zero():
    """p constant, sum of the six neighbour coefficients = 1/a3: ss = 0,
    gosa = 0, wrk2 = p (a steady state of Jacobi's method)."""
    I, J, K = 6, 7, 8
    p = np.full((I, J, K), 3.0, np.float32)
    a = np.zeros((4, I, J, K), np.float32); a[:3] = 1; a[3] = 1 / 8
    b = np.full((3, I, J, K), 5.0, np.float32)   # cross terms cancel on a constant field
    c = np.zeros((3, I, J, K), np.float32); c[:] = 1
    c[2] = 3                                      # 1+1+1 + 1+1+3 = 8 = 1/a3
    w1 = np.zeros((I, J, K), np.float32)
    bd = np.ones((I, J, K), np.float32)
    wrk2 = np.zeros((I, J, K), np.float32)
    g, gref, _ = orc.himeno_stencil(p, a, b, c, w1, bd, wrk2)
    assert g == 0 and gref == 0
    assert (wrk2[1:-1, 1:-1, 1:-1] == 3).all()


def test_himeno_bnd_masks_points():
    I, J, K = 6, 6, 6
    p, a, b, c, w1, bd, _ = _arrays(I, J, K, lambda i, j, k: i * j)
    bd[:] = 0
    wrk2 = np.zeros((I, J, K), np.float32)
    g, gref, _ = orc.himeno_stencil(p, a, b, c, w1, bd, wrk2)
    assert g == 0 and np.array_equal(wrk2[1:-1, 1:-1, 1:-1], p[1:-1, 1:-1, 1:-1])


@pytest.mark.parametrize("n", [1, 2, 3, 5, 9])
def test_himeno_filtered_planes_partition(n):
    I, J, K = 9, 5, 7
    rng = np.random.default_rng(3)
    p = rng.random((I, J, K), dtype=np.float32)
    a = rng.random((4, I, J, K), dtype=np.float32)
    b = rng.random((3, I, J, K), dtype=np.float32)
    c = rng.random((3, I, J, K), dtype=np.float32)
    w1 = rng.random((I, J, K), dtype=np.float32)
    bd = rng.random((I, J, K), dtype=np.float32)
    full = np.zeros((I, J, K), np.float32)
    _, gref, _ = orc.himeno_stencil(p, a, b, c, w1, bd, full)
    over = np.zeros((I, J, K), np.float32)
    tot = 0.0
    for d in range(n):
        lo, hi = orc.partition(I, n, d)
        w = np.zeros((I, J, K), np.float32)
        _, r, (mn, mx) = orc.himeno_stencil(p, a, b, c, w1, bd, w, planes=(lo, hi - 1))
        tot += r
        over[lo:hi] = w[lo:hi]
        a_, b_ = max(lo, 1), min(hi, I - 1)
        if a_ >= b_:
            assert (mn, mx) == (2**64 - 1, 0)
        else:
            assert (mn, mx) == ((a_ * J + 1) * K + 1, ((b_ - 1) * J + (J - 2)) * K + (K - 2))
    assert np.array_equal(over, full)
    assert tot == pytest.approx(gref, rel=1e-13)
    # copy loop
    p2 = p.copy()
    orc.himeno_copy(full, p2)
    assert np.array_equal(p2[1:-1, 1:-1, 1:-1], full[1:-1, 1:-1, 1:-1])
    assert np.array_equal(p2[0], p[0]) and np.array_equal(p2[:, :, -1], p[:, :, -1])
