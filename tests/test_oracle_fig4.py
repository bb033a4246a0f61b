"""Pins for the Fig. 4 filtered statement chain (NEXT-3).

The filtered code must reproduce the sequential loop on every device's
owned blocks of a and b (partition property) even though a and b
are divided differently, must guard the read of c like the writes it feeds
(a NaN planted where no guarded k needs it never reaches an owned result),
and duplicates the a[i] store for i in b's range (the guard a U b)."""
import numpy as np
import pytest

import oracle as orc
import synth

U64MAX = 2**64 - 1


def _inputs(n, seed):
    Ma, Mb, Mc = 2 * n + 3, 3 * n + 1, 5 * n + 7
    # k = kx[i]: injective into [n, 2n) (race-free parallel loop)
    kx = (synth.permutation_i32(n, seed, 30) + n).astype(np.int32)
    jx = synth.index_i32(n, Mc, seed, 31)
    c = synth.uniform_f64(Mc, seed, 32)
    a0 = synth.uniform_f64(Ma, seed, 33)
    b0 = synth.uniform_f64(Mb, seed, 34)
    return jx, kx, c, a0, b0


def test_fig4_sequential_closed_form():
    n, x_in = 257, 0.625
    jx, kx, c, a0, b0 = _inputs(n, 1)
    a, b = a0.copy(), b0.copy()
    orc.fig4(jx, kx, c, x_in, a, b)
    ea, eb = a0.copy(), b0.copy()
    ea[:n] = x_in
    eb[:n] = x_in
    ea[kx] = c[jx]
    eb[kx] = c[jx]
    assert np.array_equal(a, ea) and np.array_equal(b, eb)


@pytest.mark.parametrize("n", [1, 7, 64, 257])
@pytest.mark.parametrize("nd", [1, 2, 3, 5, 8])
def test_fig4_filtered_partition_property(n, nd):
    x_in = -1.5
    jx, kx, c, a0, b0 = _inputs(n, 2 + n)
    a, b = a0.copy(), b0.copy()
    orc.fig4(jx, kx, c, x_in, a, b)
    oa, ob = np.full_like(a0, np.nan), np.full_like(b0, np.nan)
    for d in range(nd):
        alo, ahi = orc.partition(a0.size, nd, d)
        blo, bhi = orc.partition(b0.size, nd, d)
        da, db = np.full_like(a0, np.nan), np.full_like(b0, np.nan)
        (amn, amx), (bmn, bmx) = orc.fig4_filtered(jx, kx, c, x_in, da, db, (alo, ahi - 1), (blo, bhi - 1))
        # brute-force write logs
        wa, wb = np.flatnonzero(~np.isnan(da)), np.flatnonzero(~np.isnan(db))
        assert (amn, amx) == ((wa.min(), wa.max()) if wa.size else (U64MAX, 0))
        assert (bmn, bmx) == ((wb.min(), wb.max()) if wb.size else (U64MAX, 0))
        # b's writes stay inside b's bounds; a's may extend over b's (guard a U b)
        assert ((wb >= blo) & (wb < bhi)).all()
        inside = lambda w: ((w >= alo) & (w < ahi)) | ((w >= blo) & (w < bhi))
        assert inside(wa).all()
        oa[alo:ahi] = np.where(np.isnan(da[alo:ahi]), a0[alo:ahi], da[alo:ahi])
        ob[blo:bhi] = np.where(np.isnan(db[blo:bhi]), b0[blo:bhi], db[blo:bhi])
    assert np.array_equal(oa, a) and np.array_equal(ob, b)


@pytest.mark.parametrize("nd", [2, 4])
def test_fig4_guarded_read_of_c(nd):
    """x = (k in a U b ranges) ? c[j] : 0: plant NaN in every c[j] whose k
    is outside this device's guard; its owned results stay NaN-free."""
    n, x_in = 128, 2.0
    jx, kx, c, a0, b0 = _inputs(n, 9)
    for d in range(nd):
        alo, ahi = orc.partition(a0.size, nd, d)
        blo, bhi = orc.partition(b0.size, nd, d)
        need = ((kx >= alo) & (kx < ahi)) | ((kx >= blo) & (kx < bhi))
        cc = c.copy()
        cc[jx[~need]] = np.nan
        cc[jx[need]] = c[jx[need]]
        da, db = a0.copy(), b0.copy()
        orc.fig4_filtered(jx, kx, cc, x_in, da, db, (alo, ahi - 1), (blo, bhi - 1))
        assert not np.isnan(da[alo:ahi]).any() and not np.isnan(db[blo:bhi]).any()
