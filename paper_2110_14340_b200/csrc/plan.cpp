// plan.cpp -- launch planning: owned blocks, clipped iteration boxes, write sets and read
//  footprints (a3)
#include "rt.hpp"

namespace jrt {

// Element intervals of the box [lo, hi) (per dim) of a row-major array with
// extents ext[0..nd); dims fully covered at the tail collapse into one
// contiguous run, so a box of whole rows / planes is a single interval.
void box_intervals(int nd, const int64_t *ext, const int64_t *lo, const int64_t *hi, int64_t base,
                   std::vector<std::pair<int64_t, int64_t>> &out) {
    for (int k = 0; k < nd; k++)
        if (hi[k] <= lo[k]) return;
    // t = first dim from which the box is contiguous
    int t = nd - 1;
    while (t > 0 && lo[t] == 0 && hi[t] == ext[t]) t--;
    int64_t inner = 1;
    for (int k = t + 1; k < nd; k++) inner *= ext[k];
    int64_t idx[8];
    for (int k = 0; k < t; k++) idx[k] = lo[k];
    for (;;) {
        int64_t f = 0;
        for (int k = 0; k < t; k++) f = f * ext[k] + idx[k];
        f = f * ext[t];
        const int64_t a = base + (f + lo[t]) * inner, b = base + (f + hi[t]) * inner;
        if (!out.empty() && out.back().second == a) out.back().second = b;
        else out.push_back({a, b});
        int k = t - 1;
        for (; k >= 0; k--) {
            if (++idx[k] < hi[k]) break;
            idx[k] = lo[k];
        }
        if (k < 0) break;
    }
}

// Footprint of a box on array r (its last nd dims), widened to the full
// extent in every dimension after the split dimension: a conservative
// superset (pulls of stale-but-unread elements are harmless) that keeps the
// interval count at one per split-dimension row instead of one per row of
// the box (a 1025x513x513 interior box would otherwise be 5e5 intervals).
void push_box(std::vector<Foot> &reads, Region *r, int nd, const int64_t *lo, const int64_t *hi,
              int64_t base = 0, int split = 0) {
    std::vector<std::pair<int64_t, int64_t>> iv;
    int64_t l[4], h[4];
    for (int k = 0; k < nd; k++) {  // clamp to the array, widen after the split dim
        const int64_t e = r->ext[r->ndims - nd + k];
        l[k] = k > split ? 0 : std::max<int64_t>(lo[k], 0);
        h[k] = k > split ? e : std::min<int64_t>(hi[k], e);
    }
    box_intervals(nd, r->ext + (r->ndims - nd), l, h, base, iv);
    for (auto &x : iv) reads.push_back({r, x.first, x.second});
}

// Box loops (Jacobi, GEMM, Himeno): the written array's split dimension
// L.split is divided equally; the iteration box is clipped to the
// owned block along it.  Write set = the clipped box; read footprints are
// boxes of the inputs (stencil halos included).
void plan_box(Launch &L, int d, int nd, int dd, DevPlan &p) {
    (void)d;
    const int id = L.D->id;
    Region *Wr = L.a[L.D->out_arg].reg;
    const int s = L.split;
    const int nb = (id == JACC_LOOP_JACOBI2D_F64 || id == JACC_LOOP_GEMM_F64) ? 2 : 3;
    int64_t lo[3], hi[3];
    for (int k = 0; k < nb; k++) {
        lo[k] = L.rg.lo[k];
        hi[k] = L.rg.hi[k];
    }
    partition(Wr->ext[s], nd, dd, p.own_lo, p.own_hi);
    lo[s] = std::max(lo[s], p.own_lo);
    hi[s] = std::min(hi[s], p.own_hi);
    p.active = true;
    for (int k = 0; k < nb; k++) {
        p.blo[k] = lo[k];
        p.bhi[k] = hi[k];
        if (hi[k] <= lo[k]) p.active = false;
    }
    p.i0 = lo[0];
    p.i1 = hi[0];
    p.j0 = lo[1];
    p.j1 = hi[1];
    if (nb == 3) {
        p.k0 = lo[2];
        p.k1 = hi[2];
    }
    if (!p.active) return;
    const int64_t *ext = Wr->ext;
    if (s == 0) {  // contiguous block: one span (its unwritten elements are owner-valid)
        int64_t f0 = 0, f1 = 0;
        for (int k = 0; k < nb; k++) {
            f0 = f0 * ext[k] + lo[k];
            f1 = f1 * ext[k] + (hi[k] - 1);
        }
        p.wlo = f0;
        p.whi = f1 + 1;
    } else {
        // superset write set for the tracker: full extent after the split
        // dim (those elements are unchanged, so owner-valid; see push_box)
        int64_t wl[3], wh[3];
        for (int k = 0; k < nb; k++) {
            wl[k] = k > s ? 0 : lo[k];
            wh[k] = k > s ? ext[k] : hi[k];
        }
        box_intervals(nb, ext, wl, wh, 0, p.wbox);
        p.wlo = p.wbox.front().first;
        p.whi = p.wbox.back().second;
    }
    if (id == JACC_LOOP_JACOBI2D_F64) {
        const int64_t rl[2] = {lo[0] - 1, lo[1] - 1}, rh[2] = {hi[0] + 1, hi[1] + 1};
        push_box(p.reads, L.a[0].reg, 2, rl, rh, 0, s);
    } else if (id == JACC_LOOP_GEMM_F64) {
        const int64_t al[2] = {lo[0], 0}, ah[2] = {hi[0], L.K};
        const int64_t bl[2] = {0, lo[1]}, bh[2] = {L.K, hi[1]};
        push_box(p.reads, L.a[0].reg, 2, al, ah, 0, s);
        push_box(p.reads, L.a[1].reg, 2, bl, bh, 0, s);
    } else if (id == JACC_LOOP_HIMENO_F32) {
        const int64_t pl[3] = {lo[0] - 1, lo[1] - 1, lo[2] - 1}, ph[3] = {hi[0] + 1, hi[1] + 1, hi[2] + 1};
        push_box(p.reads, L.a[0].reg, 3, pl, ph, 0, s);
        const int stacks[6] = {1, 4, 3, 3, 1, 1};
        const int64_t V = L.HI * L.HJ * L.HK;
        for (int k = 1; k < 6; k++)
            for (int m = 0; m < stacks[k]; m++)
                push_box(p.reads, L.a[k].reg, 3, lo, hi, m * V, s);
    } else {  // himeno copy
        push_box(p.reads, L.a[0].reg, 3, lo, hi, 0, s);
    }
}

bool is_box_loop(int id) {
    return id == JACC_LOOP_JACOBI2D_F64 || id == JACC_LOOP_GEMM_F64 || id == JACC_LOOP_HIMENO_F32 ||
           id == JACC_LOOP_HIMENO_COPY_F32;
}

// exact write intervals of a device plan
std::vector<std::pair<int64_t, int64_t>> write_intervals(const DevPlan &p) {
    if (!p.wbox.empty()) return p.wbox;
    return {{p.wlo, p.whi}};
}

// the boundary slab of d's write box at index x along split dim s
void slab_box(const Launch &L, const DevPlan &p, int64_t x, int64_t *lo, int64_t *hi) {
    for (int k = 0; k < 3; k++) {
        lo[k] = p.blo[k];
        hi[k] = p.bhi[k];
    }
    lo[L.split] = x;
    hi[L.split] = x + 1;
}

jk::Box2D make_box2d(const Region *r, int nb, const int64_t *lo, const int64_t *hi) {
    const int64_t *e = r->ext + (r->ndims - nb);
    const int64_t el = (int64_t)r->elem;
    jk::Box2D b{};
    if (nb == 2) {
        b.count = 1;
        b.height = hi[0] - lo[0];
        b.width = (hi[1] - lo[1]) * el;
        b.pitch = e[1] * el;
        b.first = (lo[0] * e[1] + lo[1]) * el;
        b.outer = 0;
    } else {
        b.count = hi[0] - lo[0];
        b.height = hi[1] - lo[1];
        b.width = (hi[2] - lo[2]) * el;
        b.pitch = e[2] * el;
        b.first = ((lo[0] * e[1] + lo[1]) * e[2] + lo[2]) * el;
        b.outer = e[1] * e[2] * el;
    }
    return b;
}

void plan_launch(Launch &L) {
    const int n = R.n;
    L.plan.assign(n, DevPlan{});
    const int id = L.D->id;
    for (int d = 0; d < n; d++) {
        DevPlan &p = L.plan[d];
        const int nd = L.dup ? 1 : n, dd = L.dup ? 0 : d;
        if (id == JACC_LOOP_SQUARE_F32) {
            // x written: split x's dim 0 (its whole region extent)
            Region *xr = L.a[1].reg;
            partition(xr->nelem, nd, dd, p.own_lo, p.own_hi);
            const int64_t xo = L.a[1].off;
            p.i0 = std::max(L.rg.lo[0], p.own_lo - xo);
            p.i1 = std::min(L.rg.hi[0], p.own_hi - xo);
            p.active = p.i1 > p.i0;
            if (p.active) {
                p.wlo = xo + p.i0;
                p.whi = xo + p.i1;
                p.reads.push_back({L.a[0].reg, L.a[0].off + p.i0, L.a[0].off + p.i1});
            }
        } else if (id == JACC_LOOP_JACOBI2D_F64) {
            plan_box(L, d, nd, dd, p);
        } else if (id == JACC_LOOP_DOT_F64 || id == JACC_LOOP_SUM_F64) {
            // reductions: filter by the outermost parallel iterator
            int64_t lo, hi;
            partition(L.rg.hi[0] - L.rg.lo[0], nd, dd, lo, hi);
            p.i0 = L.rg.lo[0] + lo;
            p.i1 = L.rg.lo[0] + hi;
            p.active = p.i1 > p.i0;
            const int narr = id == JACC_LOOP_DOT_F64 ? 2 : 1;
            if (p.active)
                for (int k = 0; k < narr; k++)
                    p.reads.push_back({L.a[k].reg, L.a[k].off + p.i0, L.a[k].off + p.i1});
        } else if (id == JACC_LOOP_GEMM_F64 || id == JACC_LOOP_HIMENO_F32 ||
                   id == JACC_LOOP_HIMENO_COPY_F32) {
            plan_box(L, d, nd, dd, p);
        } else if (id == JACC_LOOP_FIG4_F64) {
            // NEXT-3 Fig. 4: every device runs all iterations; stores are
            // guarded by the owned blocks of a and of b
            Region *ar = L.a[3].reg, *br = L.a[4].reg;
            partition(ar->nelem, nd, dd, p.own_lo, p.own_hi);
            partition(br->nelem, nd, dd, p.w2lo, p.w2hi);
            p.i0 = L.rg.lo[0];
            p.i1 = L.rg.hi[0];
            p.wlo = p.own_lo;
            p.whi = p.own_hi;
            p.active = p.i1 > p.i0;
            if (p.active) {
                for (int k = 0; k < 2; k++)
                    p.reads.push_back({L.a[k].reg, L.a[k].off + p.i0, L.a[k].off + p.i1});
                p.reads.push_back({L.a[2].reg, 0, L.a[2].reg->nelem});  // c[j]: any j
            }
        } else if (L.itersplit) {
            // NEXT-3: iterations split in blocks; a divided in word-aligned
            // owner slices, each owner adds every device's delta
            Region *ar = L.a[2].reg;
            int64_t w0, w1, b0, b1;
            partition((ar->nelem + 31) / 32, nd, dd, w0, w1);
            p.own_lo = std::min<int64_t>(32 * w0, ar->nelem);
            p.own_hi = std::min<int64_t>(32 * w1, ar->nelem);
            partition(L.rg.hi[0] - L.rg.lo[0], nd, dd, b0, b1);
            p.it0 = L.rg.lo[0] + b0;
            p.it1 = L.rg.lo[0] + b1;
            p.i0 = p.it0;
            p.i1 = p.it1;
            p.active = p.own_hi > p.own_lo || p.it1 > p.it0;
            p.wlo = p.own_lo;
            p.whi = p.own_hi;
            if (p.it1 > p.it0) {
                p.reads.push_back({L.a[0].reg, L.a[0].off + p.it0, L.a[0].off + p.it1});
                p.reads.push_back({L.a[1].reg, L.a[1].off + p.it0, L.a[1].off + p.it1});
            }
            if (p.own_hi > p.own_lo) p.reads.push_back({ar, p.own_lo, p.own_hi});
        } else {  // scatter: owned slice of a; every device scans all i
            Region *ar = L.a[2].reg;
            partition(ar->nelem, nd, dd, p.own_lo, p.own_hi);
            p.i0 = L.rg.lo[0];
            p.i1 = L.rg.hi[0];
            p.active = p.i1 > p.i0 && p.own_hi > p.own_lo;
            if (p.active) {
                p.wlo = p.own_lo;
                p.whi = p.own_hi;
                p.reads.push_back({L.a[0].reg, L.a[0].off + p.i0, L.a[0].off + p.i1});
                p.reads.push_back({L.a[1].reg, L.a[1].off + p.i0, L.a[1].off + p.i1});
                p.reads.push_back({ar, p.own_lo, p.own_hi});
            }
        }
    }
}

// HALO: which rows of device d's written block do neighbour p's next
// footprint (its written rows +- halo radius) cover?  Returns the push
// targets for the first and last written row (Jacobi).
void halo_targets(const Launch &L, int d, int &top, int &bot) {
    top = bot = -1;
    const DevPlan &me = L.plan[d];
    if (!me.active) return;
    const int s = L.split;
    for (int p = 0; p < R.n; p++) {
        if (p == d || !L.plan[p].active) continue;
        const int64_t flo = L.plan[p].blo[s] - L.D->halo_rows, fhi = L.plan[p].bhi[s] + L.D->halo_rows;
        if (me.blo[s] >= flo && me.blo[s] < fhi) top = p;
        if (me.bhi[s] - 1 >= flo && me.bhi[s] - 1 < fhi) bot = p;
    }
}


}  // namespace jrt
