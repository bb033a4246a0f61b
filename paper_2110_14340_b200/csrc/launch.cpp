// launch.cpp -- one launch end to end: pulls, per-device kernels with fused write
//  tracking, merges, reduction combine (a3-a6, a8)
#include "rt.hpp"

namespace jrt {

// Feed completed adaptive observations (FIFO) to their controllers.  An
// observation made in a mode the controller has since left is dropped.
void poll_adaptive(bool block) {
    size_t done = 0;
    for (; done < R.adapt_pending.size(); done++) {
        AdaptRec &ar = R.adapt_pending[done];
        bool ready = true;
        for (auto &e : ar.ev) {
            if (block) {
                set_dev(e.dev);
                CK(cudaEventSynchronize(e.m1));
            } else {
                cudaError_t q = cudaEventQuery(e.m1);
                if (q == cudaErrorNotReady) {
                    ready = false;
                    break;
                }
                CK(q);
            }
        }
        if (!ready) break;
        double tk = 0, tc = 0;
        for (auto &e : ar.ev) {
            float k = 0, m = 0;
            CK(cudaEventElapsedTime(&k, e.k0, e.k1));
            CK(cudaEventElapsedTime(&m, e.k1, e.m1));
            tk = std::max(tk, (double)k * 1e-3);
            tc = std::max(tc, (double)m * 1e-3);
            R.evpool.push_back(e.k0);
            R.evpool.push_back(e.k1);
            R.evpool.push_back(e.m1);
        }
        AdaptiveCtl &c = R.adapt[ar.key];
        if (ar.dup == c.dup() && c.state != AdaptiveCtl::DUP_FINAL) {
            c.h_tk.push_back(tk);
            c.h_tc.push_back(tc);
            c.h_ws.push_back(ar.ws);
            c.h_state.push_back(c.state);
            c.observe(tk, tc, ar.ws, ar.n_dev, R.peak_p2p);
        }
    }
    R.adapt_pending.erase(R.adapt_pending.begin(), R.adapt_pending.begin() + done);
}

struct Pull {
    int dst, src;
    Region *reg;
    int64_t lo, hi;
};

jacc_status do_launch(int loop_id, const jacc_range *range, const jacc_arg *args, int nargs,
                      int async_id) {
    const Desc *D = find_desc(loop_id);
    if (!D) return JACC_ERR_UNKNOWN_LOOP;
    if (R.capturing) {
        if (D->reduction) return JACC_ERR_INVALID;  // obligatory host sync cannot be captured
        async_id = 0;
    }
    invalid_if(nargs != D->nargs || (nargs > 0 && !args));
    Launch L;
    L.D = D;
    L.a.resize(nargs);
    for (int k = 0; k < nargs; k++) {
        invalid_if(args[k].kind != D->kinds[k]);
        L.a[k].kind = args[k].kind;
        if (args[k].kind == JACC_ARG_REDUCE_SUM_F64) {
            invalid_if(!args[k].ptr);
            L.red_ptr = static_cast<double *>(args[k].ptr);
            continue;
        }
        if (args[k].kind == JACC_ARG_SCALAR_F64) {
            L.scalar = args[k].f64;
            continue;
        }
        Region *r = lookup(args[k].ptr);
        if (!r) throw Fail{JACC_ERR_NOT_PRESENT};
        invalid_if(r->elem != D->elems[k]);
        const uintptr_t boff = (uintptr_t)args[k].ptr - r->base;
        invalid_if(boff % r->elem != 0);
        L.a[k].reg = r;
        L.a[k].off = (int64_t)(boff / r->elem);
    }
    // ---- shapes and ranges -------------------------------------------------
    jacc_range rg;
    memset(&rg, 0, sizeof(rg));
    const int id = D->id;
    if (id == JACC_LOOP_JACOBI2D_F64) {
        Region *s = L.a[0].reg, *t = L.a[1].reg;
        invalid_if(s->ndims != 2 || t->ndims != 2 || L.a[0].off || L.a[1].off);
        invalid_if(s->ext[0] != s->ext[1] || t->ext[0] != s->ext[0] || t->ext[1] != s->ext[1]);
        invalid_if(s == t);  // in-place stencil: a race in OpenACC (R-12)
        L.N = s->ext[0];
        rg.ndims = 2;
        rg.lo[0] = rg.lo[1] = 1;
        rg.hi[0] = rg.hi[1] = L.N - 1;
        if (range) {
            invalid_if(range->ndims != 2);
            for (int k = 0; k < 2; k++) {
                invalid_if(range->lo[k] < 1 || range->hi[k] > L.N - 1);
                rg.lo[k] = range->lo[k];
                rg.hi[k] = std::max(range->lo[k], range->hi[k]);
            }
        }
    } else if (id == JACC_LOOP_HIMENO_F32 || id == JACC_LOOP_HIMENO_COPY_F32) {
        // p, wrk1, bnd, wrk2: [I][J][K]; a: [4][I][J][K]; b, c: [3][I][J][K]
        Region *P = L.a[0].reg;
        invalid_if(P->ndims != 3);
        L.HI = P->ext[0];
        L.HJ = P->ext[1];
        L.HK = P->ext[2];
        invalid_if(L.HI < 3 || L.HJ < 3 || L.HK < 3);
        for (int k = 0; k < nargs; k++) {
            if (!L.a[k].reg) continue;
            Region *r = L.a[k].reg;
            invalid_if(L.a[k].off != 0);
            int stack = 0;
            if (id == JACC_LOOP_HIMENO_F32) stack = k == 1 ? 4 : (k == 2 || k == 3) ? 3 : 0;
            if (stack) {
                invalid_if(r->ndims != 4 || r->ext[0] != stack || r->ext[1] != L.HI ||
                           r->ext[2] != L.HJ || r->ext[3] != L.HK);
            } else {
                invalid_if(r->ndims != 3 || r->ext[0] != L.HI || r->ext[1] != L.HJ ||
                           r->ext[2] != L.HK);
            }
        }
        const int out = D->out_arg;
        for (int k = 0; k < nargs; k++)  // written array must not alias an input (R-12)
            if (k != out && L.a[k].reg) invalid_if(L.a[k].reg == L.a[out].reg);
        rg.ndims = 3;
        rg.lo[0] = rg.lo[1] = rg.lo[2] = 1;
        rg.hi[0] = L.HI - 1;
        rg.hi[1] = L.HJ - 1;
        rg.hi[2] = L.HK - 1;
        if (range) {
            invalid_if(range->ndims != 3);
            const int64_t ex[3] = {L.HI, L.HJ, L.HK};
            for (int k = 0; k < 3; k++) {
                invalid_if(range->lo[k] < 1 || range->hi[k] > ex[k] - 1);
                rg.lo[k] = range->lo[k];
                rg.hi[k] = std::max(range->lo[k], range->hi[k]);
            }
        }
    } else if (id == JACC_LOOP_GEMM_F64) {
        Region *A = L.a[0].reg, *B = L.a[1].reg, *C = L.a[2].reg;
        invalid_if(A->ndims != 2 || B->ndims != 2 || C->ndims != 2);
        invalid_if(L.a[0].off || L.a[1].off || L.a[2].off);
        L.M = A->ext[0];
        L.K = A->ext[1];
        L.Nn = B->ext[1];
        invalid_if(B->ext[0] != L.K || C->ext[0] != L.M || C->ext[1] != L.Nn);
        invalid_if(C == A || C == B);  // in-place GEMM is a race (R-12)
        rg.ndims = 2;
        rg.lo[0] = rg.lo[1] = 0;
        rg.hi[0] = L.M;
        rg.hi[1] = L.Nn;
        if (range) {
            invalid_if(range->ndims != 2);
            invalid_if(range->lo[0] < 0 || range->hi[0] > L.M || range->lo[1] < 0 ||
                       range->hi[1] > L.Nn);
            for (int k = 0; k < 2; k++) {
                rg.lo[k] = range->lo[k];
                rg.hi[k] = std::max(range->lo[k], range->hi[k]);
            }
        }
    } else {
        // 1-D loops: range over i; arrays must hold [off+lo, off+hi)
        invalid_if(!range || range->ndims != 1 || range->lo[0] < 0 || range->hi[0] < range->lo[0]);
        rg.ndims = 1;
        rg.lo[0] = range->lo[0];
        rg.hi[0] = range->hi[0];
        for (int k = 0; k < nargs; k++) {
            if (!L.a[k].reg) continue;
            if (id == JACC_LOOP_SCATTER_ADD_F64 || id == JACC_LOOP_SCATTER_ADD_I32) {
                if (k == 2) continue;  // a is indexed by idx values
            }
            if (id == JACC_LOOP_FIG4_F64 && k >= 2) continue;  // c[j], a[i|k], b[i|k]
            invalid_if(L.a[k].off + rg.hi[0] > L.a[k].reg->nelem);
        }
        if (id == JACC_LOOP_SCATTER_ADD_F64 || id == JACC_LOOP_SCATTER_ADD_I32) {
            invalid_if(L.a[2].off != 0);
            invalid_if(L.a[2].reg == L.a[0].reg || L.a[2].reg == L.a[1].reg);  // race (R-12)
        }
        if (id == JACC_LOOP_FIG4_F64) {
            invalid_if(L.a[3].off != 0 || L.a[4].off != 0 || L.a[2].off != 0);
            invalid_if(rg.hi[0] > std::min(L.a[3].reg->nelem, L.a[4].reg->nelem));
            invalid_if(L.a[3].reg == L.a[4].reg);  // a and b distinct (R-12)
            for (int k = 0; k < 3; k++)
                invalid_if(L.a[k].reg == L.a[3].reg || L.a[k].reg == L.a[4].reg);
        }
        if (id == JACC_LOOP_SQUARE_F32 && L.a[0].reg == L.a[1].reg) {
            // two pointers to one array, one read and one written:
            // duplicate computation, no communication (R-12)
            L.dup = true;
        }
    }
    L.rg = rg;
    if (is_box_loop(id)) {
        L.split = R.split_dim < 0 ? 0 : R.split_dim;  // A18: built-in loops -> leftmost (dim 0)
        invalid_if(L.split >= L.a[D->out_arg].reg->ndims);
    }
    if (R.mode == JACC_MODE_DUP) L.dup = true;
    L.itersplit = R.scatter_itersplit && R.n > 1 &&
                  (id == JACC_LOOP_SCATTER_ADD_F64 || id == JACC_LOOP_SCATTER_ADD_I32);
    // iteration-split scatter allocates and zeroes its delta arrays on first
    // use, which a capture would only record, not run
    if (L.itersplit && (R.mp || R.nq > 1 || R.capturing)) return JACC_ERR_INVALID;
    // ---- NEXT-1 adaptive utilization (single process, n > 1) ---------------
    const bool adaptive =
        R.mode == JACC_MODE_ADAPTIVE && R.n > 1 && !R.mp && !L.dup && !R.capturing;
    std::string akey;
    double adapt_ws = 0;
    if (adaptive) {
        poll_adaptive(false);
        // kernel identity: loop, argument regions/offsets, iteration range
        akey.assign((const char *)&loop_id, sizeof(loop_id));
        for (auto &ai : L.a) {
            akey.append((const char *)&ai.reg, sizeof(ai.reg));
            akey.append((const char *)&ai.off, sizeof(ai.off));
        }
        akey.append((const char *)&L.rg.ndims, sizeof(L.rg.ndims));
        akey.append((const char *)L.rg.lo, sizeof(L.rg.lo));
        akey.append((const char *)L.rg.hi, sizeof(L.rg.hi));
        R.adapt_last_key[loop_id] = akey;
        // WriteSize: bytes the busiest device would send in a multi-GPU merge
        plan_launch(L);
        if (D->out_arg >= 0) {
            Region *Wr = L.a[D->out_arg].reg;
            for (int d = 0; d < R.n; d++) {
                const DevPlan &pp = L.plan[d];
                if (!pp.active) continue;
                double b;
                if (R.policy == JACC_MERGE_EAGER)
                    b = (double)(pp.whi - pp.wlo) * Wr->elem * (R.n - 1);
                else if (D->halo_rows > 0)
                    b = 2.0 * D->halo_rows * (double)(Wr->nelem / Wr->ext[0]) * Wr->elem;
                else
                    b = 0;
                adapt_ws = std::max(adapt_ws, b);
            }
        }
        L.dup = R.adapt[akey].dup();
    }
    // duplicated execution runs every iteration on every device: nothing to split
    if (L.dup) L.itersplit = false;
    for (auto &ai : L.a)
        if (ai.reg)
            for (int d = 0; d < R.n; d++)
                if (!ai.reg->rep[d]) return JACC_ERR_STATE;  // peer replica not imported yet
    plan_launch(L);

    const int n = R.n;
    const int out = D->out_arg;
    Region *W = out >= 0 ? L.a[out].reg : nullptr;
    Region *W2 = D->out2 >= 0 ? L.a[D->out2].reg : nullptr;  // second written array
    // elements of the write block the kernel may leave untouched must be
    // current on the owner before it is declared valid there (normally a
    // no-op: an owner is the only writer of its block)
    if (W && id != JACC_LOOP_SCATTER_ADD_F64 && id != JACC_LOOP_SCATTER_ADD_I32)
        for (int d = 0; d < n; d++)
            if (L.plan[d].active) {
                for (auto &iv : write_intervals(L.plan[d]))
                    L.plan[d].reads.push_back({W, iv.first, iv.second});
                if (W2) L.plan[d].reads.push_back({W2, L.plan[d].w2lo, L.plan[d].w2hi});
            }

    // ---- pulls: stale input intervals (validity tracker) -------------------
    std::vector<Pull> pulls;
    std::vector<std::vector<char>> comm(n, std::vector<char>(n, 0));
    for (int d = 0; d < n; d++) {
        for (const Foot &f : L.plan[d].reads) {
            for (auto &m : f.reg->valid[d].missing(f.lo, f.hi)) {
                int64_t a = m.first;
                while (a < m.second) {
                    int src = -1;
                    int64_t b = m.second;
                    for (int q = 0; q < n && src < 0; q++) {
                        if (q == d) continue;
                        auto &vi = f.reg->valid[q].iv;
                        auto it = vi.upper_bound(a);
                        if (it == vi.begin()) continue;
                        --it;
                        if (it->first <= a && it->second > a) {
                            src = q;
                            b = std::min(b, it->second);
                        }
                    }
                    if (src < 0) {
                        // never written anywhere valid (uninitialised data): nothing to pull
                        break;
                    }
                    pulls.push_back({d, src, f.reg, a, b});
                    comm[d][src] = comm[src][d] = 1;
                    a = b;
                }
            }
        }
    }

    // ---- merge pattern ------------------------------------------------------
    std::vector<int> top(n, -1), bot(n, -1);
    const bool writes = W && !L.dup;
    if (writes) {
        for (int d = 0; d < n; d++) {
            if (!L.plan[d].active) continue;
            if (R.policy == JACC_MERGE_EAGER) {
                for (int p = 0; p < n; p++)
                    if (p != d) comm[d][p] = comm[p][d] = 1;
            } else if (D->halo_rows > 0) {
                halo_targets(L, d, top[d], bot[d]);
                if (top[d] >= 0) comm[d][top[d]] = comm[top[d]][d] = 1;
                if (bot[d] >= 0) comm[d][bot[d]] = comm[bot[d]][d] = 1;
            }
        }
    }
    if (R.comm_prev.empty()) R.comm_prev.assign(n, std::vector<char>(n, 0));

    // ---- NEXT-4 automated async queues ---------------------------
    // The launch joins a queue chosen from its array dependencies and waits
    // (on every device) only for the other queues it depends on; the
    // per-generation comm waits are then subsumed by the array tracker.
    struct StreamSwap {
        std::vector<cudaStream_t> saved;
        std::vector<double *> partials, part, res;
        std::vector<unsigned *> ticket;
        ~StreamSwap() {
            for (size_t d = 0; d < saved.size(); d++)
                if (saved[d]) {
                    R.dev[d].s = saved[d];
                    R.dev[d].partials = partials[d];
                    R.dev[d].part = part[d];
                    R.dev[d].res = res[d];
                    R.dev[d].ticket = ticket[d];
                }
        }
    } swap;
    int qsel = 0;
    std::vector<int> waits;
    const bool multiq = R.nq > 1;
    if (multiq) {
        std::vector<int64_t> rd, wr;
        for (int k = 0; k < nargs; k++) {
            if (!L.a[k].reg) continue;
            const int64_t key = (int64_t)(uintptr_t)L.a[k].reg;
            if (L.a[k].kind == JACC_ARG_ARRAY_IN || L.a[k].kind == JACC_ARG_ARRAY_INOUT) rd.push_back(key);
            if (L.a[k].kind == JACC_ARG_ARRAY_OUT || L.a[k].kind == JACC_ARG_ARRAY_INOUT) wr.push_back(key);
        }
        qsel = R.sched.schedule(rd, wr, async_id >= 0 ? async_id % R.nq : -1, waits);
        swap.saved.assign(n, nullptr);
        swap.partials.assign(n, nullptr);
        swap.part.assign(n, nullptr);
        swap.res.assign(n, nullptr);
        swap.ticket.assign(n, nullptr);
        for (int d = 0; d < n; d++) {
            Device &dv = R.dev[d];
            swap.saved[d] = dv.s;
            swap.partials[d] = dv.partials;
            swap.part[d] = dv.part;
            swap.res[d] = dv.res;
            swap.ticket[d] = dv.ticket;
            dv.s = dv.qs[qsel];
            if (qsel > 0) {  // queue 0 keeps the device's own scratch
                dv.partials = dv.qpartials[qsel];
                dv.part = dv.qpart[qsel];
                dv.res = dv.qres[qsel];
                dv.ticket = dv.qticket[qsel];
            }
        }
        for (int pq : waits)
            for (int d = 0; d < n; d++) {
                set_dev(d);
                for (int d2 = 0; d2 < n; d2++) CK(cudaStreamWaitEvent(R.dev[d].s, R.dev[d2].qev[pq], 0));
            }
        // a same-queue dependency is stream order only on one device: queue
        // qsel on device d must also follow the previous launch of queue qsel
        // on every peer it may exchange with (pushes into, pulls from, or
        // whose pushes it reads)
        if (n > 1)
            for (int d = 0; d < n; d++) {
                set_dev(d);
                for (int d2 = 0; d2 < n; d2++)
                    if (d2 != d) CK(cudaStreamWaitEvent(R.dev[d].s, R.dev[d2].qev[qsel], 0));
            }
    }

    // ---- enqueue per device -------------------------------------------------
    if (R.prof.size() > 30000) flush_prof();
    R.last_start = R.prof.size();
    const int cur = R.gen & 1, prev = cur ^ 1;
    const bool prof = R.profiling && !R.capturing;
    uint64_t merged_bytes = 0;
    wait_launches(R.gen);
    std::vector<ProfRec> adapt_evs;
    if (W && (id == JACC_LOOP_SCATTER_ADD_F64 || id == JACC_LOOP_SCATTER_ADD_I32)) {
        const size_t words = (size_t)((W->nelem + 31) / 32);
        for (int d = 0; d < n; d++)
            if (local(d) && !W->bitmap[d]) {
                set_dev(d);
                CK(cudaMalloc(&W->bitmap[d], words * 4));
                CK(cudaMemsetAsync(W->bitmap[d], 0, words * 4, R.dev[d].s));
            }
    }
    // GEMM under EAGER: the merge is fused into the kernel's epilogue
    const bool gemm_fused_push = id == JACC_LOOP_GEMM_F64 && writes &&
                                 R.policy == JACC_MERGE_EAGER && n > 1 && L.split == 0;
    // binned-scatter scratch is reserved before anything is enqueued, so an
    // allocation failure cannot leave a launch half-issued (the loop then
    // falls back to the direct kernel on that device)
    if (W && !R.capturing && !L.itersplit && R.nq == 1 &&
        (id == JACC_LOOP_SCATTER_ADD_F64 || id == JACC_LOOP_SCATTER_ADD_I32)) {
        for (int d = 0; d < n; d++) {
            if (!local(d) || !L.plan[d].active) continue;
            const DevPlan &p = L.plan[d];
            const int64_t lo = L.dup ? 0 : p.own_lo, hi = L.dup ? W->nelem : p.own_hi;
            const jk::ScatterPlan sp = jk::scatter_plan(p.i1 - p.i0, lo, hi, (int)W->elem, W->nelem);
            if (!sp.binned) continue;
            Device &dv = R.dev[d];
            set_dev(d);
            if (dv.scratch_bytes < sp.scratch) {
                CK(cudaStreamSynchronize(dv.s));
                // a captured graph bakes in the scratch pointer: keep the old
                // buffer alive until no graph exists (jacc_graph_destroy)
                if (dv.scratch && !R.graphs.empty()) dv.retired.push_back(dv.scratch);
                else if (dv.scratch) CK(cudaFree(dv.scratch));
                dv.scratch = nullptr;
                dv.scratch_bytes = 0;
                if (cudaMalloc(&dv.scratch, sp.scratch) == cudaSuccess) dv.scratch_bytes = sp.scratch;
                else cudaGetLastError();
            }
        }
    }
    // ---- NEXT-3 phase 1: every device scatters its iteration block into its
    // delta array (after the usual waits and pulls) ---------------------------
    std::vector<char> waited(n, 0);
    if (L.itersplit) {
        const size_t words = (size_t)((W->nelem + 31) / 32);
        for (int d = 0; d < n; d++) {
            Device &dv = R.dev[d];
            const DevPlan &p = L.plan[d];
            set_dev(d);
            if (!W->delta[d]) {
                CK(cudaMalloc(&W->delta[d], W->bytes));
                CK(cudaMalloc(&W->dbm[d], words * 4));
                CK(cudaMemsetAsync(W->delta[d], 0, W->bytes, dv.s));
                CK(cudaMemsetAsync(W->dbm[d], 0, words * 4, dv.s));
            }
            // every peer: the previous launch's phase 2 on peer q read and
            // zeroed this device's delta over peer memory, and this phase 1
            // writes it again (WAR across devices, whatever the merge policy)
            for (int q = 0; q < n; q++)
                if (q != d) CK(cudaStreamWaitEvent(dv.s, R.dev[q].ev[prev], 0));
            for (const Pull &pl : pulls) {
                if (pl.dst != d) continue;
                const size_t e = pl.reg->elem;
                CK(cudaMemcpyAsync(pl.reg->rep[d] + pl.lo * e, pl.reg->rep[pl.src] + pl.lo * e,
                                   (size_t)(pl.hi - pl.lo) * e, cudaMemcpyDefault, dv.s));
                merged_bytes += (uint64_t)(pl.hi - pl.lo) * e;
            }
            waited[d] = 1;
            if (p.it1 > p.it0) {
                const int32_t *ix = reinterpret_cast<const int32_t *>(L.a[0].reg->rep[d]) + L.a[0].off + p.it0;
                const char *bsrc = L.a[1].reg->rep[d] + (L.a[1].off + p.it0) * (int64_t)W->elem;
                if (id == JACC_LOOP_SCATTER_ADD_F64)
                    CK(jk::scatter_add_f64(dv.s, ix, reinterpret_cast<const double *>(bsrc),
                                           reinterpret_cast<double *>(W->delta[d]), p.it1 - p.it0, 0,
                                           W->nelem, W->dbm[d], dv.scr_dirty));
                else
                    CK(jk::scatter_add_i32(dv.s, ix, reinterpret_cast<const int32_t *>(bsrc),
                                           reinterpret_cast<int32_t *>(W->delta[d]), p.it1 - p.it0, 0,
                                           W->nelem, W->dbm[d], dv.scr_dirty));
            }
            CK(cudaEventRecord(dv.pe, dv.s));
        }
    }
    for (int d = 0; d < n; d++) {
        if (!local(d)) continue;
        Device &dv = R.dev[d];
        const DevPlan &p = L.plan[d];
        set_dev(d);
        // (the first launch of a capture skips them: every earlier launch is
        // complete and its events live outside the graph)
        if (!(R.capturing && R.cap.launches == 0) && !waited[d] && !multiq)
            for (int q = 0; q < n; q++)
                if (q != d && (comm[d][q] || R.comm_prev[d][q]))
                    CK(cudaStreamWaitEvent(dv.s, R.dev[q].ev[prev], 0));
        for (const Pull &pl : pulls) {
            if (pl.dst != d || waited[d]) continue;
            const size_t e = pl.reg->elem;
            // UVA: peer device pointer or CUDA-IPC mapped peer replica
            CK(cudaMemcpyAsync(pl.reg->rep[d] + pl.lo * e, pl.reg->rep[pl.src] + pl.lo * e,
                               (size_t)(pl.hi - pl.lo) * e, cudaMemcpyDefault, dv.s));
            merged_bytes += (uint64_t)(pl.hi - pl.lo) * e;
        }
        ProfRec pr{d, nullptr, nullptr, nullptr};
        if (prof) {
            pr.k0 = pool_event();
            pr.k1 = pool_event();
            pr.m1 = pool_event();
            CK(cudaEventRecord(pr.k0, dv.s));
        }
        ProfRec ap{d, nullptr, nullptr, nullptr};
        if (adaptive) {
            ap.k0 = pool_event();
            ap.k1 = pool_event();
            ap.m1 = pool_event();
            CK(cudaEventRecord(ap.k0, dv.s));
        }
        u64 *drec = nullptr;  // this launch's dirty-record slot (cleared by the previous one)
        if (W) {
            W->dslot[d] ^= 1;
            drec = W->dirty[d] + 2 * W->dslot[d];
            // nothing will write it: clear both slots (the other one is the
            // next launch's, normally cleared by this launch's kernel)
            if (!p.active) CK(cudaMemsetAsync(W->dirty[d], 0xff, 32, dv.s));
        }
        u64 *drec2 = nullptr;
        if (W2) {
            W2->dslot[d] ^= 1;
            drec2 = W2->dirty[d] + 2 * W2->dslot[d];
            if (!p.active) CK(cudaMemsetAsync(W2->dirty[d], 0xff, 32, dv.s));
        }
        if (p.active) {
            switch (id) {
            case JACC_LOOP_SQUARE_F32: {
                const float *y = reinterpret_cast<const float *>(L.a[0].reg->rep[d]) + L.a[0].off;
                float *x = reinterpret_cast<float *>(L.a[1].reg->rep[d]) + L.a[1].off;
                CK(jk::square_f32(dv.s, y, x, p.i0, p.i1, L.a[1].off, drec));
                break;
            }
            case JACC_LOOP_JACOBI2D_F64: {
                // split dim 0: the boundary rows are pushed by the stencil kernel
                // itself; other split dims push boundary slabs after it
                double *pt = (L.split == 0 && top[d] >= 0) ? reinterpret_cast<double *>(W->rep[top[d]]) : nullptr;
                double *pb = (L.split == 0 && bot[d] >= 0) ? reinterpret_cast<double *>(W->rep[bot[d]]) : nullptr;
                CK(jk::jacobi2d(dv.s, reinterpret_cast<const double *>(L.a[0].reg->rep[d]),
                                reinterpret_cast<double *>(W->rep[d]), L.N, p.i0, p.i1, p.j0, p.j1,
                                drec, pt, pb));
                int64_t rowb = (p.j1 - p.j0) * 8;
                if (pt) merged_bytes += rowb;
                if (pb) merged_bytes += rowb;
                break;
            }
            case JACC_LOOP_DOT_F64:
            case JACC_LOOP_SUM_F64: {
                const double *x = reinterpret_cast<const double *>(L.a[0].reg->rep[d]) + L.a[0].off;
                const double *y = id == JACC_LOOP_DOT_F64
                                      ? reinterpret_cast<const double *>(L.a[1].reg->rep[d]) + L.a[1].off
                                      : nullptr;
                CK(jk::reduce_f64(dv.s, x + p.i0, y ? y + p.i0 : nullptr, p.i1 - p.i0, dv.partials,
                                  dv.ticket, dv.part));
                break;
            }
            case JACC_LOOP_GEMM_F64: {
                jk::PeerPtrs push{};
                if (gemm_fused_push)
                    for (int q = 0; q < n; q++)
                        if (q != d) push.p[push.n++] = W->rep[q];
                CK(jk::gemm_f64(dv.s, reinterpret_cast<const double *>(L.a[0].reg->rep[d]),
                                reinterpret_cast<const double *>(L.a[1].reg->rep[d]),
                                reinterpret_cast<double *>(W->rep[d]), L.M, L.Nn, L.K, p.i0, p.i1,
                                p.j0, p.j1, drec, push));
                if (gemm_fused_push) merged_bytes += (uint64_t)(p.whi - p.wlo) * 8 * (n - 1);
                break;
            }
            case JACC_LOOP_FIG4_F64: {
                const int32_t *jx = reinterpret_cast<const int32_t *>(L.a[0].reg->rep[d]) + L.a[0].off;
                const int32_t *kx = reinterpret_cast<const int32_t *>(L.a[1].reg->rep[d]) + L.a[1].off;
                CK(jk::fig4(dv.s, jx, kx, reinterpret_cast<const double *>(L.a[2].reg->rep[d]),
                            L.a[2].reg->nelem, L.scalar, reinterpret_cast<double *>(W->rep[d]),
                            reinterpret_cast<double *>(W2->rep[d]), W->nelem, p.i0, p.i1, p.own_lo,
                            p.own_hi, p.w2lo, p.w2hi, drec, drec2));
                break;
            }
            case JACC_LOOP_HIMENO_F32: {
                auto F = [&](int k) { return reinterpret_cast<const float *>(L.a[k].reg->rep[d]); };
                CK(jk::himeno_stencil(dv.s, F(0), F(1), F(2), F(3), F(4), F(5),
                                      reinterpret_cast<float *>(W->rep[d]), L.HI, L.HJ, L.HK, p.i0,
                                      p.i1, p.j0, p.j1, p.k0, p.k1, (float)L.scalar,
                                      dv.partials, dv.ticket, dv.part, drec));
                break;
            }
            case JACC_LOOP_HIMENO_COPY_F32: {
                float *pt = (L.split == 0 && top[d] >= 0) ? reinterpret_cast<float *>(W->rep[top[d]]) : nullptr;
                float *pb = (L.split == 0 && bot[d] >= 0) ? reinterpret_cast<float *>(W->rep[bot[d]]) : nullptr;
                CK(jk::himeno_copy(dv.s, reinterpret_cast<const float *>(L.a[0].reg->rep[d]),
                                   reinterpret_cast<float *>(W->rep[d]), L.HI, L.HJ, L.HK, p.i0, p.i1,
                                   p.j0, p.j1, p.k0, p.k1, drec, pt, pb, dv.ticket));
                const int64_t planeb = (p.j1 - p.j0) * (p.k1 - p.k0) * 4;
                if (pt) merged_bytes += planeb;
                if (pb) merged_bytes += planeb;
                break;
            }
            case JACC_LOOP_SCATTER_ADD_F64:
            case JACC_LOOP_SCATTER_ADD_I32: {
                if (L.itersplit) {
                    // phase 2: owner of the word-aligned slice adds every delta
                    for (int q = 0; q < n; q++)
                        if (q != d) CK(cudaStreamWaitEvent(dv.s, R.dev[q].pe, 0));
                    jk::PeerPtrs dl{}, db{};
                    for (int q = 0; q < n; q++) {
                        dl.p[dl.n++] = W->delta[q];
                        db.p[db.n++] = W->dbm[q];
                    }
                    const int64_t w0 = p.own_lo >> 5, w1 = (p.own_hi + 31) >> 5;
                    if (p.own_hi > p.own_lo)
                        CK(jk::scatter_combine(dv.s, id == JACC_LOOP_SCATTER_ADD_F64, W->rep[d],
                                               W->bitmap[d], dl, db, w0, w1, W->nelem, drec));
                    else
                        CK(cudaMemsetAsync(drec, 0xff, 16, dv.s));
                    merged_bytes += (uint64_t)(p.own_hi - p.own_lo) * W->elem * (n - 1);
                    break;
                }
                const int32_t *ix = reinterpret_cast<const int32_t *>(L.a[0].reg->rep[d]) + L.a[0].off + p.i0;
                uint32_t *bm = W->bitmap[d];
                {
                    const int64_t w0 = p.own_lo >> 5, w1 = (p.own_hi + 31) >> 5;
                    CK(cudaMemsetAsync(bm + w0, 0, (size_t)(w1 - w0) * 4, dv.s));
                }
                const bool f64 = id == JACC_LOOP_SCATTER_ADD_F64;
                const char *b = L.a[1].reg->rep[d] + (L.a[1].off + p.i0) * (int64_t)W->elem;
                const int64_t lo = L.dup ? 0 : p.own_lo, hi = L.dup ? W->nelem : p.own_hi;
                jk::ScatterPlan sp = jk::scatter_plan(p.i1 - p.i0, lo, hi, (int)W->elem, W->nelem);
                if (R.nq > 1) sp.binned = false;     // per-device scratch is not per queue
                if (sp.binned && dv.scratch_bytes < sp.scratch)
                    sp.binned = false;  // scratch could not be reserved up front: direct kernel
                if (sp.binned) {
                    CK(jk::scatter_add_binned(dv.s, f64, ix, b, W->rep[d], p.i1 - p.i0, lo, hi, bm,
                                              drec, sp, dv.scratch));
                } else if (f64) {
                    CK(jk::scatter_add_f64(dv.s, ix, reinterpret_cast<const double *>(b),
                                           reinterpret_cast<double *>(W->rep[d]), p.i1 - p.i0, lo,
                                           hi, bm, drec));
                } else {
                    CK(jk::scatter_add_i32(dv.s, ix, reinterpret_cast<const int32_t *>(b),
                                           reinterpret_cast<int32_t *>(W->rep[d]), p.i1 - p.i0, lo,
                                           hi, bm, drec));
                }
                break;
            }
            }
        } else if (D->reduction) {
            CK(cudaMemsetAsync(dv.part, 0, 8, dv.s));
        }
        if (prof) CK(cudaEventRecord(pr.k1, dv.s));
        if (adaptive) CK(cudaEventRecord(ap.k1, dv.s));
        const int nbox = (id == JACC_LOOP_JACOBI2D_F64 || id == JACC_LOOP_GEMM_F64) ? 2 : 3;
        // ---- HALO with a split dim > 0: push the boundary slabs (strided) --
        if (writes && p.active && R.policy == JACC_MERGE_HALO && L.split > 0 && D->halo_rows > 0) {
            for (int side = 0; side < 2; side++) {
                const int tgt = side == 0 ? top[d] : bot[d];
                if (tgt < 0) continue;
                int64_t lo[3], hi[3];
                slab_box(L, p, side == 0 ? p.blo[L.split] : p.bhi[L.split] - 1, lo, hi);
                jk::PeerPtrs pp{};
                pp.p[pp.n++] = W->rep[tgt];
                const jk::Box2D bx = make_box2d(W, nbox, lo, hi);
                CK(jk::merge_box(dv.s, W->rep[d], pp, bx, drec, (int64_t)W->elem));
                merged_bytes += (uint64_t)(bx.count * bx.height * bx.width);
            }
        }
        // ---- EAGER merge: push the recorded dirty region to every peer ----
        if (writes && p.active && R.policy == JACC_MERGE_EAGER && n > 1 && !gemm_fused_push) {
            jk::PeerPtrs pp{};
            for (int q = 0; q < n; q++)
                if (q != d) pp.p[pp.n++] = W->rep[q];
            if (is_box_loop(id) && L.split > 0) {
                const jk::Box2D bx = make_box2d(W, nbox, p.blo, p.bhi);
                CK(jk::merge_box(dv.s, W->rep[d], pp, bx, drec, (int64_t)W->elem));
            } else if (id == JACC_LOOP_SCATTER_ADD_F64 || id == JACC_LOOP_SCATTER_ADD_I32) {
                CK(jk::merge_bitmap(dv.s, W->rep[d], pp, W->bitmap[d], (int64_t)W->elem, p.wlo, p.whi));
            } else {
                CK(jk::merge_range(dv.s, W->rep[d], pp, drec, (int64_t)W->elem, p.wlo, p.whi));
            }
            merged_bytes += (uint64_t)(p.whi - p.wlo) * W->elem * (n - 1);  // upper bound (host view)
            if (W2) {  // second written array: its own block, its own dirty record
                jk::PeerPtrs p2{};
                for (int q = 0; q < n; q++)
                    if (q != d) p2.p[p2.n++] = W2->rep[q];
                CK(jk::merge_range(dv.s, W2->rep[d], p2, drec2, (int64_t)W2->elem, p.w2lo, p.w2hi));
                merged_bytes += (uint64_t)(p.w2hi - p.w2lo) * W2->elem * (n - 1);
            }
        }
        if (prof) {
            CK(cudaEventRecord(pr.m1, dv.s));
            R.prof.push_back(pr);
        }
        if (adaptive) {
            CK(cudaEventRecord(ap.m1, dv.s));
            adapt_evs.push_back(ap);
        }
        CK(cudaEventRecord(dv.ev[cur], dv.s));
        dv.launches++;
    }
    if (R.mp) shm_store(&R.shm[R.me].launches, R.gen + 1);
    if (multiq)
        for (int d = 0; d < n; d++) {
            set_dev(d);
            CK(cudaEventRecord(R.dev[d].qev[qsel], R.dev[d].s));
        }
    if (adaptive) R.adapt_pending.push_back({akey, n, L.dup, adapt_ws, adapt_evs});

    // ---- validity bookkeeping ---------------------------------------------
    for (const Pull &pl : pulls) pl.reg->valid[pl.dst].add(pl.lo, pl.hi);
    if (W && L.dup) {
        // duplicated: every device computed (after pulling) the whole block
        for (int d = 0; d < n; d++)
            if (L.plan[d].active)
                for (auto &iv : write_intervals(L.plan[d])) W->valid[d].add(iv.first, iv.second);
    }
    if (writes && W2) {
        for (int d = 0; d < n; d++) {
            const DevPlan &p = L.plan[d];
            if (!p.active) continue;
            W2->valid[d].add(p.w2lo, p.w2hi);
            if (R.policy == JACC_MERGE_EAGER) continue;
            for (int q = 0; q < n; q++)
                if (q != d) W2->valid[q].remove(p.w2lo, p.w2hi);
        }
    }
    if (W2 && L.dup)
        for (int d = 0; d < n; d++)
            if (L.plan[d].active) W2->valid[d].add(L.plan[d].w2lo, L.plan[d].w2hi);
    if (writes) {
        for (int d = 0; d < n; d++) {
            const DevPlan &p = L.plan[d];
            if (!p.active) continue;
            const auto wiv = write_intervals(p);
            for (auto &iv : wiv) W->valid[d].add(iv.first, iv.second);
            if (R.policy == JACC_MERGE_EAGER) continue;  // every peer received the dirty set
            for (int q = 0; q < n; q++) {
                if (q == d) continue;
                // q keeps validity only on the rows / slabs pushed to it (HALO)
                std::vector<std::pair<int64_t, int64_t>> keep;
                if (D->halo_rows > 0 && L.split == 0) {
                    const int64_t unit = W->nelem / W->ext[0];  // elements per split index
                    if (top[d] == q) keep.push_back({p.i0 * unit, (p.i0 + 1) * unit});
                    if (bot[d] == q) keep.push_back({(p.i1 - 1) * unit, p.i1 * unit});
                } else if (D->halo_rows > 0) {
                    const int nb = (id == JACC_LOOP_JACOBI2D_F64) ? 2 : 3;
                    for (int side = 0; side < 2; side++) {
                        if ((side == 0 ? top[d] : bot[d]) != q) continue;
                        int64_t lo[3], hi[3];
                        slab_box(L, p, side == 0 ? p.blo[L.split] : p.bhi[L.split] - 1, lo, hi);
                        box_intervals(nb, W->ext + (W->ndims - nb), lo, hi, 0, keep);
                    }
                }
                std::vector<std::pair<int64_t, int64_t>> had;
                for (auto &k : keep) {
                    // only what q already had valid stays valid
                    IntervalSet tmp;
                    tmp.add(k.first, k.second);
                    for (auto &m : W->valid[q].missing(k.first, k.second)) tmp.remove(m.first, m.second);
                    for (auto &iv : tmp.iv) had.push_back(iv);
                }
                for (auto &iv : wiv) W->valid[q].remove(iv.first, iv.second);
                for (auto &h : had) W->valid[q].add(h.first, h.second);
            }
        }
    }
    if (prof) {
        TraceRec tr{R.trace_events++, loop_id, D->name, qsel, waits, {}, L.dup, R.policy, merged_bytes,
                    R.last_start, R.prof.size()};
        for (int q = 0; q < n; q++)
            if (!multiq && (comm[R.mp ? R.me : 0][q] || R.comm_prev[R.mp ? R.me : 0][q]) && q != (R.mp ? R.me : 0))
                tr.peers.push_back(q);
        R.trace_pending.push_back(std::move(tr));
    }
    R.dev[R.mp ? R.me : 0].bytes_merged += merged_bytes;
    R.last_bytes = merged_bytes;
    R.comm_prev = comm;
    R.gen++;
    if (R.capturing) R.cap.launches++;

    // ---- reduction combine (obligatory sync) -------------------
    if (D->reduction) {
        // the device that finishes the combine: device 0, or this rank's own
        const int h = R.mp ? R.me : 0;
        Device &d0 = R.dev[h];
        const double s_in = *L.red_ptr;
        if (L.dup) {
            // duplicated execution: every device reduced the whole range, so
            // the result is this device's own total (no cross-device sum)
            set_dev(h);
            jk::PeerPtrs pp{};
            pp.p[pp.n++] = d0.part;
            CK(jk::combine(d0.s, pp, s_in, d0.res));
        } else if (R.use_nccl) {
            NK(ncclGroupStart());
            for (int d = 0; d < n; d++)
                if (local(d))
                    NK(ncclAllReduce(R.dev[d].part, R.dev[d].res, 1, ncclDouble, ncclSum,
                                     R.dev[d].comm, R.dev[d].s));
            NK(ncclGroupEnd());
            set_dev(h);
            jk::PeerPtrs pp{};
            pp.p[0] = d0.res;
            pp.n = 1;
            CK(jk::combine(d0.s, pp, s_in, d0.res));
        } else {
            // virtual devices / no NCCL: fixed-order sum of the partials read
            // over peer memory (same GPU, P2P or CUDA-IPC mapped)
            wait_launches(R.gen);
            set_dev(h);
            for (int d = 0; d < n; d++)
                if (d != h) CK(cudaStreamWaitEvent(d0.s, R.dev[d].ev[cur], 0));
            jk::PeerPtrs pp{};
            for (int d = 0; d < n; d++) pp.p[pp.n++] = R.dev[d].part;
            CK(jk::combine(d0.s, pp, s_in, d0.res));
        }
        CK(cudaMemcpyAsync(d0.hscal, d0.res, 8, cudaMemcpyDeviceToHost, d0.s));
        CK(cudaStreamSynchronize(d0.s));
        *L.red_ptr = *d0.hscal;
        // peers read this rank's partial: nobody overwrites it before all
        // combines are done
        if (R.mp && !R.use_nccl) rank_barrier();
    }
    if (async_id == -1) sync_all();  // JACC_ASYNC_AUTO (-2) and queues >= 0 stay async
    return JACC_OK;
}


}  // namespace jrt

using namespace jrt;

extern "C" {

jacc_status jacc_launch(int loop_id, const jacc_range *range, const jacc_arg *args, int nargs,
                        int async_id) {
    const Desc *D = find_desc(loop_id);
    nvtxRangePushA(D ? D->name : "jacc_launch");  // NVTX range per launch (host issue)
    const jacc_status st = guard([&]() { return do_launch(loop_id, range, args, nargs, async_id); });
    nvtxRangePop();
    return st;
}

jacc_status jacc_wait(int async_id) {
    return guard([&]() -> jacc_status {
        if (R.capturing) return JACC_ERR_STATE;
        if (R.nq > 1 && async_id >= 0) {  // one queue, on every device
            for (int d = 0; d < R.n; d++) {
                set_dev(d);
                CK(cudaStreamSynchronize(R.dev[d].qs[async_id % R.nq]));
            }
            return JACC_OK;
        }
        sync_all();
        return JACC_OK;
    });
}


}  // extern "C"
