// abi.cpp -- C-ABI: init/finalize, settings, present table, host transfers,
//  introspection, profiling, error strings (a1, a2, a7)
#include "rt.hpp"

using namespace jrt;

extern "C" {


jacc_status jacc_init(int n_devices, const int *device_ids) {
    if (R.init) return JACC_ERR_STATE;
    return guard(
        [&]() -> jacc_status {
            int count = 0;
            if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1) return JACC_ERR_CUDA;
            if (n_devices < 1 || n_devices > JACC_MAX_DEVICES) return JACC_ERR_INVALID;
            std::vector<int> ords(n_devices);
            for (int d = 0; d < n_devices; d++) {
                ords[d] = device_ids ? device_ids[d] : d;
                if (ords[d] < 0 || ords[d] >= count) return JACC_ERR_INVALID;
            }
            R = Runtime{};
            R.n = n_devices;
            R.dev.resize(n_devices);
            for (int d = 0; d < n_devices; d++)
                for (int q = 0; q < d; q++)
                    if (ords[q] == ords[d]) R.distinct = false;
            const char *pol = getenv("JACC_MERGE");
            if (pol && !strcmp(pol, "halo")) R.policy = JACC_MERGE_HALO;
            if (const char *pk = getenv("JACC_PEAK_P2P_GBS")) R.peak_p2p = atof(pk) * 1e9;
            R.init = true;
            for (int d = 0; d < n_devices; d++) {
                Device &dv = R.dev[d];
                dv.ord = ords[d];
                set_dev(d);
                CK(cudaStreamCreateWithFlags(&dv.s, cudaStreamNonBlocking));
                CK(cudaEventCreateWithFlags(&dv.ev[0], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&dv.ev[1], cudaEventDisableTiming));
                CK(cudaEventRecord(dv.ev[0], dv.s));
                CK(cudaEventRecord(dv.ev[1], dv.s));
                CK(cudaMalloc(&dv.partials, jk::kHimenoPartials * sizeof(double)));
                CK(cudaMalloc(&dv.ticket, 64));
                CK(cudaMemset(dv.ticket, 0, 64));
                CK(cudaMalloc(&dv.part, 8));
                CK(cudaMalloc(&dv.res, 8));
                CK(cudaMemset(dv.part, 0, 8));
                CK(cudaMallocHost(&dv.hscal, 8));
                CK(cudaEventCreateWithFlags(&dv.pe, cudaEventDisableTiming));
                CK(cudaMalloc(&dv.scr_dirty, 32));
                CK(cudaMemset(dv.scr_dirty, 0xff, 32));
            }
            // peer access between distinct GPUs (NVLink / NVSwitch P2P)
            for (int d = 0; d < n_devices; d++)
                for (int q = 0; q < n_devices; q++) {
                    if (ords[d] == ords[q]) continue;
                    int ok = 0;
                    CK(cudaDeviceCanAccessPeer(&ok, ords[d], ords[q]));
                    if (!ok) {
                        R.poisoned = true;
                        return JACC_ERR_INVALID;
                    }
                    set_dev(d);
                    cudaError_t e = cudaDeviceEnablePeerAccess(ords[q], 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else CK(e);
                    R.peer_pairs++;
                }
            // JACC_FORCE_NCCL=1 builds the communicator for a single device too:
            // the NCCL combine path then runs on a one-GPU box (tests)
            if ((n_devices > 1 || getenv("JACC_FORCE_NCCL")) && R.distinct && !getenv("JACC_NO_NCCL")) {
                // NCCL allreduce for the reduction combine.  A
                // communicator that cannot be built is an error, not a silent
                // switch to the peer-memory combine (JACC_NO_NCCL=1 selects
                // that one explicitly)
                std::vector<ncclComm_t> comms(n_devices);
                const ncclResult_t nr = ncclCommInitAll(comms.data(), n_devices, ords.data());
                if (nr != ncclSuccess) {
                    fprintf(stderr, "[jacc] ncclCommInitAll: %s (set JACC_NO_NCCL=1 for the "
                            "peer-memory combine)\n", ncclGetErrorString(nr));
                    jacc_finalize();
                    return JACC_ERR_NCCL;
                }
                for (int d = 0; d < n_devices; d++) R.dev[d].comm = comms[d];
                R.use_nccl = true;
            }
            R.comm_prev.assign(n_devices, std::vector<char>(n_devices, 0));
            return JACC_OK;
        },
        false);
}

jacc_status jacc_finalize(void) {
    if (!R.init) return JACC_ERR_STATE;
    for (int d = 0; d < R.n; d++) {
        if (!local(d)) continue;
        cudaSetDevice(R.dev[d].ord);
        cudaStreamSynchronize(R.dev[d].s);
    }
    if (R.mp && !R.poisoned) {
        try {
            rank_barrier();  // no peer still reads or writes our memory
        } catch (Fail &) {
        }
    }
    if (R.capturing) {
        cudaGraph_t g = nullptr;
        cudaSetDevice(R.dev[0].ord);
        cudaStreamEndCapture(R.dev[0].s, &g);
        if (g) cudaGraphDestroy(g);
        R.capturing = false;
    }
    for (auto &g : R.graphs) destroy_graph(g.second);
    R.graphs.clear();
    for (auto &kv : R.table) free_region(kv.second.get());
    R.table.clear();
    if (!R.poisoned) {
        try {
            flush_prof();
        } catch (Fail &) {
        }
    }
    close_trace();
    for (auto &p : R.prof) {
        R.evpool.push_back(p.k0);
        R.evpool.push_back(p.k1);
        R.evpool.push_back(p.m1);
    }
    for (auto &ar : R.adapt_pending)
        for (auto &e : ar.ev) {
            R.evpool.push_back(e.k0);
            R.evpool.push_back(e.k1);
            R.evpool.push_back(e.m1);
        }
    for (auto e : R.evpool) cudaEventDestroy(e);
    for (int d = 0; d < R.n; d++) {
        Device &dv = R.dev[d];
        if (!local(d)) {
            if (dv.ev[0]) cudaEventDestroy(dv.ev[0]);
            if (dv.ev[1]) cudaEventDestroy(dv.ev[1]);
            if (dv.part) cudaIpcCloseMemHandle(dv.part);
            continue;
        }
        cudaSetDevice(dv.ord);
        if (dv.comm) ncclCommDestroy(dv.comm);
        if (dv.scratch) cudaFree(dv.scratch);
        for (void *p : dv.retired) cudaFree(p);
        dv.retired.clear();
        if (dv.pe) cudaEventDestroy(dv.pe);
        for (size_t q = 1; q < dv.qs.size(); q++) cudaStreamDestroy(dv.qs[q]);
        for (size_t q = 1; q < dv.qpartials.size(); q++) {
            cudaFree(dv.qpartials[q]);
            cudaFree(dv.qpart[q]);
            cudaFree(dv.qres[q]);
            cudaFree(dv.qticket[q]);
        }
        for (auto e : dv.qev) cudaEventDestroy(e);
        if (dv.scr_dirty) cudaFree(dv.scr_dirty);
        cudaFree(dv.partials);
        cudaFree(dv.ticket);
        cudaFree(dv.part);
        cudaFree(dv.res);
        cudaFreeHost(dv.hscal);
        cudaEventDestroy(dv.ev[0]);
        cudaEventDestroy(dv.ev[1]);
        cudaStreamDestroy(dv.s);
    }
    cudaGetLastError();
    if (R.shm) {
        munmap(R.shm, sizeof(Runtime::Slot) * JACC_MAX_DEVICES);
        if (R.me == 0) shm_unlink(R.shm_name.c_str());
    }
    R = Runtime{};
    return JACC_OK;
}

int jacc_num_devices(void) { return R.init ? R.n : 0; }

jacc_status jacc_select_split_dim(int ndims, const int *n_parallel, const int *n_sequential,
                                  int fortran_order, int *dim) {
    if (ndims < 1 || !n_parallel || !n_sequential || !dim) return JACC_ERR_INVALID;
    int best = 0;
    for (int k = 0; k < ndims; k++) best = std::max(best, n_parallel[k]);
    if (best == 0) {
        *dim = -1;  // no parallel dimension: duplicate
        return JACC_OK;
    }
    int pick = -1, fewest = 0;
    for (int k = 0; k < ndims; k++) {
        if (n_parallel[k] != best) continue;
        // strictly fewer sequential iterators wins; ties keep the leftmost
        // (C) or take the later one (Fortran: rightmost)
        if (pick < 0 || n_sequential[k] < fewest || (fortran_order && n_sequential[k] == fewest)) {
            pick = k;
            fewest = n_sequential[k];
        }
    }
    *dim = pick;
    return JACC_OK;
}

jacc_status jacc_exchange_plan(int ndims, const int64_t *extents, size_t elem, int split_dim, int n,
                               int d, jacc_copy2d_plan *out) {
    if (ndims < 1 || ndims > 8 || !extents || elem == 0 || split_dim < 0 || split_dim >= ndims ||
        n < 1 || d < 0 || d >= n || !out)
        return JACC_ERR_INVALID;
    for (int k = 0; k < ndims; k++)
        if (extents[k] < 1) return JACC_ERR_INVALID;
    int64_t lo, hi;
    partition(extents[split_dim], n, d, lo, hi);
    const Copy2D c = copy2d_plan(ndims, extents, (int64_t)elem, split_dim, lo, hi);
    out->count = c.count;
    out->height = c.height;
    out->width_bytes = c.width;
    out->pitch_bytes = c.pitch;
    out->first_offset_bytes = c.first;
    out->outer_stride_bytes = c.outer;
    return JACC_OK;
}

jacc_status jacc_partition(int64_t E, int n, int d, int64_t *lo, int64_t *hi) {
    if (E < 0 || n < 1 || d < 0 || d >= n || !lo || !hi) return JACC_ERR_INVALID;
    partition(E, n, d, *lo, *hi);
    return JACC_OK;
}

jacc_status jacc_set_merge_policy(int policy) {
    if (!R.init || R.poisoned) return JACC_ERR_STATE;
    if (policy != JACC_MERGE_EAGER && policy != JACC_MERGE_HALO) return JACC_ERR_INVALID;
    R.policy = policy;
    return JACC_OK;
}

jacc_status jacc_set_scatter_split(int iteration_split) {
    if (!R.init || R.poisoned) return JACC_ERR_STATE;
    if (iteration_split && R.mp) return JACC_ERR_INVALID;
    R.scatter_itersplit = iteration_split != 0;
    return JACC_OK;
}

jacc_status jacc_set_queues(int nq) {
    return guard([&]() -> jacc_status {
        if (R.mp || R.capturing || nq < 1 || nq > JACC_MAX_QUEUES) return JACC_ERR_INVALID;
        sync_all();
        for (int d = 0; d < R.n; d++) {
            Device &dv = R.dev[d];
            set_dev(d);
            if (dv.qs.empty()) dv.qs.push_back(dv.s);
            while ((int)dv.qs.size() < nq) {
                cudaStream_t st;
                CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
                dv.qs.push_back(st);
            }
            while ((int)dv.qev.size() < (int)dv.qs.size()) {
                cudaEvent_t e;
                CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                dv.qev.push_back(e);
            }
            if (dv.qpartials.empty()) {  // slot 0 = the device's own scratch
                dv.qpartials.push_back(dv.partials);
                dv.qpart.push_back(dv.part);
                dv.qres.push_back(dv.res);
                dv.qticket.push_back(dv.ticket);
            }
            while (dv.qpartials.size() < dv.qs.size()) {
                double *pa, *pt, *rs;
                unsigned *tk;
                CK(cudaMalloc(&pa, jk::kHimenoPartials * sizeof(double)));
                CK(cudaMalloc(&pt, 8));
                CK(cudaMalloc(&rs, 8));
                CK(cudaMalloc(&tk, 64));
                CK(cudaMemset(pt, 0, 8));
                CK(cudaMemset(tk, 0, 64));
                dv.qpartials.push_back(pa);
                dv.qpart.push_back(pt);
                dv.qres.push_back(rs);
                dv.qticket.push_back(tk);
            }
            for (size_t q = 0; q < dv.qs.size(); q++) CK(cudaEventRecord(dv.qev[q], dv.qs[q]));
        }
        R.nq = nq;
        R.sched.reset(nq);
        return JACC_OK;
    });
}

jacc_status jacc_queue_replay(int nq, int nlaunch, const int *nreads, const int64_t *reads,
                              const int *nwrites, const int64_t *writes, const int *requested,
                              int *queue_out, int *waits_out) {
    if (nq < 1 || nq > JACC_MAX_QUEUES || nlaunch < 0 || (nlaunch > 0 && (!nreads || !nwrites ||
        !requested || !queue_out || !waits_out)))
        return JACC_ERR_INVALID;
    QueueSched qs;
    qs.reset(nq);
    int64_t ri = 0, wi = 0;
    for (int l = 0; l < nlaunch; l++) {
        std::vector<int64_t> rd(reads + ri, reads + ri + nreads[l]);
        std::vector<int64_t> wr(writes + wi, writes + wi + nwrites[l]);
        ri += nreads[l];
        wi += nwrites[l];
        if (requested[l] >= nq) return JACC_ERR_INVALID;
        std::vector<int> waits;
        queue_out[l] = qs.schedule(rd, wr, requested[l], waits);
        for (int q = 0; q < nq; q++) waits_out[l * nq + q] = 0;
        for (int q : waits) waits_out[l * nq + q] = 1;
    }
    return JACC_OK;
}

jacc_status jacc_set_split_dim(int dim) {
    if (!R.init || R.poisoned) return JACC_ERR_STATE;
    if (dim < -1 || dim > 2) return JACC_ERR_INVALID;
    R.split_dim = dim;
    return JACC_OK;
}

jacc_status jacc_set_mode(int mode) {
    if (!R.init || R.poisoned) return JACC_ERR_STATE;
    if (mode != JACC_MODE_MULTI && mode != JACC_MODE_DUP && mode != JACC_MODE_ADAPTIVE)
        return JACC_ERR_INVALID;
    if (mode == JACC_MODE_ADAPTIVE && R.mp) return JACC_ERR_INVALID;  // needs every device's timing
    R.mode = mode;
    return JACC_OK;
}

jacc_status jacc_data_create(void *host, size_t bytes, size_t elem_size, int ndims,
                             const int64_t *extents) {
    return guard([&]() -> jacc_status {
        if (R.capturing) return JACC_ERR_STATE;
        if (!host || bytes == 0 || elem_size == 0 || ndims < 1 || ndims > 4 || !extents)
            return JACC_ERR_INVALID;
        int64_t prod = 1;
        for (int k = 0; k < ndims; k++) {
            if (extents[k] < 1) return JACC_ERR_INVALID;
            prod *= extents[k];
        }
        if ((size_t)prod * elem_size != bytes) return JACC_ERR_INVALID;
        const uintptr_t a = (uintptr_t)host;
        // overlap with a present region
        auto it = R.table.lower_bound(a);
        if (it != R.table.end() && it->first < a + bytes) return JACC_ERR_OVERLAP;
        if (it != R.table.begin()) {
            auto p = std::prev(it);
            if (p->second->base + p->second->bytes > a) return JACC_ERR_OVERLAP;
        }
        auto r = std::make_unique<Region>();
        r->base = a;
        r->bytes = bytes;
        r->elem = elem_size;
        r->ndims = ndims;
        for (int k = 0; k < ndims; k++) r->ext[k] = extents[k];
        r->nelem = prod;
        r->rep.assign(R.n, nullptr);
        r->dirty.assign(R.n, nullptr);
        r->bitmap.assign(R.n, nullptr);
        r->dslot.assign(R.n, 0);
        r->delta.assign(R.n, nullptr);
        r->dbm.assign(R.n, nullptr);
        r->valid.assign(R.n, IntervalSet{});
        for (int d = 0; d < R.n; d++) {
            if (!local(d)) continue;  // peers' replicas arrive via jacc_import_region
            set_dev(d);
            if (cudaMalloc(&r->rep[d], bytes) != cudaSuccess ||
                cudaMalloc(&r->dirty[d], 32) != cudaSuccess) {
                cudaGetLastError();
                free_region(r.get());
                return JACC_ERR_OOM;
            }
            CK(cudaMemset(r->dirty[d], 0xff, 32));
        }
        // pin large host buffers so update_device/update_host are DMA-direct
        if (bytes >= (1u << 20) && !getenv("JACC_NO_PIN")) {
            cudaError_t e = cudaHostRegister(host, bytes, cudaHostRegisterPortable);
            if (e == cudaSuccess) r->pinned = true;
            else cudaGetLastError();
        }
        R.table[a] = std::move(r);
        return JACC_OK;
    });
}

jacc_status jacc_data_delete(void *host) {
    return guard([&]() -> jacc_status {
        Region *r = lookup(host);
        if (!r) return JACC_ERR_NOT_PRESENT;
        if (R.capturing) return JACC_ERR_STATE;
        sync_all();
        for (auto &g : R.graphs) destroy_graph(g.second);  // they reference the replicas
        R.graphs.clear();
        free_region(r);
        R.table.erase(r->base);
        return JACC_OK;
    });
}

jacc_status jacc_update_device(void *host, size_t off, size_t bytes) {
    struct Nvtx {
        Nvtx() { nvtxRangePushA("jacc_update_device"); }
        ~Nvtx() { nvtxRangePop(); }
    } nvtx;
    return guard([&]() -> jacc_status {
        if (R.capturing) return JACC_ERR_STATE;
        Region *r = lookup(host);
        if (!r) return JACC_ERR_NOT_PRESENT;
        const size_t start = ((uintptr_t)host - r->base) + off;
        if (start + bytes > r->bytes || start % r->elem || bytes % r->elem) return JACC_ERR_INVALID;
        if (bytes == 0) return JACC_OK;
        sync_all();
        for (int d = 0; d < R.n; d++) {
            if (!local(d)) continue;
            set_dev(d);
            CK(cudaMemcpyAsync(r->rep[d] + start, (const char *)r->base + start, bytes,
                               cudaMemcpyHostToDevice, R.dev[d].s));
        }
        sync_all();
        const int64_t e0 = (int64_t)(start / r->elem), e1 = (int64_t)((start + bytes) / r->elem);
        for (int d = 0; d < R.n; d++) r->valid[d].add(e0, e1);
        return JACC_OK;
    });
}

jacc_status jacc_update_host(void *host, size_t off, size_t bytes) {
    struct Nvtx {
        Nvtx() { nvtxRangePushA("jacc_update_host"); }
        ~Nvtx() { nvtxRangePop(); }
    } nvtx;
    return guard([&]() -> jacc_status {
        if (R.capturing) return JACC_ERR_STATE;
        Region *r = lookup(host);
        if (!r) return JACC_ERR_NOT_PRESENT;
        const size_t start = ((uintptr_t)host - r->base) + off;
        if (start + bytes > r->bytes || start % r->elem || bytes % r->elem) return JACC_ERR_INVALID;
        if (bytes == 0) return JACC_OK;
        sync_all();
        const int64_t e0 = (int64_t)(start / r->elem), e1 = (int64_t)((start + bytes) / r->elem);
        // gather: pull stale intervals into the primary from a valid replica.
        // Multi-process mode: every rank's device is its own primary; all
        // ranks plan every device's pulls so the validity trackers agree.
        struct GP {
            int t, src;
            int64_t a, b;
        };
        std::vector<GP> gp;
        for (int t = 0; t < R.n; t++) {
            if (!R.mp && t != 0) continue;
            for (auto &m : r->valid[t].missing(e0, e1)) {
                int64_t a = m.first;
                while (a < m.second) {
                    int src = -1;
                    int64_t b = m.second;
                    for (int q = 0; q < R.n && src < 0; q++) {
                        if (q == t) continue;
                        auto &vi = r->valid[q].iv;
                        auto it = vi.upper_bound(a);
                        if (it == vi.begin()) continue;
                        --it;
                        if (it->first <= a && it->second > a) {
                            src = q;
                            b = std::min(b, it->second);
                        }
                    }
                    if (src < 0) break;  // never initialised anywhere
                    gp.push_back({t, src, a, b});
                    a = b;
                }
            }
        }
        const int h = R.mp ? R.me : 0;
        Device &d0 = R.dev[h];
        set_dev(h);
        for (auto &g : gp) {
            if (g.t == h)
                CK(cudaMemcpyAsync(r->rep[h] + g.a * r->elem, r->rep[g.src] + g.a * r->elem,
                                   (size_t)(g.b - g.a) * r->elem, cudaMemcpyDefault, d0.s));
        }
        for (auto &g : gp) r->valid[g.t].add(g.a, g.b);
        CK(cudaMemcpyAsync((char *)r->base + start, r->rep[h] + start, bytes, cudaMemcpyDeviceToHost,
                           d0.s));
        CK(cudaStreamSynchronize(d0.s));
        rank_barrier();  // peers may have read this rank's replica
        return JACC_OK;
    });
}

jacc_status jacc_get_dirty_range(void *host, int dev, uint64_t *mn, uint64_t *mx) {
    return guard([&]() -> jacc_status {
        if (R.capturing) return JACC_ERR_STATE;
        Region *r = lookup(host);
        if (!r) return JACC_ERR_NOT_PRESENT;
        if (dev < 0 || dev >= R.n || !mn || !mx) return JACC_ERR_INVALID;
        if (!local(dev)) return JACC_ERR_INVALID;
        local_sync();
        u64 h[2];
        set_dev(dev);
        CK(cudaMemcpy(h, r->dirty[dev] + 2 * r->dslot[dev], 16, cudaMemcpyDeviceToHost));
        *mn = h[0];
        *mx = ~h[1];
        return JACC_OK;
    });
}

jacc_status jacc_get_dirty_bitmap(void *host, int dev, uint32_t *out, size_t nwords) {
    return guard([&]() -> jacc_status {
        if (R.capturing) return JACC_ERR_STATE;
        Region *r = lookup(host);
        if (!r) return JACC_ERR_NOT_PRESENT;
        if (dev < 0 || dev >= R.n || !out) return JACC_ERR_INVALID;
        const size_t words = (size_t)((r->nelem + 31) / 32);
        if (nwords < words || !r->bitmap[dev]) return JACC_ERR_INVALID;
        if (!local(dev)) return JACC_ERR_INVALID;
        local_sync();
        set_dev(dev);
        CK(cudaMemcpy(out, r->bitmap[dev], words * 4, cudaMemcpyDeviceToHost));
        return JACC_OK;
    });
}

jacc_status jacc_get_replica(void *host, int dev, void *out, size_t bytes) {
    return guard([&]() -> jacc_status {
        if (R.capturing) return JACC_ERR_STATE;
        Region *r = lookup(host);
        if (!r) return JACC_ERR_NOT_PRESENT;
        if (dev < 0 || dev >= R.n || !out || bytes > r->bytes) return JACC_ERR_INVALID;
        if (!local(dev)) return JACC_ERR_INVALID;
        local_sync();
        set_dev(dev);
        CK(cudaMemcpy(out, r->rep[dev], bytes, cudaMemcpyDeviceToHost));
        return JACC_OK;
    });
}

jacc_status jacc_last_timing(double *tk, double *tm, uint64_t *bytes) {
    return guard([&]() -> jacc_status {
        if (R.capturing) return JACC_ERR_STATE;
        flush_prof();
        if (tk) *tk = R.last_valid ? R.last_k : 0.0;
        if (tm) *tm = R.last_valid ? R.last_m : 0.0;
        if (bytes) *bytes = R.last_bytes;
        return JACC_OK;
    });
}

jacc_status jacc_set_trace(const char *path) {
    return guard([&]() -> jacc_status {
        if (R.capturing) return JACC_ERR_STATE;
        flush_prof();
        close_trace();
        if (!path) return JACC_OK;
        R.trace = fopen(path, "w");
        if (!R.trace) return JACC_ERR_INVALID;
        R.trace_events = 0;
        R.trace_k = R.trace_c = 0;
        R.trace_modes.clear();
        R.profiling = true;
        return JACC_OK;
    });
}

jacc_status jacc_set_profiling(int on) {
    return guard([&]() -> jacc_status {
        if (R.capturing) return JACC_ERR_STATE;
        flush_prof();
        R.profiling = on != 0;
        return JACC_OK;
    });
}

jacc_status jacc_profile_totals(int dev, double *ks, double *ms, uint64_t *launches,
                                uint64_t *bytes) {
    return guard([&]() -> jacc_status {
        if (R.capturing) return JACC_ERR_STATE;
        if (dev < 0 || dev >= R.n) return JACC_ERR_INVALID;
        flush_prof();
        const Device &dv = R.dev[dev];
        if (ks) *ks = dv.kernel_s;
        if (ms) *ms = dv.merge_s;
        if (launches) *launches = dv.launches;
        if (bytes) *bytes = dv.bytes_merged;
        return JACC_OK;
    });
}

jacc_status jacc_profile_reset(void) {
    return guard([&]() -> jacc_status {
        if (R.capturing) return JACC_ERR_STATE;
        flush_prof();
        for (auto &dv : R.dev) {
            dv.kernel_s = dv.merge_s = 0;
            dv.launches = dv.bytes_merged = 0;
        }
        R.last_valid = false;
        return JACC_OK;
    });
}

jacc_status jacc_get_stream(int dev, void **stream, int *ord) {
    return guard([&]() -> jacc_status {
        if (dev < 0 || dev >= R.n || !local(dev)) return JACC_ERR_INVALID;
        if (stream) *stream = (void *)R.dev[dev].s;
        if (ord) *ord = R.dev[dev].ord;
        return JACC_OK;
    });
}

jacc_status jacc_get_info(jacc_info *out) {
    return guard([&]() -> jacc_status {
        invalid_if(!out);
        out->n_devices = R.n;
        out->distinct_gpus = R.distinct ? 1 : 0;
        out->combine = R.use_nccl ? JACC_COMBINE_NCCL : JACC_COMBINE_PEER;
        out->peer_pairs = R.mp ? -1 : R.peer_pairs;
        out->multiprocess = R.mp ? 1 : 0;
        out->rank = R.mp ? R.me : 0;
        return JACC_OK;
    });
}

jacc_status jacc_adaptive_replay(int n, double peak_p2p, int len, const double *t_kernel,
                                 const double *t_comm, const double *write_size, int *states_out) {
    if (n < 1 || peak_p2p <= 0 || len < 0 || (len > 0 && (!t_kernel || !t_comm || !write_size)) ||
        !states_out)
        return JACC_ERR_INVALID;
    AdaptiveCtl c;
    for (int i = 0; i < len; i++) {
        states_out[i] = c.state;
        c.observe(t_kernel[i], t_comm[i], write_size[i], n, peak_p2p);
    }
    states_out[len] = c.state;
    return JACC_OK;
}

jacc_status jacc_adaptive_history(int loop_id, int cap, double *t_kernel, double *t_comm,
                                  double *write_size, int *states, int *len, int *state_now) {
    return guard([&]() -> jacc_status {
        if (cap < 0 || !len) return JACC_ERR_INVALID;
        poll_adaptive(true);
        auto it = R.adapt_last_key.find(loop_id);
        if (it == R.adapt_last_key.end()) {
            *len = 0;
            if (state_now) *state_now = -1;
            return JACC_OK;
        }
        const AdaptiveCtl &c = R.adapt[it->second];
        const int m = (int)c.h_tk.size();
        *len = m;
        if (state_now) *state_now = c.state;
        for (int i = 0; i < m && i < cap; i++) {
            if (t_kernel) t_kernel[i] = c.h_tk[i];
            if (t_comm) t_comm[i] = c.h_tc[i];
            if (write_size) write_size[i] = c.h_ws[i];
            if (states) states[i] = c.h_state[i];
        }
        return JACC_OK;
    });
}

const char *jacc_error_string(jacc_status s) {
    switch (s) {
    case JACC_OK: return "JACC_OK";
    case JACC_ERR_INVALID: return "JACC_ERR_INVALID: invalid argument";
    case JACC_ERR_OVERLAP: return "JACC_ERR_OVERLAP: region overlaps a present region";
    case JACC_ERR_NOT_PRESENT: return "JACC_ERR_NOT_PRESENT: address not in any present region";
    case JACC_ERR_UNKNOWN_LOOP: return "JACC_ERR_UNKNOWN_LOOP: no such loop id";
    case JACC_ERR_OOM: return "JACC_ERR_OOM: device allocation failed";
    case JACC_ERR_CUDA: return "JACC_ERR_CUDA: CUDA error (runtime poisoned)";
    case JACC_ERR_NCCL: return "JACC_ERR_NCCL: NCCL error (runtime poisoned)";
    case JACC_ERR_STATE: return "JACC_ERR_STATE: not initialised or poisoned";
    default: return "JACC: unknown status";
    }
}


}  // extern "C"
