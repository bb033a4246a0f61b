// rt.hpp -- internal state and helpers of the libjacc.so host runtime,
// shared by plan.cpp, launch.cpp, abi.cpp, mp.cpp and graphs.cpp (not
// installed; everything here is hidden by csrc/exports.map).
//
//   a1  present table (ordered map, interior-address lookup)
//   a2  update_device: H2D into every replica
//   a3  launch planning: alias rule, owned blocks of the written
//       array's split dimension (remainder rule S:266), clipped
//       per-device iteration ranges, stale-input pulls (validity tracker)
//   a4  device kernels with fused write tracking (kernels.cu)
//   a5  reduction combine (NCCL allreduce across distinct GPUs)
//   a6  dirty-region merge (EAGER P:471/P:527, or HALO)
//   a7  update_host: gather stale owned intervals into the primary, D2H
//   a8  wait
//
// Ordering between logical devices uses one CUDA event per device per launch
// generation: launch k on device d waits for launch k-1 of every device it
// exchanged data with in launch k-1 or exchanges with in launch k ("we
// synchronize GPUs at the beginning and ending of the communication",
// P:527).  That covers RAW on pushed/pulled data and WAR on peer replicas.
#pragma once

#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "jacc.h"
#include "kernels.cuh"
#include <nvtx3/nvToolsExt.h>

namespace jrt {

using u64 = unsigned long long;

// ---------------------------------------------------------------------------
// Interval set over element indices (half-open), used for replica validity.
// ---------------------------------------------------------------------------
struct IntervalSet {
    std::map<int64_t, int64_t> iv;  // start -> end

    void add(int64_t a, int64_t b) {
        if (a >= b) return;
        auto it = iv.upper_bound(a);
        if (it != iv.begin()) {
            auto p = std::prev(it);
            if (p->second >= a) {
                a = p->first;
                b = std::max(b, p->second);
                it = iv.erase(p);
            }
        }
        while (it != iv.end() && it->first <= b) {
            b = std::max(b, it->second);
            it = iv.erase(it);
        }
        iv[a] = b;
    }
    void remove(int64_t a, int64_t b) {
        if (a >= b) return;
        auto it = iv.upper_bound(a);
        if (it != iv.begin()) --it;
        std::vector<std::pair<int64_t, int64_t>> keep;
        while (it != iv.end() && it->first < b) {
            if (it->second <= a) {
                ++it;
                continue;
            }
            if (it->first < a) keep.push_back({it->first, a});
            if (it->second > b) keep.push_back({b, it->second});
            it = iv.erase(it);
        }
        for (auto &k : keep) iv[k.first] = k.second;
    }
    // sub-intervals of [a,b) NOT covered
    std::vector<std::pair<int64_t, int64_t>> missing(int64_t a, int64_t b) const {
        std::vector<std::pair<int64_t, int64_t>> out;
        if (a >= b) return out;
        int64_t cur = a;
        auto it = iv.upper_bound(a);
        if (it != iv.begin()) --it;
        for (; it != iv.end() && it->first < b; ++it) {
            if (it->second <= cur) continue;
            if (it->first > cur) out.push_back({cur, std::min(it->first, b)});
            cur = std::max(cur, it->second);
            if (cur >= b) break;
        }
        if (cur < b) out.push_back({cur, b});
        return out;
    }
    bool covers(int64_t a, int64_t b) const { return missing(a, b).empty(); }
};

// ---------------------------------------------------------------------------
// NEXT-1: adaptive utilization controller (DESIGN R-16), one per
// kernel identity.  Starts duplicated; after the warm-up run profiles
// eff_dup (time per written byte) until Eq. (1) has held five times, then
// runs multi-GPU; switches back for good once Eq. (2) or Eq. (3) has held
// five times with a positive mean margin.
// ---------------------------------------------------------------------------
struct AdaptiveCtl {
    enum { DUP_WARMUP = 0, DUP_PROFILING = 1, MULTI = 2, DUP_FINAL = 3 };
    int state = DUP_WARMUP;
    double eff_sum = 0;
    int eff_cnt = 0, c1 = 0, c23 = 0;
    double margin_sum = 0;
    int margin_cnt = 0;
    bool dup() const { return state != MULTI; }
    // observations fed so far (for introspection / replay tests)
    std::vector<double> h_tk, h_tc, h_ws;
    std::vector<int> h_state;
    void observe(double tk, double tc, double ws, int n, double peak) {
        switch (state) {
        case DUP_WARMUP:
            state = DUP_PROFILING;  // warm-up run is not profiled
            break;
        case DUP_PROFILING:
            if (ws > 0) {
                eff_sum += tk / ws;
                eff_cnt++;
            }
            if (tk > tk / n + ws / peak) c1++;  // Eq. (1)
            if (c1 >= 5) state = MULTI;
            break;
        case MULTI: {
            const double left = tk + tc;
            const double r2 = tk * n;  // Eq. (2)
            const double r3 = (eff_cnt > 0 && ws > 0) ? (eff_sum / eff_cnt) * ws
                                                      : __builtin_inf();  // Eq. (3)
            if (left > r2 || left > r3) c23++;
            margin_sum += left - std::min(r2, r3);
            margin_cnt++;
            if (c23 >= 5 && margin_sum / margin_cnt > 0) state = DUP_FINAL;
            break;
        }
        default:
            break;
        }
    }
};

// ---------------------------------------------------------------------------
// NEXT-4: automated asynchronous execution (Fig. 2; DESIGN R-20).
// Arrays' last writer (queue, time) and last readers (per queue) give the
// RAW / WAW / WAR dependencies of a launch; it joins the queue of its most
// recent dependency (none: the least recently used queue) and waits only on
// other queues whose dependency is not already ordered before it, tracked
// in a matrix of the latest synchronisation between queues (transitive).
// ---------------------------------------------------------------------------
struct QueueSched {
    int nq = 1;
    int64_t T = 0;
    std::vector<int64_t> last_use;
    std::map<int64_t, std::pair<int, int64_t>> writer;
    std::map<int64_t, std::map<int, int64_t>> readers;
    std::vector<std::vector<int64_t>> sync;
    void reset(int q) {
        nq = q;
        T = 0;
        last_use.assign(q, -1);
        writer.clear();
        readers.clear();
        sync.assign(q, std::vector<int64_t>(q, -1));
    }
    int schedule(const std::vector<int64_t> &reads, const std::vector<int64_t> &writes, int req,
                 std::vector<int> &waits) {
        T++;
        std::vector<int64_t> touched(reads);
        touched.insert(touched.end(), writes.begin(), writes.end());
        std::sort(touched.begin(), touched.end());
        touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
        std::vector<std::pair<int, int64_t>> deps;
        for (int64_t r : touched) {
            auto it = writer.find(r);
            if (it != writer.end()) deps.push_back(it->second);
        }
        std::vector<int64_t> ws(writes);
        std::sort(ws.begin(), ws.end());
        ws.erase(std::unique(ws.begin(), ws.end()), ws.end());
        for (int64_t w : ws) {
            auto it = readers.find(w);
            if (it != readers.end())
                for (auto &kv : it->second) deps.push_back({kv.first, kv.second});
        }
        int q;
        if (req >= 0) {
            q = req;
        } else if (!deps.empty()) {
            int64_t tmax = -1;
            for (auto &d : deps) tmax = std::max(tmax, d.second);
            q = nq;
            for (auto &d : deps)
                if (d.second == tmax) q = std::min(q, d.first);
        } else {
            q = 0;
            for (int k = 1; k < nq; k++)
                if (last_use[k] < last_use[q]) q = k;
        }
        std::vector<char> w(nq, 0);
        for (auto &d : deps) {
            const int p = d.first;
            if (p == q || sync[q][p] >= d.second) continue;  // same queue / already solved
            w[p] = 1;
            sync[q][p] = last_use[p];
            for (int x = 0; x < nq; x++) sync[q][x] = std::max(sync[q][x], sync[p][x]);
        }
        waits.clear();
        for (int p = 0; p < nq; p++)
            if (w[p]) waits.push_back(p);
        for (int64_t r : reads) readers[r][q] = T;
        for (int64_t x : ws) {
            writer[x] = {q, T};
            readers[x].clear();
        }
        last_use[q] = T;
        return q;
    }
};

// ---------------------------------------------------------------------------
struct Device {
    int ord = 0;
    cudaStream_t s = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    double *partials = nullptr;  // kReduceGrid
    unsigned *ticket = nullptr;
    double *part = nullptr;      // this device's reduction partial
    double *res = nullptr;       // allreduce result / combine output
    double *hscal = nullptr;     // pinned host scalar
    ncclComm_t comm = nullptr;
    void *scratch = nullptr;     // binned-scatter pairs (grown on demand)
    // scratch buffers replaced while a captured graph may still reference
    // them (freed once no graph exists)
    std::vector<void *> retired;
    std::vector<cudaStream_t> qs;   // async queues (qs[0] = s), NEXT-4
    std::vector<cudaEvent_t> qev;   // last launch's completion per queue
    // per-queue reduction scratch (concurrent queues must not share it)
    std::vector<double *> qpartials, qpart, qres;
    std::vector<unsigned *> qticket;
    cudaEvent_t pe = nullptr;    // phase event (iteration-split scatter)
    u64 *scr_dirty = nullptr;    // scratch dirty record (phase-1 kernels)
    size_t scratch_bytes = 0;
    // profiling
    double kernel_s = 0, merge_s = 0;
    uint64_t launches = 0, bytes_merged = 0;
};

struct Region {
    uintptr_t base = 0;
    size_t bytes = 0, elem = 0;
    int ndims = 0;
    int64_t ext[4] = {1, 1, 1, 1};
    int64_t nelem = 0;
    bool pinned = false;
    std::vector<char *> rep;           // per device replica
    std::vector<u64 *> dirty;          // per device: 2 slots of [min, ~max] (32 B)
    std::vector<int> dslot;            // per device: slot of the most recent launch
    std::vector<uint32_t *> bitmap;    // per device, lazily allocated
    std::vector<char *> delta;         // per device delta array (iteration-split scatter)
    std::vector<uint32_t *> dbm;       // per device delta bitmap
    std::vector<IntervalSet> valid;    // per device
};

struct ProfRec {
    int dev;
    cudaEvent_t k0, k1, m1;
};

// D13 timing record of one launch, written as a JSON line once its events
// resolve ({event, kernel_id, queue, waits[], t_kernel_s,
// t_comm_s, mode, bytes_exchanged}; jacc_set_trace)
struct TraceRec {
    uint64_t event;
    int loop_id;
    const char *name;
    int queue;
    std::vector<int> waits;  // queues this launch waited on (NEXT-4)
    std::vector<int> peers;  // devices whose previous launch it waited on (merge ordering)
    bool dup;
    int policy;
    uint64_t bytes;
    size_t p0, p1;           // its ProfRecs: R.prof[p0, p1)
};

// one adaptive observation in flight: a launch's per-device events
struct AdaptRec {
    std::string key;
    int n_dev;
    bool dup;
    double ws;
    std::vector<ProfRec> ev;
};

// A captured launch sequence (CUDA graph over every device's stream) and
// the host-side runtime state it maps S_start -> S_end.
struct GraphRec {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
    std::map<Region *, std::vector<IntervalSet>> v_start, v_end;
    std::map<Region *, std::vector<int>> slot_start, slot_end;
    std::vector<std::vector<char>> comm_end;
};

struct Runtime {
    bool init = false;
    bool poisoned = false;
    int n = 0;
    std::vector<Device> dev;
    std::map<uintptr_t, std::unique_ptr<Region>> table;
    int policy = JACC_MERGE_EAGER;
    int mode = JACC_MODE_MULTI;
    int split_dim = -1;  // -1: A18 rule (dim 0 for the built-in loops)
    bool scatter_itersplit = false;
    int nq = 1;          // async queues per device (NEXT-4); 1 = single stream
    QueueSched sched;
    int gen = 0;
    bool distinct = true;
    bool use_nccl = false;
    int peer_pairs = 0;  // ordered pairs of distinct GPUs with P2P enabled
    std::vector<std::vector<char>> comm_prev;  // [d][q]
    bool profiling = false;
    std::vector<ProfRec> prof;                 // unresolved event records
    FILE *trace = nullptr;                     // JSON-lines trace (jacc_set_trace)
    std::vector<TraceRec> trace_pending;
    uint64_t trace_events = 0;
    double trace_k = 0, trace_c = 0;           // summary totals (max over devices per launch)
    std::map<std::string, std::pair<uint64_t, uint64_t>> trace_modes;  // name -> (multi, dup)
    size_t last_start = 0;                     // first record of the last launch
    std::vector<cudaEvent_t> evpool;
    double last_k = 0, last_m = 0;
    uint64_t last_bytes = 0;
    bool last_valid = false;
    // one-process-per-GPU mode (jacc_init_rank): this process owns logical
    // device `me`; peers' replicas and events are CUDA-IPC mapped; host
    // progress counters live in POSIX shared memory.
    bool mp = false;
    int me = 0;
    struct Slot {
        uint64_t launches;
        uint64_t barrier;
        uint64_t pad[6];
    };
    Slot *shm = nullptr;
    std::string shm_name;
    uint64_t barrier_gen = 0;
    // adaptive utilization (JACC_MODE_ADAPTIVE)
    std::map<std::string, AdaptiveCtl> adapt;
    std::map<int, std::string> adapt_last_key;  // loop_id -> most recent key
    std::vector<AdaptRec> adapt_pending;
    double peak_p2p = 770e9;  // B/s per GPU egress (measured peer copy, B200_PROFILING.md)
    // CUDA graph capture / replay of launch sequences (single process)
    bool capturing = false;
    GraphRec cap;
    std::map<int, GraphRec> graphs;
    int next_graph = 1;
};

inline Runtime R;  // the process-wide runtime state

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
struct Fail {
    jacc_status st;
};

inline void cuda_check(cudaError_t e, const char *what) {
    if (e != cudaSuccess) {
        if (getenv("JACC_DEBUG")) fprintf(stderr, "[jacc] %s: %s\n", what, cudaGetErrorString(e));
        R.poisoned = true;
        throw Fail{JACC_ERR_CUDA};
    }
}
#define CK(x) cuda_check((x), #x)

inline void nccl_check(ncclResult_t e, const char *what) {
    if (e != ncclSuccess) {
        if (getenv("JACC_DEBUG")) fprintf(stderr, "[jacc] %s: %s\n", what, ncclGetErrorString(e));
        R.poisoned = true;
        throw Fail{JACC_ERR_NCCL};
    }
}
#define NK(x) nccl_check((x), #x)

template <typename F>
jacc_status guard(F &&f, bool need_init = true) {
    if (need_init && (!R.init || R.poisoned)) return JACC_ERR_STATE;
    try {
        return f();
    } catch (Fail &e) {
        return e.st;
    } catch (std::bad_alloc &) {
        return JACC_ERR_OOM;
    }
}

inline Region *lookup(const void *p) {
    uintptr_t a = (uintptr_t)p;
    auto it = R.table.upper_bound(a);
    if (it == R.table.begin()) return nullptr;
    --it;
    Region *r = it->second.get();
    return (a >= r->base && a < r->base + r->bytes) ? r : nullptr;
}

inline bool local(int d) { return !R.mp || d == R.me; }

inline void set_dev(int d) { CK(cudaSetDevice(R.dev[d].ord)); }

// spin on a shared-memory predicate with a generous timeout (a dead peer
// must not hang the caller forever)
template <typename P>
inline void spin_until(P pred) {
    auto t0 = std::chrono::steady_clock::now();
    for (uint64_t it = 0; !pred(); it++) {
        if ((it & 1023) == 1023) {
            sched_yield();
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(300)) {
                R.poisoned = true;
                throw Fail{JACC_ERR_STATE};
            }
        }
    }
}

inline uint64_t shm_load(const uint64_t *p) { return __atomic_load_n(p, __ATOMIC_ACQUIRE); }
inline void shm_store(uint64_t *p, uint64_t v) { __atomic_store_n(p, v, __ATOMIC_RELEASE); }

// host barrier across ranks (multi-process mode only)
inline void rank_barrier() {
    if (!R.mp) return;
    const uint64_t b = ++R.barrier_gen;
    shm_store(&R.shm[R.me].barrier, b);
    spin_until([&] {
        for (int q = 0; q < R.n; q++)
            if (shm_load(&R.shm[q].barrier) < b) return false;
        return true;
    });
}

// wait until every rank has enqueued `k` launches (multi-process lockstep:
// no rank runs more than one launch ahead, so the two-slot event ring of a
// peer is never re-recorded before this rank has waited on it)
inline void wait_launches(uint64_t k) {
    if (!R.mp) return;
    spin_until([&] {
        for (int q = 0; q < R.n; q++)
            if (shm_load(&R.shm[q].launches) < k) return false;
        return true;
    });
}

// drain this process's device streams
inline void local_sync() {
    for (int d = 0; d < R.n; d++) {
        if (!local(d)) continue;
        set_dev(d);
        CK(cudaStreamSynchronize(R.dev[d].s));
        for (size_t q = 1; q < R.dev[d].qs.size(); q++) CK(cudaStreamSynchronize(R.dev[d].qs[q]));
    }
}

// drain every device's work (collective across ranks in multi-process mode)
inline void sync_all() {
    local_sync();
    rank_barrier();
}

inline cudaEvent_t pool_event() {
    if (!R.evpool.empty()) {
        cudaEvent_t e = R.evpool.back();
        R.evpool.pop_back();
        return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
}

// resolve the accumulated profiling records into totals (syncs on them;
// called only on query, so timing never adds a host sync per launch)
inline void write_trace(const std::vector<float> &ks, const std::vector<float> &ms) {
    for (auto &t : R.trace_pending) {
        double tk = 0, tc = 0;
        for (size_t i = t.p0; i < t.p1 && i < ks.size(); i++) {
            tk = std::max(tk, (double)ks[i] * 1e-3);
            tc = std::max(tc, (double)ms[i] * 1e-3);
        }
        R.trace_k += tk;
        R.trace_c += tc;
        auto &mc = R.trace_modes[t.name];
        (t.dup ? mc.second : mc.first)++;
        if (!R.trace) continue;
        std::string w, pe;
        for (size_t i = 0; i < t.waits.size(); i++) w += (i ? "," : "") + std::to_string(t.waits[i]);
        for (size_t i = 0; i < t.peers.size(); i++) pe += (i ? "," : "") + std::to_string(t.peers[i]);
        fprintf(R.trace,
                "{\"event\": %llu, \"kernel_id\": %d, \"kernel\": \"%s\", \"queue\": %d, "
                "\"waits\": [%s], \"peer_waits\": [%s], \"t_kernel_s\": %.9g, \"t_comm_s\": %.9g, "
                "\"mode\": \"%s\", \"merge\": \"%s\", \"bytes_exchanged\": %llu, \"devices\": %d}\n",
                (unsigned long long)t.event, t.loop_id, t.name, t.queue, w.c_str(), pe.c_str(), tk, tc,
                t.dup ? "dup" : "multi", t.policy == JACC_MERGE_HALO ? "halo" : "eager",
                (unsigned long long)t.bytes, R.n);
    }
    R.trace_pending.clear();
    if (R.trace) fflush(R.trace);
}

inline void close_trace() {
    if (!R.trace) return;
    std::string pm;
    for (auto &kv : R.trace_modes)
        pm += (pm.empty() ? "" : ", ") + std::string("\"") + kv.first + "\": {\"multi\": " +
              std::to_string(kv.second.first) + ", \"dup\": " + std::to_string(kv.second.second) + "}";
    fprintf(R.trace, "{\"summary\": {\"events\": %llu, \"total_kernel_s\": %.9g, \"total_comm_s\": %.9g, "
                     "\"per_kernel_modes\": {%s}}}\n",
            (unsigned long long)R.trace_events, R.trace_k, R.trace_c, pm.c_str());
    fclose(R.trace);
    R.trace = nullptr;
}

inline void flush_prof() {
    if (R.prof.empty()) {
        R.trace_pending.clear();
        return;
    }
    double kmax = 0, mmax = 0;
    std::vector<float> ks(R.prof.size()), ms(R.prof.size());
    for (size_t i = 0; i < R.prof.size(); i++) {
        auto &p = R.prof[i];
        set_dev(p.dev);
        CK(cudaEventSynchronize(p.m1));
        float k = 0, m = 0;
        CK(cudaEventElapsedTime(&k, p.k0, p.k1));
        CK(cudaEventElapsedTime(&m, p.k1, p.m1));
        ks[i] = k;
        ms[i] = m;
        R.dev[p.dev].kernel_s += k * 1e-3;
        R.dev[p.dev].merge_s += m * 1e-3;
        if (i >= R.last_start) {
            kmax = std::max(kmax, (double)k * 1e-3);
            mmax = std::max(mmax, (double)m * 1e-3);
        }
        R.evpool.push_back(p.k0);
        R.evpool.push_back(p.k1);
        R.evpool.push_back(p.m1);
    }
    if (R.last_start < R.prof.size()) {
        R.last_k = kmax;
        R.last_m = mmax;
        R.last_valid = true;
    }
    write_trace(ks, ms);
    R.prof.clear();
    R.last_start = 0;
}

inline void free_region(Region *r) {
    for (int d = 0; d < (int)r->rep.size(); d++) {
        if (!local(d)) {
            if (r->rep[d]) cudaIpcCloseMemHandle(r->rep[d]);
            continue;
        }
        set_dev(d);
        if (r->rep[d]) cudaFree(r->rep[d]);
        if (r->dirty[d]) cudaFree(r->dirty[d]);
        if (r->bitmap[d]) cudaFree(r->bitmap[d]);
        if (r->delta[d]) cudaFree(r->delta[d]);
        if (r->dbm[d]) cudaFree(r->dbm[d]);
    }
    if (r->pinned) cudaHostUnregister((void *)r->base);
}

inline void destroy_graph(GraphRec &g) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    g = GraphRec{};
}

// c4 partition ("equally dividing"; S:266 remainder rule)
inline void partition(int64_t E, int n, int d, int64_t &lo, int64_t &hi) {
    const int64_t q = E / n, r = E % n;
    lo = (int64_t)d * q + std::min<int64_t>(d, r);
    hi = (int64_t)(d + 1) * q + std::min<int64_t>(d + 1, r);
}

// A19: device d's block [lo, hi) along split dimension s of a
// row-major array decomposes into `count` 2-D copies (cudaMemcpy2D-shaped):
// copy c, row r covers bytes [first + c*outer + r*pitch, ... + width).
struct Copy2D {
    int64_t count = 0, height = 0, width = 0, pitch = 0, first = 0, outer = 0;
};

inline Copy2D copy2d_plan(int ndims, const int64_t *ext, int64_t elem, int s, int64_t lo, int64_t hi) {
    Copy2D c;
    if (hi <= lo) return c;
    int64_t inner = 1;
    for (int k = s + 1; k < ndims; k++) inner *= ext[k];
    c.width = (hi - lo) * inner * elem;
    c.first = lo * inner * elem;
    if (s == 0) {
        c.count = c.height = 1;
        c.pitch = c.outer = c.width;
        return c;
    }
    c.height = ext[s - 1];
    c.pitch = ext[s] * inner * elem;
    c.outer = c.height * c.pitch;
    c.count = 1;
    for (int k = 0; k < s - 1; k++) c.count *= ext[k];
    return c;
}

// ---------------------------------------------------------------------------
// loop descriptors (D12) and per-device plans
// ---------------------------------------------------------------------------
struct ArgInfo {
    Region *reg = nullptr;
    int64_t off = 0;  // element offset of the loop's array inside the region
    int kind = 0;
};

struct Foot {  // read footprint: region, element interval
    Region *reg;
    int64_t lo, hi;
};

struct DevPlan {
    bool active = false;
    int64_t i0 = 0, i1 = 0, j0 = 0, j1 = 0;  // iteration sub-range
    int64_t k0 = 0, k1 = 0;                  // (3-D loops)
    int64_t it0 = 0, it1 = 0;                // iteration block (iteration-split scatter)
    int64_t w2lo = 0, w2hi = 0;              // owned block of the second written array
    int64_t blo[3] = {0, 0, 0}, bhi[3] = {0, 0, 0};  // write box (box loops)
    std::vector<std::pair<int64_t, int64_t>> wbox;   // exact write intervals (split dim > 0)
    int64_t wlo = 0, whi = 0;                // write bound (elements of written region), [wlo,whi)
    int64_t own_lo = 0, own_hi = 0;          // owned block of the split extent
    std::vector<Foot> reads;
};

struct Desc {
    int id;
    const char *name;
    int nargs;
    int kinds[9];
    size_t elems[9];   // required element sizes (0 = n/a)
    int out_arg;       // index of written array (-1 none)
    bool reduction;
    int halo_rows;     // stencil radius along the split dim (HALO prediction)
    int out2 = -1;     // second written array (Fig. 4 chain), -1 none
};

inline const Desc kDescs[] = {
    {JACC_LOOP_SQUARE_F32, "square_f32", 2, {JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_OUT, 0}, {4, 4, 0}, 1, false, 0},
    {JACC_LOOP_JACOBI2D_F64, "jacobi2d_f64", 2, {JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_OUT, 0}, {8, 8, 0}, 1, false, 1},
    {JACC_LOOP_DOT_F64, "dot_f64", 3, {JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_IN, JACC_ARG_REDUCE_SUM_F64}, {8, 8, 0}, -1, true, 0},
    {JACC_LOOP_SUM_F64, "sum_f64", 2, {JACC_ARG_ARRAY_IN, JACC_ARG_REDUCE_SUM_F64, 0}, {8, 0, 0}, -1, true, 0},
    {JACC_LOOP_GEMM_F64, "gemm_f64", 3, {JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_OUT}, {8, 8, 8}, 2, false, 0},
    {JACC_LOOP_SCATTER_ADD_F64, "scatter_add_f64", 3, {JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_INOUT}, {4, 8, 8}, 2, false, 0},
    {JACC_LOOP_SCATTER_ADD_I32, "scatter_add_i32", 3, {JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_INOUT}, {4, 4, 4}, 2, false, 0},
    {JACC_LOOP_HIMENO_F32, "himeno_f32", 9,
     {JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_IN,
      JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_OUT, JACC_ARG_REDUCE_SUM_F64, JACC_ARG_SCALAR_F64},
     {4, 4, 4, 4, 4, 4, 4, 0, 0}, 6, true, 0},
    {JACC_LOOP_HIMENO_COPY_F32, "himeno_copy_f32", 2, {JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_OUT}, {4, 4}, 1, false, 1},
    {JACC_LOOP_FIG4_F64, "fig4_f64", 6,
     {JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_IN, JACC_ARG_ARRAY_OUT, JACC_ARG_ARRAY_OUT,
      JACC_ARG_SCALAR_F64},
     {4, 4, 8, 8, 8, 0}, 3, false, 0, 4},
};

inline const Desc *find_desc(int id) {
    for (auto &d : kDescs)
        if (d.id == id) return &d;
    return nullptr;
}

inline void invalid_if(bool c) {
    if (c) throw Fail{JACC_ERR_INVALID};
}

// ---------------------------------------------------------------------------
// the launch
// ---------------------------------------------------------------------------
struct Launch {
    const Desc *D;
    std::vector<ArgInfo> a;
    jacc_range rg;
    bool dup = false;
    std::vector<DevPlan> plan;
    double *red_ptr = nullptr;
    // loop-specific shapes
    int64_t n1 = 0;            // 1-D length (square, dot, sum, scatter iterations)
    int64_t N = 0;             // jacobi grid
    int64_t M = 0, Nn = 0, K = 0;  // gemm
    int64_t HI = 0, HJ = 0, HK = 0;  // himeno grid
    int split = 0;                   // split dimension of the written array (A18)
    bool itersplit = false;          // NEXT-3 iteration-split scatter
    double scalar = 0;               // SCALAR_F64 argument (himeno omega)
};


// ---------------------------------------------------------------------------
// planning (plan.cpp), adaptive feedback and the launch (launch.cpp)
// ---------------------------------------------------------------------------
void box_intervals(int nd, const int64_t *ext, const int64_t *lo, const int64_t *hi, int64_t base,
                   std::vector<std::pair<int64_t, int64_t>> &out);
bool is_box_loop(int id);
std::vector<std::pair<int64_t, int64_t>> write_intervals(const DevPlan &p);
void slab_box(const Launch &L, const DevPlan &p, int64_t x, int64_t *lo, int64_t *hi);
jk::Box2D make_box2d(const Region *r, int nb, const int64_t *lo, const int64_t *hi);
void plan_launch(Launch &L);
void halo_targets(const Launch &L, int d, int &top, int &bot);
void poll_adaptive(bool block);
jacc_status do_launch(int loop_id, const jacc_range *range, const jacc_arg *args, int nargs,
                      int async_id);

}  // namespace jrt
