// runtime.cpp -- host runtime of libjacc.so: the C-ABI of include/jacc.h.
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

namespace {

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
    std::vector<uint8_t *> bytemap;    // per device epoch byte-map (binned scatter)
    std::vector<char *> delta;         // per device delta array (iteration-split scatter)
    std::vector<uint32_t *> dbm;       // per device delta bitmap
    std::vector<uint8_t> epoch;
    std::vector<IntervalSet> valid;    // per device
};

struct ProfRec {
    int dev;
    cudaEvent_t k0, k1, m1;
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
    std::vector<std::vector<char>> comm_prev;  // [d][q]
    bool profiling = false;
    std::vector<ProfRec> prof;                 // unresolved event records
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

Runtime R;

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
struct Fail {
    jacc_status st;
};

void cuda_check(cudaError_t e, const char *what) {
    if (e != cudaSuccess) {
        if (getenv("JACC_DEBUG")) fprintf(stderr, "[jacc] %s: %s\n", what, cudaGetErrorString(e));
        R.poisoned = true;
        throw Fail{JACC_ERR_CUDA};
    }
}
#define CK(x) cuda_check((x), #x)

void nccl_check(ncclResult_t e, const char *what) {
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

Region *lookup(const void *p) {
    uintptr_t a = (uintptr_t)p;
    auto it = R.table.upper_bound(a);
    if (it == R.table.begin()) return nullptr;
    --it;
    Region *r = it->second.get();
    return (a >= r->base && a < r->base + r->bytes) ? r : nullptr;
}

bool local(int d) { return !R.mp || d == R.me; }

void set_dev(int d) { CK(cudaSetDevice(R.dev[d].ord)); }

// spin on a shared-memory predicate with a generous timeout (a dead peer
// must not hang the caller forever)
template <typename P>
void spin_until(P pred) {
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

uint64_t shm_load(const uint64_t *p) { return __atomic_load_n(p, __ATOMIC_ACQUIRE); }
void shm_store(uint64_t *p, uint64_t v) { __atomic_store_n(p, v, __ATOMIC_RELEASE); }

// host barrier across ranks (multi-process mode only)
void rank_barrier() {
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
void wait_launches(uint64_t k) {
    if (!R.mp) return;
    spin_until([&] {
        for (int q = 0; q < R.n; q++)
            if (shm_load(&R.shm[q].launches) < k) return false;
        return true;
    });
}

// drain this process's device streams
void local_sync() {
    for (int d = 0; d < R.n; d++) {
        if (!local(d)) continue;
        set_dev(d);
        CK(cudaStreamSynchronize(R.dev[d].s));
        for (size_t q = 1; q < R.dev[d].qs.size(); q++) CK(cudaStreamSynchronize(R.dev[d].qs[q]));
    }
}

// drain every device's work (collective across ranks in multi-process mode)
void sync_all() {
    local_sync();
    rank_barrier();
}

cudaEvent_t pool_event() {
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
void flush_prof() {
    if (R.prof.empty()) return;
    double kmax = 0, mmax = 0;
    for (size_t i = 0; i < R.prof.size(); i++) {
        auto &p = R.prof[i];
        set_dev(p.dev);
        CK(cudaEventSynchronize(p.m1));
        float k = 0, m = 0;
        CK(cudaEventElapsedTime(&k, p.k0, p.k1));
        CK(cudaEventElapsedTime(&m, p.k1, p.m1));
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
    R.prof.clear();
    R.last_start = 0;
}

void free_region(Region *r) {
    for (int d = 0; d < (int)r->rep.size(); d++) {
        if (!local(d)) {
            if (r->rep[d]) cudaIpcCloseMemHandle(r->rep[d]);
            continue;
        }
        set_dev(d);
        if (r->rep[d]) cudaFree(r->rep[d]);
        if (r->dirty[d]) cudaFree(r->dirty[d]);
        if (r->bitmap[d]) cudaFree(r->bitmap[d]);
        if (r->bytemap[d]) cudaFree(r->bytemap[d]);
        if (r->delta[d]) cudaFree(r->delta[d]);
        if (r->dbm[d]) cudaFree(r->dbm[d]);
    }
    if (r->pinned) cudaHostUnregister((void *)r->base);
}

void destroy_graph(GraphRec &g) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    g = GraphRec{};
}

// c4 partition ("equally dividing"; S:266 remainder rule)
void partition(int64_t E, int n, int d, int64_t &lo, int64_t &hi) {
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

Copy2D copy2d_plan(int ndims, const int64_t *ext, int64_t elem, int s, int64_t lo, int64_t hi) {
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

const Desc kDescs[] = {
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

const Desc *find_desc(int id) {
    for (auto &d : kDescs)
        if (d.id == id) return &d;
    return nullptr;
}

void invalid_if(bool c) {
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
    if (L.itersplit && (R.mp || R.nq > 1)) return JACC_ERR_INVALID;
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
    const bool multiq = R.nq > 1;
    if (multiq) {
        std::vector<int64_t> rd, wr;
        for (int k = 0; k < nargs; k++) {
            if (!L.a[k].reg) continue;
            const int64_t key = (int64_t)(uintptr_t)L.a[k].reg;
            if (L.a[k].kind == JACC_ARG_ARRAY_IN || L.a[k].kind == JACC_ARG_ARRAY_INOUT) rd.push_back(key);
            if (L.a[k].kind == JACC_ARG_ARRAY_OUT || L.a[k].kind == JACC_ARG_ARRAY_INOUT) wr.push_back(key);
        }
        std::vector<int> waits;
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
            const jk::ScatterPlan sp = jk::scatter_plan(p.i1 - p.i0, lo, hi, (int)W->elem);
            if (!sp.binned) continue;
            Device &dv = R.dev[d];
            set_dev(d);
            if (dv.scratch_bytes < sp.scratch) {
                CK(cudaStreamSynchronize(dv.s));
                if (dv.scratch) CK(cudaFree(dv.scratch));
                dv.scratch = nullptr;
                dv.scratch_bytes = 0;
                if (cudaMalloc(&dv.scratch, sp.scratch) == cudaSuccess) dv.scratch_bytes = sp.scratch;
                else cudaGetLastError();
            }
            const size_t bmap = (size_t)((W->nelem + 31) / 32) * 32;  // whole region
            if (!W->bytemap[d]) {
                if (cudaMalloc(&W->bytemap[d], bmap) == cudaSuccess) {
                    CK(cudaMemsetAsync(W->bytemap[d], 0, bmap, dv.s));
                    W->epoch[d] = 0;
                } else {
                    W->bytemap[d] = nullptr;
                    cudaGetLastError();
                }
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
            if (!multiq)
                for (int q = 0; q < n; q++)
                    if (q != d && (comm[d][q] || R.comm_prev[d][q]))
                        CK(cudaStreamWaitEvent(dv.s, R.dev[q].ev[prev], 0));
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
            if (!p.active) CK(cudaMemsetAsync(drec, 0xff, 16, dv.s));  // nothing will write it
        }
        u64 *drec2 = nullptr;
        if (W2) {
            W2->dslot[d] ^= 1;
            drec2 = W2->dirty[d] + 2 * W2->dslot[d];
            if (!p.active) CK(cudaMemsetAsync(drec2, 0xff, 16, dv.s));
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
                jk::ScatterPlan sp = jk::scatter_plan(p.i1 - p.i0, lo, hi, (int)W->elem);
                if (R.capturing) sp.binned = false;  // epoch byte-map state is host-side
                if (R.nq > 1) sp.binned = false;     // per-device scratch is not per queue
                if (sp.binned && (dv.scratch_bytes < sp.scratch || !W->bytemap[d]))
                    sp.binned = false;  // scratch could not be reserved up front: direct kernel
                if (sp.binned) {
                    if (W->epoch[d] == 255) {  // wrap: clear stale epochs
                        CK(cudaMemsetAsync(W->bytemap[d], 0, (size_t)((W->nelem + 31) / 32) * 32, dv.s));
                        W->epoch[d] = 0;
                    }
                    W->epoch[d]++;
                    CK(jk::scatter_add_binned(dv.s, f64, ix, b, W->rep[d], p.i1 - p.i0, lo, hi, bm,
                                              drec, sp, dv.scratch, W->bytemap[d],
                                              W->epoch[d]));
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

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
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
                }
            if (n_devices > 1 && R.distinct && !getenv("JACC_NO_NCCL")) {
                // NCCL allreduce for the reduction combine; if the communicator
                // cannot be built the fixed-order peer-memory combine (P2P
                // loads of every device's partial) is used instead
                std::vector<ncclComm_t> comms(n_devices);
                const ncclResult_t nr = ncclCommInitAll(comms.data(), n_devices, ords.data());
                if (nr == ncclSuccess) {
                    for (int d = 0; d < n_devices; d++) R.dev[d].comm = comms[d];
                    R.use_nccl = true;
                } else if (getenv("JACC_DEBUG")) {
                    fprintf(stderr, "[jacc] ncclCommInitAll: %s; peer-memory combine\n",
                            ncclGetErrorString(nr));
                }
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
        r->bytemap.assign(R.n, nullptr);
        r->delta.assign(R.n, nullptr);
        r->dbm.assign(R.n, nullptr);
        r->epoch.assign(R.n, 0);
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

jacc_status jacc_launch(int loop_id, const jacc_range *range, const jacc_arg *args, int nargs,
                        int async_id) {
    return guard([&]() { return do_launch(loop_id, range, args, nargs, async_id); });
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

// ---------------------------------------------------------------------------
// one process per GPU
// ---------------------------------------------------------------------------
jacc_status jacc_unique_id(void *out, size_t bytes) {
    if (!out || bytes < JACC_UNIQUE_ID_BYTES) return JACC_ERR_INVALID;
    static_assert(sizeof(ncclUniqueId) <= JACC_UNIQUE_ID_BYTES, "nccl id size");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return JACC_ERR_NCCL;
    memset(out, 0, bytes);
    memcpy(out, &id, sizeof(id));
    return JACC_OK;
}

jacc_status jacc_init_rank(int rank, int world, int cuda_ordinal, const void *unique_id,
                           const char *shm_name) {
    if (R.init) return JACC_ERR_STATE;
    return guard(
        [&]() -> jacc_status {
            int count = 0;
            if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1) return JACC_ERR_CUDA;
            if (world < 1 || world > JACC_MAX_DEVICES || rank < 0 || rank >= world ||
                cuda_ordinal < 0 || cuda_ordinal >= count || !shm_name || !*shm_name)
                return JACC_ERR_INVALID;
            R = Runtime{};
            R.n = world;
            R.mp = true;
            R.me = rank;
            R.dev.resize(world);
            R.init = true;
            const char *pol = getenv("JACC_MERGE");
            if (pol && !strcmp(pol, "halo")) R.policy = JACC_MERGE_HALO;
            // host progress counters (zero-filled on creation)
            R.shm_name = shm_name[0] == '/' ? shm_name : std::string("/") + shm_name;
            int fd = shm_open(R.shm_name.c_str(), O_CREAT | O_RDWR, 0600);
            if (fd < 0) return JACC_ERR_INVALID;
            const size_t sz = sizeof(Runtime::Slot) * JACC_MAX_DEVICES;
            if (ftruncate(fd, (off_t)sz) != 0) {
                close(fd);
                return JACC_ERR_INVALID;
            }
            void *m = mmap(nullptr, sz, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
            close(fd);
            if (m == MAP_FAILED) return JACC_ERR_INVALID;
            R.shm = static_cast<Runtime::Slot *>(m);
            Device &dv = R.dev[rank];
            dv.ord = cuda_ordinal;
            set_dev(rank);
            CK(cudaStreamCreateWithFlags(&dv.s, cudaStreamNonBlocking));
            for (int k = 0; k < 2; k++) {
                CK(cudaEventCreateWithFlags(&dv.ev[k], cudaEventDisableTiming | cudaEventInterprocess));
                CK(cudaEventRecord(dv.ev[k], dv.s));
            }
            CK(cudaMalloc(&dv.partials, jk::kHimenoPartials * sizeof(double)));
            CK(cudaMalloc(&dv.ticket, 64));
            CK(cudaMemset(dv.ticket, 0, 64));
            CK(cudaMalloc(&dv.part, 8));
            CK(cudaMalloc(&dv.res, 8));
            CK(cudaMemset(dv.part, 0, 8));
            CK(cudaMallocHost(&dv.hscal, 8));
            CK(cudaStreamSynchronize(dv.s));
            if (unique_id && world > 1) {
                ncclUniqueId id;
                memcpy(&id, unique_id, sizeof(id));
                NK(ncclCommInitRank(&dv.comm, world, id, rank));
                R.use_nccl = true;
            }
            R.comm_prev.assign(world, std::vector<char>(world, 0));
            return JACC_OK;
        },
        false);
}

jacc_status jacc_export_runtime(void *out, size_t bytes) {
    return guard([&]() -> jacc_status {
        if (!R.mp || !out || bytes < JACC_RUNTIME_HANDLE_BYTES) return JACC_ERR_INVALID;
        static_assert(3 * sizeof(cudaIpcMemHandle_t) <= JACC_RUNTIME_HANDLE_BYTES, "handle size");
        Device &dv = R.dev[R.me];
        set_dev(R.me);
        char *o = static_cast<char *>(out);
        memset(o, 0, bytes);
        cudaIpcEventHandle_t e0, e1;
        cudaIpcMemHandle_t mp;
        CK(cudaIpcGetEventHandle(&e0, dv.ev[0]));
        CK(cudaIpcGetEventHandle(&e1, dv.ev[1]));
        CK(cudaIpcGetMemHandle(&mp, dv.part));
        memcpy(o, &e0, sizeof(e0));
        memcpy(o + 64, &e1, sizeof(e1));
        memcpy(o + 128, &mp, sizeof(mp));
        return JACC_OK;
    });
}

jacc_status jacc_import_runtime(int peer, const void *in, size_t bytes) {
    return guard([&]() -> jacc_status {
        if (!R.mp || !in || bytes < JACC_RUNTIME_HANDLE_BYTES || peer < 0 || peer >= R.n ||
            peer == R.me)
            return JACC_ERR_INVALID;
        const char *p = static_cast<const char *>(in);
        Device &pv = R.dev[peer];
        set_dev(R.me);
        cudaIpcEventHandle_t e0, e1;
        cudaIpcMemHandle_t mp;
        memcpy(&e0, p, sizeof(e0));
        memcpy(&e1, p + 64, sizeof(e1));
        memcpy(&mp, p + 128, sizeof(mp));
        CK(cudaIpcOpenEventHandle(&pv.ev[0], e0));
        CK(cudaIpcOpenEventHandle(&pv.ev[1], e1));
        void *ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, mp, cudaIpcMemLazyEnablePeerAccess));
        pv.part = static_cast<double *>(ptr);
        pv.ord = -1;
        return JACC_OK;
    });
}

jacc_status jacc_export_region(void *host, void *out, size_t bytes) {
    return guard([&]() -> jacc_status {
        if (!R.mp || !out || bytes < JACC_REGION_HANDLE_BYTES) return JACC_ERR_INVALID;
        Region *r = lookup(host);
        if (!r) return JACC_ERR_NOT_PRESENT;
        set_dev(R.me);
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, r->rep[R.me]));
        memset(out, 0, bytes);
        memcpy(out, &h, sizeof(h));
        return JACC_OK;
    });
}

jacc_status jacc_import_region(void *host, int peer, const void *in, size_t bytes) {
    return guard([&]() -> jacc_status {
        if (!R.mp || !in || bytes < JACC_REGION_HANDLE_BYTES || peer < 0 || peer >= R.n ||
            peer == R.me)
            return JACC_ERR_INVALID;
        Region *r = lookup(host);
        if (!r) return JACC_ERR_NOT_PRESENT;
        if (r->rep[peer]) return JACC_ERR_STATE;
        set_dev(R.me);
        cudaIpcMemHandle_t h;
        memcpy(&h, in, sizeof(h));
        void *ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        r->rep[peer] = static_cast<char *>(ptr);
        return JACC_OK;
    });
}

int jacc_rank(void) { return R.init ? (R.mp ? R.me : 0) : -1; }

// ---------------------------------------------------------------------------
// CUDA graphs of launch sequences
// ---------------------------------------------------------------------------
namespace {
void snapshot(std::map<Region *, std::vector<IntervalSet>> &v, std::map<Region *, std::vector<int>> &sl) {
    v.clear();
    sl.clear();
    for (auto &kv : R.table) {
        v[kv.second.get()] = kv.second->valid;
        sl[kv.second.get()] = kv.second->dslot;
    }
}
bool same_validity(const std::map<Region *, std::vector<IntervalSet>> &v) {
    if (v.size() != R.table.size()) return false;
    for (auto &kv : R.table) {
        auto it = v.find(kv.second.get());
        if (it == v.end()) return false;
        for (int d = 0; d < R.n; d++)
            if (it->second[d].iv != kv.second->valid[d].iv) return false;
    }
    return true;
}
// make stream s (on device h) wait for every device's current work
void join_into(int h) {
    for (int d = 0; d < R.n; d++) {
        if (d == h) continue;
        set_dev(d);
        cudaEvent_t e = pool_event();
        CK(cudaEventRecord(e, R.dev[d].s));
        set_dev(h);
        CK(cudaStreamWaitEvent(R.dev[h].s, e, 0));
        R.evpool.push_back(e);  // safe: a recorded event may be re-recorded later
    }
}
}  // namespace

jacc_status jacc_graph_begin(void) {
    return guard([&]() -> jacc_status {
        if (R.mp || R.capturing || R.mode == JACC_MODE_ADAPTIVE || R.nq > 1) return JACC_ERR_INVALID;
        sync_all();
        flush_prof();
        R.cap = GraphRec{};
        snapshot(R.cap.v_start, R.cap.slot_start);
        // everything before the capture is complete: no waits on older events
        R.comm_prev.assign(R.n, std::vector<char>(R.n, 0));
        set_dev(0);
        CK(cudaStreamBeginCapture(R.dev[0].s, cudaStreamCaptureModeRelaxed));
        // fork: every other device stream joins the capture
        cudaEvent_t fork = pool_event();
        CK(cudaEventRecord(fork, R.dev[0].s));
        for (int d = 1; d < R.n; d++) {
            set_dev(d);
            CK(cudaStreamWaitEvent(R.dev[d].s, fork, 0));
        }
        R.evpool.push_back(fork);
        R.capturing = true;
        return JACC_OK;
    });
}

jacc_status jacc_graph_end(int *graph_id) {
    return guard([&]() -> jacc_status {
        if (!R.capturing || !graph_id) return JACC_ERR_INVALID;
        R.capturing = false;
        join_into(0);
        set_dev(0);
        cudaGraph_t g = nullptr;
        CK(cudaStreamEndCapture(R.dev[0].s, &g));
        R.cap.graph = g;
        CK(cudaGraphInstantiate(&R.cap.exec, g, 0));
        snapshot(R.cap.v_end, R.cap.slot_end);
        R.cap.comm_end = R.comm_prev;
        const int id = R.next_graph++;
        R.graphs[id] = R.cap;
        R.cap = GraphRec{};
        // the captured work has NOT run: restore the pre-capture state
        for (auto &kv : R.table) {
            Region *r = kv.second.get();
            r->valid = R.graphs[id].v_start[r];
            r->dslot = R.graphs[id].slot_start[r];
        }
        R.gen -= R.graphs[id].launches;
        R.comm_prev.assign(R.n, std::vector<char>(R.n, 0));
        // events last recorded inside the capture: re-record them outside
        for (int d = 0; d < R.n; d++) {
            set_dev(d);
            CK(cudaEventRecord(R.dev[d].ev[0], R.dev[d].s));
            CK(cudaEventRecord(R.dev[d].ev[1], R.dev[d].s));
        }
        *graph_id = id;
        return JACC_OK;
    });
}

jacc_status jacc_graph_replay(int graph_id, int count) {
    return guard([&]() -> jacc_status {
        auto it = R.graphs.find(graph_id);
        if (it == R.graphs.end() || count < 0 || R.capturing) return JACC_ERR_INVALID;
        GraphRec &g = it->second;
        if (!same_validity(g.v_start)) return JACC_ERR_STATE;  // not the captured state
        if (count == 0) return JACC_OK;
        // dirty-record slots: the first captured launch of each region writes
        // slot start^1, which the previous launch must have cleared
        for (auto &kv : R.table) {
            Region *r = kv.second.get();
            for (int d = 0; d < R.n; d++)
                if (r->dslot[d] != g.slot_start[r][d]) {
                    set_dev(d);
                    CK(cudaMemsetAsync(r->dirty[d] + 2 * (g.slot_start[r][d] ^ 1), 0xff, 16,
                                       R.dev[d].s));
                }
        }
        join_into(0);
        set_dev(0);
        for (int k = 0; k < count; k++) CK(cudaGraphLaunch(g.exec, R.dev[0].s));
        // order every device stream after the replay and refresh its event
        cudaEvent_t done = pool_event();
        CK(cudaEventRecord(done, R.dev[0].s));
        R.gen += g.launches * count;
        for (int d = 0; d < R.n; d++) {
            set_dev(d);
            if (d) CK(cudaStreamWaitEvent(R.dev[d].s, done, 0));
            CK(cudaEventRecord(R.dev[d].ev[(R.gen - 1) & 1], R.dev[d].s));
            R.dev[d].launches += (uint64_t)g.launches * count;
        }
        R.evpool.push_back(done);
        for (auto &kv : R.table) {
            Region *r = kv.second.get();
            r->valid = g.v_end[r];
            r->dslot = g.slot_end[r];
        }
        R.comm_prev = g.comm_end;
        return JACC_OK;
    });
}

jacc_status jacc_graph_destroy(int graph_id) {
    return guard([&]() -> jacc_status {
        auto it = R.graphs.find(graph_id);
        if (it == R.graphs.end()) return JACC_ERR_INVALID;
        destroy_graph(it->second);
        R.graphs.erase(it);
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
