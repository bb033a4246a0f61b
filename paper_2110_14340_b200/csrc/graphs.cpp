// graphs.cpp -- CUDA graphs of launch sequences (capture, replay with the validity snapshot)
#include "rt.hpp"

using namespace jrt;

extern "C" {

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
        // back-to-back replays need the graph to map the captured state onto
        // itself (its pulls were planned for S_start)
        if (count > 1) {
            for (auto &kv : R.table)
                for (int d = 0; d < R.n; d++)
                    if (g.v_end[kv.second.get()][d].iv != g.v_start[kv.second.get()][d].iv)
                        return JACC_ERR_STATE;
        }
        // dirty-record slots: the first captured launch of each region writes
        // slot start^1, which the previous launch must have cleared.  When a
        // region is written an odd number of times per replay the slot parity
        // flips, so each replay gets its own clear.
        bool flips = false;
        for (auto &kv : R.table)
            for (int d = 0; d < R.n; d++)
                flips |= g.slot_end[kv.second.get()][d] != g.slot_start[kv.second.get()][d];
        for (int k = 0; k < count; k++) {
            bool cleared = false;
            for (auto &kv : R.table) {
                Region *r = kv.second.get();
                for (int d = 0; d < R.n; d++)
                    if (r->dslot[d] != g.slot_start[r][d]) {
                        set_dev(d);
                        CK(cudaMemsetAsync(r->dirty[d] + 2 * (g.slot_start[r][d] ^ 1), 0xff, 16,
                                           R.dev[d].s));
                        cleared = true;
                    }
            }
            if (k == 0 || cleared) join_into(0);
            set_dev(0);
            if (!flips) {  // parity stable: all replays back to back
                for (; k < count; k++) CK(cudaGraphLaunch(g.exec, R.dev[0].s));
                break;
            }
            CK(cudaGraphLaunch(g.exec, R.dev[0].s));
            // the replay's last writes leave the slots of S_end; the other
            // device streams follow device 0 before the next clear
            for (auto &kv : R.table) kv.second->dslot = g.slot_end[kv.second.get()];
            if (k + 1 < count) {
                cudaEvent_t e = pool_event();
                CK(cudaEventRecord(e, R.dev[0].s));
                for (int d = 1; d < R.n; d++) {
                    set_dev(d);
                    CK(cudaStreamWaitEvent(R.dev[d].s, e, 0));
                }
                R.evpool.push_back(e);
            }
        }
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
        if (R.graphs.empty())  // scratch a graph might still have referenced
            for (int d = 0; d < R.n; d++) {
                if (R.dev[d].retired.empty()) continue;
                set_dev(d);
                CK(cudaStreamSynchronize(R.dev[d].s));
                for (void *p : R.dev[d].retired) CK(cudaFree(p));
                R.dev[d].retired.clear();
            }
        return JACC_OK;
    });
}


}  // extern "C"
