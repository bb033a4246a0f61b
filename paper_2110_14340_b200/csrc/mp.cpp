// mp.cpp -- one process per GPU: bootstrap, CUDA-IPC replica and event exchange,
//  shared-memory lockstep
#include "rt.hpp"

using namespace jrt;

extern "C" {

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
        static_assert(3 * sizeof(cudaIpcMemHandle_t) + 16 <= JACC_RUNTIME_HANDLE_BYTES, "handle size");
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
        // the GPU's UUID: importers learn whether two ranks share a GPU
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, dv.ord));
        memcpy(o + 192, &prop.uuid, 16);
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
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, R.dev[R.me].ord));
        if (!memcmp(p + 192, &prop.uuid, 16)) R.distinct = false;  // reported by jacc_get_info
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


}  // extern "C"
