// Probe: global RED throughput on sm_100a for the scatter apply phase.
// Random 8-byte (or 4-byte) REDs into a window of `a` that slides with a
// global chunk counter (the binned apply's access pattern), with keys either
// hashed in registers (RED issue only) or loaded from a pair stream (the
// apply).  Timing only; not product code.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/red_probe tools/red_probe.cu
#include <cstdint>
#include <cstdio>
typedef unsigned long long u64;

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    return x ^ (x >> 16);
}

// MODE 0: hashed keys (no loads); 1: keys+vals loaded from the pair stream
// (pairs grouped by window, like the partition's output); 2: MODE 1 with all
// of a thread's loads issued before its REDs (PER pairs per thread per chunk)
template <typename T, int MODE, int PER>
__global__ void apply(const int32_t *__restrict__ pk, const T *__restrict__ pv, int64_t m,
                      int ch, int lw, u64 *work, T *a) {
    __shared__ u64 chunk;
    const int64_t nch = (m + ch - 1) / ch;
    for (;;) {
        if (threadIdx.x == 0) chunk = atomicAdd(work, 1ull);
        __syncthreads();
        const int64_t c = (int64_t)chunk;
        __syncthreads();
        if (c >= nch) break;
        const int64_t p0 = c * ch;
        const int64_t p1 = p0 + ch < m ? p0 + ch : m;
        if (MODE == 0) {
            const int64_t w0 = (p0 >> lw) << lw;
            for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
                const int32_t k = (int32_t)(w0 + (hsh((uint32_t)p) & ((1u << lw) - 1)));
                atomicAdd(a + k, (T)1);
            }
        } else if (MODE == 1) {
#pragma unroll 4
            for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
                const int32_t k = __ldcs(pk + p);
                atomicAdd(a + k, __ldcs(pv + p));
            }
        } else {
            for (int64_t q = p0 + threadIdx.x; q < p1; q += (int64_t)blockDim.x * PER) {
                int32_t k[PER];
                T v[PER];
#pragma unroll
                for (int j = 0; j < PER; j++) {
                    const int64_t p = q + (int64_t)j * blockDim.x;
                    k[j] = p < p1 ? __ldcs(pk + p) : -1;
                }
#pragma unroll
                for (int j = 0; j < PER; j++) {
                    const int64_t p = q + (int64_t)j * blockDim.x;
                    if (p < p1) v[j] = __ldcs(pv + p);
                }
#pragma unroll
                for (int j = 0; j < PER; j++)
                    if (k[j] >= 0) atomicAdd(a + k[j], v[j]);
            }
        }
    }
}

template <typename T>
__global__ void gen(int32_t *k, T *v, int64_t n, int lw) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t h = hsh((uint32_t)p * 2654435761u + 12345u);
        k[p] = (int32_t)(((p >> lw) << lw) | (int64_t)(h & ((1u << lw) - 1)));
        v[p] = (T)(h >> 22);
    }
}

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            printf("%s: %s\n", #x, cudaGetErrorString(e_));                                \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

template <typename T, int MODE, int PER>
int run(const char *name, const int32_t *k, const T *v, int64_t n, int lw, T *a, u64 *work,
        int thr, int bps, int ch) {
    auto kern = apply<T, MODE, PER>;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; rep++) {
        CK(cudaMemsetAsync(work, 0, 8));
        cudaEventRecord(e0);
        kern<<<148 * bps, thr>>>(k, v, n, ch, lw, work, a);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
    }
    CK(cudaGetLastError());
    printf("%-10s elem=%zu window=2^%d thr=%4d bps=%d ch=%5d : %.3f ms  %.1f G RED/s\n", name,
           sizeof(T), lw, thr, bps, ch, best, n / (best * 1e6));
    return 0;
}

int main() {
    const int64_t n = 1ll << 28;
    int32_t *k;
    double *v, *a;
    u64 *work;
    CK(cudaMalloc(&k, n * 4));
    CK(cudaMalloc(&v, n * 8));
    CK(cudaMalloc(&a, n * 8));
    CK(cudaMalloc(&work, 8));
    CK(cudaMemset(a, 0, n * 8));
    const int lws[] = {17, 20, 22};
    for (int lw : lws) {
        gen<double><<<148 * 8, 256>>>(k, v, n, lw);
        CK(cudaDeviceSynchronize());
        for (int cfg = 0; cfg < 6; cfg++) {
            const int thr[] = {256, 256, 256, 512, 1024, 256};
            const int bps[] = {2, 3, 4, 2, 1, 8};
            run<double, 0, 1>("hash-f64", k, v, n, lw, a, work, thr[cfg], bps[cfg], 4096);
            run<double, 1, 1>("load-f64", k, v, n, lw, a, work, thr[cfg], bps[cfg], 4096);
            run<double, 2, 4>("batch4-f64", k, v, n, lw, a, work, thr[cfg], bps[cfg], 4096);
            run<double, 2, 8>("batch8-f64", k, v, n, lw, a, work, thr[cfg], bps[cfg], 8192);
        }
    }
    // 4-byte REDs (the int32 scatter)
    int32_t *vi = reinterpret_cast<int32_t *>(v), *ai = reinterpret_cast<int32_t *>(a);
    gen<int32_t><<<148 * 8, 256>>>(k, vi, n, 21);
    CK(cudaDeviceSynchronize());
    for (int cfg = 0; cfg < 3; cfg++) {
        const int thr[] = {256, 256, 512};
        const int bps[] = {3, 4, 2};
        run<int32_t, 0, 1>("hash-i32", k, vi, n, 21, ai, work, thr[cfg], bps[cfg], 4096);
        run<int32_t, 1, 1>("load-i32", k, vi, n, 21, ai, work, thr[cfg], bps[cfg], 4096);
        run<int32_t, 2, 4>("batch4-i32", k, vi, n, 21, ai, work, thr[cfg], bps[cfg], 4096);
    }
    return 0;
}
