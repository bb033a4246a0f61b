// Probe: shared-memory update throughput on sm_100a (random addresses in a
// 16K-element fp64 slice): fp64 atomicAdd (CAS loop), u32 atomicAdd, plain
// racy load-add-store, and warp match_any.  Timing only; not product code.
#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
__device__ __forceinline__ unsigned hsh(unsigned x) { x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; return x ^ (x >> 16); }
template <int MODE>
__global__ void __launch_bounds__(512) k(double *out, int iters) {
    __shared__ double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0;
    __syncthreads();
    unsigned x = blockIdx.x * 1024 + threadIdx.x;
    unsigned acc = 0;
    for (int it = 0; it < iters; it++) {
        x = hsh(x + it);
        const unsigned o = x & 4095;
        if (MODE == 0) atomicAdd(&s[o], 1.0);
        else if (MODE == 1) atomicAdd(reinterpret_cast<unsigned *>(s) + o, 1u);
        else if (MODE == 2) { s[o] = s[o] + 1.0; }
        else if (MODE == 3) { acc += __match_any_sync(0xffffffffu, o >> 7); }
        else if (MODE == 4) { atomicOr(reinterpret_cast<unsigned *>(s) + (o >> 5), 1u << (o & 31)); }
    }
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = s[threadIdx.x] + acc;
}
int main() {
    double *o;
    cudaMalloc(&o, 148 * 4 * 512 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096;
    const char *nm[] = {"f64 atomicAdd (CAS)", "u32 atomicAdd", "plain f64 RMW", "match_any", "u32 atomicOr"};
    for (int m = 0; m < 5; m++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(a);
            if (m == 0) k<0><<<148, 512>>>(o, iters);
            if (m == 1) k<1><<<148, 512>>>(o, iters);
            if (m == 2) k<2><<<148, 512>>>(o, iters);
            if (m == 3) k<3><<<148, 512>>>(o, iters);
            if (m == 4) k<4><<<148, 512>>>(o, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("%-22s %.3f ms  %.2f G updates/s/SM  (%.2f lanes/clk/SM at 1.9 GHz)\n", nm[m], ms,
                            512.0 * iters / (ms * 1e6), 512.0 * iters / (ms * 1e-3) / 1.9e9);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
