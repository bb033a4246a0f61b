// Probe: the apply phase of the binned scatter (pairs already grouped by
// bucket of `a`), L2 fp64 atomics vs a thread-block cluster whose shared
// memories hold one bucket of `a` (DSMEM remote fp64 adds).  Timing only;
// not part of the product.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//   -o /tmp/scat_apply_probe tools/scat_apply_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
namespace cg = cooperative_groups;
typedef unsigned long long u64;

__device__ __forceinline__ u64 mix(u64 x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// pairs grouped by bucket of 2^lb elements: exactly 2^lb pairs per bucket
__global__ void gen(int32_t *k, double *v, int64_t n, int lb) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const u64 h = mix((u64)p);
        k[p] = (int32_t)(((p >> lb) << lb) | (int64_t)(h & ((1ull << lb) - 1)));
        v[p] = (double)(h >> 54) / 1024.0;
    }
}

constexpr int CH = 4096;
__global__ void __launch_bounds__(256) apply_l2(const int32_t *__restrict__ pk,
                                                const double *__restrict__ pv, int64_t m,
                                                u64 *work, double *a, uint8_t *bm, int useb) {
    __shared__ u64 chunk;
    const int64_t nch = (m + CH - 1) / CH;
    for (;;) {
        if (threadIdx.x == 0) chunk = atomicAdd(work, 1ull);
        __syncthreads();
        const int64_t c = (int64_t)chunk;
        __syncthreads();
        if (c >= nch) break;
        const int64_t p0 = c * CH, p1 = p0 + CH < m ? p0 + CH : m;
#pragma unroll 4
        for (int64_t p = p0 + threadIdx.x; p < p1; p += 256) {
            const int32_t k = __ldcs(pk + p);
            atomicAdd(a + k, __ldcs(pv + p));
            if (useb) bm[k] = 1;
        }
    }
}


// dirty bits kept in a shared-memory window of 2^WB elements aligned at the
// chunk's first key; merged with one word-OR per window word per chunk
template <int WB>
__global__ void __launch_bounds__(256) apply_l2_sbits(const int32_t *__restrict__ pk,
                                                      const double *__restrict__ pv, int64_t m,
                                                      int ch, u64 *work, double *a, uint32_t *bits) {
    __shared__ uint32_t sb[1 << (WB - 5)];
    __shared__ u64 chunk;
    const int64_t nch = (m + ch - 1) / ch;
    for (;;) {
        if (threadIdx.x == 0) chunk = atomicAdd(work, 1ull);
        for (int i = threadIdx.x; i < (1 << (WB - 5)); i += 256) sb[i] = 0;
        __syncthreads();
        const int64_t c = (int64_t)chunk;
        if (c >= nch) break;
        const int64_t p0 = c * ch, p1 = p0 + ch < m ? p0 + ch : m;
        const int64_t w0 = ((int64_t)__ldg(pk + p0) >> WB) << WB;
#pragma unroll 4
        for (int64_t p = p0 + threadIdx.x; p < p1; p += 256) {
            const int32_t k = __ldcs(pk + p);
            atomicAdd(a + k, __ldcs(pv + p));
            const int64_t o = (int64_t)k - w0;
            if (o >= 0 && o < (1 << WB)) atomicOr(&sb[o >> 5], 1u << (o & 31));
            else atomicOr(&bits[k >> 5], 1u << (k & 31));
        }
        __syncthreads();
        for (int i = threadIdx.x; i < (1 << (WB - 5)); i += 256)
            if (sb[i]) atomicOr(&bits[(w0 >> 5) + i], sb[i]);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) apply_l2_gor(const int32_t *__restrict__ pk,
                                                    const double *__restrict__ pv, int64_t m,
                                                    u64 *work, double *a, uint32_t *bits) {
    __shared__ u64 chunk;
    const int64_t nch = (m + CH - 1) / CH;
    for (;;) {
        if (threadIdx.x == 0) chunk = atomicAdd(work, 1ull);
        __syncthreads();
        const int64_t c = (int64_t)chunk;
        __syncthreads();
        if (c >= nch) break;
        const int64_t p0 = c * CH, p1 = p0 + CH < m ? p0 + CH : m;
#pragma unroll 4
        for (int64_t p = p0 + threadIdx.x; p < p1; p += 256) {
            const int32_t k = __ldcs(pk + p);
            atomicAdd(a + k, __ldcs(pv + p));
            atomicOr(&bits[k >> 5], 1u << (k & 31));
        }
    }
}

// cluster of C CTAs; CTA r holds a[e0 + r*L, e0 + (r+1)*L) of bucket e0 = B*C*L
template <int C, int L, int MODE>
__global__ void __launch_bounds__(512) apply_dsm(const int32_t *__restrict__ pk,
                                                 const double *__restrict__ pv, int64_t nbk,
                                                 double *a, uint32_t *bits) {
    extern __shared__ __align__(16) unsigned char sm[];
    double *sa = reinterpret_cast<double *>(sm);
    uint8_t *sf = sm + L * 8;
    cg::cluster_group cl = cg::this_cluster();
    const int r = (int)cl.block_rank();
    const int64_t ncl = gridDim.x / C, cid = blockIdx.x / C;
    const int64_t BS = (int64_t)C * L;
    for (int64_t B = cid; B < nbk; B += ncl) {
        const int64_t e0 = B * BS + (int64_t)r * L;
        const double2 *src = reinterpret_cast<const double2 *>(a + e0);
        for (int i = threadIdx.x; i < L / 2; i += blockDim.x) reinterpret_cast<double2 *>(sa)[i] = src[i];
        for (int i = threadIdx.x; i < L / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sf)[i] = make_uint4(0, 0, 0, 0);
        cl.sync();
        // this CTA's share of the bucket's BS pairs
        const int64_t q0 = B * BS + (int64_t)r * L, q1 = q0 + L;
#pragma unroll 4
        for (int64_t p = q0 + threadIdx.x; p < q1; p += blockDim.x) {
            const int32_t k = __ldcs(pk + p);
            const double v = __ldcs(pv + p);
            const int64_t off = (int64_t)k - B * BS;
            const unsigned dr = (unsigned)(off / L), o = (unsigned)(off % L);
            if (MODE == 0) {
                double *rp = cl.map_shared_rank(sa, dr);
                atomicAdd(rp + o, v);
                uint8_t *rf = cl.map_shared_rank(sf, dr);
                rf[o] = 1;
            } else {
                unsigned la = (unsigned)__cvta_generic_to_shared(sa + o), ra;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(dr));
                asm volatile("red.shared::cluster.add.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
                unsigned lf = (unsigned)__cvta_generic_to_shared(sf + o), rf;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rf) : "r"(lf), "r"(dr));
                asm volatile("st.shared::cluster.u8 [%0], %1;" ::"r"(rf), "h"((unsigned short)1) : "memory");
            }
        }
        cl.sync();
        double2 *dst = reinterpret_cast<double2 *>(a + e0);
        for (int i = threadIdx.x; i < L / 2; i += blockDim.x) dst[i] = reinterpret_cast<double2 *>(sa)[i];
        for (int w = threadIdx.x; w < L / 32; w += blockDim.x) {
            const uint4 *f = reinterpret_cast<const uint4 *>(sf + 32 * w);
            const uint4 q0 = f[0], q1 = f[1];
            const uint32_t wd[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
            uint32_t b = 0;
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 4; j++)
                    if ((wd[i] >> (8 * j)) & 0xffu) b |= 1u << (4 * i + j);
            bits[e0 / 32 + w] = b;
        }
        __syncthreads();
    }
}

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

template <int C, int L, int MODE>
int run_dsm(const int32_t *k, const double *v, int64_t n, double *a, uint32_t *bits) {
    auto kern = apply_dsm<C, L, MODE>;
    const int smem = L * 9;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (C > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(C);
    int ncl = 0;
    CK(cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg));
    cfg.gridDim = dim3(ncl * C);
    const int64_t nbk = n / ((int64_t)C * L);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    CK(cudaLaunchKernelEx(&cfg, kern, k, v, nbk, a, bits));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < 5; i++) CK(cudaLaunchKernelEx(&cfg, kern, k, v, nbk, a, bits));
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("dsm C=%d L=%d mode=%d clusters=%d: %.3f ms\n", C, L, MODE, ncl, ms / 5);
    return 0;
}

int main() {
    const int64_t n = 1ll << 28;
    int32_t *k;
    double *v, *a;
    uint8_t *bm;
    uint32_t *bits;
    u64 *work;
    CK(cudaMalloc(&k, n * 4));
    CK(cudaMalloc(&v, n * 8));
    CK(cudaMalloc(&a, n * 8));
    CK(cudaMalloc(&bm, n));
    CK(cudaMalloc(&bits, n / 8));
    CK(cudaMalloc(&work, 8));
    CK(cudaMemset(a, 0, n * 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char *name, auto fn) {
        float tot = 0;
        for (int it = 0; it < 6; it++) {
            cudaMemset(work, 0, 8);
            cudaMemset(bits, 0, n / 8);
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaDeviceSynchronize();
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it) tot += ms;
        }
        cudaError_t e = cudaGetLastError();
        printf("%s: %.3f ms %s\n", name, tot / 5, e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    char nm[128];
    for (int lb : {21, 18, 17}) {
        gen<<<148 * 8, 256>>>(k, v, n, lb);
        for (int useb = 1; useb >= 0; useb--) {
            snprintf(nm, sizeof nm, "l2 bucket 2^%d bytemap=%d", lb, useb);
            timeit(nm, [&] { apply_l2<<<148 * 8, 256>>>(k, v, n, work, a, bm, useb); });
        }
        snprintf(nm, sizeof nm, "l2 bucket 2^%d global RED.OR bits", lb);
        timeit(nm, [&] { apply_l2_gor<<<148 * 8, 256>>>(k, v, n, work, a, bits); });
        for (int ch : {8192, 16384, 32768}) {
            if (lb <= 18) {
                snprintf(nm, sizeof nm, "l2 bucket 2^%d smem bits win 2^%d ch %d", lb, lb, ch);
                if (lb == 18) timeit(nm, [&] { apply_l2_sbits<18><<<148 * 6, 256>>>(k, v, n, ch, work, a, bits); });
                if (lb == 17) timeit(nm, [&] { apply_l2_sbits<17><<<148 * 8, 256>>>(k, v, n, ch, work, a, bits); });
            }
        }
    }
    return 0;
}
