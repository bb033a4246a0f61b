// Probe: BK5 merge kernel variants on one B200 (peer replica = another
// buffer on the same GPU, so every byte is an HBM read + write).  Range
// merge = contiguous copy of the recorded dirty span; bitmap merge = copy of
// exactly the elements whose dirty bit is set (dense ~63 % and sparse
// ~0.4 % bitmaps).  Timing only; not product code.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/merge_probe tools/merge_probe.cu
#include <cstdint>
#include <cstdio>
#include <vector>
typedef unsigned long long u64;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            printf("%s: %s\n", #x, cudaGetErrorString(e_));                                \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

// (a) int4 grid-stride, U-way unrolled (the product kernel uses U = 4)
template <int U>
__global__ void __launch_bounds__(256) copy_unroll(const int4 *__restrict__ s, int4 *__restrict__ d, int64_t n) {
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; q + (U - 1) * nth < n; q += U * nth) {
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; u++) v[u] = __ldcs(s + q + u * nth);
#pragma unroll
        for (int u = 0; u < U; u++) __stcs(d + q + u * nth, v[u]);
    }
    for (; q < n; q += nth) __stcs(d + q, __ldcs(s + q));
}

// (b) TMA bulk copies: each CTA streams chunks of CH bytes global -> shared
// -> global through an S-stage ring (one elected thread issues everything)
template <int CH, int S>
__global__ void __launch_bounds__(32) copy_bulk(const char *__restrict__ s, char *__restrict__ d, int64_t bytes) {
    extern __shared__ __align__(128) unsigned char buf[];
    __shared__ __align__(8) u64 bar[S];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < S; i++) {
        unsigned a = (unsigned)__cvta_generic_to_shared(&bar[i]);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    const int64_t nch = bytes / CH;
    unsigned phase[S] = {};
    int64_t c = blockIdx.x;
    int issued = 0;
    int64_t ids[S];
    // prologue
    for (int i = 0; i < S && c < nch; i++, c += gridDim.x) {
        unsigned sb = (unsigned)__cvta_generic_to_shared(buf + i * CH);
        unsigned ba = (unsigned)__cvta_generic_to_shared(&bar[i]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(CH));
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sb), "l"(s + c * CH), "r"(CH), "r"(ba) : "memory");
        ids[i] = c;
        issued++;
    }
    for (int k = 0; issued > 0; k = (k + 1) % S) {
        unsigned ba = (unsigned)__cvta_generic_to_shared(&bar[k]);
        unsigned sb = (unsigned)__cvta_generic_to_shared(buf + k * CH);
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                     ::"r"(ba), "r"(phase[k]));
        phase[k] ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(d + ids[k] * CH), "r"(sb), "r"(CH) : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        issued--;
        if (c < nch) {
            // the slot is reused: wait until its store has read the buffer
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(CH));
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(sb), "l"(s + c * CH), "r"(CH), "r"(ba) : "memory");
            ids[k] = c;
            c += gridDim.x;
            issued++;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// bitmap merge: (c) the product kernel (warp walks 32 words, one word at a time)
__global__ void __launch_bounds__(256) bm_walk(const double *__restrict__ src, double *dst,
                                               const uint32_t *__restrict__ bm, int64_t words) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w0 = gw * 32; w0 < words; w0 += nw * 32) {
        const uint32_t mine = (w0 + lane < words) ? __ldg(bm + w0 + lane) : 0u;
        unsigned any = __ballot_sync(0xffffffffu, mine != 0u);
        while (any) {
            const int j = __ffs(any) - 1;
            any &= any - 1;
            const uint32_t bits = __shfl_sync(0xffffffffu, mine, j);
            if ((bits >> lane) & 1u) {
                const int64_t e = ((w0 + j) << 5) + lane;
                dst[e] = src[e];
            }
        }
    }
}

// (d) batched: words in batches of 8 (8 independent predicated loads in
// flight per lane), and for sparse groups each lane walks its own word's bits
__global__ void __launch_bounds__(256) bm_batch(const double *__restrict__ src, double *dst,
                                                const uint32_t *__restrict__ bm, int64_t words) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w0 = gw * 32; w0 < words; w0 += nw * 32) {
        const uint32_t mine = (w0 + lane < words) ? __ldg(bm + w0 + lane) : 0u;
        const int tot = __reduce_add_sync(0xffffffffu, __popc(mine));
        if (tot == 0) continue;
        if (tot <= 96) {
            // sparse: each lane copies its own word's set bits
            uint32_t m = mine;
            while (m) {
                const int bpos = __ffs(m) - 1;
                m &= m - 1;
                const int64_t e = ((w0 + lane) << 5) + bpos;
                dst[e] = src[e];
            }
            continue;
        }
#pragma unroll 1
        for (int j0 = 0; j0 < 32; j0 += 8) {
            double v[8];
            bool on[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const uint32_t bits = __shfl_sync(0xffffffffu, mine, j0 + u);
                on[u] = (bits >> lane) & 1u;
                if (on[u]) v[u] = __ldcs(src + ((w0 + j0 + u) << 5) + lane);
            }
#pragma unroll
            for (int u = 0; u < 8; u++)
                if (on[u]) dst[((w0 + j0 + u) << 5) + lane] = v[u];
        }
    }
}

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; return x ^ (x >> 16);
}
__global__ void gen_bits(uint32_t *bm, int64_t words, int64_t nset, int64_t m) {
    // nset random bits in m elements (with collisions), via atomicOr
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nset; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = ((uint64_t)hsh((uint32_t)i) << 32 | hsh((uint32_t)i ^ 0x9e3779b9u)) % (uint64_t)m;
        atomicOr(bm + (k >> 5), 1u << (k & 31));
    }
}

template <typename F>
float timeit(F f, int reps = 5) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; r++) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    return best;
}

int main() {
    const int64_t bytes = 1ll << 30;
    char *s, *d;
    CK(cudaMalloc(&s, bytes));
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemset(s, 1, bytes));
    const int64_t n4 = bytes / 16;
    float ms;
    ms = timeit([&] { cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice); });
    printf("range  cudaMemcpy D2D          %.1f us  %.0f GB/s (r+w)\n", ms * 1e3, 2 * bytes / ms / 1e6);
    for (int bps : {4, 8, 16}) {
        ms = timeit([&] { copy_unroll<4><<<148 * bps, 256>>>((const int4 *)s, (int4 *)d, n4); });
        printf("range  int4 unroll4 %2d/SM       %.1f us  %.0f GB/s\n", bps, ms * 1e3, 2 * bytes / ms / 1e6);
        ms = timeit([&] { copy_unroll<8><<<148 * bps, 256>>>((const int4 *)s, (int4 *)d, n4); });
        printf("range  int4 unroll8 %2d/SM       %.1f us  %.0f GB/s\n", bps, ms * 1e3, 2 * bytes / ms / 1e6);
    }
    ms = timeit([&] { copy_unroll<1><<<(int)((n4 + 255) / 256), 256>>>((const int4 *)s, (int4 *)d, n4); });
    printf("range  int4 one-per-thread      %.1f us  %.0f GB/s\n", ms * 1e3, 2 * bytes / ms / 1e6);
    {
        auto k = copy_bulk<32768, 4>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768));
        for (int g : {148, 296, 444}) {
            ms = timeit([&] { k<<<g, 32, 4 * 32768>>>(s, d, bytes); });
            printf("range  TMA bulk 32K x4 grid %d  %.1f us  %.0f GB/s\n", g, ms * 1e3, 2 * bytes / ms / 1e6);
        }
        auto k2 = copy_bulk<16384, 6>;
        CK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 16384));
        for (int g : {296, 444, 592}) {
            ms = timeit([&] { k2<<<g, 32, 6 * 16384>>>(s, d, bytes); });
            printf("range  TMA bulk 16K x6 grid %d  %.1f us  %.0f GB/s\n", g, ms * 1e3, 2 * bytes / ms / 1e6);
        }
        CK(cudaGetLastError());
    }
    // bitmap merges over 2^27 f64 elements (1 GiB), dense and sparse
    const int64_t m = 1ll << 27, words = m / 32;
    uint32_t *bm;
    CK(cudaMalloc(&bm, words * 4));
    for (int64_t nset : {m, (int64_t)1 << 20}) {
        CK(cudaMemset(bm, 0, words * 4));
        gen_bits<<<148 * 8, 256>>>(bm, words, nset, m);
        CK(cudaDeviceSynchronize());
        std::vector<uint32_t> h(words);
        CK(cudaMemcpy(h.data(), bm, words * 4, cudaMemcpyDeviceToHost));
        int64_t pop = 0;
        for (auto w : h) pop += __builtin_popcount(w);
        const double mv = 2.0 * 8 * pop + 4.0 * words;
        for (int bps : {4, 8}) {
            ms = timeit([&] { bm_walk<<<148 * bps, 256>>>((const double *)s, (double *)d, bm, words); });
            printf("bitmap pop %10lld walk  %d/SM  %.1f us  %.0f GB/s (2x8B per set bit + bitmap)\n", (long long)pop, bps, ms * 1e3, mv / ms / 1e6);
            ms = timeit([&] { bm_batch<<<148 * bps, 256>>>((const double *)s, (double *)d, bm, words); });
            printf("bitmap pop %10lld batch %d/SM  %.1f us  %.0f GB/s\n", (long long)pop, bps, ms * 1e3, mv / ms / 1e6);
        }
    }
    CK(cudaGetLastError());
    return 0;
}
