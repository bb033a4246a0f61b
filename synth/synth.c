/*
 * synth.c -- seeded synthetic input generators shared by the oracle side
 * and the CUDA side (the ONLY module both may use).  Holds none of the
 * method's arithmetic: just counter-based random numbers and the PolyBench
 * jacobi-2d initial field.
 *
 * Counter-based: element i of array `aid` under `seed` is
 *   r = splitmix64(seed ^ (aid << 40) ^ i)
 * (SURVEY 8(d) recipe), so any sub-range can be generated independently and
 * in parallel, and results never depend on thread count.
 */
#include <stdint.h>
#include <stddef.h>

static inline uint64_t splitmix64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t key(uint64_t seed, uint64_t aid, uint64_t i)
{
    return splitmix64(seed ^ (aid << 40) ^ i);
}

uint64_t syn_splitmix64(uint64_t x) { return splitmix64(x); }

/* uniform [0,1) binary64 with 53 random bits */
void syn_uniform_f64(double *out, int64_t n, int64_t off, uint64_t seed, uint64_t aid)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++)
        out[i] = (double)(key(seed, aid, (uint64_t)(off + i)) >> 11) * 0x1.0p-53;
}

/* uniform [0,1) binary32 with 24 random bits */
void syn_uniform_f32(float *out, int64_t n, int64_t off, uint64_t seed, uint64_t aid)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++)
        out[i] = (float)(key(seed, aid, (uint64_t)(off + i)) >> 40) * 0x1.0p-24f;
}

/* dyadic k/1024, k uniform in [0,1024) */
void syn_dyadic_f64(double *out, int64_t n, int64_t off, uint64_t seed, uint64_t aid)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++)
        out[i] = (double)(key(seed, aid, (uint64_t)(off + i)) >> 54) * 0x1.0p-10;
}

/* int32 uniform in [0, m), m <= 2^31 (multiply-shift range reduction) */
void syn_index_i32(int32_t *out, int64_t n, int64_t off, uint64_t seed, uint64_t aid, int64_t m)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++)
        out[i] = (int32_t)(((key(seed, aid, (uint64_t)(off + i)) >> 32) * (uint64_t)m) >> 32);
}

/* int32 uniform in [lo, hi] */
void syn_int_i32(int32_t *out, int64_t n, int64_t off, uint64_t seed, uint64_t aid,
                 int64_t lo, int64_t hi)
{
    uint64_t span = (uint64_t)(hi - lo + 1);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++)
        out[i] = (int32_t)(lo + (int64_t)(((key(seed, aid, (uint64_t)(off + i)) >> 32) * span) >> 32));
}

/* random permutation of [0, m) (sequential Fisher-Yates driven by the
 * counter-based stream; deterministic for a given seed) */
void syn_permutation_i32(int32_t *out, int64_t m, uint64_t seed, uint64_t aid)
{
    for (int64_t i = 0; i < m; i++)
        out[i] = (int32_t)i;
    for (int64_t i = m - 1; i > 0; i--) {
        uint64_t j = ((key(seed, aid, (uint64_t)i) >> 32) * (uint64_t)(i + 1)) >> 32;
        int32_t t = out[i];
        out[i] = out[j];
        out[j] = t;
    }
}

/* PolyBench/C 4.2 jacobi-2d init_array:
 *   A[i][j] = ((DATA_TYPE) i*(j+2) + 2) / n;
 *   B[i][j] = ((DATA_TYPE) i*(j+3) + 3) / n;
 * rows [row0, row0+nrows) of an N x N row-major grid. */
void syn_polybench_jacobi2d(double *A, double *B, int64_t N, int64_t row0, int64_t nrows)
{
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrows; r++) {
        int64_t i = row0 + r;
        for (int64_t j = 0; j < N; j++) {
            if (A) A[r * N + j] = ((double)i * (double)(j + 2) + 2.0) / (double)N;
            if (B) B[r * N + j] = ((double)i * (double)(j + 3) + 3.0) / (double)N;
        }
    }
}

/* Himeno benchmark initial state (himenoBMT initmt): a0..a2 = 1, a3 = 1/6,
 * b = 0, c = 1, p[i][j][k] = (float)(i*i) / (float)((I-1)*(I-1)),
 * wrk1 = 0, bnd = 1.  a: [4][I][J][K], b, c: [3][I][J][K]. */
void syn_himeno_init(float *p, float *a, float *b, float *c, float *wrk1, float *bnd,
                     int64_t I, int64_t J, int64_t K)
{
    const int64_t V = I * J * K, P = J * K;
    const float den = (float)((I - 1) * (I - 1));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < I; i++) {
        const float pv = (float)(i * i) / den;
        for (int64_t x = i * P; x < (i + 1) * P; x++) {
            p[x] = pv;
            a[x] = 1.0f; a[V + x] = 1.0f; a[2 * V + x] = 1.0f; a[3 * V + x] = (float)(1.0 / 6.0);
            b[x] = 0.0f; b[V + x] = 0.0f; b[2 * V + x] = 0.0f;
            c[x] = 1.0f; c[V + x] = 1.0f; c[2 * V + x] = 1.0f;
            wrk1[x] = 0.0f;
            bnd[x] = 1.0f;
        }
    }
}
