/*
 * oracle.c -- plain, slow, sequential CPU oracle for the JACC multi-GPU
 * `parallel loop` hot path (Matsumura, Garcia De Gonzalo, Pena,
 * arXiv 2110.14340).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2110_14340_b200/csrc); neither side includes or links the other.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (see
 * __graft_entry__.build()).  IEEE binary64, round-to-nearest-even, no FMA
 * contraction, so every expression rounds exactly as written.
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n, "DESIGN R-k"
 * = reading k in DESIGN.md (where the paper is silent).
 *
 * Every function below has a pin in tests/test_oracle.py (closed forms,
 * invariants, brute force, library special cases); none is "parity unpinned".
 */
#include <stdint.h>
#include <string.h>
#include <math.h>

/* ------------------------------------------------------------------ */
/* c4  Partition of a split extent E over n devices.                   */
/* "equally dividing parallel dimensions among GPUs" (Sec 4.2);  */
/* remainder rule: the first E mod n blocks get one extra element       */
/* (DESIGN R-2).  Listing 2 drops the remainder --   */
/* that bug is deliberately not reproduced.  Half-open [lo, hi).        */
/* ------------------------------------------------------------------ */
void orc_partition(int64_t E, int n, int d, int64_t *lo, int64_t *hi)
{
    int64_t q = E / n;
    int64_t r = E % n;
    *lo = (int64_t)d * q + (d < r ? d : r);
    *hi = (int64_t)(d + 1) * q + ((d + 1) < r ? (d + 1) : r);
}

/* ------------------------------------------------------------------ */
/* K1  Listing 1: for(i=0;i<N;i++) x[i] = y[i]*y[i];  fp32 */
/* ------------------------------------------------------------------ */
void orc_square_f32(int64_t n, const float *y, float *x)
{
    for (int64_t i = 0; i < n; i++)
        x[i] = y[i] * y[i];
}

/* Filtered form of K1 for one device: the write x[i] is guarded by the
 * device's bounds, "(a_lb <= i && a_ub >= i) ? a[i]=... : a[i]"
 * (P:463-464), bounds inclusive.  Records the stored flat indices'
 * min/max (the write log of S:453-460).  Empty => min = UINT64_MAX, max = 0. */
void orc_square_f32_filtered(int64_t n, const float *y, float *x,
                             int64_t x_lb, int64_t x_ub,
                             uint64_t *wmin, uint64_t *wmax)
{
    uint64_t mn = UINT64_MAX, mx = 0;
    for (int64_t i = 0; i < n; i++) {
        if (x_lb <= i && x_ub >= i) {
            x[i] = y[i] * y[i];
            if ((uint64_t)i < mn) mn = (uint64_t)i;
            if ((uint64_t)i > mx) mx = (uint64_t)i;
        }
    }
    *wmin = mn; *wmax = mx;
}

/* ------------------------------------------------------------------ */
/* c1  Jacobi-2D (PolyBench/C jacobi-2d; not in the paper, whose stencil */
/* analogue is Himeno "Jacobi's method"; DESIGN R-1).     */
/* One sweep = one `parallel loop` launch:                              */
/*   for i in [1,N-1) for j in [1,N-1):                                 */
/*     dst[i][j] = 0.2 * (src[i][j] + src[i][j-1] + src[i][j+1]         */
/*                        + src[i+1][j] + src[i-1][j]);                 */
/* adds left to right, then one multiply by the binary64 literal 0.2.   */
/* Row-major N x N.  Boundary rows/columns are never written.           */
/* ------------------------------------------------------------------ */
void orc_jacobi2d_sweep(int64_t N, const double *src, double *dst)
{
    for (int64_t i = 1; i < N - 1; i++)
        for (int64_t j = 1; j < N - 1; j++)
            dst[i * N + j] = 0.2 * (src[i * N + j] + src[i * N + (j - 1)]
                                    + src[i * N + (j + 1)]
                                    + src[(i + 1) * N + j]
                                    + src[(i - 1) * N + j]);
}

/* PolyBench kernel_jacobi_2d: each timestep is two sweeps, A->B then B->A
 * (two launches per timestep; DESIGN R-1). */
void orc_jacobi2d(int64_t T, int64_t N, double *A, double *B)
{
    for (int64_t t = 0; t < T; t++) {
        orc_jacobi2d_sweep(N, A, B);
        orc_jacobi2d_sweep(N, B, A);
    }
}

/* Predicate-filtered sweep for one device: the loop runs over
 * the WHOLE iteration space, and the write dst[i][j] is guarded by the
 * device's bounds on dst's split dimension (dim 0, the leftmost parallel
 * dimension), inclusive [row_lb, row_ub].  Records min/max of
 * the flat indices actually stored (write log). */
void orc_jacobi2d_sweep_filtered(int64_t N, const double *src, double *dst,
                                 int64_t row_lb, int64_t row_ub,
                                 uint64_t *wmin, uint64_t *wmax)
{
    uint64_t mn = UINT64_MAX, mx = 0;
    for (int64_t i = 1; i < N - 1; i++)
        for (int64_t j = 1; j < N - 1; j++) {
            if (row_lb <= i && row_ub >= i) {
                dst[i * N + j] = 0.2 * (src[i * N + j] + src[i * N + (j - 1)]
                                        + src[i * N + (j + 1)]
                                        + src[(i + 1) * N + j]
                                        + src[(i - 1) * N + j]);
                uint64_t f = (uint64_t)(i * N + j);
                if (f < mn) mn = f;
                if (f > mx) mx = f;
            }
        }
    *wmin = mn; *wmax = mx;
}

/* ------------------------------------------------------------------ */
/* c2  Reductions (reduction clause semantics, DESIGN R-9):              */
/*   s = s_in; for i<n: s += x[i]*y[i];   (dot)                          */
/*   s = s_in; for i<n: s += x[i];        (sum)                          */
/* in double, in loop order, product rounded before the add.             */
/* ------------------------------------------------------------------ */
double orc_dot_f64(int64_t n, const double *x, const double *y, double s_in)
{
    double s = s_in;
    for (int64_t i = 0; i < n; i++)
        s += x[i] * y[i];
    return s;
}

double orc_sum_f64(int64_t n, const double *x, double s_in)
{
    double s = s_in;
    for (int64_t i = 0; i < n; i++)
        s += x[i];
    return s;
}

/* Accuracy reference for c2/c8 (DESIGN R-10): the same loops with
 * Neumaier's compensated summation (Neumaier 1974, "improved Kahan"):
 *   t = s + v; if |s| >= |v|: c += (s - t) + v else c += (v - t) + s; s = t
 * result s + c.  The product x[i]*y[i] is formed exactly by splitting it
 * into its rounded value p and error e = fma(x, y, -p) (exact for binary64,
 * no overflow/underflow in the configs), both summed compensated. */
static void neu_add(double *s, double *c, double v)
{
    double t = *s + v;
    if (fabs(*s) >= fabs(v))
        *c += (*s - t) + v;
    else
        *c += (v - t) + *s;
    *s = t;
}

double orc_dot_neumaier(int64_t n, const double *x, const double *y, double s_in)
{
    double s = s_in, c = 0.0;
    for (int64_t i = 0; i < n; i++) {
        double p = x[i] * y[i];
        double e = fma(x[i], y[i], -p);
        neu_add(&s, &c, p);
        neu_add(&s, &c, e);
    }
    return s + c;
}

double orc_sum_neumaier(int64_t n, const double *x, double s_in)
{
    double s = s_in, c = 0.0;
    for (int64_t i = 0; i < n; i++)
        neu_add(&s, &c, x[i]);
    return s + c;
}

/* Per-device partial of a reduction: "we filter the computation based on
 * the range of the outermost parallel iterator".  Private copy
 * starts at the identity 0 (DESIGN R-9); iterator bounds inclusive. */
double orc_dot_f64_filtered(int64_t n, const double *x, const double *y,
                            int64_t it_lb, int64_t it_ub)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; i++)
        if (it_lb <= i && it_ub >= i)
            s += x[i] * y[i];
    return s;
}

double orc_sum_f64_filtered(int64_t n, const double *x, int64_t it_lb, int64_t it_ub)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; i++)
        if (it_lb <= i && it_ub >= i)
            s += x[i];
    return s;
}

/* c8  Reduction combine: s_out = s_in + sum_d partial_d, partials in
 * device order ("multi-GPU reduction code"). */
double orc_reduce_combine(double s_in, int n, const double *partials)
{
    double t = 0.0;
    for (int d = 0; d < n; d++)
        t += partials[d];
    return s_in + t;
}

/* ------------------------------------------------------------------ */
/* c3  Dense GEMM loop nest (DESIGN R-11; alpha = 1, beta = 0):          */
/*   for i<M for j<N { c = 0.0; for k<K: c += A[i][k]*B[k][j]; C[i][j]=c; } */
/* Row-major A[M][K], B[K][N], C[M][N]; product rounded, then added, in   */
/* k order.                                                              */
/* ------------------------------------------------------------------ */
void orc_gemm_f64(int64_t M, int64_t N, int64_t K,
                  const double *A, const double *B, double *C)
{
    for (int64_t i = 0; i < M; i++)
        for (int64_t j = 0; j < N; j++) {
            double c = 0.0;
            for (int64_t k = 0; k < K; k++)
                c += A[i * K + k] * B[k * N + j];
            C[i * N + j] = c;
        }
}

/* Same loop nest in i-k-j order with C accumulated in memory.  Every C
 * element still sees its products in increasing k with the same rounding,
 * so the result is bit-identical to orc_gemm_f64 (DESIGN R-11); it only
 * exists because it is ~10x faster for the timed CPU baseline. */
void orc_gemm_f64_ikj(int64_t M, int64_t N, int64_t K,
                      const double *A, const double *B, double *C)
{
    for (int64_t i = 0; i < M; i++) {
        for (int64_t j = 0; j < N; j++)
            C[i * N + j] = 0.0;
        for (int64_t k = 0; k < K; k++) {
            double a = A[i * K + k];
            for (int64_t j = 0; j < N; j++)
                C[i * N + j] += a * B[k * N + j];
        }
    }
}

/* Filtered GEMM for one device: writes to C guarded on C's split dim
 * (rows), inclusive [row_lb, row_ub]; records min/max stored
 * flat index. */
void orc_gemm_f64_filtered(int64_t M, int64_t N, int64_t K,
                           const double *A, const double *B, double *C,
                           int64_t row_lb, int64_t row_ub,
                           uint64_t *wmin, uint64_t *wmax)
{
    uint64_t mn = UINT64_MAX, mx = 0;
    for (int64_t i = 0; i < M; i++)
        for (int64_t j = 0; j < N; j++) {
            double c = 0.0;
            for (int64_t k = 0; k < K; k++)
                c += A[i * K + k] * B[k * N + j];
            if (row_lb <= i && row_ub >= i) {
                C[i * N + j] = c;
                uint64_t f = (uint64_t)(i * N + j);
                if (f < mn) mn = f;
                if (f > mx) mx = f;
            }
        }
    *wmin = mn; *wmax = mx;
}

/* ------------------------------------------------------------------ */
/* c5  Indirect scatter: for i<n: a[idx[i]] += b[i];                     */
/* fp64: sums in loop order.  int32: wrapping (uint32) arithmetic.       */
/* ------------------------------------------------------------------ */
void orc_scatter_add_f64(int64_t n, const int32_t *idx, const double *b, double *a)
{
    for (int64_t i = 0; i < n; i++)
        a[idx[i]] += b[i];
}

void orc_scatter_add_i32(int64_t n, const int32_t *idx, const int32_t *b, int32_t *a)
{
    for (int64_t i = 0; i < n; i++)
        a[idx[i]] = (int32_t)((uint32_t)a[idx[i]] + (uint32_t)b[i]);
}

/* Filtered scatter for one device: the write index idx[i] is
 * computed outside the filter on every device; the update
 * (an OpenACC atomic in the parallel loop) is "predicated around the
 * operation" on the computed index against a's inclusive bounds.
 * Records the write log as a dirty bitmap over all of a (bit k of word w
 * <-> element 32w+k, DESIGN D10) plus min/max. */
static void bitmap_set(uint32_t *bm, uint64_t e)
{
    bm[e >> 5] |= (uint32_t)1u << (e & 31u);
}

void orc_scatter_add_f64_filtered(int64_t n, const int32_t *idx, const double *b,
                                  double *a, int64_t a_lb, int64_t a_ub,
                                  uint32_t *bitmap, uint64_t *wmin, uint64_t *wmax)
{
    uint64_t mn = UINT64_MAX, mx = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t k = idx[i];                       /* duplicated index computation */
        if (a_lb <= k && a_ub >= k) {
            a[k] += b[i];
            bitmap_set(bitmap, (uint64_t)k);
            if ((uint64_t)k < mn) mn = (uint64_t)k;
            if ((uint64_t)k > mx) mx = (uint64_t)k;
        }
    }
    *wmin = mn; *wmax = mx;
}

void orc_scatter_add_i32_filtered(int64_t n, const int32_t *idx, const int32_t *b,
                                  int32_t *a, int64_t a_lb, int64_t a_ub,
                                  uint32_t *bitmap, uint64_t *wmin, uint64_t *wmax)
{
    uint64_t mn = UINT64_MAX, mx = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t k = idx[i];
        if (a_lb <= k && a_ub >= k) {
            a[k] = (int32_t)((uint32_t)a[k] + (uint32_t)b[i]);
            bitmap_set(bitmap, (uint64_t)k);
            if ((uint64_t)k < mn) mn = (uint64_t)k;
            if ((uint64_t)k > mx) mx = (uint64_t)k;
        }
    }
    *wmin = mn; *wmax = mx;
}

/* ------------------------------------------------------------------ */
/* c7  Coherence exchange, EAGER policy ("Updated data are sent to */
/* all other GPUs after each kernel execution"): copy each owner's      */
/* written flat range [wmin, wmax] from its replica into every other    */
/* replica.  replicas[d] points at device d's copy (elem bytes each).   */
/* ------------------------------------------------------------------ */
void orc_exchange_range(int n, void **replicas, size_t elem,
                        const uint64_t *wmin, const uint64_t *wmax)
{
    for (int d = 0; d < n; d++) {
        if (wmin[d] > wmax[d]) continue;                /* empty write set */
        size_t off = (size_t)wmin[d] * elem;
        size_t len = (size_t)(wmax[d] - wmin[d] + 1) * elem;
        for (int p = 0; p < n; p++)
            if (p != d)
                memcpy((char *)replicas[p] + off, (char *)replicas[d] + off, len);
    }
}

/* Same, driven by per-device dirty bitmaps: copy exactly the marked
 * elements from owner d to every other replica. */
void orc_exchange_bitmap(int n, void **replicas, size_t elem, int64_t nelem,
                         uint32_t **bitmaps)
{
    for (int d = 0; d < n; d++)
        for (int64_t e = 0; e < nelem; e++)
            if (bitmaps[d][e >> 5] & ((uint32_t)1u << (e & 31)))
                for (int p = 0; p < n; p++)
                    if (p != d)
                        memcpy((char *)replicas[p] + e * elem,
                               (char *)replicas[d] + e * elem, elem);
}

/* ------------------------------------------------------------------ */
/* NEXT-2 workload: Himeno benchmark (Table 1 "Himeno   */
/* 19-point Jacobian Stencil Computation", Size XL 1024x512x512 fp32;  */
/* P:704 "Himeno iteratively updates a 19-point stencil grid according */
/* to Jacobi's method"; Fig. 10).  The loop bodies follow   */
/* the benchmark's public source (DESIGN R-17): one Jacobi iteration =  */
/* the stencil loop (writes wrk2, reduces gosa) then the copy loop      */
/* (p = wrk2), both over the interior i in [1,I-1), j in [1,J-1),       */
/* k in [1,K-1) of row-major [I][J][K] fp32 arrays.  a holds 4 arrays,  */
/* b and c 3 each, [m][I][J][K].  Expression order exactly as written,  */
/* fp32 arithmetic (FLT_EVAL_METHOD 0), no contraction.                */
/* ------------------------------------------------------------------ */
#define HI(m, i, j, k) ((((int64_t)(m) * I + (i)) * J + (j)) * K + (k))

static float himeno_point(int64_t I, int64_t J, int64_t K, const float *p, const float *a,
                          const float *b, const float *c, const float *wrk1, const float *bnd,
                          int64_t i, int64_t j, int64_t k, float *ss_out)
{
    float s0 = a[HI(0, i, j, k)] * p[HI(0, i + 1, j, k)]
             + a[HI(1, i, j, k)] * p[HI(0, i, j + 1, k)]
             + a[HI(2, i, j, k)] * p[HI(0, i, j, k + 1)]
             + b[HI(0, i, j, k)]
               * (p[HI(0, i + 1, j + 1, k)] - p[HI(0, i + 1, j - 1, k)]
                  - p[HI(0, i - 1, j + 1, k)] + p[HI(0, i - 1, j - 1, k)])
             + b[HI(1, i, j, k)]
               * (p[HI(0, i, j + 1, k + 1)] - p[HI(0, i, j - 1, k + 1)]
                  - p[HI(0, i, j + 1, k - 1)] + p[HI(0, i, j - 1, k - 1)])
             + b[HI(2, i, j, k)]
               * (p[HI(0, i + 1, j, k + 1)] - p[HI(0, i - 1, j, k + 1)]
                  - p[HI(0, i + 1, j, k - 1)] + p[HI(0, i - 1, j, k - 1)])
             + c[HI(0, i, j, k)] * p[HI(0, i - 1, j, k)]
             + c[HI(1, i, j, k)] * p[HI(0, i, j - 1, k)]
             + c[HI(2, i, j, k)] * p[HI(0, i, j, k - 1)]
             + wrk1[HI(0, i, j, k)];
    float ss = (s0 * a[HI(3, i, j, k)] - p[HI(0, i, j, k)]) * bnd[HI(0, i, j, k)];
    *ss_out = ss;
    return ss;
}

/* stencil loop over planes [i_lb, i_ub] (inclusive; the whole interior
 * for the sequential oracle), writes wrk2, returns gosa_in + sum ss*ss
 * accumulated in fp32 in loop order; *gosa_ref (if non-NULL) receives the
 * Neumaier-compensated fp64 sum of the same fp32 terms (accuracy
 * reference, DESIGN R-17).  Records the write log min/max. */
float orc_himeno_stencil(int64_t I, int64_t J, int64_t K, const float *p, const float *a,
                         const float *b, const float *c, const float *wrk1, const float *bnd,
                         float *wrk2, float omega, int64_t i_lb, int64_t i_ub, float gosa_in,
                         double *gosa_ref, uint64_t *wmin, uint64_t *wmax)
{
    float gosa = gosa_in;
    double s = 0.0, cmp = 0.0;
    uint64_t mn = UINT64_MAX, mx = 0;
    for (int64_t i = 1; i < I - 1; i++)
        for (int64_t j = 1; j < J - 1; j++)
            for (int64_t k = 1; k < K - 1; k++) {
                if (!(i_lb <= i && i_ub >= i)) continue;   /* filter */
                float ss;
                himeno_point(I, J, K, p, a, b, c, wrk1, bnd, i, j, k, &ss);
                gosa += ss * ss;
                neu_add(&s, &cmp, (double)(ss * ss));
                wrk2[HI(0, i, j, k)] = p[HI(0, i, j, k)] + omega * ss;
                uint64_t f = (uint64_t)HI(0, i, j, k);
                if (f < mn) mn = f;
                if (f > mx) mx = f;
            }
    if (gosa_ref) *gosa_ref = (double)gosa_in + (s + cmp);
    if (wmin) *wmin = mn;
    if (wmax) *wmax = mx;
    return gosa;
}

/* copy loop p = wrk2 over interior planes [i_lb, i_ub] */
void orc_himeno_copy(int64_t I, int64_t J, int64_t K, const float *wrk2, float *p,
                     int64_t i_lb, int64_t i_ub, uint64_t *wmin, uint64_t *wmax)
{
    uint64_t mn = UINT64_MAX, mx = 0;
    for (int64_t i = 1; i < I - 1; i++)
        for (int64_t j = 1; j < J - 1; j++)
            for (int64_t k = 1; k < K - 1; k++) {
                if (!(i_lb <= i && i_ub >= i)) continue;
                p[HI(0, i, j, k)] = wrk2[HI(0, i, j, k)];
                uint64_t f = (uint64_t)HI(0, i, j, k);
                if (f < mn) mn = f;
                if (f > mx) mx = f;
            }
    if (wmin) *wmin = mn;
    if (wmax) *wmax = mx;
}
#undef HI

/* ------------------------------------------------------------------ */
/* NEXT-3  Fig. 4 predicate-filtered statement chain.       */
/* Loop body (x is firstprivate, initialised to x_in every iteration):  */
/*   a[i]=x; b[i]=a[i]; x=c[j]; a[k]=x; b[k]=a[k];                      */
/* with j = jx[i], k = kx[i] (index arrays).  Sequential oracle:        */
/* ------------------------------------------------------------------ */
void orc_fig4(int64_t n, const int32_t *jx, const int32_t *kx, const double *c, double x_in,
              double *a, double *b)
{
    for (int64_t i = 0; i < n; i++) {
        double x = x_in;
        int64_t j = jx[i], k = kx[i];
        a[i] = x;
        b[i] = a[i];
        x = c[j];
        a[k] = x;
        b[k] = a[k];
    }
}

/* The filtered code of Fig. 4 (bottom) for one device, guards verbatim:
 *   ((a_lb<=i && a_ub>=i)||(b_lb<=i && b_ub>=i)) ? a[i]=x : a[i];
 *   ((b_lb<=i && b_ub>=i)) ? b[i]=a[i] : b[i];
 *   x = ((a_lb<=k && a_ub>=k)||(b_lb<=k && b_ub>=k)) ? c[j] : 0;
 *   ((a_lb<=k && a_ub>=k)||(b_lb<=k && b_ub>=k)) ? a[k]=x : a[k];
 *   ((b_lb<=k && b_ub>=k)) ? b[k]=a[k] : b[k];
 * Bounds inclusive.  Records the write logs of a and b (min/max
 * of every executed store, including the duplicated stores to a outside
 * a's own bounds that the guards of b require). */
void orc_fig4_filtered(int64_t n, const int32_t *jx, const int32_t *kx, const double *c,
                       double x_in, double *a, double *b, int64_t a_lb, int64_t a_ub,
                       int64_t b_lb, int64_t b_ub, uint64_t *amin, uint64_t *amax,
                       uint64_t *bmin, uint64_t *bmax)
{
    uint64_t an = UINT64_MAX, ax = 0, bn = UINT64_MAX, bx = 0;
#define LOGW(mn, mx, f) do { if ((uint64_t)(f) < mn) mn = (uint64_t)(f); \
                             if ((uint64_t)(f) > mx) mx = (uint64_t)(f); } while (0)
    for (int64_t i = 0; i < n; i++) {
        double x = x_in;
        int64_t j = jx[i], k = kx[i];
        if ((a_lb <= i && a_ub >= i) || (b_lb <= i && b_ub >= i)) { a[i] = x; LOGW(an, ax, i); }
        if (b_lb <= i && b_ub >= i) { b[i] = a[i]; LOGW(bn, bx, i); }
        x = ((a_lb <= k && a_ub >= k) || (b_lb <= k && b_ub >= k)) ? c[j] : 0;
        if ((a_lb <= k && a_ub >= k) || (b_lb <= k && b_ub >= k)) { a[k] = x; LOGW(an, ax, k); }
        if (b_lb <= k && b_ub >= k) { b[k] = a[k]; LOGW(bn, bx, k); }
    }
#undef LOGW
    *amin = an; *amax = ax; *bmin = bn; *bmax = bx;
}
