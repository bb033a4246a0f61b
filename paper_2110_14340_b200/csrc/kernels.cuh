// kernels.cuh -- launch wrappers of the sm_100a device kernels (internal to
// libjacc.so; not part of the C-ABI).  Every wrapper enqueues on `s` and
// returns the launch error.  Dirty records are two u64 in device memory:
// d[0] = min stored flat index, d[1] = ~max stored flat index; all-ones is
// the empty set (UINT64_MAX, 0) (DESIGN R-3, R-15).  Each record is one
// slot of a 32-byte-aligned pair; a writing kernel fills its slot and
// clears the other one (slot address ^ 16) for the next launch.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace jk {

using u64 = unsigned long long;
constexpr int kMaxPeers = 16;

struct PeerPtrs {
    void *p[kMaxPeers];
    int n;
};

// BK6  Listing 1: x[i] = y[i]*y[i] for i in [i0, i1); x and y
// are the loop's arrays (already offset); dirty indices are x_off + i.
cudaError_t square_f32(cudaStream_t s, const float *y, float *x, int64_t i0, int64_t i1,
                       int64_t x_off, u64 *dirty);

// BK1  PolyBench jacobi-2d sweep (DESIGN R-1) over rows [r0,r1) x cols
// [c0,c1) of an N x N grid, with fused dirty-range tracking and fused HALO
// push: row r0 is also stored into push_top, row r1-1 into push_bot (peer
// replicas of dst, same layout; nullptr = no push).
cudaError_t jacobi2d(cudaStream_t s, const double *src, double *dst, int64_t N,
                     int64_t r0, int64_t r1, int64_t c0, int64_t c1, u64 *dirty,
                     double *push_top, double *push_bot);

// BK2  Fixed-order reduction of sum x[i]*y[i] (y != nullptr) or sum x[i]
// over [0, n); result written to *out.  `partials` holds kReduceGrid
// doubles, `ticket` one zeroed u32 (left zeroed on exit).
constexpr int kReduceGrid = 148 * 4;  // (partials buffers hold kHimenoPartials)
cudaError_t reduce_f64(cudaStream_t s, const double *x, const double *y, int64_t n,
                       double *partials, unsigned *ticket, double *out);

// c8 combine on one device: *out = s_in + sum_d *parts[d] (device order).
cudaError_t combine(cudaStream_t s, PeerPtrs parts, double s_in, double *out);

// BK3  C[r0:r1, c0:c1] = A[r0:r1, :] * B[:, c0:c1] on the fp64 tensor pipe
// (DMMA via mma.sync m8n8k4 f64), dirty-range tracking fused.
// push: peer replicas of C that receive every finished tile in the
// epilogue (the EAGER merge fused with the GEMM; n = 0: none).
cudaError_t gemm_f64(cudaStream_t s, const double *A, const double *B, double *C,
                     int64_t M, int64_t N, int64_t K, int64_t r0, int64_t r1,
                     int64_t c0, int64_t c1, u64 *dirty, PeerPtrs push);

// BK4  Owner-filtered scatter: for i in [0,n):
// k = idx[i]; if lo <= k < hi: a[k] += b[i] (atomic); bitmap bit k set
// (warp-aggregated atomicOr), dirty min/max of k.  a, bitmap indexed by
// element of the whole region.
cudaError_t scatter_add_f64(cudaStream_t s, const int32_t *idx, const double *b, double *a,
                            int64_t n, int64_t lo, int64_t hi, uint32_t *bitmap, u64 *dirty);
cudaError_t scatter_add_i32(cudaStream_t s, const int32_t *idx, const int32_t *b, int32_t *a,
                            int64_t n, int64_t lo, int64_t hi, uint32_t *bitmap, u64 *dirty);

// BK4b Same loop, executed as a destination-binned pipeline for arrays far
// larger than L2: (1) histogram of the owned keys per 2^20-element bucket,
// (2) scan, (3) partition of the (k, b[i]) pairs into bucket-contiguous
// streams through shared-memory staging (coalesced, full-line writes),
// (4) apply the pairs in stream order, so the read-modify-writes of a hit
// L2 and every line of a moves to/from HBM about once, (5) dirty bits per
// bucket part in shared memory, each bitmap word written once (EAGER:
// merge_bitmap follows).  Dirty range fused into (4).  is_f64: T = double,
// else int32.
struct ScatterPlan {
    bool binned;
    bool all_owned;     // [lo, hi) covers every element of a (one device / duplicated)
    int shift, nb;      // bucket = 2^shift elements, nb buckets
    bool spec;          // speculative fixed-capacity layout first (no histogram pass)
    u64 cap;            // its pairs per bucket (bucket b at [b*cap, (b+1)*cap))
    size_t slots;       // pair slots: max(n, nb*cap)
    size_t hdr;         // bytes of counters/bases at the start of the scratch
    size_t scratch;     // total scratch bytes (header + slots keys + slots values)
};
ScatterPlan scatter_plan(int64_t n, int64_t lo, int64_t hi, int elem, int64_t m_total);
cudaError_t scatter_add_binned(cudaStream_t s, bool is_f64, const int32_t *idx, const void *b,
                               void *a, int64_t n, int64_t lo, int64_t hi, uint32_t *bitmap,
                               u64 *dirty, const ScatterPlan &pl, void *scratch);

// NEXT-2  Himeno benchmark (DESIGN R-17), fp32, row-major
// [I][J][K] arrays (a: 4, b and c: 3 stacked arrays).  Stencil loop over
// planes [i0,i1) x [j0,j1) x [k0,k1): wrk2 = p + omega*ss, partial
// gosa = sum ss*ss accumulated in fp64 in a fixed order (block partials in
// `partials`, capacity kHimenoPartials, last block finishes) -> *out;
// dirty range of wrk2 fused.  Copy loop p = wrk2 over the same box, dirty
// range of p fused, HALO push of planes i0 / i1-1 into peer replicas of p.
constexpr int kHimenoPartials = 16384;
cudaError_t himeno_stencil(cudaStream_t s, const float *p, const float *a, const float *b,
                           const float *c, const float *wrk1, const float *bnd, float *wrk2,
                           int64_t I, int64_t J, int64_t K, int64_t i0, int64_t i1, int64_t j0,
                           int64_t j1, int64_t k0, int64_t k1, float omega, double *partials,
                           unsigned *ticket, double *out, u64 *dirty);
cudaError_t himeno_copy(cudaStream_t s, const float *wrk2, float *p, int64_t I, int64_t J,
                        int64_t K, int64_t i0, int64_t i1, int64_t j0, int64_t j1, int64_t k0,
                        int64_t k1, u64 *dirty, float *push_top, float *push_bot,
                        unsigned *ticket);  // ticket: the device's zeroed counter block

// NEXT-3  Iteration-split scatter with an additive merge.  Phase 1 (every
// device, its block of iterations): the scatter kernels above with
// lo = 0, hi = M into a zero-kept delta array + delta bitmap.  Phase 2
// (owner of the word-aligned slice [32*w0, 32*w1) of a): for every word
// dirty in any device's delta bitmap, a[e] += sum_q delta_q[e] in device
// order, read over peer memory; the consumed deltas and delta-bitmap words
// are zeroed (so they stay zero for the next launch); the union bitmap is
// the owner's dirty bitmap, min/max its dirty range.
cudaError_t scatter_combine(cudaStream_t s, bool is_f64, void *a, uint32_t *bm_out,
                            PeerPtrs deltas, PeerPtrs dbms, int64_t w0, int64_t w1, int64_t M,
                            u64 *dirty);

// NEXT-3  Fig. 4 statement chain, filtered for one device:
// for i in [i0,i1): x = x_in; j = jx[i]; k = kx[i];
//   (i in A|B) ? a[i] = x;  (i in B) ? b[i] = a[i];
//   x = (k in A|B) ? c[j] : 0;  (k in A|B) ? a[k] = x;  (k in B) ? b[k] = a[k];
// A = [alo,ahi), B = [blo,bhi) (half-open owned blocks of a and b); every
// executed store is logged (dirty a / dirty b), duplicated a stores included.
cudaError_t fig4(cudaStream_t s, const int32_t *jx, const int32_t *kx, const double *c, int64_t nc,
                 double x_in, double *a, double *b, int64_t na, int64_t i0, int64_t i1, int64_t alo,
                 int64_t ahi, int64_t blo, int64_t bhi, u64 *adirty, u64 *bdirty);

// BK5  Dirty-region merge over peer memory.  merge_range copies the
// recorded span [dirty min, dirty max] (clamped to [lo, hi)) of src into
// every peer replica; `max_elems` bounds the grid (host-known write bound).
cudaError_t merge_range(cudaStream_t s, const void *src, PeerPtrs dsts, const u64 *dirty,
                        int64_t elem, int64_t lo, int64_t hi);
// merge_box copies a strided box (2-D or 3-D sub-box of a row-major array,
// described as `count` pitched 2-D copies, all in bytes) from src to every
// peer, restricted to the device-recorded dirty span when dirty != nullptr
// (split dimensions > 0: the paper's cudaMemcpy2DAsync exchange
// done with peer stores).
struct Box2D {
    int64_t count, height, width, pitch, first, outer;
};
cudaError_t merge_box(cudaStream_t s, const void *src, PeerPtrs dsts, Box2D b, const u64 *dirty,
                      int64_t elem);
// merge_bitmap copies exactly the elements whose dirty bit is set within
// [lo, hi) into every peer replica (elem = 4 or 8 bytes).
cudaError_t merge_bitmap(cudaStream_t s, const void *src, PeerPtrs dsts, const uint32_t *bitmap,
                         int64_t elem, int64_t lo, int64_t hi);

}  // namespace jk
