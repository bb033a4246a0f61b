/*
 * jacc.h -- C-ABI of the B200-native JACC multi-GPU `parallel loop` runtime
 * (libjacc.so).  Reimplements, from the paper's statement of the problem,
 * the hot path of arXiv 2110.14340 (Matsumura, Garcia De Gonzalo, Pena):
 * one OpenACC `parallel loop` distributed automatically over the GPUs of a
 * single box by predicate-based filtering (Sec 4).
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, R-k = reading k
 * in DESIGN.md.
 *
 * Conventions (all entry points):
 *   - Return codes only; no exceptions cross the ABI.  JACC_OK == 0,
 *     errors are negative; jacc_error_string() gives stable text.
 *   - A CUDA error poisons the runtime: every later call returns
 *     JACC_ERR_STATE until jacc_finalize() + jacc_init().
 *   - One host thread drives the API (not thread-safe).
 *   - "host" pointers are caller-owned host memory; the caller keeps them
 *     valid between jacc_data_create() and jacc_data_delete(); the library
 *     never frees them.  The library owns device replicas, dirty records,
 *     streams, events and communicators.
 *   - Index ranges are half-open [lo, hi) (R-3); recorded dirty ranges are
 *     inclusive [min, max] in flat element indices, empty <=> min > max,
 *     reported as (UINT64_MAX, 0).
 *   - Devices are LOGICAL devices 0..n-1 (device 0 is the primary, R-13);
 *     each maps to a CUDA ordinal.  Several logical devices may share one
 *     ordinal ("virtual devices": separate replicas on one GPU) so the
 *     multi-device path can be exercised on a single B200.
 */
#ifndef JACC_H
#define JACC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int jacc_status;

enum {
    JACC_OK = 0,
    JACC_ERR_INVALID = -1,      /* bad argument, size, extent or loop shape */
    JACC_ERR_OVERLAP = -2,      /* data_create overlaps a present region */
    JACC_ERR_NOT_PRESENT = -3,  /* pointer not inside any present region (P:209 `present`) */
    JACC_ERR_UNKNOWN_LOOP = -4, /* loop_id not in the descriptor table */
    JACC_ERR_OOM = -5,          /* device allocation failed */
    JACC_ERR_CUDA = -6,         /* CUDA runtime error (runtime is now poisoned) */
    JACC_ERR_NCCL = -7,         /* NCCL error (runtime is now poisoned) */
    JACC_ERR_STATE = -8         /* not initialised, double init, or poisoned */
};

/* ---------------------------------------------------------------------- */
/* Lifetime                                                                */
/* ---------------------------------------------------------------------- */

/* Initialise n_devices logical devices.  device_ids[d] is the CUDA ordinal
 * of logical device d (NULL = 0..n-1).  Repeated ordinals create virtual
 * devices on one GPU.  Peer access is enabled between distinct ordinals
 * (NVLink/NVSwitch P2P); an NCCL communicator is created when n > 1 and all
 * ordinals are distinct (reduction combine).  The paper drives its
 * GPUs from OpenMP threads inside the library; here each logical
 * device has its own CUDA stream and the runtime enqueues asynchronously.
 * Errors: JACC_ERR_STATE if already initialised, JACC_ERR_INVALID for
 * n_devices < 1 or > JACC_MAX_DEVICES or a bad ordinal. */
#define JACC_MAX_DEVICES 16
jacc_status jacc_init(int n_devices, const int *device_ids);

/* Synchronise, free every replica and runtime object.  Present regions
 * still registered are dropped (host memory untouched). */
jacc_status jacc_finalize(void);

/* Number of logical devices (0 if not initialised). */
int jacc_num_devices(void);

/* Merge policy for loops that write arrays (R-5):
 *   JACC_MERGE_EAGER: after each launch every device pushes its recorded
 *     dirty region of every written array to all other replicas
 *     ("Updated data are sent to all other GPUs after each kernel
 *     execution"; sync at start and end): a range record
 *     moves its [min, max] span, a bitmap record its dirty elements, with
 *     32-element words holding >= 8 dirty elements inside the device's
 *     owned block moved whole (same values, full sectors; DESIGN R-22).
 *   JACC_MERGE_HALO: push only the dirty rows the neighbouring devices read
 *     in a launch of the same loop shape (the config's boundary-row
 *     dirty-range merge; the paper's manual halo comparison P:909,
 *     P:933-939).  Replicas stay stale elsewhere; stale intervals are
 *     pulled on demand before a launch that reads them and by
 *     jacc_update_host().  Results are identical under both policies. */
enum { JACC_MERGE_EAGER = 0, JACC_MERGE_HALO = 1 };
jacc_status jacc_set_merge_policy(int policy);

/* Execution mode: JACC_MODE_MULTI splits by owned blocks
 * (default); JACC_MODE_DUP runs the full loop on every device with no
 * exchange ("duplicating computation on all GPUs and performing no
 * GPU-to-GPU communication").  The alias rule (R-12) forces DUP per launch.
 * JACC_MODE_ADAPTIVE (single-process mode only): every kernel
 * identity (loop, argument regions, range) starts duplicated, is profiled
 * with CUDA events, switches to multi-GPU after Eq. (1) has held five
 * times, and back to duplication for good after Eq. (2) or (3) has held
 * five times with a positive mean margin (controller below; DESIGN R-16).
 * peak_P2P defaults to 770 GB/s (env JACC_PEAK_P2P_GBS). */
enum { JACC_MODE_MULTI = 0, JACC_MODE_DUP = 1, JACC_MODE_ADAPTIVE = 2 };
jacc_status jacc_set_mode(int mode);

/* Split dimension of the written array for the multidimensional loops
 * (Jacobi-2D, GEMM, Himeno): -1 (default) applies the P:524-525 rule, which
 * for these loop bodies selects dim 0 (contiguous row / plane blocks, fused
 * boundary pushes); dim 1 or 2 divides columns / the innermost dimension
 * instead: every device's block is then strided, write sets
 * are boxes, and merges are pitched box copies over peer memory
 * (EAGER: the dirty box; HALO: the boundary slabs).  Other loops are 1-D
 * and always split dim 0.  Errors: JACC_ERR_INVALID outside [-1, 2]; a
 * launch whose written array has no such dimension: JACC_ERR_INVALID. */
jacc_status jacc_set_split_dim(int dim);

/* NEXT-3 scatter distribution.  0 (default): the paper's owner filter
 * (R-6): every device scans all iterations and applies
 * the updates whose index falls in its slice of `a`.  1: iteration split
 * with an additive merge: each device scatters its block of iterations
 * into a private zero-kept delta array (+ delta bitmap); then the owner of
 * each word-aligned slice of `a` adds every device's delta for the words
 * dirty anywhere, in device order, reading them over peer memory, and the
 * merge policy distributes the result (its dirty bitmap = the union).
 * Single-process mode only; a duplicated launch (JACC_MODE_DUP, or DUP
 * chosen by JACC_MODE_ADAPTIVE) runs every iteration on every device and
 * ignores the setting.  Errors: JACC_ERR_INVALID in multi-process mode, or
 * at launch with several async queues. */
jacc_status jacc_set_scatter_split(int iteration_split);

/* Owned block [lo, hi) of logical device d when an extent E is split over
 * n devices: "equally dividing parallel dimensions among GPUs",
 * the first E mod n blocks one element larger (R-2).  Pure host
 * logic; needs no GPU and no jacc_init.  Errors: JACC_ERR_INVALID for
 * E < 0, n < 1, d outside [0, n) or NULL outputs. */
jacc_status jacc_partition(int64_t E, int n, int d, int64_t *lo, int64_t *hi);

/* A18 parallel-dimension selection: n_parallel[k] /
 * n_sequential[k] = number of parallel / sequential loop iterators in the
 * index expression of dimension k of an updated array.  *dim = the
 * dimension with the most parallel iterators, among those the fewest
 * sequential ones, ties to the leftmost (C, fortran_order = 0) or rightmost
 * (Fortran); -1 when no dimension holds a parallel iterator (the array is
 * computed in duplicate).  Pure host logic.  Errors: JACC_ERR_INVALID. */
jacc_status jacc_select_split_dim(int ndims, const int *n_parallel, const int *n_sequential,
                                  int fortran_order, int *dim);

/* A19 exchange plan ("GPU-to-GPU communication through
 * cudaMemcpy2DAsync"): device d's owned block along split_dim of a
 * row-major array (extents[0..ndims), elem bytes) as `count` pitched 2-D
 * copies; copy c, row r (r < height) covers the bytes
 * [first + c*outer + r*pitch, + width).  split_dim 0 gives one contiguous
 * copy; an empty block gives count 0.  Pure host logic. */
typedef struct {
    int64_t count, height, width_bytes, pitch_bytes, first_offset_bytes, outer_stride_bytes;
} jacc_copy2d_plan;
jacc_status jacc_exchange_plan(int ndims, const int64_t *extents, size_t elem, int split_dim, int n,
                               int d, jacc_copy2d_plan *out);

/* ---------------------------------------------------------------------- */
/* Present table ("managed in a red-black tree ... to accept any */
/* address of declared data")                       */
/* ---------------------------------------------------------------------- */

/* Register [host, host+bytes) and allocate one replica of `bytes` on every
 * logical device ("Device-memory allocations ... are replicated on
 * all the GPUs").  No copy is made (OpenACC `create`).  elem_size is the
 * element size in bytes; extents[0..ndims) the row-major shape (ndims 1..4)
 * whose product times elem_size must equal bytes.
 * Errors: JACC_ERR_INVALID (bytes == 0, bad shape, host NULL),
 * JACC_ERR_OVERLAP, JACC_ERR_OOM. */
jacc_status jacc_data_create(void *host, size_t bytes, size_t elem_size,
                             int ndims, const int64_t *extents);

/* Unregister the region containing `host` (any interior address) and free
 * its replicas.  Errors: JACC_ERR_NOT_PRESENT. */
jacc_status jacc_data_delete(void *host);

/* Copy host bytes [offset, offset+bytes) of the region containing `host`
 * into EVERY replica ("host-to-GPU communications are replicated")
 * and mark them valid.  `host` may be any interior address; offset is
 * relative to it.  Synchronous w.r.t. the host buffer (it may be reused on
 * return).  Errors: JACC_ERR_NOT_PRESENT, JACC_ERR_INVALID (out of range). */
jacc_status jacc_update_device(void *host, size_t offset_bytes, size_t bytes);

/* Make the primary replica coherent over the range (pull stale intervals
 * from their owners over P2P) and copy it to host ("the primary
 * GPU is used for GPU-to-host transfers").  Waits for all outstanding work.
 * Errors as jacc_update_device. */
jacc_status jacc_update_host(void *host, size_t offset_bytes, size_t bytes);

/* ---------------------------------------------------------------------- */
/* Loop launch (jacc_kernel_push)                    */
/* ---------------------------------------------------------------------- */

/* Precompiled loop bodies (the paper's experiments embed pre-filtered
 * kernel strings).  Argument order per loop:
 *   JACC_LOOP_SQUARE_F32      (Listing 1): y IN f32[n], x OUT f32[n];
 *       for i in range: x[i] = y[i]*y[i].  range: 1-D over [0,n).
 *   JACC_LOOP_JACOBI2D_F64    (R-1): src IN f64[N][N], dst OUT f64[N][N];
 *       for i,j in range: dst[i][j] = 0.2*(src[i][j]+src[i][j-1]+src[i][j+1]
 *       +src[i+1][j]+src[i-1][j]).  range: 2-D within [1,N-1)^2 (NULL = all).
 *   JACC_LOOP_DOT_F64         : x IN f64, y IN f64, s REDUCE_SUM_F64;
 *       s = s + sum_{i in range} x[i]*y[i].
 *   JACC_LOOP_SUM_F64         : x IN f64, s REDUCE_SUM_F64; s = s + sum x[i].
 *   JACC_LOOP_GEMM_F64        (R-11): A IN f64[M][K], B IN f64[K][N],
 *       C OUT f64[M][N]; C = A*B.  range: 2-D over [0,M)x[0,N) (NULL = all).
 *   JACC_LOOP_SCATTER_ADD_F64 (R-6..R-8): idx IN i32[n], b IN f64[n],
 *       a INOUT f64[M]; for i in range: a[idx[i]] += b[i] (atomic).
 *   JACC_LOOP_SCATTER_ADD_I32 : idx IN i32[n], b IN i32[n], a INOUT i32[M].
 *   JACC_LOOP_HIMENO_F32      (NEXT-2, Himeno stencil loop, P:654, P:704,
 *       R-17): p IN f32[I][J][K], a IN f32[4][I][J][K], b IN f32[3][I][J][K],
 *       c IN f32[3][I][J][K], wrk1 IN, bnd IN, wrk2 OUT (f32[I][J][K]),
 *       gosa REDUCE_SUM_F64, omega SCALAR_F64 (.f64 field); for the 19-point
 *       stencil over range (3-D within [1,I-1)x[1,J-1)x[1,K-1), NULL = all):
 *       ss = (s0*a3 - p)*bnd; gosa += ss*ss; wrk2 = p + omega*ss (fp32 as
 *       written; gosa accumulated in fp64).
 *   JACC_LOOP_HIMENO_COPY_F32 : wrk2 IN, p OUT; p = wrk2 over the range.
 *   JACC_LOOP_FIG4_F64        (NEXT-3, Fig. 4): jx IN i32[n],
 *       kx IN i32[n], c IN f64, a OUT f64, b OUT f64, x SCALAR_F64; for i in
 *       range: x = x_in; a[i]=x; b[i]=a[i]; x=c[jx[i]]; a[kx[i]]=x;
 *       b[kx[i]]=a[kx[i]] -- two written arrays divided separately, every
 *       store guarded as in Fig. 4 (a's stores by a's and b's blocks, b's
 *       by b's, the read of c by the guard of the stores it feeds).  The
 *       loop must be race-free (kx injective, disjoint from the range).
 * 1-D array arguments may point inside a region (the loop's array starts
 * there); multi-dimensional arguments must point at the region base. */
enum {
    JACC_LOOP_SQUARE_F32 = 1,
    JACC_LOOP_JACOBI2D_F64 = 2,
    JACC_LOOP_DOT_F64 = 3,
    JACC_LOOP_SUM_F64 = 4,
    JACC_LOOP_GEMM_F64 = 5,
    JACC_LOOP_SCATTER_ADD_F64 = 6,
    JACC_LOOP_SCATTER_ADD_I32 = 7,
    JACC_LOOP_HIMENO_F32 = 8,
    JACC_LOOP_HIMENO_COPY_F32 = 9,
    JACC_LOOP_FIG4_F64 = 10
};

/* Iteration range, half-open per dimension (R-3). */
typedef struct {
    int ndims;
    int64_t lo[3];
    int64_t hi[3];
} jacc_range;

typedef enum {
    JACC_ARG_ARRAY_IN = 0,
    JACC_ARG_ARRAY_OUT = 1,
    JACC_ARG_ARRAY_INOUT = 2,
    JACC_ARG_SCALAR_F64 = 3,
    JACC_ARG_SCALAR_I64 = 4,
    /* reduction(+:s): ptr is a host double* holding s_in on entry and
     * s_out = s_in + sum on return (R-9); the launch is synchronous
     * (obligatory sync). */
    JACC_ARG_REDUCE_SUM_F64 = 5
} jacc_arg_kind;

typedef struct {
    int kind;      /* jacc_arg_kind */
    void *ptr;     /* host address inside a present region (arrays), or host double* (reductions) */
    double f64;    /* scalar value (SCALAR_F64) */
    int64_t i64;   /* scalar value (SCALAR_I64) */
} jacc_arg;

/* Distribute one loop over the logical devices:
 * resolve every array argument in the present table, apply the alias rule
 * (R-12), partition the written array's split dimension into n contiguous
 * owned blocks (dim 0; remainder rule R-2) -- or, for
 * reductions, the outermost iteration range -- clip each
 * device's iterations to its block, pull stale input intervals, run the
 * device kernel with fused write-set tracking (dirty min/max range, or a
 * dirty bitmap for the scatter, R-15), merge the recorded dirty regions
 * into the other replicas per the merge policy, and combine reductions
 * (NCCL allreduce when the devices are distinct GPUs).
 * async_id: -1 = synchronous (returns after completion); >= 0 = returns
 * after enqueue (reductions are always synchronous).
 * Errors: JACC_ERR_UNKNOWN_LOOP, JACC_ERR_INVALID (arg count/kind/shape,
 * in-place stencil or GEMM), JACC_ERR_NOT_PRESENT, JACC_ERR_CUDA/NCCL. */
jacc_status jacc_launch(int loop_id, const jacc_range *range,
                        const jacc_arg *args, int nargs, int async_id);

/* Wait for outstanding work (async_id -1 = all queues; with several async
 * queues, async_id >= 0 waits for that queue on every device). */
jacc_status jacc_wait(int async_id);

/* NEXT-4 automated asynchronous execution (Fig. 2).  With
 * nq > 1 queues (CUDA streams per device; the paper uses 16) every
 * launch is scheduled by its array dependencies: RAW/WAW on the last
 * writer of an array it touches, WAR on the last readers of an array it
 * writes.  async_id = JACC_ASYNC_AUTO (or -1): the queue of the most recent
 * dependency, or the least recently used queue when there is none;
 * async_id >= 0: that queue.  The launch waits only for the other queues
 * whose dependencies are not already ordered before it (a matrix of the
 * latest synchronisation between queues, transitive).  Single-process mode,
 * not during a graph capture.  nq = 1 restores the single stream.  With
 * several queues each queue has its own reduction scratch, scatters use the
 * direct kernel (the binned pipeline's scratch is per device) and the
 * iteration-split scatter is refused (JACC_ERR_INVALID). */
#define JACC_MAX_QUEUES 32
#define JACC_ASYNC_AUTO (-2)
jacc_status jacc_set_queues(int nq);

/* Pure host logic of the scheduler (no GPU): replay `nlaunch` launches with
 * nreads[l] / nwrites[l] array ids (concatenated in reads / writes) and
 * requested[l] (queue, or -1 = automatic); queue_out[l] = chosen queue,
 * waits_out[l*nq + q] = 1 if launch l waits for queue q. */
jacc_status jacc_queue_replay(int nq, int nlaunch, const int *nreads, const int64_t *reads,
                              const int *nwrites, const int64_t *writes, const int *requested,
                              int *queue_out, int *waits_out);

/* ---------------------------------------------------------------------- */
/* Introspection (parity tests and measurement)                            */
/* ---------------------------------------------------------------------- */

/* Dirty range recorded on device `dev` for the region containing `host`
 * by the most recent launch that wrote it (inclusive flat element
 * indices; empty = (UINT64_MAX, 0)).  Waits for outstanding work. */
jacc_status jacc_get_dirty_range(void *host, int dev, uint64_t *min, uint64_t *max);

/* Dirty bitmap of device `dev` for the region (bit k of word w <-> element
 * 32w+k), recorded by the most recent scatter launch; nwords must be
 * >= ceil(elements/32).  JACC_ERR_INVALID if no bitmap was recorded. */
jacc_status jacc_get_dirty_bitmap(void *host, int dev, uint32_t *out, size_t nwords);

/* D2H copy of `bytes` from the start of device `dev`'s replica of the
 * region containing `host` (no coherence action).  Waits for all work. */
jacc_status jacc_get_replica(void *host, int dev, void *out, size_t bytes);

/* Timing of the most recent launch (requires jacc_set_profiling(1)):
 * max over devices of kernel time and of merge time (seconds), and the
 * bytes moved device-to-device by its merge and pulls. */
jacc_status jacc_last_timing(double *t_kernel_s, double *t_merge_s, uint64_t *bytes_merged);

/* Record CUDA events around every loop kernel and merge (D13 timing
 * records).  Accumulated totals since the last reset: */
jacc_status jacc_set_profiling(int on);
jacc_status jacc_profile_totals(int dev, double *kernel_s, double *merge_s,
                                uint64_t *launches, uint64_t *bytes_merged);
jacc_status jacc_profile_reset(void);

/* D13 trace: with a path, turn profiling on and append one JSON
 * line per launch to the file once its CUDA events resolve:
 *   {"event", "kernel_id", "kernel", "queue", "waits": [queues waited on],
 *    "peer_waits": [devices whose previous launch it waited on],
 *    "t_kernel_s", "t_comm_s" (max over devices), "mode": "multi"|"dup",
 *    "merge": "eager"|"halo", "bytes_exchanged", "devices"}
 * NULL (or jacc_finalize) closes the file after a summary line
 *   {"summary": {"events", "total_kernel_s", "total_comm_s",
 *                "per_kernel_modes": {name: {"multi": k, "dup": m}}}}.
 * Every jacc_launch is also an NVTX range named after its loop.
 * Errors: JACC_ERR_INVALID (file cannot be opened), JACC_ERR_STATE while
 * capturing a graph. */
jacc_status jacc_set_trace(const char *path);

/* The CUDA stream (cudaStream_t) logical device `dev` runs on, and its
 * CUDA ordinal, so callers can time the path with their own events. */
jacc_status jacc_get_stream(int dev, void **stream, int *cuda_ordinal);

/* What a measurement must state about the runtime: the
 * logical devices, whether they are distinct GPUs, which reduction combine
 * runs (NCCL allreduce across distinct GPUs; otherwise the
 * fixed-order sum over peer memory), how many ordered pairs of distinct
 * GPUs have peer access (NVLink P2P loads/stores of the merges) and
 * the one-process-per-GPU mode.  With distinct GPUs an NCCL communicator
 * that cannot be built makes jacc_init / jacc_init_rank fail with
 * JACC_ERR_NCCL (never a silent switch of combine); JACC_NO_NCCL=1 asks
 * for the peer-memory combine explicitly.
 * Errors: JACC_ERR_STATE before init, JACC_ERR_INVALID for NULL. */
enum { JACC_COMBINE_PEER = 0, JACC_COMBINE_NCCL = 1 };
typedef struct {
    int n_devices;
    int distinct_gpus;   /* 1 if no two logical devices share a GPU */
    int combine;         /* JACC_COMBINE_PEER or JACC_COMBINE_NCCL */
    int peer_pairs;      /* ordered pairs (d, q), distinct GPUs, P2P enabled;
                            -1 in one-process-per-GPU mode (CUDA-IPC mappings
                            of the peers' memory carry the P2P there) */
    int multiprocess;    /* 1 in one-process-per-GPU mode */
    int rank;            /* this process's logical device (0: single process) */
} jacc_info;
jacc_status jacc_get_info(jacc_info *out);

/* ---------------------------------------------------------------------- */
/* One process per GPU (the launch model of bench.py under torchrun)       */
/* ---------------------------------------------------------------------- */
/* In this mode each process ("rank") owns ONE logical device (d = rank)
 * of `world`, every rank issues the same API calls in the same order
 * (SPMD), and the runtime reaches the other devices' replicas through
 * CUDA IPC mappings of their memory (NVLink P2P loads/stores on distinct
 * GPUs; plain device memory when ranks share one GPU).  Cross-device
 * ordering uses CUDA IPC events plus per-rank progress counters in POSIX
 * shared memory (no rank enqueues launch k before every rank has enqueued
 * launch k-1).  The caller moves the opaque byte blobs below between ranks
 * with any transport (bench.py uses torch.distributed): that is plumbing,
 * no data-path bytes travel through it.
 *
 * Protocol:
 *   rank 0: jacc_unique_id(id)            (optional: NCCL reduction combine,
 *                                          only when ranks are distinct GPUs)
 *   all:    jacc_init_rank(rank, world, ordinal, id or NULL, shm_name)
 *   all:    jacc_export_runtime(blob) -> all-gather -> jacc_import_runtime(peer, blob_peer)
 *   per array, all ranks in the same order:
 *           jacc_data_create(...); jacc_export_region(host, blob) -> all-gather
 *           -> jacc_import_region(host, peer, blob_peer) for every peer
 * Then the ordinary API applies.  jacc_update_device/update_host/wait/
 * data_delete/finalize and reductions are collective; update_host makes
 * the caller's own replica coherent and copies it to the caller's host
 * buffer.  Introspection calls accept only the caller's device. */
#define JACC_UNIQUE_ID_BYTES 128
#define JACC_RUNTIME_HANDLE_BYTES 256
#define JACC_REGION_HANDLE_BYTES 64

/* NCCL unique id for the reduction communicator (out: >= 128 bytes). */
jacc_status jacc_unique_id(void *out, size_t bytes);

/* Initialise this process as logical device `rank` of `world` on CUDA
 * ordinal `cuda_ordinal`.  unique_id: NULL = combine reductions over CUDA
 * IPC (required when ranks share a GPU), else the NCCL id from rank 0.
 * shm_name: name of the POSIX shared-memory segment for progress counters,
 * identical on all ranks and unique per job.  Errors: JACC_ERR_STATE if
 * initialised, JACC_ERR_INVALID, JACC_ERR_CUDA, JACC_ERR_NCCL. */
jacc_status jacc_init_rank(int rank, int world, int cuda_ordinal, const void *unique_id,
                           const char *shm_name);

/* Opaque handle blob of this rank's events, reduction buffer and GPU UUID
 * (>= JACC_RUNTIME_HANDLE_BYTES) / import a peer's (a peer on the same GPU
 * makes jacc_get_info report distinct_gpus = 0). */
jacc_status jacc_export_runtime(void *out, size_t bytes);
jacc_status jacc_import_runtime(int peer, const void *in, size_t bytes);

/* Opaque handle of this rank's replica of the region containing `host`
 * (>= JACC_REGION_HANDLE_BYTES) / map a peer's replica.  A launch that uses
 * a region before every peer replica is imported fails with JACC_ERR_STATE. */
jacc_status jacc_export_region(void *host, void *out, size_t bytes);
jacc_status jacc_import_region(void *host, int peer, const void *in, size_t bytes);

/* This process's logical device (0 in single-process mode, -1 before init). */
int jacc_rank(void);

/* ---------------------------------------------------------------------- */
/* Adaptive utilization controller (NEXT-1)                     */
/* ---------------------------------------------------------------------- */
/* Controller states: 0 DUP_WARMUP, 1 DUP_PROFILING, 2 MULTI, 3 DUP_FINAL. */
/* Pure host logic, no GPU: feed `len` observations (kernel time, comm time
 * [s], WriteSize [bytes] -- WriteSize = bytes the busiest device sends in
 * a multi-GPU merge) to a fresh controller for n devices and peak_p2p
 * [B/s]; states_out[i] = state before observation i, states_out[len] =
 * final state (len + 1 entries).  Errors: JACC_ERR_INVALID. */
jacc_status jacc_adaptive_replay(int n, double peak_p2p, int len, const double *t_kernel,
                                 const double *t_comm, const double *write_size, int *states_out);

/* Observations fed so far to the controller of the most recent kernel
 * identity launched with `loop_id` under JACC_MODE_ADAPTIVE (waits for
 * outstanding observations): up to `cap` entries, *len = total count,
 * *state_now = current state (-1 if none). */
jacc_status jacc_adaptive_history(int loop_id, int cap, double *t_kernel, double *t_comm,
                                  double *write_size, int *states, int *len, int *state_now);

/* ---------------------------------------------------------------------- */
/* CUDA graphs of launch sequences (single-process mode)                   */
/* ---------------------------------------------------------------------- */
/* Capture the device work of the launches issued between
 * jacc_graph_begin() and jacc_graph_end() (every device's stream, merges
 * and pulls included) into one CUDA graph; nothing executes during the
 * capture.  The graph maps the runtime state at begin (replica validity,
 * dirty-record slots) to the state at end; jacc_graph_replay runs it
 * `count` times and requires the current state to equal the captured
 * start state (true for a steady stencil ping-pong), else JACC_ERR_STATE.
 * Launches with a reduction cannot be captured (obligatory host sync) and
 * return JACC_ERR_INVALID; synchronous calls during a capture return
 * JACC_ERR_STATE.  jacc_data_delete() destroys every graph. */
jacc_status jacc_graph_begin(void);
jacc_status jacc_graph_end(int *graph_id);
jacc_status jacc_graph_replay(int graph_id, int count);
jacc_status jacc_graph_destroy(int graph_id);

const char *jacc_error_string(jacc_status s);

#ifdef __cplusplus
}
#endif
#endif /* JACC_H */
