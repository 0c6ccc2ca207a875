/* knn.h — C ABI of libknn.so: B200-native (sm_100a) brute-force k-NN search and
 * k-NN-graph construction, the data-parallel hot path of arXiv 1309.5478
 * ("Fast k-NNG construction with GPU-based quick multi-select").
 *
 * Problem statement (§Introduction): given a corpus of N points and a set
 * of M query points, k-NN finds for each query the k nearest corpus points; in the
 * k-NN graph (k-NNG) every corpus point is also a query.  Method:
 * (1) the M×N distance matrix, computed as a matrix product (PAPER.md:73-83,
 *     d^2 = ||x||^2 + ||y||^2 - 2 x.y), then
 * (2) a per-row multi-select of the k smallest distances and their indices
 *     ("GPU-based quick multi-select").
 *
 * Conventions (all entry points)
 *  - Layout: point sets are row-major fp32, one point per row, row stride = d
 *    ("vector-contiguous"; the paper's vectors are the columns of X).
 *    Outputs are M×k row-major: out_idx[i*k + r] (int32), out_dist[i*k + r] (fp32).
 *  - Order: each output row is sorted ascending by the total order
 *        (distance ascending, -0 == +0, NaN after +inf; ties by smaller index)
 *    (readings R1, R2, R6).  Results are deterministic and bit-identical
 *    across runs, launch configurations and GPU shardings.
 *  - Pointers: every float / int pointer argument is a DEVICE pointer on the ctx's
 *    device unless stated otherwise; `stream` is a cudaStream_t passed as void*
 *    (NULL = legacy default stream).  The caller owns all inputs and outputs; the
 *    library never frees or retains caller pointers after return.  Workspace is owned
 *    by the ctx, grown on demand, freed by knn_ctx_destroy.
 *  - Errors: status codes only, never exceptions/aborts across the ABI.  Argument
 *    errors are detected before any launch.  On error outputs are unspecified and
 *    knn_last_error(ctx) describes the failure.
 *  - Threading: a ctx is not thread-safe; distinct ctxs are independent.
 */
#ifndef KNN_B200_H
#define KNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KNN_ABI_VERSION 2

typedef struct knn_ctx* knn_ctx_t;

/* Distance metrics.  L2SQ = d^2, L2 = d_E = sqrt(d^2)
 * (PAPER.md:61).  COSINE: the key 1 - x.y / (||x|| ||y||) (PAPER.md:63-66 gives the
 * similarity d_C; 1 - d_C makes "k smallest" mean nearest), in [0, 2];
 * a zero-norm vector gets the key 3.0 against everything.  PEARSON: the
 * cosine key of the mean-centred vectors (a constant vector has zero
 * centred norm: 3.0).  COSINE / PEARSON need the tensor-core path (KNN_ERR_UNSUPPORTED
 * under KNN_GEMM=simt).  Keys are within 1e-5 (absolute) of the fp64 definition. */
typedef enum { KNN_L2SQ = 0, KNN_L2 = 1, KNN_COSINE = 2, KNN_PEARSON = 3 } knn_metric;

typedef enum {
    KNN_OK = 0,
    KNN_ERR_ARG = 1,          /* invalid argument (sizes, k range, null pointer, alignment) */
    KNN_ERR_UNSUPPORTED = 2,  /* valid request the library does not implement (metric, k > 1024) */
    KNN_ERR_NONFINITE = 3,    /* input holds NaN/inf, or a squared norm >= FLT_MAX/4 (R8) */
    KNN_ERR_OOM = 4,          /* device workspace allocation failed */
    KNN_ERR_CUDA = 5,         /* a CUDA runtime/driver call failed */
    KNN_ERR_NCCL = 6,         /* a collective failed (NCCL or the host transport), or NCCL missing */
    KNN_ERR_INTERNAL = 7
} knn_status;

/* "No self exclusion" value for the self_shift arguments below. */
#define KNN_NO_SELF INT64_MIN
/* Largest supported k. */
#define KNN_MAX_K 1024

int         knn_abi_version(void);
/* Create a context bound to CUDA device `device`. */
knn_status  knn_ctx_create(int device, knn_ctx_t* out);
knn_status  knn_ctx_destroy(knn_ctx_t ctx);
/* Message for the last non-OK status of this ctx (static storage inside ctx). */
const char* knn_last_error(knn_ctx_t ctx);

/* ---------------------------------------------------------------- top level ------
 * Blocking: return after the work queued on `stream` has completed, so the status is
 * final (including KNN_ERR_NONFINITE from the input validation of knn_rownorms).
 *
 * knn_graph: the k-NNG of X (N×d).  Row i lists the k nearest OTHER points of x_i:
 * self is excluded by position (reading R3), so 1 <= k <= min(N-1, 1024).
 * metric: any knn_metric.  out_idx/out_dist: N×k. */
knn_status knn_graph(knn_ctx_t ctx, const float* X, int64_t N, int32_t d, int32_t k,
                     int32_t metric, int32_t* out_idx, float* out_dist, void* stream);

/* knn_search: for each of the M queries Q (M×d), its k nearest points of X (N×d) under
 * squared Euclidean distance (the north-star signature knn_search(query, M, corpus, N,
 * d, k)).  1 <= k <= min(N, 1024).  out_idx/out_dist: M×k. */
knn_status knn_search(knn_ctx_t ctx, const float* Q, int64_t M, const float* X, int64_t N,
                      int32_t d, int32_t k, int32_t* out_idx, float* out_dist, void* stream);

/* knn_search_block: the general block both sharded drivers are built from.  Query i of
 * Q against corpus point j of X, with
 *   - self exclusion by position: pair (i, j) is dropped when j == i + self_shift
 *     (self_shift = KNN_NO_SELF: nothing dropped).  A row whose valid corpus points
 *     number fewer than k is padded with (+inf, excluded index) entries, which sort
 *     after every finite distance;
 *   - idx_offset added to every returned index (global index of X's first row).
 * 1 <= k <= min(N, 1024).  metric: any knn_metric.  Blocking, like knn_graph. */
knn_status knn_search_block(knn_ctx_t ctx, const float* Q, int64_t M, const float* X,
                            int64_t N, int32_t d, int32_t k, int32_t metric,
                            int64_t self_shift, int64_t idx_offset,
                            int32_t* out_idx, float* out_dist, void* stream);

/* Same computation with HOST input/output buffers (pageable or pinned): copies Q and X
 * to the device, runs knn_search_block, copies the M×k results back; all inside the
 * call.  This is the end-to-end entry point a host application uses. */
knn_status knn_search_block_host(knn_ctx_t ctx, const float* Q_host, int64_t M,
                                 const float* X_host, int64_t N, int32_t d, int32_t k,
                                 int32_t metric, int64_t self_shift, int64_t idx_offset,
                                 int32_t* out_idx_host, float* out_dist_host, void* stream);

/* ---------------------------------------------------------------- building blocks --
 * Stream-ordered (asynchronous): they validate arguments, enqueue kernels on `stream`
 * and return.  Used by the tests and the benchmark. */

/* Out-of-core k-NN (NEXT-4; "batch execution with data partitioning for
 * large corpus data that do not fit into GPU memory ... overlap computation with data
 * transfer ... merging of results between executions").  Q_host (M×d) and X_host (N×d)
 * stay in HOST memory (pageable or pinned; pageable ranges are page-locked with
 * cudaHostRegister for the duration of the call); the device holds one block of at
 * most query_block queries and two staging buffers of corpus chunks of chunk_points
 * points.  Chunk c+1 is copied host->device on a separate stream while chunk c is
 * processed (prep, GEMM, select with global indices), and each chunk's partial top-k is
 * merged into the running result with the a-S6 merge.  graph != 0: the k-NNG of X
 * (requires Q_host == X_host, M == N; self excluded by position, k <= N-1).  Results
 * (M×k, host) are bit-identical to knn_search / knn_graph on device-resident inputs:
 * per-pair values do not depend on the chunking and the merge is exact under the total
 * order.  chunk_points, query_block <= 0 pick defaults (131072 points; all queries up
 * to a 2 GiB block).  A trailing chunk with fewer than k+1 points is folded into the
 * previous one.  Blocking. */
knn_status knn_search_streamed(knn_ctx_t ctx, const float* Q_host, int64_t M, const float* X_host,
                               int64_t N, int32_t d, int32_t k, int32_t metric, int32_t graph,
                               int64_t chunk_points, int64_t query_block, int32_t* out_idx_host,
                               float* out_dist_host);

/* ||x_j||^2 = sum_t x_j[t]^2 for j < N, accumulated in fp64, rounded to fp32
 * (norms by reduction; reading R15).  out_sqn: N floats.
 * Also writes *out_flag (device int32, may be NULL) = 1 when some x is non-finite or
 * some ||x||^2 >= FLT_MAX/4, else leaves it unchanged (caller zeroes it). */
knn_status knn_rownorms(knn_ctx_t ctx, const float* X, int64_t N, int32_t d, float* out_sqn,
                        int32_t* out_flag, void* stream);

/* The distance matrix: for i < M, j < N
 *   D[i*ldD + j] = max(||q_i||^2 + ||x_j||^2 - 2 q_i.x_j, 0)   (metric KNN_L2SQ)
 *                 sqrt of that                                (metric KNN_L2)
 *                 the cosine / Pearson key                     (KNN_COSINE / KNN_PEARSON)
 * with the dot products from the FP32-accurate split tensor-core GEMM
 * and +inf where j == i + self_shift.  ldD >= N.  D: M×ldD floats. */
knn_status knn_distances(knn_ctx_t ctx, const float* Q, int64_t M, const float* X, int64_t N,
                         int32_t d, int32_t metric, int64_t self_shift, float* D, int64_t ldD,
                         void* stream);

/* The per-row multi-select: for each row i < M of D (row stride ldD,
 * N columns), the k smallest (D[i,j], j) under the total order above, written sorted.
 * Values are written canonicalised (-0 -> +0, NaN -> +NaN).  1 <= k <= min(N, 1024),
 * ldD >= N.  Exact: bit-identical to sorting the row. */
knn_status knn_select(knn_ctx_t ctx, const float* D, int64_t M, int64_t N, int64_t ldD,
                      int32_t k, int32_t* out_idx, float* out_dist, void* stream);
/* Which kernel the last knn_select-style launch of this process used (diagnostic):
 * *kind = 0 warp per row (k <= 128, many rows), 1 CTA per row (persistent ring), 2 CTA per
 * row on unaligned rows, 3 a thread-block cluster per row (few rows: one
 * block per query cannot fill the GPU below ~#SM rows; NEXT-3), with *splits = the
 * cluster size (row segments merged over distributed shared memory), else 1; 4 two-pass
 * warp per row (k <= 32, 1024 <= N <= 131072: pivot = the k-th smallest group minimum,
 * PAPER.md:56). */
knn_status knn_last_select_kernel(int32_t* kind, int32_t* splits);

/* ABLATION, not the product path: the paper's quick multi-select as written
 * (PAPER.md:49-56): one warp per row, repeated ballot/popc partitions around a pivot into
 * two global auxiliary arrays with two coalesced writes per 32 elements, recursion into
 * the side holding the K-th element with a stack of references to the kept left sides,
 * direct sort below 1024 elements.  Same contract and results as knn_select (pairs are
 * (value, index) under the total order, so it is exact); used by scripts/select_sweep.py to
 * measure the paper's algorithm on B200.  Workspace: 16 bytes per element of a row block
 * (ctx-owned, rows processed in blocks of at most 4 GiB). */
knn_status knn_select_paper(knn_ctx_t ctx, const float* D, int64_t M, int64_t N, int64_t ldD,
                            int32_t k, int32_t* out_idx, float* out_dist, void* stream);

/* k-way merge of partial lists ("Batch execution will obviously require
 * merging of results"): part_dist / part_idx are G blocks laid out [G][M][k]; list g's
 * indices are shifted by offsets_host[g] (a HOST array of G int64) before the merge.
 * Output: the first k of the union under the total order (global index tie-break),
 * M×k.  Equal to the unsharded select when the G lists come from contiguous column
 * shards.  1 <= G <= 64, 1 <= k <= 1024. */
knn_status knn_merge(knn_ctx_t ctx, const float* part_dist, const int32_t* part_idx, int32_t G,
                     int64_t M, int32_t k, const int64_t* offsets_host, int32_t* out_idx,
                     float* out_dist, void* stream);

/* The merge over a table of G list pointers (host arrays of G device pointers): list g
 * of row row0 + r starts at dist_lists[g] + (row0 + r) * k (idx_lists likewise), its
 * indices shifted by offsets_host[g]; output rows r < M.  The pointers may be local or
 * mapped from a peer GPU's memory with knn_ipc_open: the corpus-sharded k-NNG (Par-2,
 * PAPER.md:102) merges its own row block straight from its peers' partial lists over
 * NVLink, with no all-to-all copy.  Same results as knn_merge.  1 <= G <= 64. */
knn_status knn_merge_lists(knn_ctx_t ctx, const float* const* dist_lists,
                           const int32_t* const* idx_lists, int32_t G, int64_t row0, int64_t M,
                           int32_t k, const int64_t* offsets_host, int32_t* out_idx,
                           float* out_dist, void* stream);

/* Symmetric multi-GPU k-NNG (Par-3): the pivot plan's phases, so that the
 * ranks of a job split the UPPER TRIANGLE of the distance matrix (the transpose reuse of
 * PAPER.md:83 survives sharding) instead of splitting rows (which doubles the per-rank
 * multiply work).  X is the full N×d point set on every rank (device).
 *  1. knn_graph_pivots: pivots of rows [row0, row0+rows) (the sample pass of §6.5) into
 *     thr[row0 .. row0+rows).  The caller all-gathers thr over the ranks; thr must hold
 *     roundup(N, 256) floats, NaN past N.  Asynchronous.
 *  2. knn_graph_partition: the partition GEMM over the triangle units [unit_lo, unit_hi)
 *     (knn_graph_units(N) in total), appending candidates of ANY row to the caller's lists
 *     cnt[N] (zeroed here) and cent[N][cap] (cap = knn_graph_list_cap(k)): 64-bit entries
 *     (key << 32 | column), key = the order-preserving bits of the distance (IEEE bits
 *     with the sign bit set, for values >= +0).  Asynchronous.  Directly after
 *     knn_graph_pivots on the same ctx, points, metric and stream it reuses the operands
 *     that call prepared (no second pass over X).
 *     For k <= 32 and the L2 metrics (unless KNN_PLAN_PIVOT_EXACT or KNN_PIVOT1=0) it
 *     queues, as knn_graph does, the single-product partition (keys = lower bounds of the
 *     distance) next to the FP32-accurate one, the device choosing one from all N pivots
 *     (thr must then hold every rank's pivots); the choice is kept in the ctx.
 *  3. knn_graph_gather_select: for rows [row0, row0+rows), concatenates the G ranks' lists
 *     (host arrays of G device pointers; peers' lists mapped with knn_ipc_open, read over
 *     NVLink inside the kernel) and runs the exact candidate select into out (rows×k) —
 *     after a single-product partition on this ctx, the fp32 re-evaluation of the rows'
 *     survivors from the points X and the pivots thr passed to knn_graph_partition (both
 *     must still be alive).
 *     Blocking; returns KNN_ERR_INTERNAL when a list overflowed or a row's certificate
 *     failed (fewer than k candidates): the caller then falls back to another plan.
 * k <= N-1; N >= 16384 and 1 <= k <= 1024 (else KNN_ERR_UNSUPPORTED); tensor-core path. */
int64_t knn_graph_units(int64_t N);
int32_t knn_graph_list_cap(int32_t k);
/* The pivot plans' column-sample size for N corpus points and k: the
 * chunk-minimum sample of k <= 32 (N / 8, 12 or 16 by N; env KNN_PIVOT_DIV overrides) or
 * the quantile sample of k > 32, rounded up to 256 columns.  (Introspection: bench.py's
 * flop accounting of the sample pass.) */
int64_t knn_pivot_sample_size(knn_ctx_t ctx, int64_t N, int32_t k);
knn_status knn_graph_pivots(knn_ctx_t ctx, const float* X, int64_t N, int32_t d, int32_t k, int32_t metric,
                            int64_t row0, int64_t rows, float* thr, void* stream);
knn_status knn_graph_partition(knn_ctx_t ctx, const float* X, int64_t N, int32_t d, int32_t k,
                               int32_t metric, const float* thr, int64_t unit_lo, int64_t unit_hi,
                               int32_t* cnt, uint64_t* cent, int32_t cap, void* stream);
knn_status knn_graph_gather_select(knn_ctx_t ctx, int32_t G, const int32_t* const* cnts,
                                   const uint64_t* const* cents, int32_t cap, int64_t N, int32_t k,
                                   int64_t row0, int64_t rows, int32_t* out_idx, float* out_dist, void* stream);

/* CUDA IPC plumbing for knn_merge_lists across processes (one process per GPU):
 * knn_ipc_export writes the 64-byte IPC handle of the allocation holding dev_ptr and the
 * byte offset of dev_ptr inside it; a peer process passes both to knn_ipc_open, which maps
 * the allocation (once per ctx; later opens of the same handle reuse the mapping) and
 * returns the peer-visible pointer.  knn_ipc_close_all unmaps everything this ctx opened
 * (also done by knn_ctx_destroy).  The exporter must keep the memory alive while mapped. */
knn_status knn_ipc_export(knn_ctx_t ctx, const void* dev_ptr, uint8_t handle[64], int64_t* offset);
knn_status knn_ipc_open(knn_ctx_t ctx, const uint8_t handle[64], int64_t offset, void** dev_ptr);
knn_status knn_ipc_close_all(knn_ctx_t ctx);

/* ---------------------------------------------------------------- multi-GPU ---------
 * One process per GPU, each with its own ctx (PAPER.md:102:
 * "batch execution with data partitioning ... merging of results"; the
 * queries are independent, coarse-grained parallelism).  The caller creates the
 * communicator once per ctx, then every rank makes the SAME sharded call with the same
 * arguments (collective semantics: a rank that does not call blocks the others).
 *
 * knn_comm_unique_id: an NCCL unique id (128 bytes) made on ONE rank; the caller ships it
 *   to the others (e.g. torch.distributed.broadcast_object_list).  NCCL is loaded at run
 *   time (dlopen "libnccl.so.2", else the build-time path, else env KNN_NCCL_LIB);
 *   KNN_ERR_NCCL if it cannot be loaded.
 * knn_comm_init: joins the communicator of `nranks` ranks as `rank` on the ctx's device
 *   (blocking, collective).  Collectives then run on the caller's stream over NVLink /
 *   NVSwitch.  Re-initialising replaces the previous communicator.
 * knn_comm_init_ops: the same with a caller-supplied HOST transport instead of NCCL (for
 *   process groups NCCL cannot serve, e.g. several ranks sharing one GPU in tests): the
 *   library synchronises the stream, stages the data through pinned host memory and calls
 *   the callbacks, which must perform the collective over all ranks and return 0 (nonzero:
 *   the call fails with KNN_ERR_NCCL).  All pointers passed to the callbacks are HOST
 *   pointers; `bytes` counts are per rank.  The ops struct is copied; `user` is passed back.
 * knn_comm_destroy: releases the communicator (also done by knn_ctx_destroy).
 * knn_comm_info: *backend = 0 none, 1 NCCL, 2 host callbacks; *rank, *nranks. */
typedef struct knn_comm_ops {
    int (*allgather)(void* user, const void* send, void* recv, int64_t bytes);  /* recv: nranks*bytes */
    int (*broadcast)(void* user, void* buf, int64_t bytes, int root);
    int (*alltoall)(void* user, const void* send, void* recv, int64_t bytes);   /* block g -> rank g */
    int (*allreduce_max_i32)(void* user, int32_t* buf, int64_t count);
    void* user;
} knn_comm_ops;
knn_status knn_comm_unique_id(uint8_t id[128]);
knn_status knn_comm_init(knn_ctx_t ctx, int32_t rank, int32_t nranks, const uint8_t id[128]);
knn_status knn_comm_init_ops(knn_ctx_t ctx, int32_t rank, int32_t nranks, const knn_comm_ops* ops);
knn_status knn_comm_destroy(knn_ctx_t ctx);
knn_status knn_comm_info(knn_ctx_t ctx, int32_t* backend, int32_t* rank, int32_t* nranks);

/* Contiguous block r of ceil(n/parts)-sized blocks of [0, n): [*lo, *hi) (possibly empty).
 * The split every sharded call uses for rows, columns and triangle units.  Host only. */
void knn_shard_range(int64_t n, int32_t parts, int32_t r, int64_t* lo, int64_t* hi);

/* Sharded calls.  shard_mode:
 *   KNN_SHARD_QUERY  (Par-1): query rows split in contiguous blocks; each rank runs the
 *                    whole single-GPU hot path (knn_search_block) on its rows against all
 *                    N points; results all-gathered.
 *   KNN_SHARD_CORPUS (Par-2): corpus columns split; each rank computes partial top-k lists
 *                    of EVERY query row against its columns (global self exclusion and
 *                    indices), an all-to-all hands each rank the nranks partial lists of its
 *                    own rows, the k-way merge kernel (a-S6) reduces them, results
 *                    all-gathered.  Needs k <= the smallest column block.
 *   KNN_SHARD_SYM    (Par-3, knn_graph_sharded only; N >= 16384 on the tensor-core path):
 *                    the ranks split the UPPER TRIANGLE of the k-NNG's distance matrix (the
 *                    transpose reuse of PAPER.md:83 survives sharding): pivots of own rows
 *                    (all-gathered), the partition GEMM over 1/nranks of the triangle's
 *                    256x256 blocks appending candidates of any row to rank-local lists,
 *                    then each rank's select reads the lists of its rows from every rank
 *                    directly in peer memory (CUDA IPC mappings, exchanged once over the
 *                    communicator; NVLink loads inside the kernel); results all-gathered.
 *                    Falls back to KNN_SHARD_QUERY (on every rank alike) when peer mappings
 *                    are unavailable, N < 16384, or a certificate fails.
 * Inputs: X (N×d) and Q (M×d) are device buffers on every rank; their contents on rank 0
 * are broadcast into them on the other ranks inside the call (so they must be writable).
 * Outputs: the full M×k (N×k) lists on EVERY rank, bit-identical to the single-GPU calls
 * for every mode and rank count.  Blocking.  Without a communicator they run as one rank;
 * one rank runs the single-GPU call directly (env KNN_SHARD_G1_PHASES=1: the sharded
 * phases anyway, for tests).
 * Argument rules as knn_search_block / knn_graph.  knn_search_sharded: squared L2,
 * modes QUERY / CORPUS.  Collective failures return KNN_ERR_NCCL; a rank whose local
 * computation fails makes every rank return an error (statuses agreed by an all-reduce). */
#define KNN_SHARD_QUERY 0
#define KNN_SHARD_CORPUS 1
#define KNN_SHARD_SYM 2
knn_status knn_graph_sharded(knn_ctx_t ctx, int32_t shard_mode, float* X, int64_t N, int32_t d, int32_t k,
                             int32_t metric, int32_t* out_idx, float* out_dist, void* stream);
knn_status knn_search_sharded(knn_ctx_t ctx, int32_t shard_mode, float* Q, int64_t M, float* X, int64_t N,
                              int32_t d, int32_t k, int32_t* out_idx, float* out_dist, void* stream);
/* Mode the last sharded call of this ctx actually ran (after fallbacks), -1 none. */
int knn_last_shard_mode(knn_ctx_t ctx);

/* DIAGNOSTIC (not the hot path): the distance GEMM of X against itself (sym != 0: the
 * symmetric upper-triangle schedule) with an epilogue that only drains the TMEM
 * accumulators — the tensor-core mainloop's own rate.  Runs `reps` timed launches after one
 * warm-up and returns the mean launch time in *ms.  Blocking. */
knn_status knn_diag_mainloop(knn_ctx_t ctx, const float* X, int64_t N, int32_t d, int32_t sym,
                             int32_t reps, double* ms);

/* ---------------------------------------------------------------- introspection ----
 * Number of kernel launches this ctx has issued so far (for benchmarks). */
int64_t knn_launch_count(knn_ctx_t ctx);

/* Which distance-GEMM plan this ctx uses: 0 = tcgen05 split-fp16 tensor-core GEMM
 * (gemm_tc.cu), 1 = SIMT FP32 FFMA (gemm_simt.cu; selected by env KNN_GEMM=simt at
 * ctx creation, or when the device is not sm_100). */
int knn_gemm_path(knn_ctx_t ctx);
/* Plan of the top-level calls (PAPER.md:56 quick multi-select):
 * KNN_PLAN_AUTO (default): for N >= 16384 and M >= 256 on the tensor-core path the pivot
 * (partition) plan — a sampled per-row pivot, the GEMM epilogue keeping only elements below
 * it, an exact select of the candidates, the call redone on the full matrix if a row's
 * certificate fails; otherwise the materialised distances (symmetric upper-triangle GEMM
 * for the k-NNG) + select.  KNN_PLAN_MATERIALISED: never the pivot plan.  KNN_PLAN_FUSED
 * is reserved: round 1's per-row-list fused kernel was retired (4.5x slower than the pivot
 * plan, which is the fused GEMM+select); setting it returns KNN_ERR_UNSUPPORTED.
 * For k <= 32 and the L2 metrics the AUTO pivot plan may partition on the single hi.hi
 * product with its error bound and re-evaluate the survivors near the k-th from the fp32
 * inputs (chosen on the device per call when that bound is narrow against
 * the pivots): its distances are then the direct fp32 sum of squared differences (more
 * accurate than the split-fp16 contraction, within the same tolerance of the exact value,
 * but not the same bits).  KNN_PLAN_PIVOT_EXACT: the pivot plan with the FP32-accurate
 * 3-product partition only; it, MATERIALISED and the symmetric plan give bit-identical
 * results.
 * Environment, read at ctx creation: KNN_FUSED=0 (MATERIALISED), KNN_PIVOT=0
 * (no pivot plan), KNN_SYM=0 (no symmetric GEMM), KNN_PIVOT_DIV=n (sample N/n columns,
 * default 8), KNN_PIVOT_CAP (candidate list capacity), KNN_D_BUDGET_MB (distance block
 * budget), KNN_GEMM=simt (FFMA cross-check GEMM), KNN_PIVOT_MARGIN (tests: override the
 * sample's error margin), KNN_PIVOT1=1 / 0 (k <= 32, L2: always / never the single-product
 * partition; unset: chosen on the device), KNN_PIVOT1_RATIO (the choice's largest bound
 * width relative to the mean pivot, default 0.02), KNN_PIVOT_RANK (0: the certified pivot
 * rank k+1; r: rank r). */
typedef enum {
    KNN_PLAN_AUTO = 0,
    KNN_PLAN_FUSED = 1,
    KNN_PLAN_MATERIALISED = 2,
    KNN_PLAN_PIVOT_EXACT = 3
} knn_plan;
knn_status knn_set_plan(knn_ctx_t ctx, int32_t plan);
/* Plan the last top-level call of this ctx executed: 0 = blocked distances + select,
 * 1 = (retired fused plan, never reported), 2 = symmetric k-NNG distances (upper triangle of 256x256 blocks,
 * each written directly and transposed) + select, 3 = pivot plan,
 * symmetric, 4 = pivot plan, general block, 5 / 6 = the same with the single-product
 * partition and the fp32 re-evaluation (L2 metrics, k <= 32), -1 = none yet.  The pivot plan (k <= 32,
 * N >= 16384) is the quick multi-select partition of PAPER.md:56 applied at matrix scale:
 * a sample pass over the first N/8 corpus points (one fp16 product plus a bound of its
 * error) gives each row the minimum of every 32-column chunk; the row pivot is the k-th
 * smallest of those minima (>= the row's k-th distance); the FP32-accurate GEMM keeps
 * only elements <= pivot (for rows and, in the symmetric plan, transposed for columns);
 * an exact select of the candidates follows.  Rows with fewer than k candidates (a
 * failed certificate) or a candidate-buffer overflow make the call redo itself on the
 * full matrix. */
int knn_last_plan(knn_ctx_t ctx);
/* Total candidates the last pivot-plan call kept (sum over rows of the partition's
 * survivors; 0 for the other plans, -1 for a null ctx).  Diagnostic: the bench reports
 * the candidate select's algorithmic bytes from it. */
int64_t knn_last_candidates(knn_ctx_t ctx);

/* Per-kernel device timing for benchmarks: when enabled, every launch is bracketed by
 * CUDA events recorded on the launch stream.  knn_profile_enable(ctx, 1) also resets
 * the counters.  knn_profile_read waits for the recorded events and returns the summed
 * duration (ms) and the launch count of one kernel class.  Classes: PREP (a-S2), GEMM
 * (materialised distance GEMM, or the pivot plans' sample pass), SELECT (a-S4 select, or
 * the pivot select), MERGE (the pivot plans' candidate select; the streamed merge),
 * FUSED (the partition GEMM of the pivot plans), SHARD_MERGE (the k-way merge of the
 * corpus-sharded calls). */
typedef enum { KNN_KERNEL_PREP = 0, KNN_KERNEL_GEMM = 1, KNN_KERNEL_SELECT = 2,
               KNN_KERNEL_MERGE = 3, KNN_KERNEL_FUSED = 4, KNN_KERNEL_SHARD_MERGE = 5 } knn_kernel;
knn_status knn_profile_enable(knn_ctx_t ctx, int32_t on);
knn_status knn_profile_read(knn_ctx_t ctx, int32_t kernel, double* total_ms, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* KNN_B200_H */
