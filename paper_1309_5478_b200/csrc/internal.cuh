// internal.cuh — shared device helpers and launcher declarations of libknn.so.
// Product code only; nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdint>

namespace knn {

constexpr int kMaxK = 1024;
constexpr uint32_t kKeyMax = 0xFFFFFFFFu;  // larger than every key (used as "accept all")

// Order-preserving map float -> uint32 for the total order of include/knn.h:
// -0 == +0 (reading R6), every NaN -> +NaN, which sorts after +inf.
__device__ __forceinline__ uint32_t ukey(float x) {
    uint32_t b = __float_as_uint(x);
    b = (b == 0x80000000u) ? 0u : b;                       // -0 -> +0
    b = ((b & 0x7FFFFFFFu) > 0x7F800000u) ? 0x7FC00000u : b;  // NaN -> +NaN
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ukey_to_float(uint32_t u) {
    uint32_t b = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
    return __uint_as_float(b);
}

__host__ __device__ constexpr int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ constexpr int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// The K padding of the split operands: one 128-byte swizzle atom of fp16 = 64 elements.
constexpr int kSplitKAlign = 64;
// Per-point arrays read by the tensor-core GEMMs (norms, scales, pivots) are allocated and
// zero-padded to a multiple of one column tile.
constexpr int kColPad = 256;

// ---------------------------------------------------------------- launchers --------
// prep.cu: row norms (fp64 accumulate) + non-finite flag; optionally the scaled fp16
// hi/lo split for the tensor-core GEMM (hi/lo may be null).
// eps2 (optional, L2 metrics with the split): per point ||s x - hi||^2 / ||s x||^2 rounded
// up (0 on the padding to kColPad); tmax2 (optional): atomically raised to the max eps2.
cudaError_t launch_prep(const float* X, int64_t N, int32_t d, int32_t d_pad, float* sqn,
                        float* rscale, __half* hi, __half* lo, int32_t* flag, int32_t metric,
                        cudaStream_t s, float* eps2 = nullptr, float* tmax2 = nullptr);
// Per-point single-product bound terms from prep's eps2 and the call's *tmax2 (prep.cu,
// DESIGN.md §6.5): nsc = sqn (1 - F1) rounded down (the partition's lower-bound norms; may be null),
// ninf = sqn (1 + Fs) rounded up (the sample's upper-bound norms; may be null), bnd =
// sqn F1 rounded up (may be null).  |u_hh - D| <= Fs_q sqn_q + Fs_x sqn_x <= F1_q .. for
// every pair of points prepared with the same *tmax2.
cudaError_t launch_bound_norms(const float* sqn, const float* eps2, int64_t n, const float* tmax2, int32_t d_pad,
                               float* nsc, float* ninf, float* bnd, cudaStream_t s);

// prep.cu: the pivot plans' column sample: S points perm(j) = (j * sample_stride(N)) mod N,
// their split operands and epilogue terms copied contiguously (column arrays padded).
int64_t sample_stride(int64_t N);
// smax (device float, may be null): the max of the sample's sqn terms.
cudaError_t launch_gather_sample(const __half* hi, const __half* lo, const float* sqn, const float* rs,
                                 int64_t N, int64_t S, int32_t d_pad, __half* shi, __half* slo, float* ssqn,
                                 float* srs, float* smax, cudaStream_t s);

// *out = max(0, v[0..n)) (the sample pass's XMAX for a sample prepared in place).
cudaError_t launch_max_nonneg(const float* v, int64_t n, float* out, cudaStream_t s);

// gemm_simt.cu: FP32 FFMA distance GEMM with the fused epilogue.
cudaError_t launch_dist_simt(const float* Q, const float* qn, int64_t M, const float* X,
                             const float* xn, int64_t N, int32_t d, int32_t metric,
                             int64_t self_shift, float* D, int64_t ldD, cudaStream_t s);

// gemm_tc.cu: tcgen05 3-pass split-fp16 distance GEMM with the fused epilogue.
struct TcOperands {
    const __half* q_hi; const __half* q_lo; const float* qn; const float* q_rs; int64_t M;
    const __half* x_hi; const __half* x_lo; const float* xn; const float* x_rs; int64_t N;
    int32_t d_pad;
};
cudaError_t launch_dist_tc(const TcOperands& op, int32_t metric, int64_t self_shift, float* D,
                           int64_t ldD, int num_sms, cudaStream_t s);
// Symmetric k-NNG distances (queries = corpus, self excluded): the whole N x N matrix from
// the upper triangle of 256x256 blocks, each also written transposed.
cudaError_t launch_dist_tc_sym(const TcOperands& op, int32_t metric, float* D, int64_t ldD,
                               int num_sms, cudaStream_t s);
// Pivot (partition) plan: the GEMM keeps, per row, the elements at or below thr[row]
// (squared domain) as candidates cent[row*cap + i], i < cnt[row], entries (ukey << 32 | col)
// (the ukey of the distance: order-preserving bits); SYM also records the transposed
// element for the column's row.  flag |= 2 on candidate overflow.
// unit_lo / unit_hi (sym only): the triangle's units [unit_lo, unit_hi); -1 = all.
// col_major (sym only): units in column-major order (the units of column blocks [0, J) are
// [0, J (J + 1) / 2)): the host-pipelined k-NNG partitions the triangle as chunks arrive.
cudaError_t launch_dist_tc_pivot(const TcOperands& op, int32_t metric, int64_t self_shift, bool sym,
                                 const float* thr, int32_t* cnt, uint64_t* cent,
                                 int32_t cap, int32_t* flag, int num_sms, cudaStream_t s,
                                 int64_t unit_lo = -1, int64_t unit_hi = -1, bool col_major = false,
                                 int32_t gate = -1);
// The same partition from the single hi.hi product (L2 metrics): kept iff the lower bound
// L = u_hh - F1_q ||q||^2 - F1_x ||x||^2 <= thr[row] (resp. thr[col]); the key is L.
// op.qn / op.xn must be launch_bound_norms' nsc terms (prep norms scaled by 1 - F1).
cudaError_t launch_dist_tc_pivot1(const TcOperands& op, int32_t metric, int64_t self_shift, bool sym,
                                  const float* thr, int32_t* cnt, uint64_t* cent,
                                  int32_t cap, int32_t* flag, int num_sms, cudaStream_t s, int32_t gate = -1,
                                  int64_t unit_lo = -1, int64_t unit_hi = -1, bool col_major = false);
// Device-side choice of the pivot plan's partition: flag[1] = 1 (single
// product + re-evaluation) iff the single-product bound is narrow against the pivots,
// 2 F (mean qn + mean xn) <= ratio * mean(finite pivots), else 0 (3 products); the callers
// pass the bnd terms of launch_bound_norms with F = 1.
// part: pivot1_decide_ws_bytes() of device scratch; counter: a device uint zeroed before the call.
size_t pivot1_decide_ws_bytes();
cudaError_t launch_pivot1_decide(const float* thr, const float* qn, int64_t M, const float* xn, int64_t N,
                                 float F, float ratio, int32_t* flag, double* part, unsigned* counter,
                                 cudaStream_t s);
// Diagnostic: the 3-product GEMM with an epilogue that only drains TMEM (mainloop rate).
cudaError_t launch_dist_tc_null(const TcOperands& op, bool sym, int num_sms, cudaStream_t s);
// Pivot sample pass: mins[c][i] = min distance of query i over corpus points 32c..32c+31
// (N a multiple of 32; self pair excluded).
// The sample is S columns (a multiple of 256): S/256 full column blocks of op's N columns,
// spread evenly over them (block j * ((N/256) / (S/256))), so that ordered data (e.g. points
// sorted by cluster) still gives every row a representative sample.
// xmax: device pointer to an upper bound of the columns' sqn terms (the sample's max).
// bounded_norms: op.qn / op.xn are launch_bound_norms' ninf terms (L2; no constant margin).
cudaError_t launch_dist_tc_mins(const TcOperands& op, int64_t S, int32_t metric, int64_t self_shift, float* mins,
                                float margin_override, int num_sms, cudaStream_t s, const float* xmax,
                                bool bounded_norms = false);
// Quantile-pivot sample for k > 32: Ds[i][j] (ldS) = the single-product upper bound of u(i, j)
// for corpus points j < op.N (self pair +inf), unclamped.
cudaError_t launch_dist_tc_sample(const TcOperands& op, int64_t S, int32_t metric, int64_t self_shift, float* Ds,
                                  int64_t ldS, float margin_override, int num_sms, cudaStream_t s,
                                  bool bounded_norms = false);
// select.cu: pivots = k-th smallest chunk minimum per row; exact select over candidates.
// thr[M .. pad_end) (relative to thr) is zero-filled: the SYM partition reads whole 256-row
// tiles of pivots; pad_end must not pass the caller's allocation (absolute limit).
cudaError_t launch_pivot_from_mins(const float* mins, int64_t nchunk, int64_t M, int64_t pad_end, int32_t k,
                                   int32_t metric, float* thr, int32_t* cnt, cudaStream_t s);
// gate >= 0: the kernel runs only if flag[1] == gate (the device-side plan choice of
// launch_pivot1_decide; both partitions and both candidate selects are queued, one runs).
cudaError_t launch_candidate_select(const int32_t* cnt, const uint64_t* cent,
                                    int32_t cap, int64_t M, int32_t k, int64_t idx_offset,
                                    int32_t* out_idx, float* out_dist, int32_t* flag, cudaStream_t s,
                                    int32_t gate = -1);
// k > 32 pivot plan: per-row pivot with >= r of the S sampled upper bounds at or below it;
// exact select over the partition's candidate lists (CTA per row; flag |= 2 on a failed
// certificate or an overflowed list).
cudaError_t launch_pivot_from_sample(const float* Ds, int64_t M, int64_t S, int64_t ldS, int32_t r,
                                     float* thr, cudaStream_t s);
// Exact top-k (k <= 32, L2 metrics) of the single-product partition's lists (lower bounds):
// re-evaluates the few candidates whose bounds reach the k-th upper bound in fp64 from the
// fp32 inputs Q [M][d] / X [N][d]; qn the rows' prep norms, bq / bx the rows' / columns'
// launch_bound_norms bnd terms (U = L + 2 (bq + bx) >= D).
// flag |= 2 when the partition is not certified exact for some row (the caller redoes).
cudaError_t launch_candidate_recompute(const int32_t* cnt, const uint64_t* cent,
                                       int32_t cap, int64_t M, int32_t k, int64_t idx_offset, const float* Q,
                                       const float* X, int32_t d, const float* qn, const float* bq,
                                       const float* bx, const float* thr, int32_t metric, int32_t* out_idx,
                                       float* out_dist, int32_t* flag, cudaStream_t s, int32_t gate = -1);
// redo: M + 1 int32 of workspace for the warp-per-row form (null: CTA per row only).
cudaError_t launch_candidate_select_large(const int32_t* cnt, const uint64_t* cent,
                                          int32_t cap, int64_t M, int32_t k, int64_t idx_offset,
                                          int32_t* out_idx, float* out_dist, int32_t* flag, int32_t* redo,
                                          cudaStream_t s);
// Multi-GPU symmetric k-NNG: concatenate G (possibly peer-mapped) candidate lists per row.
cudaError_t launch_gather_lists(const int32_t* const* cnts, const uint64_t* const* ents,
                                int32_t G, int32_t cap_src, int64_t row0, int64_t rows, int32_t cap_dst,
                                int32_t* cnt_dst, uint64_t* ent_dst, int32_t* flag, cudaStream_t s);
bool tc_supported();  // device is sm_100 and the driver entry point for TMA maps exists


// select.cu
// redo: workspace of M + 1 int32 for the sampled-pivot plan of the CTA-per-row select (null:
// plain running threshold).
cudaError_t launch_select(const float* D, int64_t M, int64_t N, int64_t ldD, int32_t k,
                          int64_t idx_offset, int32_t* out_idx, float* out_dist, int32_t* redo,
                          cudaStream_t s);
// select_paper.cu: the paper's quick multi-select (ablation); ws of ws_bytes for the aux arrays.
size_t select_paper_ws_bytes(int64_t rows, int64_t N);
cudaError_t launch_select_paper(const float* D, int64_t M, int64_t N, int64_t ldD, int32_t k,
                                void* ws, size_t ws_bytes, int32_t* out_idx, float* out_dist,
                                cudaStream_t s);
// The kernel of the last launch_select (knn_last_select_kernel).
extern int g_last_select_kind, g_last_select_splits;
// Merge over a table of list pointers (local or peer-mapped): list g of row row0 + r at
// dist_lists[g] + (row0 + r) * k; output rows r < M.
cudaError_t launch_merge_lists(const float* const* dist_lists, const int32_t* const* idx_lists, int32_t G,
                               int64_t row0, int64_t M, int32_t k, const int64_t* offsets_host,
                               int32_t* out_idx, float* out_dist, cudaStream_t s);
cudaError_t launch_merge(const float* part_dist, const int32_t* part_idx, int32_t G, int64_t M,
                         int32_t k, const int64_t* offsets_host, int32_t* out_idx,
                         float* out_dist, cudaStream_t s);

}  // namespace knn
