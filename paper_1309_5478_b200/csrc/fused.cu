// fused.cu — a-S5: distance GEMM with the per-row k-select fused into the epilogue, so
// the M×N distance matrix never reaches HBM (BASELINE.json north_star (d)).
//
// Paper: the two steps of the brute-force k-NN — the distance matrix as a matrix product
// and the per-row multi-select — run back to back
// through a materialised matrix; "Batch execution will obviously require merging of
// results" covers the split-N partial lists below.
//
// Design:
//  * Mainloop = gemm_tc.cu's (tc_common.cuh): 2-CTA clusters, B multicast, 3-segment
//    split-fp16 tcgen05 MMAs into a double-buffered TMEM accumulator.
//  * Work unit = a row-block pair against one of S column splits; the CTA keeps the state
//    of its 128 rows for the whole split.
//  * 4 epilogue warps; thread = one query row (its TMEM lane).  Each row keeps a sorted
//    best-32 list in shared memory (threshold T = its k-th entry) and an unsorted survivor
//    buffer.  Per 32-column chunk: the unclamped distance u (its clamp max(u,0)+0 is the
//    materialised value, so u < T whenever that value is; for L2 the test runs against
//    RU(T^2)), one min-vote per chunk, one vote per column that holds a survivor, and the
//    survivor's exact value (same expression as gemm_tc.cu, hence bit-identical results)
//    appended to its row's buffer.  A buffer past 32 entries is folded into the sorted
//    list by the whole warp (bitonic sort of 32 + merge, warpsel.cuh), lowering T.
//  * End of unit: fold the rest; the first k list entries are the row's answer, written
//    as final lists (S = 1) or as partial lists merged by knn_merge (S > 1).
#include "tc_common.cuh"
#include "warpsel.cuh"

#include <climits>

namespace knn {
namespace {

using namespace tc;

constexpr int FSTAGES = 2;
constexpr int FEPI_WARPS = 4;                 // one thread per row of the 128-row block
constexpr int FTHREADS = 64 + 32 * FEPI_WARPS;
constexpr int FK = 32;                        // largest k of the fused plan
constexpr int FCAP = 64;                      // survivor buffer per row (folded when > 32)
constexpr int BMP = BM + 1;                   // padded row stride of the survivor buffers
constexpr int BEST_BYTES = BM * 32 * 8;       // sorted best-32 per row, [BM][32] x u64
constexpr int BUF_BYTES = FCAP * BMP * 4;     // one of key / idx buffers, [FCAP][BMP]
constexpr int FSMEM_BYTES = FSTAGES * STAGE_BYTES + BEST_BYTES + 2 * BUF_BYTES + 1024 /*align*/ +
                            1024 /*barriers*/;

struct FusedArgs {
    const float* qn; const float* q_rs; int64_t M;
    const float* xn; const float* x_rs; int64_t N;
    int64_t self_shift; int64_t idx_offset; int k;
    int32_t* out_idx; float* out_dist;  // [S][M][k]
};

template <int METRIC>
__global__ void __cluster_dims__(CLUSTER, 1, 1) __launch_bounds__(FTHREADS, 1)
knn_fused_kernel(const __grid_constant__ CUtensorMap map_qh, const __grid_constant__ CUtensorMap map_ql,
                 const __grid_constant__ CUtensorMap map_xh, const __grid_constant__ CUtensorMap map_xl,
                 int num_kb, SplitSched sched, FusedArgs a) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(16) float col_n[2][BN];
    __shared__ __align__(16) float col_s[2][BN];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    uint8_t* stage_base = smem;
    uint64_t* best = reinterpret_cast<uint64_t*>(smem + FSTAGES * STAGE_BYTES);  // [BM][32]
    uint32_t* bkey = reinterpret_cast<uint32_t*>(best + BM * 32);                 // [FCAP][BMP]
    uint32_t* bidx = bkey + FCAP * BMP;
    uint64_t* bars = reinterpret_cast<uint64_t*>(bidx + FCAP * BMP);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * FSTAGES + 4);
    const Bars b{smem_u32(bars), smem_u32(bars + FSTAGES), smem_u32(bars + 2 * FSTAGES),
                 smem_u32(bars + 2 * FSTAGES + 2)};

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tmem_base = setup(bars, FSTAGES, FEPI_WARPS, tmem_slot, &map_qh, 1);
    const uint32_t crank = cluster_rank();
    const int64_t cid = blockIdx.x / CLUSTER, ncl = gridDim.x / CLUSTER;

    if (warp == 0) {
        if (lane == 0)
            producer_loop<FSTAGES>(&map_qh, &map_ql, &map_xh, &map_xl, stage_base, b, sched, num_kb,
                                   crank, cid, ncl, a.self_shift);
        __syncwarp();
    } else if (warp == 1) {
#ifdef KNN_MMA_CONVERGED
        mma_loop<FSTAGES>(stage_base, b, sched, num_kb, tmem_base, cid, ncl, a.self_shift);
#else
        if (lane == 0) mma_loop<FSTAGES>(stage_base, b, sched, num_kb, tmem_base, cid, ncl, a.self_shift);
#endif
        __syncwarp();
    } else {
        // -------------------------------------------------------- epilogue -----------
        // Each thread owns one row: a sorted best-32 list best[row][:] (key << 32 | idx;
        // threshold = its (k-1)-th entry) and an unsorted survivor buffer; a buffer with
        // more than 32 entries is folded into the list by the whole warp (warp_merge32).
        const int quad = warp & 3;           // TMEM lane quadrant = rows quad*32 .. +32
        const int etid = threadIdx.x - 64;   // 0..127
        const int rl = quad * 32 + lane;     // this thread's row within the block
        const int k = a.k;
        const float kInf = __int_as_float(0x7F800000);
        // fold row rr's survivor buffer (all lanes); returns the row's new threshold
        auto fold = [&](int rr, int n) -> float {
            const int rrl = quad * 32 + rr;
            uint64_t L = best[rrl * 32 + lane];
            for (int o = 0; o < n; o += 32)
                L = ws::warp_merge32<BMP>(L, bkey + o * BMP + rrl, bidx + o * BMP + rrl,
                                          n - o < 32 ? n - o : 32);
            best[rrl * 32 + lane] = L;
            const uint32_t tk = (uint32_t)(__shfl_sync(ws::FULL, L, k - 1) >> 32);
            __syncwarp();
            if (tk == 0xFFFFFFFFu) return kInf;
            const float t = ukey_to_float(tk);
            // the filter runs on squared distances: for L2, sqrt(x) < t implies x < t^2 <=
            // RU(t*t), so rounding the square up never rejects a true neighbour
            return METRIC == 1 ? __fmul_ru(t, t) : t;
        };
        int it = 0;
        for (auto cur = sched.first(cid); sched.valid(cur); sched.next(cur, ncl)) {
            const Unit w = sched.unit(cur);
            const int64_t row0 = (2 * w.mp + crank) * BM + quad * 32;  // warp's first row
            const int64_t row = row0 + lane;
            const bool row_ok = row < a.M;
            const float qn = row_ok ? __ldg(a.qn + row) : 0.0f;
            const float cq = row_ok ? -2.0f * __ldg(a.q_rs + row) : 0.0f;
            const int64_t self_col = row + a.self_shift;  // wraps harmlessly for no-self
            int cnt = 0;
            float tf = kInf;  // accept every finite distance until k are known
            for (int rr = 0; rr < 32; ++rr) best[(quad * 32 + rr) * 32 + lane] = ~0ull;
            __syncwarp();
            for (int64_t nb = w.nb0; nb < w.nb1; ++nb)
            for (int pass = 0, cls = tile_class(w.mp, nb, a.self_shift); pass < tile_passes(cls);
                 ++pass, ++it) {
                const int tmask = tile_mask(cls, pass);  // mixed block: one side per pass
                const int buf = it & 1;
                const uint32_t tphase = (it >> 1) & 1;
                const int64_t n0 = nb * BN;
                for (int c = etid; c < BN; c += 32 * FEPI_WARPS) {
                    const int64_t j = n0 + c;
                    col_n[buf][c] = j < a.N ? __ldg(a.xn + j) : 0.0f;
                    col_s[buf][c] = j < a.N ? __ldg(a.x_rs + j) : 0.0f;
                }
                named_bar(1, 32 * FEPI_WARPS);
                const bool diag = a.self_shift != INT64_MIN && row0 + a.self_shift < n0 + BN &&
                                  row0 + 31 + a.self_shift >= n0;
                const bool tail = n0 + BN > a.N;
                mbar_wait(b.tfull0 + 8 * buf, tphase);
                tc_fence_after();
                const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + buf * BN;
                #pragma unroll 1
                for (int ch = 0; ch < BN / 32; ++ch) {
                    uint32_t r[32];
                    tmem_ld32(taddr + ch * 32, r);
                    if (ch == BN / 32 - 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(b.tempty0 + 8 * buf);
                    }
                    const int cb = ch * 32;
                    const float4* cn4 = reinterpret_cast<const float4*>(&col_n[buf][cb]);
                    const float4* cs4 = reinterpret_cast<const float4*>(&col_s[buf][cb]);
                    // unclamped distance u: the materialised value is max(u, 0) + 0, so
                    // u < tf whenever that value is < tf (no false negatives).
                    float v[32];
                    #pragma unroll
                    for (int c4 = 0; c4 < 8; ++c4) {
                        const float4 nn = cn4[c4];
                        const float4 ss = cs4[c4];
                        const float na[4] = {nn.x, nn.y, nn.z, nn.w};
                        const float sa4[4] = {ss.x, ss.y, ss.z, ss.w};
                        #pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int c = 4 * c4 + e;
                            v[c] = fmaf(__uint_as_float(r[c]) * cq, sa4[e], qn + na[e]);
                        }
                    }
                    const int64_t c0 = n0 + cb;
                    if (diag || tail || tmask) {
                        #pragma unroll
                        for (int c = 0; c < 32; ++c) {
                            const bool lower = row + a.self_shift > c0 + c;  // i+shift > j
                            if (c0 + c == self_col || c0 + c >= a.N || (tmask && lower != (tmask == 2)))
                                v[c] = kInf;
                        }
                    }
                    float m[16];
                    #pragma unroll
                    for (int c = 0; c < 16; ++c) m[c] = fminf(v[c], v[c + 16]);
                    #pragma unroll
                    for (int wdt = 8; wdt > 0; wdt >>= 1)
                        #pragma unroll
                        for (int c = 0; c < wdt; ++c) m[c] = fminf(m[c], m[c + wdt]);
                    if (!__any_sync(ws::FULL, m[0] < tf)) continue;
                    // per column: the rows (lanes) holding a survivor append it to their own
                    // buffer; columns without any survivor cost one vote
                    #pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        const bool ok = v[c] < tf;
                        if (__any_sync(ws::FULL, ok)) {
                            if (ok) {
                                float dd = fmaxf(v[c], 0.0f) + 0.0f;
                                if (METRIC == 1) dd = sqrtf(dd);
                                bkey[cnt * BMP + rl] = __float_as_uint(dd) | 0x80000000u;  // ukey(dd >= 0)
                                bidx[cnt * BMP + rl] = (uint32_t)(c0 + c);
                                ++cnt;
                            }
                        }
                    }
                    uint32_t need = __ballot_sync(ws::FULL, cnt > 32);
                    if (need) {
                        __syncwarp();
                        while (need) {
                            const int rr = __ffs(need) - 1;
                            need &= need - 1;
                            const int n = __shfl_sync(ws::FULL, cnt, rr);
                            const float t = fold(rr, n);
                            if (lane == rr) {
                                cnt = 0;
                                tf = t;
                            }
                        }
                    }
                }
            }
            // ---- end of unit: fold what is left, write the first k of each sorted list
            __syncwarp();
            const int64_t split = w.nb0 / sched.per;
            for (int rr = 0; rr < 32; ++rr) {
                const int64_t grow = row0 + rr;
                if (grow >= a.M) break;
                const int n = __shfl_sync(ws::FULL, cnt, rr);
                if (n > 0) fold(rr, n);
                const uint64_t L = best[(quad * 32 + rr) * 32 + lane];
                if (lane < k) {
                    const size_t o = ((size_t)split * a.M + grow) * k + lane;
                    const uint32_t key = (uint32_t)(L >> 32);
                    if (key == 0xFFFFFFFFu) {  // fewer than k columns in this split
                        a.out_idx[o] = -1;
                        a.out_dist[o] = kInf;
                    } else {
                        a.out_idx[o] = (int32_t)((int64_t)(uint32_t)L + a.idx_offset);
                        a.out_dist[o] = ukey_to_float(key);
                    }
                }
            }
            __syncwarp();
        }
    }
    teardown(tmem_base);
}

}  // namespace

int fused_max_k() { return FK; }

int fused_splits(int64_t M, int64_t N, int num_sms) {
    const int64_t n_mp = ceil_div(ceil_div(M, BM), 2), n_nb = ceil_div(N, BN);
    const int64_t ncl = num_sms / CLUSTER;
    int best = 1;
    int64_t best_cost = INT64_MAX;
    for (int S = 1; S <= 8 && S <= n_nb; ++S) {
        const int64_t cost = ceil_div(n_mp * S, ncl) * ceil_div(n_nb, S);
        if (cost < best_cost) {
            best_cost = cost;
            best = S;
        }
    }
    return best;
}

cudaError_t launch_knn_fused(const TcOperands& op, int32_t metric, int64_t self_shift, int32_t k,
                             int64_t idx_offset, int S, int32_t* out_idx, float* out_dist,
                             int num_sms, cudaStream_t s) {
    if (op.M == 0) return cudaSuccess;
    if (k < 1 || k > FK) return cudaErrorInvalidValue;
    CUtensorMap mqh, mql, mxh, mxl;
    if (!tc_make_operand_map(&mqh, op.q_hi, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mql, op.q_lo, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mxh, op.x_hi, op.N, op.d_pad, BN / 2) ||
        !tc_make_operand_map(&mxl, op.x_lo, op.N, op.d_pad, BN / 2))
        return cudaErrorInvalidValue;
    const int64_t n_mp = ceil_div(ceil_div(op.M, BM), 2), n_nb = ceil_div(op.N, BN);
    const int64_t per = ceil_div(n_nb, S);
    SplitSched sched{n_mp, n_nb, ceil_div(n_nb, per), per};
    const int64_t units = n_mp * sched.S;
    const int64_t pairs = units < num_sms / CLUSTER ? units : num_sms / CLUSTER;
    FusedArgs fa{op.qn, op.q_rs, op.M, op.xn, op.x_rs, op.N, self_shift, idx_offset, k, out_idx, out_dist};
    auto kern = metric == 1 ? knn_fused_kernel<1> : knn_fused_kernel<0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FSMEM_BYTES);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)(pairs * CLUSTER), FTHREADS, FSMEM_BYTES, s>>>(mqh, mql, mxh, mxl, op.d_pad / BK,
                                                                 sched, fa);
    return cudaGetLastError();
}

}  // namespace knn
