// gemm_tc.cu — a-S3: the distance matrix as a dense contraction on the 5th-generation
// tensor cores (tcgen05 + TMEM + TMA), FP32-accurate, with the distance assembly fused
// into the epilogue.
//
// Paper: "the n×m dot products x_i.y_j ... are easily formulated as a matrix product
// X^T Y"; "d^2_ij = ||x_i||^2 + ||y_j||^2 - 2 x_i.y_j";
// d_E = sqrt(d^2).  The paper used a library SGEMM on Fermi FP32 cores.
//
// B200 design:
//  * Operands are the per-vector power-of-two-scaled fp16 halves of prep.cu:
//    s_q q = qh + ql,  s_x x = xh + xl.  The dot is recovered FP32-accurately from three
//    fp16 products with fp32 accumulation in TMEM:  ql.xh + qh.xl + qh.xh  (the
//    dropped ql.xl and the split residuals are <= ~3*2^-22 relative per term), issued
//    as three K-segments of one accumulation, smallest terms first.  fp16 runs at twice
//    the TF32 tensor rate, so this costs what 1.5 TF32 passes would (vs 3 for 3xTF32).
//  * Warp-specialised persistent kernel, one CTA per SM, 6 warps:
//      warp 0  TMA producer: per K-block loads qh, ql (BM×BK) and xh, xl (BN×BK) tiles,
//              (the xh, xl halves multicast across the CTA pair of the cluster),
//              swizzled K-major, into a STAGES-deep ring (each stage feeds 3 MMA
//              segments, so the hi tiles are loaded once and used twice);
//      warp 1  TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=256, K=16);
//      warps 2-9 epilogue: tcgen05.ld (32x32b.x32) -> registers -> fused distance
//              assembly -> streaming 128-bit stores of the fp32 distance row.  Two
//              warps per TMEM lane quadrant (32 rows), each owning half the columns.
//    The accumulator is double-buffered in TMEM (2 × 256 columns), so the epilogue of
//    tile t overlaps the MMAs of tile t+1.
//  * Epilogue (per element): acc*(-2 rs_q) is exact (power-of-two scale), so
//      D = max(fma(acc * (-2 rs_q), rs_x, ||q||^2 + ||x||^2), 0) + 0
//    rounds once; +0 canonicalises -0 (R6); sqrt for L2; +inf on the excluded self pair.
#include "tc_common.cuh"

#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace knn {
namespace {

using namespace tc;

constexpr int STAGES = 3;
constexpr int EPI_WARPS = 8;     // 2 per TMEM lane quadrant, each owning BN/2 columns
constexpr int COL_WARP = 2 + EPI_WARPS;  // column-data producer (one elected thread)
constexpr int THREADS = 64 + 32 * EPI_WARPS + 32;
constexpr int STG_BYTES = 32 * 32 * 4;  // one 32x32 fp32 output chunk (TMA-store staging)
// Column data of a tile (||x_j||^2, 2^-sh_j and, SYM PIVOT, the column pivots), bulk-copied
// by COL_WARP into an NCOL-deep ring so the epilogue warps never wait on each other.
constexpr int NCOL = 4;
constexpr int COL_BYTES = 3 * BN * 4;
constexpr int SMEM_BYTES = RING_BYTES + EPI_WARPS * 2 * STG_BYTES + NCOL * COL_BYTES +
                           1024 /*align*/ + 1024 /*barriers*/;
// SYM (symmetric k-NNG): each warp's two staging buffers hold the direct and the transposed
// chunk of the same 32x32 block.

struct EpiArgs {
    const float* qn; const float* q_rs; int64_t M;
    const float* xn; const float* x_rs; int64_t N;  // column arrays padded to 256 entries
    int32_t metric; int64_t self_shift; float* D; int64_t ldD;
    // PIVOT (partition epilogue): per-row pivots in the squared domain; per-row candidate
    // lists cent[row * cap + i], i < cnt[row], entries (ukey << 32 | col)
    const float* thr; int32_t* cnt; uint64_t* cent; int32_t cap; int32_t* flag;
    float margin;  // MINS: error bound of the hi.hi value, relative to ||q||^2 + ||x||^2
    // MINS / SAMPLE with a strided column sample: matrix column block nb is output column
    // block nb / nb_stride
    int64_t nb_stride = 1;
    const float* xmax = nullptr;  // MINS: upper bound of every column's sqn term (device scalar)
    int32_t gate = -1;  // PIVOT modes: run only if flag[1] == gate (device plan choice), -1 always
    int32_t dbg = 0;  // DIAGNOSTIC (env KNN_DBG_EPI, wrong results): 1 skip column test, 2 skip appends,
                      // 4 skip both tests, 8 skip global flushes, 16 staging without appends
};

// Distance from the unclamped value u = ||q||^2 + ||x||^2 - 2 q.x (one rounding): the
// materialised value max(u, 0) + 0 (+0 canonicalises -0), sqrt for L2.
// METRIC 2 (cosine / Pearson): u = 1 - cos in [0, 2]; the zero-norm sentinel terms (5/2
// per vector, prep.cu) clamp to 3.
template <int METRIC>
__device__ __forceinline__ float finalize_dist(float u) {
    float dd = fmaxf(u, 0.0f) + 0.0f;
    if (METRIC == 1) dd = sqrtf(dd);
    if (METRIC == 2) dd = fminf(dd, 3.0f);
    return dd;
}

// kernel template argument of a metric: 0 squared L2, 1 L2 (sqrt), 2 cosine / Pearson
inline int metric_kind(int32_t metric) { return metric == 1 ? 1 : metric >= 2 ? 2 : 0; }

// Append candidate (key, column) to row r's global list; counts overflow.
__device__ __forceinline__ void pivot_append(const EpiArgs& ep, int64_t r, uint32_t key, uint32_t col) {
    const int pos = atomicAdd(ep.cnt + r, 1);
    if (pos < ep.cap) {
        ep.cent[r * ep.cap + pos] = (uint64_t)key << 32 | col;
    } else {
        *ep.flag |= 2;  // overflow: the caller redoes the problem with the full matrix
    }
}

// Candidates found by a warp are first appended to a warp-private shared list (SoA: row,
// col, key) and flushed to the global per-row lists in batches of up to PEND_CAP, four
// returning atomics in flight per lane, so their latency is paid once per batch.
constexpr int PEND_CAP = 320;
// KNN_DIAG_EPI builds (scripts/epi_cost.py) honour env KNN_DBG_EPI; product builds compile
// the diagnostic switches out of the epilogue
#ifdef KNN_DIAG_EPI
#define EPI_DBG(bit) (ep.dbg & (bit))
#else
#define EPI_DBG(bit) 0
#endif
#ifndef KNN_EPI_REG
#define KNN_EPI_REG 1  // survivor slots by warp scan, padded staging rows (1), or round 1's path (0)
#endif
constexpr int SROW = 36;  // staged floats per lane row (KNN_EPI_REG): 144-byte rows  // 3 x 320 x 4 B in one 4 KB staging buffer

// Deferred flush (PIVOT modes): the pending list is moved into registers (J entries per
// lane) and its slots reserved with returning atomics, but the entries are written only at
// the next flush, when those atomics have long returned — the warp never waits for them.
template <int J>
struct DeferredFlush {
    uint32_t r[J], c[J], k[J];
    int pos[J];
    __device__ __forceinline__ void init() {
        #pragma unroll
        for (int j = 0; j < J; ++j) pos[j] = -1;
    }
    __device__ __forceinline__ void complete(const EpiArgs& ep) {
        #pragma unroll
        for (int j = 0; j < J; ++j) {
            if (pos[j] >= 0) {
                if (pos[j] < ep.cap) {
                    // one 8-byte store per entry (two 4-byte lists cost twice the scattered
                    // L2 transactions and left twice the partially written sectors, which
                    // HBM3 fills by read-modify-write: profiles/r02_partition_traffic.txt)
                    ep.cent[(int64_t)r[j] * ep.cap + pos[j]] = (uint64_t)k[j] << 32 | c[j];
                } else {
                    *ep.flag |= 2;
                }
            }
            pos[j] = -1;
        }
    }
    __device__ __forceinline__ void flush(const EpiArgs& ep, const uint4* pent, int n) {
        const int lane = threadIdx.x & 31;
        complete(ep);
        __syncwarp();
        #pragma unroll
        for (int j = 0; j < J; ++j) {
            const int i = 32 * j + lane;
            if (i < n) {
                const uint4 e = pent[i];  // {row, col, key, -}: one 16-byte load per entry
                r[j] = e.x;
                c[j] = e.y;
                k[j] = e.z;
                pos[j] = atomicAdd(ep.cnt + r[j], 1);
            }
        }
        __syncwarp();
    }
};

// Per-mode epilogue shape.  The partition (PIVOT) epilogue is latency-bound (2 warps per
// SM sub-partition issue ~45% of cycles), so it runs 12 warps — 3 per TMEM lane quadrant,
// owning 3/3/2 of the tile's eight 32-column chunks — with a smaller pending list and a
// 3-deep column ring to fit the shared memory; the other modes keep 8 warps (BN/2 each).
// ARES (A-panel-resident sample pass, PanelSched): the operand region holds two A panels
// (d_pad <= 256) and a 5-stage B ring, using the staging slabs the MINS epilogue does not
// need (it stores its chunk minima directly).
constexpr int ARES_KB = CTA2 ? 10 : 5;      // B ring stages
constexpr int ARES_PANEL = 8 * A_BYTES;     // one A panel: BM x 256 fp16
template <int MODE, bool ARES = false>
#ifndef KNN_MINS_WARPS
#define KNN_MINS_WARPS 8  // epilogue warps of the chunk-minimum sample pass (8 or 16)
#endif
#ifndef KNN_PV1_WARPS
#define KNN_PV1_WARPS 16  // epilogue warps of the single-product partition (12, 16 or 20; 20 with
                          // 80 registers, a 3-stage ring and 64-entry pending lists measured
                          // slower: 1.42 -> 1.48 ms)
#endif
struct EpiCfg {
    static constexpr bool PV = MODE == 1 || MODE == 5;  // MODE_PIVOT, MODE_PIVOT1
    // the single-product partition is bound by its epilogue's latency: 16 warps (4 per TMEM
    // lane quadrant, 2 chunks each) over a 4-stage operand ring (the MMA is not its limit)
    static constexpr bool PV20 = MODE == 5 && KNN_PV1_WARPS == 20;  // (5 per quadrant; one idles per tile)
    static constexpr bool PV16 = MODE == 5 && (KNN_PV1_WARPS == 16 || PV20);
    static constexpr int WARPS = PV20 ? 20 : PV16 || (MODE == 2 && KNN_MINS_WARPS == 16) ? 16 : PV ? 12 : EPI_WARPS;
    static constexpr int PARTS = WARPS / 4;
    static constexpr int CPW = (BN / 32 + PARTS - 1) / PARTS;  // chunks per warp (last: fewer)
    // PV staging: 32 rows of SROW floats (KNN_EPI_REG) or a swizzled 32x32 chunk
    static constexpr int STG_PV = KNN_EPI_REG ? 32 * SROW * 4 : STG_BYTES;
    static constexpr int PEND = PV20 ? 64 : PV16 ? 96 : PV ? (KNN_EPI_REG ? (CTA2 ? 160 : 96) : 128) : PEND_CAP;
    static constexpr int SLAB = PV ? STG_PV + 16 * PEND : MODE == 2 ? 0 : 2 * STG_BYTES;  // per warp
    static constexpr int NCOLS = PV16 ? 6 : PV ? 3 : NCOL;  // column-data ring slots
    static constexpr int THREADS = 64 + 32 * WARPS + 32;
    static constexpr int RING = ARES ? 2 * ARES_PANEL + ARES_KB * B_TILE
                                     : PV20 ? 3 * (A_BYTES + B_TILE) : PV16 ? 4 * (A_BYTES + B_TILE) : RING_BYTES;
    static constexpr int SMEM = RING + WARPS * SLAB + NCOLS * COL_BYTES + 1024 + 1024;
    static_assert(SMEM <= 232448, "shared memory");
    static_assert(SLAB % 16 == 0, "slab alignment");
};
__device__ __forceinline__ void pivot_flush(const EpiArgs& ep, const uint4* pent, int n) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    for (int i0 = 0; i0 < n; i0 += 128) {
        int pos[4];
        uint32_t r[4];
        #pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = i0 + 32 * j + lane;
            if (i < n) {
                r[j] = pent[i].x;
                pos[j] = atomicAdd(ep.cnt + r[j], 1);
            }
        }
        #pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = i0 + 32 * j + lane;
            if (i < n) {
                if (pos[j] < ep.cap) {
                    ep.cent[(int64_t)r[j] * ep.cap + pos[j]] = (uint64_t)pent[i].z << 32 | pent[i].y;
                } else {
                    *ep.flag |= 2;
                }
            }
        }
    }
    __syncwarp();
}

// Epilogue modes: MODE_STORE writes D; MODE_PIVOT keeps the partition's candidates;
// MODE_MINS writes, per row, the minimum distance of every 32-column chunk; MODE_SAMPLE
// writes the single-product upper bound v >= u of every element (the quantile pivot's
// sample for k > 32), unclamped, in the u domain.
enum { MODE_STORE = 0, MODE_PIVOT = 1, MODE_MINS = 2, MODE_SAMPLE = 3, MODE_NULL = 4, MODE_PIVOT1 = 5 };
// MODE_PIVOT1: the partition from the single hi.hi product; the kept key is the lower bound
// u_hh - F1_q ||q||^2 - F1_x ||x||^2 <= the exact distance (computed as the u of the per-point
// norms scaled by 1 - F1, prep.cu launch_bound_norms), so every element at or below the pivot is kept; the
// candidate select re-evaluates the survivors exactly (select.cu).
// MODE_NULL (diagnostic, knn_diag_mainloop): the epilogue only drains TMEM (tcgen05.ld) and
// frees the accumulator, so the kernel runs at the mainloop's own rate.

template <int METRIC, bool SYM, int MODE, class Sched>
__global__ void __cluster_dims__(CLUSTER, 1, 1) __launch_bounds__(EpiCfg<MODE, Sched::kResidentA>::THREADS, 1)
dist_tc_kernel(const __grid_constant__ CUtensorMap map_qh, const __grid_constant__ CUtensorMap map_ql,
               const __grid_constant__ CUtensorMap map_xh, const __grid_constant__ CUtensorMap map_xl,
               const __grid_constant__ CUtensorMap map_d, int use_tma_store, int num_kb,
               Sched sched, EpiArgs ep) {
    // SYM: upper-triangle pair blocks only, O1 everywhere (every element has i < j or is
    // mirrored from one), so the mainloop sees no self shift.
    constexpr bool PIVOT1 = MODE == MODE_PIVOT1;
    constexpr bool PIVOT = MODE == MODE_PIVOT || PIVOT1;
    constexpr bool MINS = MODE == MODE_MINS;
    constexpr bool SAMPLE = MODE == MODE_SAMPLE;
    constexpr int NCOLARR = PIVOT && SYM ? 3 : 2;  // column arrays per tile
    constexpr bool ARES = Sched::kResidentA;
    using E = EpiCfg<MODE, ARES>;
    constexpr int NCOL = E::NCOLS;
    constexpr int EPI_WARPS = E::WARPS;
    constexpr int COL_WARP = 2 + EPI_WARPS;
    constexpr int PEND_CAP = E::PEND;
    // MINS (approximate pivot sample): one hi.hi product per K-block, twice the stages
    constexpr int NSEG = MINS || SAMPLE || PIVOT1 ? 1 : 3;
    constexpr int KSTAGES = ARES ? ARES_KB : E::RING / stage_bytes<NSEG>();
    static_assert(ARES || KSTAGES * stage_bytes<NSEG>() <= E::RING, "smem layout");
    static_assert(!ARES || (MODE == MODE_MINS && !SYM), "A-resident mainloop: sample pass only");
    // the single product is orientation-free: no two-pass blocks on the diagonal
    const int64_t ml_shift = SYM || NSEG == 1 ? INT64_MIN : ep.self_shift;
    extern __shared__ uint8_t smem_raw[];
    // 1024-align by pointer arithmetic (keeps the shared address space visible to the compiler)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* stage_base = smem;
    uint8_t* stg_base = smem + E::RING;  // [EPI_WARPS] slabs of E::SLAB bytes
    float* col_base = reinterpret_cast<float*>(stg_base + EPI_WARPS * E::SLAB);  // [NCOL][3][BN]
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(col_base) + NCOL * COL_BYTES);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * KSTAGES + 4);
    const uint32_t colfull0 = smem_u32(bars + 2 * KSTAGES + 5);
    const uint32_t colempty0 = colfull0 + 8 * NCOL;
    const uint32_t afull0 = colempty0 + 8 * NCOL, aempty0 = afull0 + 16;  // ARES panel buffers
    // per column slot, the work item it belongs to (written by COL_WARP before the slot's
    // expect_tx, read by the epilogue after the slot's full barrier): {mp, nb, cls | pass << 8,
    // unit index}; mp = -1 ends the stream.  The epilogue warps then never run the scheduler.
    int4* col_hdr = reinterpret_cast<int4*>(bars + 2 * KSTAGES + 5 + 2 * NCOL + 4 + 1);
    const Bars b{smem_u32(bars), smem_u32(bars + KSTAGES), smem_u32(bars + 2 * KSTAGES),
                 smem_u32(bars + 2 * KSTAGES + 2)};
    const uint32_t tfull0 = b.tfull0, tempty0 = b.tempty0;

    // the other partition was chosen on the device: every CTA of the pair leaves before any
    // barrier, TMEM allocation or cluster synchronisation
    if (PIVOT && ep.gate >= 0 && ep.flag[1] != ep.gate) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < NCOL; ++i) {
            mbar_init(colfull0 + 8 * i, 1);
            mbar_init(colempty0 + 8 * i, EPI_WARPS);
        }
        if (ARES)
            for (int i = 0; i < 2; ++i) {
                mbar_init(afull0 + 8 * i, 1);
                mbar_init(aempty0 + 8 * i, 1);
            }
    }
    const uint32_t tmem_base = setup(bars, KSTAGES, EPI_WARPS, tmem_slot, &map_qh, 1);
    const uint32_t crank = cluster_rank();
    const int64_t cid = blockIdx.x / CLUSTER, ncl = gridDim.x / CLUSTER;

    if (warp == 0) {
        if (lane == 0) {
            if constexpr (ARES)
                producer_loop_ares<KSTAGES>(&map_qh, &map_xh, stage_base, stage_base + 2 * ARES_PANEL, b, afull0,
                                            aempty0, sched, num_kb, crank, cid, ncl);
            else
                producer_loop<KSTAGES, Sched, NSEG>(&map_qh, &map_ql, &map_xh, &map_xl, stage_base, b, sched,
                                                    num_kb, crank, cid, ncl, ml_shift);
        }
        __syncwarp();
    } else if (warp == 1) {
        if (CTA2 && crank != 0) {
            // the pair's MMAs are issued by the leader CTA only
        } else if constexpr (ARES) {
            if (lane == 0)
                mma_loop_ares<KSTAGES>(stage_base, stage_base + 2 * ARES_PANEL, b, afull0, aempty0, sched, num_kb,
                                       tmem_base, cid, ncl);
        } else {
#ifdef KNN_MMA_CONVERGED
        mma_loop<KSTAGES, Sched, NSEG>(stage_base, b, sched, num_kb, tmem_base, cid, ncl, ml_shift);
#else
        if (lane == 0)
            mma_loop<KSTAGES, Sched, NSEG>(stage_base, b, sched, num_kb, tmem_base, cid, ncl, ml_shift);
#endif
        }
        __syncwarp();
    } else if (warp == COL_WARP) {
        // ------------------------------------------- column data of each work item --
        if (lane == 0) {
            int it = 0, ui = 0;
            for (auto cur = sched.first(cid); sched.valid(cur); sched.next(cur, ncl), ++ui) {
                const tc::Unit wu = sched.unit(cur);
                for (int64_t nbu = wu.nb0; nbu < wu.nb1; ++nbu) {  // (one tile per unit but PanelSched)
                const tc::Unit w{wu.mp, nbu, nbu + 1};
                const int cls = tile_class(w.mp, w.nb0, ml_shift);
                const int64_t n0 = w.nb0 * BN;
                for (int pass = 0; pass < tile_passes(cls); ++pass, ++it) {
                    const int slot = it % NCOL;
                    mbar_wait(colempty0 + 8 * slot, ((it / NCOL) & 1) ^ 1);
                    // the epilogue's generic-proxy reads of this slot (ordered by the
                    // mbarrier) before the async-proxy writes of the refill
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    const uint32_t fb = colfull0 + 8 * slot;
                    const uint32_t dst = smem_u32(col_base + slot * 3 * BN);
                    col_hdr[slot] = make_int4((int)w.mp, (int)w.nb0, cls | pass << 8, ui);
                    mbar_expect_tx(fb, NCOLARR * BN * 4);
                    bulk_load(dst, ep.xn + n0, BN * 4, fb);
                    bulk_load(dst + BN * 4, ep.x_rs + n0, BN * 4, fb);
                    if (PIVOT && SYM) bulk_load(dst + 2 * BN * 4, ep.thr + n0, BN * 4, fb);
                }
                }
            }
            // end of the stream: a header-only item
            const int slot = it % NCOL;
            mbar_wait(colempty0 + 8 * slot, ((it / NCOL) & 1) ^ 1);
            col_hdr[slot] = make_int4(-1, 0, 0, 0);
            mbar_arrive(colfull0 + 8 * slot);
        }
        __syncwarp();
    } else {
        // -------------------------------------------- epilogue (EPI_WARPS warps) --
        const int quad = warp & 3;                  // TMEM lane quadrant this warp may access
        const int part = (warp - 2) >> 2;           // which chunks of 32 columns it owns
        int wi = 0;  // work items seen: rotates the short share of chunks among the warps
        uint8_t* slab = stg_base + (warp - 2) * E::SLAB;
        const bool vec_ok = (ep.ldD % 4) == 0 && ((reinterpret_cast<uintptr_t>(ep.D) & 15) == 0);
        int sbsel = 0;  // which of the warp's two staging buffers
        int it = 0;
        // PIVOT: the warp's pending-candidate list lives in its second staging buffer
        // pending entries {row, col, key, -}, one 16-byte store / load each
        uint4* pent = reinterpret_cast<uint4*>(slab + E::STG_PV);
        int pend_n = 0;  // warp-uniform
        DeferredFlush<(E::PEND + 31) / 32> dfl;  // PIVOT: the previous flush's entries
        dfl.init();
        __shared__ int s_pend[EPI_WARPS];  // PIVOT: each warp's pending-list length (slot allocator)
        if (PIVOT && lane == 0) s_pend[warp - 2] = 0;
        __syncwarp();
        // the row terms of the last work item: consecutive items of a CTA often share the row
        // block (row-major triangle schedule), so the three loads are skipped then
        int64_t row_c = -1;
        float qn_c = 0.0f, cq_c = 0.0f, trow_c = -1.0f;
        for (;; ++it) {
            const int slot = it % NCOL;
            mbar_wait(colfull0 + 8 * slot, (it / NCOL) & 1);
            const int4 hdr = col_hdr[slot];
            if (hdr.x < 0) break;  // end of the work items
            wi = hdr.w;
            const tc::Unit w{hdr.x, hdr.y, hdr.y + 1};
            const int cls = hdr.z & 0xFF;
            const int pass = hdr.z >> 8;
            // this warp's chunks of the tile (3 warps per quadrant: 3/3/2, the short share
            // rotating per work item so that a warp can run ahead into the other accumulator)
            const int ch0 = ((E::PV ? part + wi : part) % E::PARTS) * E::CPW;
            const int nch = (BN / 32 - ch0) < E::CPW ? (BN / 32 - ch0) : E::CPW;
            const int64_t nb = w.nb0;
            const int64_t mb = 2 * w.mp + crank;
            const int64_t n0 = nb * BN;
            const int64_t n0_out = (nb / ep.nb_stride) * BN;  // MINS / SAMPLE output column base
            const int64_t row0 = mb * BM + quad * 32;
            const int64_t row = row0 + lane;
            const bool row_ok = row < ep.M;
            if (row != row_c) {
                row_c = row;
                qn_c = row_ok ? __ldg(ep.qn + row) : 0.0f;
                cq_c = row_ok ? -2.0f * __ldg(ep.q_rs + row) : 0.0f;
                trow_c = PIVOT && row_ok ? __ldg(ep.thr + row) : -1.0f;  // row pivot
            }
            const float qn = qn_c, cq = cq_c, trow = trow_c;
            const uint64_t cq2 = f2_pack(cq, cq), qn2 = f2_pack(qn, qn), trow2 = f2_pack(trow, trow);
            // MINS: qn (1 + m) + m XMAX, and the cosine sentinel cap 3 + m (qn + XMAX)
            const float xmx = MINS ? __ldg(ep.xmax) : 0.0f;
            const float mins_row_term = MINS ? fmaf(ep.margin, qn + xmx, qn) * (1.0f + 0x1p-22f) : 0.0f;
            const float mins_cos_cap = MINS ? fmaf(ep.margin, qn + xmx, 3.0f) : 0.0f;
            const int64_t c_lo = n0 + ch0 * 32;
            // does this warp's 32 x (32 nch) block touch the excluded self pairs?
            const bool diag = ep.self_shift != INT64_MIN &&
                              row0 + ep.self_shift < c_lo + 32 * nch && row0 + 31 + ep.self_shift >= c_lo;
            const int64_t self_col = row + ep.self_shift;
            float* drow = ep.D + row * ep.ldD;
        {
            const int tmask = tile_mask(cls, pass);  // mixed block: keep one side only
            const int buf = it & 1;
            const uint32_t tphase = (it >> 1) & 1;
            const float* col_n = col_base + slot * 3 * BN;
            const float* col_s = col_n + BN;
            const float* col_t = col_n + 2 * BN;
            mbar_wait(tfull0 + 8 * buf, tphase);
            tc_fence_after();
            if (nch <= 0) {  // (E::PV20: this warp's share of the tile is empty; it still frees it)
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty0 + 8 * buf);
            }
            const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + buf * BN + ch0 * 32;
            #pragma unroll 1  // (unrolling the two chunks of the 16-warp partition: 1.45 -> 1.59 ms)
            for (int ch = 0; ch < nch; ++ch) {
                uint32_t r[32];
                tmem_ld32(taddr + ch * 32, r);
                if (ch == nch - 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (CTA2)
                            mbar_arrive_leader(tempty0 + 8 * buf);  // the leader's MMA waits for both CTAs
                        else
                            mbar_arrive(tempty0 + 8 * buf);
                    }
                }
                if constexpr (MODE == MODE_NULL) {
                    asm volatile("" ::"r"(r[0]), "r"(r[31]));  // keep the TMEM load
                    continue;
                }
                const int cb = (ch0 + ch) * 32;  // first column of the chunk in the tile
                const float4* cn4 = reinterpret_cast<const float4*>(col_n + cb);
                const float4* cs4 = reinterpret_cast<const float4*>(col_s + cb);
                if constexpr (MINS) {
                    // pivot sample pass: an upper bound of the chunk's minimum distance for
                    // this row in three operations per element.  With a_j = acc_j 2^-sh_j and
                    // w_j = cq a_j + xn_j (cq = -2^(1-sh_q): the single-product u_j - qn),
                    // value = min_j w_j + qn (1 + m) + m XMAX >= u_j* + m (qn + xn_j*) for the
                    // minimising j*, i.e. >= the hi.hi value of element j* plus its error bound,
                    // so at least one element of the chunk has an FP32-accurate u at or below
                    // it (XMAX >= every xn_j).  No self pair: the sample is a
                    // gathered column subset.
                    float m[8];
                    #pragma unroll
                    for (int c4 = 0; c4 < 8; ++c4) {
                        const float4 nn = cn4[c4];
                        const float4 ss = cs4[c4];
                        const float w0 = fmaf(cq, __uint_as_float(r[4 * c4]) * ss.x, nn.x);
                        const float w1 = fmaf(cq, __uint_as_float(r[4 * c4 + 1]) * ss.y, nn.y);
                        const float w2 = fmaf(cq, __uint_as_float(r[4 * c4 + 2]) * ss.z, nn.z);
                        const float w3 = fmaf(cq, __uint_as_float(r[4 * c4 + 3]) * ss.w, nn.w);
                        m[c4] = fminf(fminf(w0, w1), fminf(w2, w3));
                    }
                    #pragma unroll
                    for (int wdt = 4; wdt > 0; wdt >>= 1)
                        #pragma unroll
                        for (int c = 0; c < wdt; ++c) m[c] = fminf(m[c], m[c + wdt]);
                    const int64_t c0m = n0 + cb;
                    if (row_ok && c0m < ep.N) {
                        float val = m[0] + mins_row_term;
                        if (METRIC == 2) val = fminf(val, mins_cos_cap);
                        float* dst = ep.D + ((n0_out + cb) >> 5) * ep.ldD + row;  // mins[chunk][row]
                        *dst = finalize_dist<METRIC>(val);
                    }
                    continue;
                }
                float v[32];
                if constexpr (SAMPLE) {
                    #pragma unroll
                    for (int c4 = 0; c4 < 8; ++c4) {
                        const float4 nn = cn4[c4];
                        const float4 ss = cs4[c4];
                        const float na[4] = {nn.x, nn.y, nn.z, nn.w};
                        const float sa4[4] = {ss.x, ss.y, ss.z, ss.w};
                        #pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int c = 4 * c4 + e;
                            const float nsum = qn + na[e];
                            float u = fmaf(__uint_as_float(r[c]) * cq, sa4[e], nsum);
                            if (METRIC == 2) u = fminf(u, 3.0f);
                            // the hi.hi value plus a bound of its error, so that it is never
                            // below the FP32-accurate u of the partition
                            v[c] = fmaf(nsum, ep.margin, u);
                        }
                    }
                } else {
                    // u = fl(fl(acc cq) s_j + fl(qn + xn_j)), two columns per FMUL2 / FADD2 /
                    // FFMA2 (each half rounds as the scalar op: the same bits as before)
                    // (PIVOT1: qn, xn arrive scaled by 1 - F, so u is already the lower bound)
                    #pragma unroll
                    for (int c4 = 0; c4 < 8; ++c4) {
                        const float4 nn = cn4[c4];
                        const float4 ss = cs4[c4];
                        #pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int c = 4 * c4 + 2 * h;
                            const uint64_t acc2 = f2_pack(__uint_as_float(r[c]), __uint_as_float(r[c + 1]));
                            const uint64_t sj = h ? f2_pack(ss.z, ss.w) : f2_pack(ss.x, ss.y);
                            const uint64_t ns = f2_add(qn2, h ? f2_pack(nn.z, nn.w) : f2_pack(nn.x, nn.y));
                            // L2: fl(fl(acc cq) s_j + ns) — the scales are powers of two, so
                            // the two orientations of a pair agree exactly.  Cosine / Pearson:
                            // the scales are not, so the scale product is formed first,
                            // fl(acc fl(cq s_j) + ns), symmetric in (q, x): the blocked and the
                            // symmetric (mirrored) plans then give the same bits
                            const uint64_t u2 = METRIC == 2 ? f2_fma(acc2, f2_mul(cq2, sj), ns)
                                                            : f2_fma(f2_mul(acc2, cq2), sj, ns);
                            float u0, u1;
                            f2_unpack(u2, u0, u1);
                            // cosine: the sentinel clamp before any comparison (key <= T => u <= T)
                            if (METRIC == 2) {
                                u0 = fminf(u0, 3.0f);
                                u1 = fminf(u1, 3.0f);
                            }
                            v[c] = PIVOT ? u0 : finalize_dist<METRIC>(u0);
                            v[c + 1] = PIVOT ? u1 : finalize_dist<METRIC>(u1);
                        }
                    }
                }
                const int64_t c0 = n0 + cb;
                if (diag) {
                    #pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (c0 + c == self_col) v[c] = __int_as_float(0x7F800000);
                }
                if constexpr (MINS) {
                    // pivot sample pass: the chunk's minimum distance for this row (the self
                    // pair was set to +inf above; a block straddling the diagonal comes in two
                    // masked passes, the second folds into the first's value)
                    if (tmask) {
                        #pragma unroll
                        for (int c = 0; c < 32; ++c) {
                            const bool lower = row + ep.self_shift > c0 + c;
                            if (lower != (tmask == 2)) v[c] = __int_as_float(0x7F800000);
                        }
                    }
                    float m[16];
                    #pragma unroll
                    for (int c = 0; c < 16; ++c) m[c] = fminf(v[c], v[c + 16]);
                    #pragma unroll
                    for (int wdt = 8; wdt > 0; wdt >>= 1)
                        #pragma unroll
                        for (int c = 0; c < wdt; ++c) m[c] = fminf(m[c], m[c + wdt]);
                    if (row_ok && c0 < ep.N) {
                        float* dst = ep.D + ((n0_out + cb) >> 5) * ep.ldD + row;  // mins[chunk][row]
                        float mn = m[0] == __int_as_float(0x7F800000) ? m[0] : finalize_dist<METRIC>(m[0]);
                        if (tmask == 2) mn = fminf(mn, *dst);
                        *dst = mn;
                    }
                    continue;
                }
                if constexpr (PIVOT) {
                    // Partition (quickselect): keep the elements at or below the
                    // row's pivot as candidates; in SYM mode also the transposed element for
                    // the column's row.  u is unclamped: max(u,0)+0 <= T implies u <= T.
                    if (!row_ok) {  // rows past M are masked, not skipped: the warp votes below
                        #pragma unroll
                        for (int c = 0; c < 32; ++c) v[c] = __int_as_float(0x7F800000);
                    }
                    if (SYM) {
                        // (32-bit compares: indices are < 2^31, include/knn.h)
                        if ((int32_t)c0 < (int32_t)row0) continue;  // lower chunks: produced by their mirror
                        if ((int32_t)c0 == (int32_t)row0) {        // diagonal chunk: keep col > row only
                            #pragma unroll
                            for (int c = 0; c < 32; ++c)
                                if (c <= lane) v[c] = __int_as_float(0x7F800000);
                        }
                    } else if (tmask || diag) {
                        #pragma unroll
                        for (int c = 0; c < 32; ++c) {
                            const bool lower = row + ep.self_shift > c0 + c;
                            if (c0 + c == self_col || (tmask && lower != (tmask == 2)))
                                v[c] = __int_as_float(0x7F800000);
                        }
                    }
                    if ((uint32_t)c0 + 32u > (uint32_t)ep.N) {
                        #pragma unroll
                        for (int c = 0; c < 32; ++c)
                            if ((int32_t)c0 + c >= (int32_t)ep.N) v[c] = __int_as_float(0x7F800000);
                    }
                    // this row's survivors in the chunk: row side (hr) and column side (hc)
                    uint32_t hr = 0, hc = 0;
                    if (EPI_DBG(4)) {
                        asm volatile("" ::"f"(v[0]), "f"(v[31]));
                        continue;
                    }
                    // Kept iff u < thr, i.e. u <= pivot: the pivot kernels store nextup(pivot)
                    // in thr (select.cu).  fl(u - t) is negative iff u < t (exact sign of a
                    // rounded difference; inf - inf is the canonical, positive NaN), so each
                    // test is an FADD and a funnel shift of its sign bit into the mask, c
                    // descending so that bit c ends at position c.  (One combined test
                    // against max(row pivot, column pivot) measured slower: 2.92 vs 2.84 ms;
                    // so did one superset test per element against max(row pivot, the chunk's
                    // largest column pivot) with exact sides per superset element: single-product
                    // partition 1.45 -> 1.81 ms, 3-product 2.30 -> 2.44 ms.)
                    // (the differences two at a time: FADD2)
                    #pragma unroll
                    for (int c = 30; c >= 0; c -= 2) {
                        float d0, d1;
                        f2_unpack(f2_sub(f2_pack(v[c], v[c + 1]), trow2), d0, d1);
                        hr = __funnelshift_l(__float_as_uint(d1), hr, 1);
                        hr = __funnelshift_l(__float_as_uint(d0), hr, 1);
                    }
                    if (SYM && !EPI_DBG(1)) {
                        const float4* ct4 = reinterpret_cast<const float4*>(col_t + cb);
                        #pragma unroll
                        for (int c4 = 7; c4 >= 0; --c4) {
                            const float4 tt = ct4[c4];
                            float d0, d1, d2, d3;
                            f2_unpack(f2_sub(f2_pack(v[4 * c4 + 2], v[4 * c4 + 3]), f2_pack(tt.z, tt.w)), d2, d3);
                            f2_unpack(f2_sub(f2_pack(v[4 * c4], v[4 * c4 + 1]), f2_pack(tt.x, tt.y)), d0, d1);
                            hc = __funnelshift_l(__float_as_uint(d3), hc, 1);
                            hc = __funnelshift_l(__float_as_uint(d2), hc, 1);
                            hc = __funnelshift_l(__float_as_uint(d1), hc, 1);
                            hc = __funnelshift_l(__float_as_uint(d0), hc, 1);
                        }
                    }
                    const uint32_t hm = hr | hc;
                    if (EPI_DBG(2)) {
                        asm volatile("" ::"r"(hm));
                        continue;
                    }
                    if (!__any_sync(0xFFFFFFFFu, hm != 0)) continue;
#if KNN_EPI_REG
                    // each lane's slots in the warp's pending list from a warp prefix sum of
                    // the lanes' counts (no shared atomic on one counter, which serialises
                    // the ~10 lanes holding survivors); survivor values staged by the lanes that
                    // have some, rows padded to 36 floats (conflict-free 16-byte stores at
                    // immediate offsets, no swizzle arithmetic), then read back by index
                    const int mine = __popc(hr) + __popc(hc);
                    int incl = mine;
                    #pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
                    float* srow = reinterpret_cast<float*>(slab) + lane * SROW;
                    if (hm) {
                        #pragma unroll
                        for (int u = 0; u < 8; ++u)
                            *reinterpret_cast<float4*>(srow + 4 * u) =
                                make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                    }
                    if (EPI_DBG(16)) {  // DIAGNOSTIC: tests, slot scan and staging only
                        __syncwarp();
                        continue;
                    }
                    if (pend_n + total > PEND_CAP) {
                        if (!EPI_DBG(8)) dfl.flush(ep, pent, pend_n);
                        pend_n = 0;
                    }
                    uint32_t h = hm;
                    if (total <= PEND_CAP) {
                        int pos = pend_n + incl - mine;
                        while (h) {
                            const int c = __ffs(h) - 1;
                            h &= h - 1;
                            const float x = srow[c];
                            const uint32_t key = __float_as_uint(PIVOT1 ? fmaxf(x, 0.0f) : finalize_dist<METRIC>(x)) | 0x80000000u;
                            if ((hr >> c) & 1) {
                                pent[pos] = make_uint4((uint32_t)row, (uint32_t)(c0 + c), key, 0u);
                                ++pos;
                            }
                            if (SYM && ((hc >> c) & 1)) {
                                pent[pos] = make_uint4((uint32_t)(c0 + c), (uint32_t)row, key, 0u);
                                ++pos;
                            }
                        }
                        pend_n += total;
                    } else {  // more survivors than the list holds (adversarial ties): direct
                        while (h) {
                            const int c = __ffs(h) - 1;
                            h &= h - 1;
                            const float x = srow[c];
                            const uint32_t key = __float_as_uint(PIVOT1 ? fmaxf(x, 0.0f) : finalize_dist<METRIC>(x)) | 0x80000000u;
                            if ((hr >> c) & 1) pivot_append(ep, row, key, (uint32_t)(c0 + c));
                            if (SYM && ((hc >> c) & 1)) pivot_append(ep, c0 + c, key, (uint32_t)row);
                        }
                    }
                    __syncwarp();
                    continue;
#else
                    // stage the chunk's values (swizzled) so that each lane can walk its own
                    // survivors with dynamic indices.  Only lanes with survivors store (a lane
                    // reads back only its own row): ~5 of 32 lanes, so each store is about one
                    // shared-memory wavefront instead of four — the tensor core's operand reads
                    // already take most of the shared-memory bandwidth.
                    float* svp = reinterpret_cast<float*>(slab);
                    const uint32_t sv = smem_u32(svp);
                    if (hm) {
                        #pragma unroll
                        for (int u = 0; u < 8; ++u)
                            sts128(sv + lane * 128 + ((u ^ (lane & 7)) << 4), v[4 * u], v[4 * u + 1],
                                   v[4 * u + 2], v[4 * u + 3]);
                    }
                    if (EPI_DBG(16)) {  // DIAGNOSTIC: staging only
                        __syncwarp();
                        continue;
                    }
                    // staged element c of this lane's row: 16-byte unit (c >> 2) ^ (lane & 7)
                    // of the row, i.e. index lane * 32 + (c ^ ((lane & 7) << 2))
                    const float* srow = svp + lane * 32;
                    const int sx = (lane & 7) << 2;
                    // slots of this lane's entries in the warp's pending list: the warp total
                    // by one reduction, each lane's base by a shared atomic on the warp's
                    // running count (order inside the list is irrelevant)
                    const int mine = __popc(hr) + __popc(hc);
                    const int total = __reduce_add_sync(0xFFFFFFFFu, mine);
                    if (pend_n + total > PEND_CAP) {
                        if (!EPI_DBG(8)) dfl.flush(ep, pent, pend_n);
                        pend_n = 0;
                        if (lane == 0) s_pend[warp - 2] = 0;
                    }
                    __syncwarp();
                    uint32_t h = hm;
                    if (total <= PEND_CAP) {
                        int pos = mine ? atomicAdd(&s_pend[warp - 2], mine) : 0;
                        while (h) {
                            const int c = __ffs(h) - 1;
                            h &= h - 1;
                            const float x = srow[c ^ sx];
                            const uint32_t key = __float_as_uint(PIVOT1 ? fmaxf(x, 0.0f) : finalize_dist<METRIC>(x)) | 0x80000000u;
                            if ((hr >> c) & 1) {
                                pent[pos] = make_uint4((uint32_t)row, (uint32_t)(c0 + c), key, 0u);
                                ++pos;
                            }
                            if (SYM && ((hc >> c) & 1)) {
                                pent[pos] = make_uint4((uint32_t)(c0 + c), (uint32_t)row, key, 0u);
                                ++pos;
                            }
                        }
                        pend_n += total;
                    } else {  // more survivors than the list holds (adversarial ties): direct
                        while (h) {
                            const int c = __ffs(h) - 1;
                            h &= h - 1;
                            const float x = svp[lane * 32 + (((c >> 2) ^ (lane & 7)) << 2) + (c & 3)];
                            const uint32_t key = __float_as_uint(PIVOT1 ? fmaxf(x, 0.0f) : finalize_dist<METRIC>(x)) | 0x80000000u;
                            if ((hr >> c) & 1) pivot_append(ep, row, key, (uint32_t)(c0 + c));
                            if (SYM && ((hc >> c) & 1)) pivot_append(ep, c0 + c, key, (uint32_t)row);
                        }
                    }
                    __syncwarp();
                    continue;
#endif
                }
                if constexpr (SYM) {
                    // chunk rows [row0, +32) x cols [c0, +32), both global.  Below the
                    // diagonal: produced by the mirror chunk.  Above: stored directly and
                    // transposed.  On it: lower triangle mirrored from the upper in smem.
                    if (c0 < row0) continue;
                    const uint32_t sd = smem_u32(slab);
                    const uint32_t st = sd + STG_BYTES;
                    if (lane == 0) bulk_wait_read<0>();  // both buffers' previous stores read
                    __syncwarp();
                    #pragma unroll
                    for (int u = 0; u < 8; ++u)
                        sts128(sd + lane * 128 + ((u ^ (lane & 7)) << 4), v[4 * u], v[4 * u + 1],
                               v[4 * u + 2], v[4 * u + 3]);
                    if (c0 == row0) {
                        __syncwarp();
                        float* sp = reinterpret_cast<float*>(slab);
                        for (int j = 0; j < lane; ++j)  // (lane, j) <- (j, lane)
                            sp[lane * 32 + (((j >> 2) ^ (lane & 7)) << 2) + (j & 3)] =
                                sp[j * 32 + (((lane >> 2) ^ (j & 7)) << 2) + (lane & 3)];
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&map_d, sd, (int)c0, (int)row0);
                        bulk_commit();
                    }
                    if (c0 == row0) continue;
                    if (lane == 0) bulk_wait_read<1>();  // transposed buffer's previous store read
                    __syncwarp();
                    #pragma unroll
                    for (int j = 0; j < 32; ++j)  // element (row j, col lane) of the transpose
                        asm volatile("st.shared.f32 [%0], %1;" ::"r"(st + j * 128 + ((((lane >> 2) ^ (j & 7))) << 4) +
                                                                   (lane & 3) * 4),
                                     "f"(v[j])
                                     : "memory");
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&map_d, st, (int)row0, (int)c0);
                        bulk_commit();
                    }
                    continue;
                }
                if (tmask) {
                    // one orientation pass of a block straddling the diagonal: store only
                    // the elements this orientation owns (rare; plain stores)
                    if (!row_ok) continue;
                    #pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        const bool lower = row + ep.self_shift > c0 + c;  // i+shift > j
                        if (c0 + c < ep.N && lower == (tmask == 2)) drow[c0 + c] = v[c];
                    }
                    continue;
                }
                if (use_tma_store) {
                    // stage the 32x32 chunk in 128B-swizzled smem (row = lane: 16-byte
                    // unit u of the row lives at unit u ^ (row & 7)), then one TMA store;
                    // rows >= M / columns >= N are clipped by the TMA unit.
                    if (lane == 0) bulk_wait_read<1>();  // this buffer's previous store read
                    __syncwarp();
                    const uint32_t sbuf = smem_u32(slab + sbsel * STG_BYTES);
                    #pragma unroll
                    for (int u = 0; u < 8; ++u)
                        sts128(sbuf + lane * 128 + ((u ^ (lane & 7)) << 4), v[4 * u], v[4 * u + 1],
                               v[4 * u + 2], v[4 * u + 3]);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&map_d, sbuf, (int)(SAMPLE ? n0_out + cb : c0), (int)row0);
                        bulk_commit();
                    }
                    sbsel ^= 1;
                    continue;
                }
                if (!row_ok) continue;
                if (vec_ok && c0 + 32 <= ep.N) {
                    #pragma unroll
                    for (int c = 0; c < 32; c += 4)
                        st_cs4(drow + c0 + c, v[c], v[c + 1], v[c + 2], v[c + 3]);
                } else {
                    #pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (c0 + c < ep.N) drow[c0 + c] = v[c];
                }
            }
            // this work item's column data fully read
            __syncwarp();
            if (lane == 0) mbar_arrive(colempty0 + 8 * slot);
        }
        }
        if (use_tma_store && lane == 0) bulk_wait_all();
        if constexpr (PIVOT) {
            dfl.complete(ep);
            pivot_flush(ep, pent, pend_n);
        }
    }
    teardown(tmem_base);
}

// ------------------------------------------------------------ host side -------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_once;

// Rows per group of the symmetric schedule (SymSched::gm): group-major once the split
// operands (hi + lo, 4 bytes per coordinate) outgrow ~2/3 of the 126 MB L2, row-major below
// (measured: N = 65536, d = 256 (64 MB): row-major 2.70 vs 2.77 ms; C4 (128 MB): 2.67 ->
// 2.42 ms with 16 rows; C5 (128 MB): 11.6 -> 11.1 ms).  Env KNN_SYM_GROUP overrides.
int64_t sym_group_rows(int64_t N, int32_t d_pad) {
    static const int64_t env = [] {
        const char* v = getenv("KNN_SYM_GROUP");
        return v ? (int64_t)atoi(v) : (int64_t)-1;
    }();
    if (env >= 0) return env;
    return (double)N * d_pad * 4.0 > 80e6 ? 16 : 0;
}

void init_encode() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    else
        cudaGetLastError();
}

}  // namespace

// Output map: fp32 D (rows x N, row stride ldD), 32x32 boxes, 128B swizzle (the staging
// layout of the epilogue).
bool tc_make_output_map(CUtensorMap* m, float* D, int64_t rows, int64_t N, int64_t ldD) {
    std::call_once(g_once, init_encode);
    if (!g_encode) return false;
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ldD * 4};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, D, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool tc_make_operand_map(CUtensorMap* m, const __half* base, int64_t rows, int32_t d_pad, int box_rows) {
    std::call_once(g_once, init_encode);
    if (!g_encode) return false;
    cuuint64_t dims[2] = {(cuuint64_t)d_pad, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)d_pad * 2};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapSwizzle swz = SWZ == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                   : SWZ == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                               : CU_TENSOR_MAP_SWIZZLE_32B;
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool tc_supported() {
    std::call_once(g_once, init_encode);
    if (!g_encode) return false;
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    return major == 10 && minor == 0;
}

cudaError_t launch_dist_tc(const TcOperands& op, int32_t metric, int64_t self_shift, float* D,
                           int64_t ldD, int num_sms, cudaStream_t s) {
    if (op.M == 0 || op.N == 0) return cudaSuccess;
    std::call_once(g_once, init_encode);
    if (!g_encode) return cudaErrorNotSupported;
    CUtensorMap mqh, mql, mxh, mxl;
    if (!tc_make_operand_map(&mqh, op.q_hi, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mql, op.q_lo, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mxh, op.x_hi, op.N, op.d_pad, BN / 2) ||
        !tc_make_operand_map(&mxl, op.x_lo, op.N, op.d_pad, BN / 2))
        return cudaErrorInvalidValue;
    TileSched tiles{ceil_div(ceil_div(op.M, BM), 2), ceil_div(op.N, BN)};
    const int64_t num_tiles = tiles.n_mp * tiles.n_nb;  // work units per CTA pair
    const int64_t pairs = num_tiles < num_sms / CLUSTER ? num_tiles : num_sms / CLUSTER;
    const int grid = (int)(pairs * CLUSTER);
    EpiArgs ep{op.qn, op.q_rs, op.M, op.xn, op.x_rs, op.N, metric, self_shift, D, ldD,
               nullptr, nullptr, nullptr, 0, nullptr};
    auto kern = metric_kind(metric) == 1 ? dist_tc_kernel<1, false, MODE_STORE, TileSched> : metric_kind(metric) == 2 ? dist_tc_kernel<2, false, MODE_STORE, TileSched> : dist_tc_kernel<0, false, MODE_STORE, TileSched>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    CUtensorMap md;
    const bool tma_store = (ldD % 4) == 0 && (reinterpret_cast<uintptr_t>(D) & 15) == 0 &&
                           tc_make_output_map(&md, D, op.M, op.N, ldD);
    if (!tma_store) memset(&md, 0, sizeof md);
    kern<<<grid, THREADS, SMEM_BYTES, s>>>(mqh, mql, mxh, mxl, md, tma_store ? 1 : 0, op.d_pad / BK,
                                           tiles, ep);
    return cudaGetLastError();
}

cudaError_t launch_dist_tc_sym(const TcOperands& op, int32_t metric, float* D, int64_t ldD, int num_sms,
                               cudaStream_t s) {
    if (op.N == 0) return cudaSuccess;
    if (op.M != op.N || ldD % 4 != 0 || (reinterpret_cast<uintptr_t>(D) & 15) != 0)
        return cudaErrorInvalidValue;
    CUtensorMap mqh, mql, mxh, mxl, md;
    if (!tc_make_operand_map(&mqh, op.q_hi, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mql, op.q_lo, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mxh, op.x_hi, op.N, op.d_pad, BN / 2) ||
        !tc_make_operand_map(&mxl, op.x_lo, op.N, op.d_pad, BN / 2) ||
        !tc_make_output_map(&md, D, op.N, op.N, ldD))
        return cudaErrorInvalidValue;
    SymSched sched{ceil_div(op.N, BN)};
    sched.gm = sym_group_rows(op.N, op.d_pad);
    const int64_t units = sched.n * (sched.n + 1) / 2;
    const int64_t pairs = units < num_sms / CLUSTER ? units : num_sms / CLUSTER;
    EpiArgs ep{op.qn, op.q_rs, op.M, op.xn, op.x_rs, op.N, metric, 0, D, ldD,
               nullptr, nullptr, nullptr, 0, nullptr};
    auto kern = metric_kind(metric) == 1 ? dist_tc_kernel<1, true, MODE_STORE, SymSched> : metric_kind(metric) == 2 ? dist_tc_kernel<2, true, MODE_STORE, SymSched> : dist_tc_kernel<0, true, MODE_STORE, SymSched>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)(pairs * CLUSTER), THREADS, SMEM_BYTES, s>>>(mqh, mql, mxh, mxl, md, 1, op.d_pad / BK,
                                                                sched, ep);
    return cudaGetLastError();
}

cudaError_t launch_dist_tc_mins(const TcOperands& op, int64_t S, int32_t metric, int64_t self_shift, float* mins,
                                float margin_override, int num_sms, cudaStream_t s, const float* xmax,
                                bool bounded_norms) {
    if (!xmax || self_shift != INT64_MIN) return cudaErrorInvalidValue;  // gathered samples only
    if (op.M == 0 || op.N == 0) return cudaSuccess;
    // S sampled columns = S/256 full column blocks spread evenly over the op.N columns
    const int64_t ns = S / BN, nfull = op.N / BN;
    if (S % BN != 0 || ns < 1 || ns > nfull) return cudaErrorInvalidValue;
    CUtensorMap mqh, mql, mxh, mxl, md;
    memset(&md, 0, sizeof md);
    if (!tc_make_operand_map(&mqh, op.q_hi, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mql, op.q_lo, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mxh, op.x_hi, op.N, op.d_pad, BN / 2) ||
        !tc_make_operand_map(&mxl, op.x_lo, op.N, op.d_pad, BN / 2))
        return cudaErrorInvalidValue;
    // mins is [S/32][M]: ep.D / ep.ldD reused as its base / row stride.  Error of the single
    // hi.hi product (prep.cu split, |lo| <= 2^-11 |x| per component): |2 q.x - 2 qh.xh| <=
    // (2^-10 (1 + 2^-10) + d 2^-23) 2|q||x| (the d term bounds fp32 accumulation), and
    // 2|q||x| <= ||q||^2 + ||x||^2; + 2^-20 covers the roundings of both u values.
    // bounded_norms: op.qn / op.xn already carry the per-point bound (launch_bound_norms'
    // ninf = sqn (1 + Fs)), so no margin is added
    float margin = bounded_norms ? 0.0f
                                 : (float)(std::ldexp(1.0, -10) * (1.0 + std::ldexp(1.0, -10)) +
                                           op.d_pad * std::ldexp(1.0, -23) + std::ldexp(1.0, -20));
    if (!std::isnan(margin_override)) margin = margin_override;  // tests: force bad pivots
    EpiArgs ep{op.qn, op.q_rs, op.M, op.xn, op.x_rs, op.N, metric, self_shift, mins, op.M,
               nullptr, nullptr, nullptr, 0, nullptr, margin, nfull / ns, xmax};
    const int64_t n_mp = ceil_div(ceil_div(op.M, BM), 2);
    static const bool ares_env = [] {
        const char* v = getenv("KNN_MINS_RESIDENT");  // 0: stream A with every tile (round 1)
        return !(v && atoi(v) == 0);
    }();
    if (ares_env && nfull == ns && op.d_pad <= 256) {
        // A-panel-resident: units of `run` column blocks per row-block pair, run chosen so
        // that the units spread evenly over the clusters (>= 8 units per cluster)
        const int64_t ncl = num_sms / CLUSTER;
        int64_t run = ns;
        while (run > 2 && n_mp * ceil_div(ns, run) < 8 * ncl) run = ceil_div(run, 2);
        PanelSched sched{n_mp, ns, run};
        const int64_t units = n_mp * ceil_div(ns, run);
        const int64_t pairs = units < ncl ? units : ncl;
        auto kern = metric_kind(metric) == 1 ? dist_tc_kernel<1, false, MODE_MINS, PanelSched>
                    : metric_kind(metric) == 2 ? dist_tc_kernel<2, false, MODE_MINS, PanelSched>
                                               : dist_tc_kernel<0, false, MODE_MINS, PanelSched>;
        constexpr int smem = EpiCfg<MODE_MINS, true>::SMEM;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        kern<<<(unsigned)(pairs * CLUSTER), EpiCfg<MODE_MINS, true>::THREADS, smem, s>>>(mqh, mql, mxh, mxl, md, 0, op.d_pad / BK, sched,
                                                               ep);
        return cudaGetLastError();
    }
    TileSched sched{n_mp, ns, nfull / ns};
    const int64_t units = sched.n_mp * sched.n_nb;
    const int64_t pairs = units < num_sms / CLUSTER ? units : num_sms / CLUSTER;
    auto kern = metric_kind(metric) == 1 ? dist_tc_kernel<1, false, MODE_MINS, TileSched> : metric_kind(metric) == 2 ? dist_tc_kernel<2, false, MODE_MINS, TileSched> : dist_tc_kernel<0, false, MODE_MINS, TileSched>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         EpiCfg<MODE_MINS>::SMEM);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)(pairs * CLUSTER), EpiCfg<MODE_MINS>::THREADS, EpiCfg<MODE_MINS>::SMEM, s>>>(mqh, mql, mxh, mxl, md, 0, op.d_pad / BK,
                                                                sched, ep);
    return cudaGetLastError();
}

cudaError_t launch_dist_tc_sample(const TcOperands& op, int64_t S, int32_t metric, int64_t self_shift, float* Ds,
                                  int64_t ldS, float margin_override, int num_sms, cudaStream_t s,
                                  bool bounded_norms) {
    if (op.M == 0 || op.N == 0) return cudaSuccess;
    const int64_t ns = S / BN, nfull = op.N / BN;
    if (S % BN != 0 || ns < 1 || ns > nfull) return cudaErrorInvalidValue;
    if (ldS % 4 != 0 || (reinterpret_cast<uintptr_t>(Ds) & 15) != 0) return cudaErrorInvalidValue;
    CUtensorMap mqh, mql, mxh, mxl, md;
    if (!tc_make_operand_map(&mqh, op.q_hi, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mql, op.q_lo, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mxh, op.x_hi, op.N, op.d_pad, BN / 2) ||
        !tc_make_operand_map(&mxl, op.x_lo, op.N, op.d_pad, BN / 2) ||
        !tc_make_output_map(&md, Ds, op.M, S, ldS))
        return cudaErrorInvalidValue;
    // the same single-product error bound as the chunk-minimum sample (launch_dist_tc_mins)
    // (bounded_norms: the per-point bound is in op.qn / op.xn, launch_bound_norms' ninf)
    float margin = bounded_norms ? 0.0f
                                 : (float)(std::ldexp(1.0, -10) * (1.0 + std::ldexp(1.0, -10)) +
                                           op.d_pad * std::ldexp(1.0, -23) + std::ldexp(1.0, -20));
    if (!std::isnan(margin_override)) margin = margin_override;
    EpiArgs ep{op.qn, op.q_rs, op.M, op.xn, op.x_rs, op.N, metric, self_shift, Ds, ldS,
               nullptr, nullptr, nullptr, 0, nullptr, margin, nfull / ns};
    TileSched sched{ceil_div(ceil_div(op.M, BM), 2), ns, nfull / ns};
    const int64_t units = sched.n_mp * sched.n_nb;
    const int64_t pairs = units < num_sms / CLUSTER ? units : num_sms / CLUSTER;
    auto kern = metric_kind(metric) == 1 ? dist_tc_kernel<1, false, MODE_SAMPLE, TileSched> : metric_kind(metric) == 2 ? dist_tc_kernel<2, false, MODE_SAMPLE, TileSched> : dist_tc_kernel<0, false, MODE_SAMPLE, TileSched>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)(pairs * CLUSTER), THREADS, SMEM_BYTES, s>>>(mqh, mql, mxh, mxl, md, 1, op.d_pad / BK,
                                                                sched, ep);
    return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_pivot_impl(const TcOperands& op, int32_t metric, int64_t self_shift, bool sym,
                              const float* thr, int32_t* cnt, uint64_t* cent,
                              int32_t cap, int32_t* flag, int num_sms, cudaStream_t s,
                              int64_t unit_lo, int64_t unit_hi, float margin, bool col_major = false,
                              int32_t gate = -1) {
    if (op.M == 0 || op.N == 0) return cudaSuccess;
    if (sym && op.M != op.N) return cudaErrorInvalidValue;
    CUtensorMap mqh, mql, mxh, mxl, md;
    memset(&md, 0, sizeof md);
    if (!tc_make_operand_map(&mqh, op.q_hi, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mql, op.q_lo, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mxh, op.x_hi, op.N, op.d_pad, BN / 2) ||
        !tc_make_operand_map(&mxl, op.x_lo, op.N, op.d_pad, BN / 2))
        return cudaErrorInvalidValue;
    EpiArgs ep{op.qn, op.q_rs, op.M, op.xn, op.x_rs, op.N, metric, sym ? 0 : self_shift, nullptr, 0,
               thr, cnt, cent, cap, flag, margin};
    ep.gate = gate;
    if (const char* dv = getenv("KNN_DBG_EPI")) ep.dbg = atoi(dv);
    cudaError_t e;
    if (sym) {
        SymSched sched{ceil_div(op.N, BN)};
        sched.gm = col_major ? -1 : sym_group_rows(op.N, op.d_pad);
        const int64_t all = sched.n * (sched.n + 1) / 2;
        sched.u_lo = unit_lo < 0 ? 0 : unit_lo;
        sched.u_hi = unit_hi < 0 || unit_hi > all ? all : unit_hi;
        if (sched.u_hi <= sched.u_lo) return cudaSuccess;
        const int64_t units = sched.u_hi - sched.u_lo;
        const int64_t pairs = units < num_sms / CLUSTER ? units : num_sms / CLUSTER;
        auto kern = metric_kind(metric) == 1 ? dist_tc_kernel<1, true, MODE, SymSched> : metric_kind(metric) == 2 ? dist_tc_kernel<MODE == MODE_PIVOT ? 2 : 0, true, MODE, SymSched> : dist_tc_kernel<0, true, MODE, SymSched>;
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, EpiCfg<MODE>::SMEM)) !=
            cudaSuccess)
            return e;
        kern<<<(unsigned)(pairs * CLUSTER), EpiCfg<MODE>::THREADS, EpiCfg<MODE>::SMEM, s>>>(
            mqh, mql, mxh, mxl, md, 0, op.d_pad / BK, sched, ep);
    } else {
        TileSched sched{ceil_div(ceil_div(op.M, BM), 2), ceil_div(op.N, BN)};
        const int64_t units = sched.n_mp * sched.n_nb;
        const int64_t pairs = units < num_sms / CLUSTER ? units : num_sms / CLUSTER;
        auto kern = metric_kind(metric) == 1 ? dist_tc_kernel<1, false, MODE, TileSched> : metric_kind(metric) == 2 ? dist_tc_kernel<MODE == MODE_PIVOT ? 2 : 0, false, MODE, TileSched> : dist_tc_kernel<0, false, MODE, TileSched>;
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, EpiCfg<MODE>::SMEM)) !=
            cudaSuccess)
            return e;
        kern<<<(unsigned)(pairs * CLUSTER), EpiCfg<MODE>::THREADS, EpiCfg<MODE>::SMEM, s>>>(
            mqh, mql, mxh, mxl, md, 0, op.d_pad / BK, sched, ep);
    }
    return cudaGetLastError();
}

cudaError_t launch_dist_tc_pivot(const TcOperands& op, int32_t metric, int64_t self_shift, bool sym,
                                 const float* thr, int32_t* cnt, uint64_t* cent,
                                 int32_t cap, int32_t* flag, int num_sms, cudaStream_t s,
                                 int64_t unit_lo, int64_t unit_hi, bool col_major, int32_t gate) {
    return launch_pivot_impl<MODE_PIVOT>(op, metric, self_shift, sym, thr, cnt, cent, cap, flag, num_sms,
                                         s, unit_lo, unit_hi, 0.0f, col_major, gate);
}

cudaError_t launch_dist_tc_pivot1(const TcOperands& op, int32_t metric, int64_t self_shift, bool sym,
                                  const float* thr, int32_t* cnt, uint64_t* cent,
                                  int32_t cap, int32_t* flag, int num_sms, cudaStream_t s, int32_t gate,
                                  int64_t unit_lo, int64_t unit_hi, bool col_major) {
    if (metric_kind(metric) == 2) return cudaErrorInvalidValue;  // L2 metrics only
    return launch_pivot_impl<MODE_PIVOT1>(op, metric, self_shift, sym, thr, cnt, cent, cap, flag,
                                          num_sms, s, unit_lo, unit_hi, 0.0f, col_major, gate);
}

cudaError_t launch_dist_tc_null(const TcOperands& op, bool sym, int num_sms, cudaStream_t s) {
    if (op.M == 0 || op.N == 0) return cudaSuccess;
    CUtensorMap mqh, mql, mxh, mxl, md;
    memset(&md, 0, sizeof md);
    if (!tc_make_operand_map(&mqh, op.q_hi, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mql, op.q_lo, op.M, op.d_pad, BM) ||
        !tc_make_operand_map(&mxh, op.x_hi, op.N, op.d_pad, BN / 2) ||
        !tc_make_operand_map(&mxl, op.x_lo, op.N, op.d_pad, BN / 2))
        return cudaErrorInvalidValue;
    EpiArgs ep{op.qn, op.q_rs, op.M, op.xn, op.x_rs, op.N, 0, INT64_MIN, nullptr, 0,
               nullptr, nullptr, nullptr, 0, nullptr};
    cudaError_t e;
    if (sym) {
        SymSched sched{ceil_div(op.N, BN)};
        sched.gm = sym_group_rows(op.N, op.d_pad);
        const int64_t units = sched.n * (sched.n + 1) / 2;
        const int64_t pairs = units < num_sms / CLUSTER ? units : num_sms / CLUSTER;
        auto kern = dist_tc_kernel<0, true, MODE_NULL, SymSched>;
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES)) != cudaSuccess)
            return e;
        kern<<<(unsigned)(pairs * CLUSTER), THREADS, SMEM_BYTES, s>>>(mqh, mql, mxh, mxl, md, 0, op.d_pad / BK,
                                                                    sched, ep);
    } else {
        TileSched sched{ceil_div(ceil_div(op.M, BM), 2), ceil_div(op.N, BN)};
        const int64_t units = sched.n_mp * sched.n_nb;
        const int64_t pairs = units < num_sms / CLUSTER ? units : num_sms / CLUSTER;
        auto kern = dist_tc_kernel<0, false, MODE_NULL, TileSched>;
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES)) != cudaSuccess)
            return e;
        kern<<<(unsigned)(pairs * CLUSTER), THREADS, SMEM_BYTES, s>>>(mqh, mql, mxh, mxl, md, 0, op.d_pad / BK,
                                                                    sched, ep);
    }
    return cudaGetLastError();
}

}  // namespace knn
