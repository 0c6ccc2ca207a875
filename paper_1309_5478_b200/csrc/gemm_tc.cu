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
#include "internal.cuh"
#include "ptx.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

namespace knn {
namespace {

constexpr int BM = 128;          // rows per tile (TMEM lanes)
constexpr int BN = 256;          // columns per tile (TMEM columns per accumulator)
constexpr int BK = 32;           // fp16 K elements per stage = one 64-byte swizzle row
constexpr int SWZ = BK * 2;      // swizzle span in bytes (64)
constexpr int STAGES = 3;
constexpr int UMMA_K = 16;
constexpr int EPI_WARPS = 8;     // 2 per TMEM lane quadrant, each owning BN/2 columns
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr int A_BYTES = BM * BK * 2;  // one fp16 A tile (16 KB)
constexpr int B_BYTES = BN * BK * 2;  // one fp16 B tile (32 KB)
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // hi+lo of both operands
constexpr int TMEM_COLS = 512;   // 2 accumulators × BN fp32 columns
constexpr int STG_BYTES = 32 * 32 * 4;  // one 32x32 fp32 output chunk (TMA-store staging)
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_WARPS * 2 * STG_BYTES + 1024 /*align*/ +
                           1024 /*barriers*/;
constexpr int GROUP_M = 8;       // tile-order swizzle: 8 row-block pairs share a column sweep
constexpr int CLUSTER = 2;       // CTA pair along M: the B operand is TMA-multicast to both

// Instruction descriptor (PTX ISA, tcgen05 "Instruction descriptor", kind::f16):
// [4,6) D format = F32 (1); [7,10) A = F16 (0); [10,13) B = F16 (0); bit 15/16 = 0:
// both K-major; [17,23) N>>3; [24,29) M>>4.
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
// Multicast variant: the box lands at the same smem offset in every CTA of ctaMask and
// completes tx bytes on the mbarrier at the same offset in each of them.
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                               int c0, int c1, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "h"(mask)
        : "memory");
}
// Commit this CTA's prior MMAs to the mbarrier at `bar` in every CTA of ctaMask.
__device__ __forceinline__ void tc_commit_mc(uint32_t bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(c0), "r"(c1), "r"(src)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void sts128(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
// Shared-memory matrix descriptor, K-major, SWZ-byte swizzle (PTX ISA "Matrix
// descriptor"): [0,14) start>>4; [16,30) LBO>>4 (unused for swizzled K-major: 1);
// [32,46) SBO>>4 = 8 rows * SWZ bytes between 8-row core-matrix groups; [46,48)
// version = 1; [49,52) base offset = 0 (tiles are 1024-aligned); [61,64) layout:
// 2 = SWIZZLE_128B, 4 = SWIZZLE_64B, 6 = SWIZZLE_32B.
constexpr uint64_t SDESC_LAYOUT = SWZ == 128 ? 2 : SWZ == 64 ? 4 : 6;
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) |
           ((uint64_t)((8 * SWZ) >> 4) << 32) | ((uint64_t)1 << 46) | (SDESC_LAYOUT << 61);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_cs4(float* p, float a, float b, float c, float d) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}

// Work unit of a 2-CTA cluster: a pair of row blocks (2*mp, 2*mp+1) against one column
// block nb; CTA rank r of the pair computes row block 2*mp + r.  Units are ordered in
// groups of GROUP_M pairs sweeping all column blocks (L2 reuse of the B panel).
struct TileMap {
    int64_t n_mp, n_nb;  // row-block pairs, column blocks
    __device__ __forceinline__ void get(int64_t t, int64_t& mp, int64_t& nb) const {
        const int64_t per_group = (int64_t)GROUP_M * n_nb;
        const int64_t g = t / per_group;
        const int64_t r = t - g * per_group;
        const int64_t m0 = g * GROUP_M;
        const int64_t gm = (n_mp - m0) < GROUP_M ? (n_mp - m0) : GROUP_M;
        mp = m0 + r % gm;
        nb = r / gm;
    }
};

struct EpiArgs {
    const float* qn; const float* q_rs; int64_t M;
    const float* xn; const float* x_rs; int64_t N;
    int32_t metric; int64_t self_shift; float* D; int64_t ldD;
};

template <int METRIC>
__global__ void __cluster_dims__(CLUSTER, 1, 1) __launch_bounds__(THREADS, 1)
dist_tc_kernel(const __grid_constant__ CUtensorMap map_qh, const __grid_constant__ CUtensorMap map_ql,
               const __grid_constant__ CUtensorMap map_xh, const __grid_constant__ CUtensorMap map_xl,
               const __grid_constant__ CUtensorMap map_d, int use_tma_store, int num_kb,
               TileMap tiles, int64_t num_tiles, EpiArgs ep) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(16) float col_n[2][BN];  // ||x_j||^2 of the tile's columns
    __shared__ __align__(16) float col_s[2][BN];  // 2^-sh_j of the tile's columns
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    uint8_t* stage_base = smem;
    uint8_t* stg_base = smem + STAGES * STAGE_BYTES;  // [EPI_WARPS][2] output chunks
    uint64_t* bars = reinterpret_cast<uint64_t*>(stg_base + EPI_WARPS * 2 * STG_BYTES);
    // bars: full[STAGES], empty[STAGES], tfull[2], tempty[2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES);
    const uint32_t tfull0 = smem_u32(bars + 2 * STAGES), tempty0 = smem_u32(bars + 2 * STAGES + 2);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, CLUSTER);  // both CTAs' MMAs must release a stage
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull0 + 8 * b, 1);
            mbar_init(tempty0 + 8 * b, EPI_WARPS);  // one arrive per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_qh)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ql)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_xh)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_xl)));
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();  // barriers of both CTAs initialised before any multicast
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t crank = cluster_rank();
    const int64_t cid = blockIdx.x / CLUSTER, ncl = gridDim.x / CLUSTER;

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer --------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = cid; t < num_tiles; t += ncl) {
                int64_t mp, nb;
                tiles.get(t, mp, nb);
                const int row_a = (int)((2 * mp + crank) * BM);
                const int row_b = (int)(nb * BN + crank * (BN / 2));  // this CTA's half of B
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(empty0 + 8 * stage, phase ^ 1);
                    const uint32_t fb = full0 + 8 * stage;
                    mbar_expect_tx(fb, STAGE_BYTES);
                    const uint32_t sb = smem_u32(stage_base + (size_t)stage * STAGE_BYTES);
                    const uint32_t boff = crank * (B_BYTES / 2);
                    tma_load_2d(sb, &map_qh, fb, kb * BK, row_a);
                    tma_load_2d(sb + A_BYTES, &map_ql, fb, kb * BK, row_a);
                    tma_load_2d_mc(sb + 2 * A_BYTES + boff, &map_xh, fb, kb * BK, row_b, 0x3);
                    tma_load_2d_mc(sb + 2 * A_BYTES + B_BYTES + boff, &map_xl, fb, kb * BK, row_b, 0x3);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer ----------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int64_t t = cid; t < num_tiles; t += ncl, ++it) {
                const int buf = it & 1;
                const uint32_t tphase = (it >> 1) & 1;
                mbar_wait(tempty0 + 8 * buf, tphase ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + buf * BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(full0 + 8 * stage, phase);
                    tc_fence_after();
                    const uint32_t sb = smem_u32(stage_base + (size_t)stage * STAGE_BYTES);
                    const uint32_t qh = sb, ql = sb + A_BYTES, xh = sb + 2 * A_BYTES,
                                   xl = sb + 2 * A_BYTES + B_BYTES;
                    // three K-segments, smallest terms first: ql.xh, qh.xl, qh.xh
                    const uint32_t sa[3] = {ql, qh, qh};
                    const uint32_t sbx[3] = {xh, xl, xh};
                    #pragma unroll
                    for (int seg = 0; seg < 3; ++seg) {
                        #pragma unroll
                        for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                            const uint32_t acc = (kb | seg | kk) != 0;
                            tc_mma(tmem_d, sdesc(sa[seg] + kk * UMMA_K * 2),
                                   sdesc(sbx[seg] + kk * UMMA_K * 2), acc);
                        }
                    }
                    // frees the smem stage (in both CTAs: B halves were multicast) when done
                    tc_commit_mc(empty0 + 8 * stage, 0x3);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit(tfull0 + 8 * buf);  // accumulator ready for the epilogue
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------ epilogue (8 warps) --
        const int quad = warp & 3;                  // TMEM lane quadrant this warp may access
        const int half = (warp - 2) >> 2;           // which BN/2 columns it owns
        const int etid = threadIdx.x - 64;          // 0..255
        const bool vec_ok = (ep.ldD % 4) == 0 && ((reinterpret_cast<uintptr_t>(ep.D) & 15) == 0);
        int sbsel = 0;  // which of the warp's two staging buffers
        int it = 0;
        for (int64_t t = cid; t < num_tiles; t += ncl, ++it) {
            int64_t mp, nb;
            tiles.get(t, mp, nb);
            const int64_t mb = 2 * mp + crank;
            const int buf = it & 1;
            const uint32_t tphase = (it >> 1) & 1;
            const int64_t n0 = nb * BN;
            // stage the tile's column norms and scales (double-buffered by `buf`)
            {
                const int64_t j = n0 + etid;
                col_n[buf][etid] = j < ep.N ? __ldg(ep.xn + j) : 0.0f;
                col_s[buf][etid] = j < ep.N ? __ldg(ep.x_rs + j) : 0.0f;
            }
            named_bar(1, 32 * EPI_WARPS);
            const int64_t row0 = mb * BM + quad * 32;
            const int64_t row = row0 + lane;
            const bool row_ok = row < ep.M;
            const float qn = row_ok ? __ldg(ep.qn + row) : 0.0f;
            const float cq = row_ok ? -2.0f * __ldg(ep.q_rs + row) : 0.0f;
            const int64_t c_lo = n0 + half * (BN / 2);
            // does this warp's 32x(BN/2) block touch the excluded self pairs?
            const bool diag = ep.self_shift != INT64_MIN &&
                              row0 + ep.self_shift < c_lo + BN / 2 && row0 + 31 + ep.self_shift >= c_lo;
            const int64_t self_col = row + ep.self_shift;
            float* drow = ep.D + row * ep.ldD;

            mbar_wait(tfull0 + 8 * buf, tphase);
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + buf * BN + half * (BN / 2);
            #pragma unroll 1
            for (int ch = 0; ch < BN / 64; ++ch) {
                uint32_t r[32];
                tmem_ld32(taddr + ch * 32, r);
                if (ch == BN / 64 - 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tempty0 + 8 * buf);
                }
                const int cb = half * (BN / 2) + ch * 32;  // first column of the chunk in the tile
                const float4* cn4 = reinterpret_cast<const float4*>(&col_n[buf][cb]);
                const float4* cs4 = reinterpret_cast<const float4*>(&col_s[buf][cb]);
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
                        float dd = fmaf(__uint_as_float(r[c]) * cq, sa4[e], qn + na[e]);
                        dd = fmaxf(dd, 0.0f) + 0.0f;
                        if (METRIC == 1) dd = sqrtf(dd);
                        v[c] = dd;
                    }
                }
                const int64_t c0 = n0 + cb;
                if (diag) {
                    #pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (c0 + c == self_col) v[c] = __int_as_float(0x7F800000);
                }
                if (use_tma_store) {
                    // stage the 32x32 chunk in 128B-swizzled smem (row = lane: 16-byte
                    // unit u of the row lives at unit u ^ (row & 7)), then one TMA store;
                    // rows >= M / columns >= N are clipped by the TMA unit.
                    if (lane == 0) bulk_wait_read<1>();  // this buffer's previous store read
                    __syncwarp();
                    const uint32_t sbuf = smem_u32(stg_base + ((warp - 2) * 2 + sbsel) * STG_BYTES);
                    #pragma unroll
                    for (int u = 0; u < 8; ++u)
                        sts128(sbuf + lane * 128 + ((u ^ (lane & 7)) << 4), v[4 * u], v[4 * u + 1],
                               v[4 * u + 2], v[4 * u + 3]);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&map_d, sbuf, (int)c0, (int)row0);
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
        }
        if (use_tma_store && lane == 0) bulk_wait_all();
    }
    tc_fence_before();
    cluster_sync_all();  // no CTA leaves while its peer may still multicast into it
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(TMEM_COLS));
    }
}

// ------------------------------------------------------------ host side -------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_once;

void init_encode() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    else
        cudaGetLastError();
}

// Output map: fp32 D (rows x N, row stride ldD), 32x32 boxes, 128B swizzle (the staging
// layout of the epilogue).
bool make_dmap(CUtensorMap* m, float* D, int64_t rows, int64_t N, int64_t ldD) {
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ldD * 4};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, D, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_map(CUtensorMap* m, const __half* base, int64_t rows, int32_t d_pad, int box_rows) {
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

}  // namespace

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
    if (!make_map(&mqh, op.q_hi, op.M, op.d_pad, BM) || !make_map(&mql, op.q_lo, op.M, op.d_pad, BM) ||
        !make_map(&mxh, op.x_hi, op.N, op.d_pad, BN / 2) || !make_map(&mxl, op.x_lo, op.N, op.d_pad, BN / 2))
        return cudaErrorInvalidValue;
    TileMap tiles{ceil_div(ceil_div(op.M, BM), 2), ceil_div(op.N, BN)};
    const int64_t num_tiles = tiles.n_mp * tiles.n_nb;  // work units per CTA pair
    const int64_t pairs = num_tiles < num_sms / CLUSTER ? num_tiles : num_sms / CLUSTER;
    const int grid = (int)(pairs * CLUSTER);
    EpiArgs ep{op.qn, op.q_rs, op.M, op.xn, op.x_rs, op.N, metric, self_shift, D, ldD};
    auto kern = metric == 1 ? dist_tc_kernel<1> : dist_tc_kernel<0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    CUtensorMap md;
    const bool tma_store = (ldD % 4) == 0 && (reinterpret_cast<uintptr_t>(D) & 15) == 0 &&
                           make_dmap(&md, D, op.M, op.N, ldD);
    if (!tma_store) memset(&md, 0, sizeof md);
    kern<<<grid, THREADS, SMEM_BYTES, s>>>(mqh, mql, mxh, mxl, md, tma_store ? 1 : 0, op.d_pad / BK,
                                           tiles, num_tiles, ep);
    return cudaGetLastError();
}

}  // namespace knn
