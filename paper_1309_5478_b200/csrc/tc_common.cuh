// tc_common.cuh — the shared tcgen05 mainloop of the distance GEMMs (materialised
// gemm_tc.cu and fused fused.cu): tile constants, PTX wrappers, work schedulers, the TMA
// producer loop and the single-thread MMA issuer loop.  See gemm_tc.cu for the design.
#pragma once
#include "internal.cuh"
#include "ptx.cuh"

#include <cuda.h>

namespace knn {
namespace tc {

// KNN_CTA2 (default): the CTA pair runs ONE tcgen05.mma.cta_group::2 of M = 256 (each CTA
// holds its 128 rows of A and its 128-column half of B, issued by the pair's leader CTA)
// instead of one M = 128 MMA per CTA over a B operand multicast to both.  Per CTA the tensor
// core then reads 8 KB of shared memory per 128-cycle MMA instead of 12 KB and the TMA writes
// a third less — the operand traffic was above the 128 B/clk shared-memory port.
#ifndef KNN_CTA2
#define KNN_CTA2 0
#endif
constexpr bool CTA2 = KNN_CTA2 != 0;
constexpr int BM = 128;          // rows per tile (TMEM lanes)
constexpr int BN = 256;          // columns per tile (TMEM columns per accumulator)
constexpr int BK = 32;           // fp16 K elements per stage = one 64-byte swizzle row
constexpr int SWZ = BK * 2;      // swizzle span in bytes (64)
constexpr int UMMA_K = 16;
constexpr int A_BYTES = BM * BK * 2;  // one fp16 A tile (8 KB)
constexpr int B_BYTES = BN * BK * 2;  // one fp16 B tile (16 KB)
constexpr int B_TILE = CTA2 ? B_BYTES / 2 : B_BYTES;  // per-CTA bytes of one B tile
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_TILE;  // hi+lo of both operands (32 / 48 KB)
// the operand region: 3 stages of 48 KB (1-CTA) or 4 of 32 KB (CTA2)
constexpr int RING_BYTES = CTA2 ? 4 * STAGE_BYTES : 3 * (2 * A_BYTES + 2 * B_BYTES);
constexpr int TMEM_COLS = 512;   // 2 accumulators x BN fp32 columns
constexpr int CLUSTER = 2;       // CTA pair along M: the B operand is TMA-multicast to both
constexpr int GROUP_M = 8;       // tile order: 8 row-block pairs share a column sweep

// Instruction descriptor (PTX ISA, tcgen05 "Instruction descriptor", kind::f16):
// [4,6) D format = F32 (1); [7,10) A = F16 (0); [10,13) B = F16 (0); bit 15/16 = 0:
// both K-major; [17,23) N>>3; [24,29) M>>4.
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((CTA2 ? 2 * BM : BM) >> 4) << 24);

// Operand tiles are re-read by many tiles: keep them in L2 (evict-last).
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(policy_evict_last())
        : "memory");
}
// Multicast variant: the box lands at the same smem offset in every CTA of ctaMask and
// completes tx bytes on the mbarrier at the same offset in each of them.
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                               int c0, int c1, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5, %6;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "h"(mask), "l"(policy_evict_last())
        : "memory");
}
// Commit this CTA's prior MMAs to the mbarrier at `bar` in every CTA of ctaMask.
__device__ __forceinline__ void tc_commit_mc(uint32_t bar, uint16_t mask) {
#ifdef KNN_MMA_CONVERGED
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;\n\t}" ::"r"(bar), "h"(mask)
        : "memory");
#else
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar), "h"(mask)
        : "memory");
#endif
}
// TMA store of a box with an L2 eviction-priority hint (evict-first for the streamed
// distance matrix, so it does not push the reused operands out of L2).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(c0), "r"(c1), "r"(src), "l"(pol)
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
#ifdef KNN_MMA_CONVERGED
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
                 : "memory");
#else
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
#endif
}
// KNN_MMA_CONVERGED: the whole MMA warp runs the issue loop (warp-uniform descriptors, which
// the compiler can keep in uniform registers) and one lane, picked by elect.sync inside the
// instruction sequence, issues each tcgen05 instruction.
#ifdef KNN_MMA_CONVERGED
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
#else
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
#endif
// shared::cluster address of the same shared-memory offset in the pair's leader CTA (rank 0):
// a CTA's own shared window address carries its rank in bit 24
__device__ __forceinline__ uint32_t leader_addr(uint32_t a) { return a & 0xFEFFFFFFu; }
// TMA load into this CTA's shared memory whose completion is counted on the LEADER's
// mbarrier (cta_group::2: the leader's MMA consumes both CTAs' halves)
__device__ __forceinline__ void tma_load_2d_2sm(uint32_t dst, const CUtensorMap* map, uint32_t bar_leader,
                                                int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_leader), "l"(policy_evict_last())
        : "memory");
}
__device__ __forceinline__ void tc_mma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
// commit the pair's prior cta_group::2 MMAs to the mbarrier at `bar` in both CTAs
__device__ __forceinline__ void tc_commit2_mc(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
        ::"r"(bar), "h"((uint16_t)0x3) : "memory");
}
// arrive on the leader CTA's copy of a barrier (release at cluster scope)
__device__ __forceinline__ void mbar_arrive_leader(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(leader_addr(bar)) : "memory");
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

// ------------------------------------------------------------------ schedulers -------
// A work unit of a 2-CTA cluster: the row-block pair mp (CTA rank r computes row block
// 2*mp + r) against column blocks [nb0, nb1).
struct Unit {
    int64_t mp, nb0, nb1;
};

// Materialised GEMM: one tile per unit, groups of GROUP_M pairs sweep all column blocks.
struct TileSched {
    static constexpr bool kResidentA = false;
    int64_t n_mp, n_nb;
    int64_t nb_stride = 1;  // column block nb of the schedule is block nb * nb_stride of the matrix
    __device__ __forceinline__ int64_t units() const { return n_mp * n_nb; }
    __device__ __forceinline__ Unit get(int64_t t) const {
        const int64_t per_group = (int64_t)GROUP_M * n_nb;
        const int64_t g = t / per_group;
        const int64_t r = t - g * per_group;
        const int64_t m0 = g * GROUP_M;
        const int64_t gm = (n_mp - m0) < GROUP_M ? (n_mp - m0) : GROUP_M;
        const int64_t nb = (r / gm) * nb_stride;
        return {m0 + r % gm, nb, nb + 1};
    }
    // Cursor: each CTA walks t = cid, cid + ncl, ... incrementally (no 64-bit divisions
    // per work item): group g, offset r inside it.
    struct Cur {
        int64_t t, g, r;
    };
    __device__ __forceinline__ Cur first(int64_t t) const {
        const int64_t g = t / ((int64_t)GROUP_M * n_nb);
        return {t, g, t - g * GROUP_M * n_nb};
    }
    __device__ __forceinline__ bool valid(const Cur& c) const { return c.t < units(); }
    __device__ __forceinline__ void next(Cur& c, int64_t step) const {
        c.t += step;
        c.r += step;
        while (c.g * GROUP_M < n_mp) {
            const int64_t rem = n_mp - c.g * GROUP_M;
            const int64_t pg = (rem < GROUP_M ? rem : GROUP_M) * n_nb;
            if (c.r < pg) break;
            c.r -= pg;
            ++c.g;
        }
    }
    __device__ __forceinline__ Unit unit(const Cur& c) const {
        const int64_t m0 = c.g * GROUP_M;
        const uint32_t gm = (uint32_t)((n_mp - m0) < GROUP_M ? (n_mp - m0) : GROUP_M);
        const uint32_t nb = (uint32_t)c.r / gm;
        const int64_t nbg = (int64_t)nb * nb_stride;
        return {m0 + ((uint32_t)c.r - nb * gm), nbg, nbg + 1};
    }
};

// Symmetric k-NNG (queries = corpus): the upper triangle of 256x256 pair blocks, nb >= mp;
// each block is also written transposed.  Unit order: gm == 0, row by row (consecutive
// units share the A panel); gm > 0, GROUP-MAJOR: groups of gm triangle rows [m0, m0+gm)
// sweep the column blocks nb >= m0, the rows of the group that reach nb taking column nb in
// turn, so every B block is used by up to gm row blocks while it is L2-resident (operand
// sets larger than L2: C4 / C5 re-read B from HBM for every triangle row otherwise).
struct SymSched {
    static constexpr bool kResidentA = false;
    int64_t n;  // pair blocks per side
    // units [u_lo, u_hi) of the triangle only (the multi-GPU symmetric k-NNG splits it)
    int64_t u_lo = 0, u_hi = INT64_MAX;
    int64_t gm = 0;  // rows per group (0: row-major; -1: COLUMN-major, unit u of column j =
                     // row block u - j(j+1)/2: the units of columns [0, J) are a prefix, so a
                     // caller can partition the triangle as the columns' points arrive)
    __device__ __forceinline__ int64_t units() const { return n * (n + 1) / 2; }
    __device__ __forceinline__ int64_t end() const { return u_hi < units() ? u_hi : units(); }
    // row m of the triangle starts at unit s(m) = m*n - m(m-1)/2: the largest m with
    // s(m) <= u is the smaller root of m^2 - (2n+1) m + 2u = 0, rounded down and corrected
    __device__ __forceinline__ int64_t start(int64_t m) const { return m * n - m * (m - 1) / 2; }
    __device__ __forceinline__ Unit get(int64_t u) const {
        const double bq = 2.0 * (double)n + 1.0;
        int64_t m = (int64_t)((bq - sqrt(bq * bq - 8.0 * (double)u)) * 0.5);
        m = m < 0 ? 0 : m > n - 1 ? n - 1 : m;
        while (m > 0 && start(m) > u) --m;
        while (m < n - 1 && start(m + 1) <= u) ++m;
        const int64_t nb = m + (u - start(m));
        return {m, nb, nb + 1};
    }
    // group g: rows [g gm, min(n, g gm + gm)); its units: the triangle part (columns below
    // the group's last row) then gr units per column
    __device__ __forceinline__ int64_t gsize(int64_t g) const {
        const int64_t m0 = g * gm, gr = (n - m0) < gm ? (n - m0) : gm;
        return gr * (gr - 1) / 2 + (n - (m0 + gr - 1)) * gr;
    }
    // Cursor: row-major (m, o) or group-major (g, o = unit index inside the group, sz)
    struct Cur {
        int64_t t, m, o, sz;
    };
    __device__ __forceinline__ Cur first(int64_t t) const {
        t += u_lo;
        if (t >= end()) return {t, n, 0, 0};
        if (gm < 0) {  // column j: the largest j with j (j + 1) / 2 <= t
            int64_t j = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
            while (j > 0 && j * (j + 1) / 2 > t) --j;
            while ((j + 1) * (j + 2) / 2 <= t) ++j;
            return {t, j, t - j * (j + 1) / 2, 0};
        }
        if (gm > 0) {
            int64_t g = 0, o = t, sz = gsize(0);
            while (o >= sz) {
                o -= sz;
                sz = gsize(++g);
            }
            return {t, g, o, sz};
        }
        const Unit w = get(t);
        return {t, w.mp, w.nb0 - w.mp, 0};
    }
    __device__ __forceinline__ bool valid(const Cur& c) const { return c.t < end(); }
    __device__ __forceinline__ void next(Cur& c, int64_t step) const {
        c.t += step;
        c.o += step;
        if (gm < 0) {
            while (c.t < end() && c.o > c.m) {
                c.o -= c.m + 1;
                ++c.m;
            }
            return;
        }
        if (gm > 0) {
            while (c.t < end() && c.o >= c.sz) {
                c.o -= c.sz;
                c.sz = gsize(++c.m);
            }
            return;
        }
        while (c.m < n && c.o >= n - c.m) {
            c.o -= n - c.m;
            ++c.m;
        }
    }
    __device__ __forceinline__ Unit unit(const Cur& c) const {
        if (gm < 0) return {c.o, c.m, c.m + 1};  // (row block o, column block m), o <= m
        if (gm > 0) {
            const int64_t m0 = c.m * gm, gr = (n - m0) < gm ? (n - m0) : gm;
            const int64_t tri = gr * (gr - 1) / 2;
            int64_t nb, m;
            if (c.o < tri) {  // column m0 + a holds rows m0 .. m0 + a
                int64_t a = 0;
                while ((a + 1) * (a + 2) / 2 <= c.o) ++a;
                nb = m0 + a;
                m = m0 + (c.o - a * (a + 1) / 2);
            } else {
                const int64_t v = c.o - tri;
                nb = m0 + gr - 1 + v / gr;
                m = m0 + v % gr;
            }
            return {m, nb, nb + 1};
        }
        return {c.m, c.m + c.o, c.m + c.o + 1};
    }
};

// Fused GEMM+select: a unit is a row-block pair against one of S column splits; units of
// the same split are consecutive so concurrent clusters sweep the same B panel.
struct SplitSched {
    static constexpr bool kResidentA = false;
    int64_t n_mp, n_nb, S, per;  // per = column blocks per split
    __device__ __forceinline__ int64_t units() const { return n_mp * S; }
    __device__ __forceinline__ Unit get(int64_t u) const {
        const int64_t s = u / n_mp;
        const int64_t nb0 = s * per;
        const int64_t nb1 = nb0 + per < n_nb ? nb0 + per : n_nb;
        return {u % n_mp, nb0, nb1};
    }
    struct Cur {
        int64_t t;
    };
    __device__ __forceinline__ Cur first(int64_t t) const { return {t}; }
    __device__ __forceinline__ bool valid(const Cur& c) const { return c.t < units(); }
    __device__ __forceinline__ void next(Cur& c, int64_t step) const { c.t += step; }
    __device__ __forceinline__ Unit unit(const Cur& c) const { return get(c.t); }
};

// A-panel-resident GEMM (the single-product sample pass, d_pad <= 256): a unit is a row-block
// pair against a RUN of `run` consecutive column blocks; each CTA loads its 128-row A panel
// (all of K) once per unit into one of two panel buffers and streams only the B tiles, so
// the operand traffic from L2 per tile halves (A was re-read for every tile).  Units are
// mp-major: consecutive units (concurrent clusters) cover a few row-block pairs and every run.
struct PanelSched {
    static constexpr bool kResidentA = true;
    int64_t n_mp, n_nb, run;  // (column blocks are matrix blocks: no sampling stride)
    __device__ __forceinline__ int64_t nruns() const { return (n_nb + run - 1) / run; }
    __device__ __forceinline__ int64_t units() const { return n_mp * nruns(); }
    struct Cur {
        int64_t t;
    };
    __device__ __forceinline__ Cur first(int64_t t) const { return {t}; }
    __device__ __forceinline__ bool valid(const Cur& c) const { return c.t < units(); }
    __device__ __forceinline__ void next(Cur& c, int64_t step) const { c.t += step; }
    __device__ __forceinline__ Unit unit(const Cur& c) const {
        const int64_t nr = nruns();
        const int64_t mp = c.t / nr, r = c.t - mp * nr;
        const int64_t nb0 = r * run, nb1 = nb0 + run < n_nb ? nb0 + run : n_nb;
        return {mp, nb0, nb1};
    }
};

// ------------------------------------------------------------------ orientation -------
// Canonical orientation: the value of pair (query i, corpus j) is always
// computed with the LOWER point index as the first split operand, so that when queries
// and corpus are one point set (j == i + shift is the self pair) D[i][j] and D[j][i] are
// the same bits in every plan.  Segment order O1 = (ql.xh, qh.xl, qh.xh) for i+shift < j,
// O2 = (qh.xl, ql.xh, qh.xh) for i+shift > j (the same products in the transposed order).
// A 256x256 pair block straddling the diagonal is computed twice, O1 keeping only
// i+shift <= j and O2 keeping only i+shift > j.
enum { TILE_ABOVE = 0, TILE_BELOW = 1, TILE_MIXED = 2 };
__device__ __forceinline__ int tile_class(int64_t mp, int64_t nb, int64_t shift) {
    if (shift == INT64_MIN) return TILE_ABOVE;
    const int64_t r_lo = 2 * BM * mp + shift, r_hi = r_lo + 2 * BM - 1;  // shifted row range
    const int64_t c_lo = nb * BN, c_hi = c_lo + BN - 1;
    if (r_hi < c_lo) return TILE_ABOVE;
    if (r_lo > c_hi) return TILE_BELOW;
    return TILE_MIXED;
}
__device__ __forceinline__ int tile_passes(int cls) { return cls == TILE_MIXED ? 2 : 1; }
__device__ __forceinline__ int tile_orient(int cls, int pass) { return cls == TILE_MIXED ? pass : cls; }
// 0: keep all; 1: keep i+shift <= j (O1 pass of a mixed block); 2: keep i+shift > j
__device__ __forceinline__ int tile_mask(int cls, int pass) {
    return cls == TILE_MIXED ? 1 + pass : 0;
}

// ------------------------------------------------------------------ mainloop ---------
// Barriers: full[s] (1 arrival + tx bytes), empty[s] (CLUSTER arrivals: both CTAs' MMAs),
// tfull[2] (MMA commit), tempty[2] (one arrival per epilogue warp).
struct Bars {
    uint32_t full0, empty0, tfull0, tempty0;
};

// TMA producer (one elected thread): per K-block, the CTA's own qh/ql rows and its half of
// the xh/xl rows multicast to both CTAs of the pair.  NSEG = 1 (the single hi.hi product of
// the approximate pivot sample pass) loads only qh and xh: stage = [qh | xh].
template <int NSEG>
constexpr int stage_bytes() { return NSEG == 3 ? STAGE_BYTES : A_BYTES + B_TILE; }
template <int NSEG>
constexpr int ring_stages() { return RING_BYTES / stage_bytes<NSEG>(); }
template <int STAGES, class Sched, int NSEG = 3>
__device__ __forceinline__ void producer_loop(const CUtensorMap* map_qh, const CUtensorMap* map_ql,
                                              const CUtensorMap* map_xh, const CUtensorMap* map_xl,
                                              uint8_t* stage_base, const Bars& b, const Sched& sched,
                                              int num_kb, uint32_t crank, int64_t cid, int64_t ncl,
                                              int64_t shift) {
    int stage = 0;
    uint32_t phase = 0;
    for (auto cur = sched.first(cid); sched.valid(cur); sched.next(cur, ncl)) {
        const Unit w = sched.unit(cur);
        const int row_a = (int)((2 * w.mp + crank) * BM);
        for (int64_t nb = w.nb0; nb < w.nb1; ++nb)
        for (int pass = 0; pass < tile_passes(tile_class(w.mp, nb, shift)); ++pass) {
            const int row_b = (int)(nb * BN + crank * (BN / 2));  // this CTA's half of B
            for (int kb = 0; kb < num_kb; ++kb) {
                mbar_wait(b.empty0 + 8 * stage, phase ^ 1);
                const uint32_t fb = b.full0 + 8 * stage;
                const uint32_t sb = smem_u32(stage_base + (size_t)stage * stage_bytes<NSEG>());
                if constexpr (CTA2) {
                    // own A rows and own B half into own shared memory, completion counted on
                    // the leader's barrier (the leader expects both CTAs' bytes)
                    if (crank == 0) mbar_expect_tx(fb, 2 * stage_bytes<NSEG>());
                    const uint32_t fl = leader_addr(fb);
                    if (NSEG == 3) {
                        tma_load_2d_2sm(sb, map_qh, fl, kb * BK, row_a);
                        tma_load_2d_2sm(sb + A_BYTES, map_ql, fl, kb * BK, row_a);
                        tma_load_2d_2sm(sb + 2 * A_BYTES, map_xh, fl, kb * BK, row_b);
                        tma_load_2d_2sm(sb + 2 * A_BYTES + B_TILE, map_xl, fl, kb * BK, row_b);
                    } else {
                        tma_load_2d_2sm(sb, map_qh, fl, kb * BK, row_a);
                        tma_load_2d_2sm(sb + A_BYTES, map_xh, fl, kb * BK, row_b);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                    continue;
                }
                mbar_expect_tx(fb, stage_bytes<NSEG>());
                const uint32_t boff = crank * (B_BYTES / 2);
                if (NSEG == 3) {
                    tma_load_2d(sb, map_qh, fb, kb * BK, row_a);
                    tma_load_2d(sb + A_BYTES, map_ql, fb, kb * BK, row_a);
                    tma_load_2d_mc(sb + 2 * A_BYTES + boff, map_xh, fb, kb * BK, row_b, 0x3);
                    tma_load_2d_mc(sb + 2 * A_BYTES + B_BYTES + boff, map_xl, fb, kb * BK, row_b, 0x3);
                } else {
                    tma_load_2d(sb, map_qh, fb, kb * BK, row_a);
                    tma_load_2d_mc(sb + A_BYTES + boff, map_xh, fb, kb * BK, row_b, 0x3);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    }
}

// Single-thread MMA issuer: per tile, waits for a free TMEM accumulator, then per K-block
// issues the three split segments (ql.xh, qh.xl, qh.xh; smallest first) and frees the
// stage in both CTAs; finally signals the epilogue.
template <int STAGES, class Sched, int NSEG = 3>
__device__ __forceinline__ void mma_loop(uint8_t* stage_base, const Bars& b, const Sched& sched,
                                         int num_kb, uint32_t tmem_base, int64_t cid, int64_t ncl,
                                         int64_t shift) {
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (auto cur = sched.first(cid); sched.valid(cur); sched.next(cur, ncl)) {
        const Unit w = sched.unit(cur);
        for (int64_t nb = w.nb0; nb < w.nb1; ++nb)
        for (int pass = 0, cls = tile_class(w.mp, nb, shift); pass < tile_passes(cls); ++pass, ++it) {
            const bool o2 = tile_orient(cls, pass) == TILE_BELOW;
            const int buf = it & 1;
            const uint32_t tphase = (it >> 1) & 1;
            mbar_wait(b.tempty0 + 8 * buf, tphase ^ 1);
            tc_fence_after();
            const uint32_t tmem_d = tmem_base + buf * BN;
            for (int kb = 0; kb < num_kb; ++kb) {
                mbar_wait(b.full0 + 8 * stage, phase);
                tc_fence_after();
                const uint32_t sb = smem_u32(stage_base + (size_t)stage * stage_bytes<NSEG>());
                const uint32_t qh = sb, ql = sb + A_BYTES, xh = sb + (NSEG == 3 ? 2 * A_BYTES : A_BYTES),
                               xl = sb + 2 * A_BYTES + B_TILE;
                // O1: ql.xh, qh.xl, qh.xh   O2: qh.xl, ql.xh, qh.xh  (smallest terms first);
                // NSEG = 1: qh.xh only
                const uint32_t sa[3] = {NSEG == 1 ? qh : o2 ? qh : ql, o2 ? ql : qh, qh};
                const uint32_t sbx[3] = {NSEG == 1 ? xh : o2 ? xl : xh, o2 ? xh : xl, xh};
                #pragma unroll
                for (int seg = 0; seg < NSEG; ++seg) {
                    #pragma unroll
                    for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                        const uint32_t acc = (kb | seg | kk) != 0;
                        if constexpr (CTA2)
                            tc_mma2(tmem_d, sdesc(sa[seg] + kk * UMMA_K * 2), sdesc(sbx[seg] + kk * UMMA_K * 2), acc);
                        else
                            tc_mma(tmem_d, sdesc(sa[seg] + kk * UMMA_K * 2), sdesc(sbx[seg] + kk * UMMA_K * 2),
                                   acc);
                    }
                }
                if constexpr (CTA2)
                    tc_commit2_mc(b.empty0 + 8 * stage);  // stage free in both CTAs
                else
                    tc_commit_mc(b.empty0 + 8 * stage, 0x3);  // stage free in both CTAs
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if constexpr (CTA2)
                tc_commit2_mc(b.tfull0 + 8 * buf);  // both CTAs' accumulators ready
            else
                tc_commit(b.tfull0 + 8 * buf);  // accumulator ready for the epilogue
        }
    }
}

// A-resident mainloop (PanelSched, single product qh.xh): per unit the CTA's A panel
// (num_kb tiles of BM x BK) lands in panel buffer (unit & 1) on afull[buf]; B tiles stream
// through a KB-stage ring (the B halves multicast to both CTAs, as above).  The MMA warp
// releases a panel buffer by committing aempty[buf] after the unit's last MMA.
template <int KB, class Sched>
__device__ __forceinline__ void producer_loop_ares(const CUtensorMap* map_qh, const CUtensorMap* map_xh,
                                                   uint8_t* abase, uint8_t* bbase, const Bars& b,
                                                   uint32_t afull0, uint32_t aempty0, const Sched& sched,
                                                   int num_kb, uint32_t crank, int64_t cid, int64_t ncl) {
    int stage = 0;
    uint32_t phase = 0;
    int ui = 0;
    for (auto cur = sched.first(cid); sched.valid(cur); sched.next(cur, ncl), ++ui) {
        const Unit w = sched.unit(cur);
        const int row_a = (int)((2 * w.mp + crank) * BM);
        const int ab = ui & 1;
        mbar_wait(aempty0 + 8 * ab, ((ui >> 1) & 1) ^ 1);
        const uint32_t pa = smem_u32(abase + (size_t)ab * num_kb * A_BYTES);
        if constexpr (CTA2) {
            if (crank == 0) mbar_expect_tx(afull0 + 8 * ab, (uint32_t)(2 * num_kb * A_BYTES));
            for (int kb = 0; kb < num_kb; ++kb)
                tma_load_2d_2sm(pa + kb * A_BYTES, map_qh, leader_addr(afull0 + 8 * ab), kb * BK, row_a);
        } else {
            mbar_expect_tx(afull0 + 8 * ab, (uint32_t)(num_kb * A_BYTES));
            for (int kb = 0; kb < num_kb; ++kb)
                tma_load_2d(pa + kb * A_BYTES, map_qh, afull0 + 8 * ab, kb * BK, row_a);
        }
        for (int64_t nb = w.nb0; nb < w.nb1; ++nb) {
            const int row_b = (int)(nb * BN + crank * (BN / 2));
            for (int kb = 0; kb < num_kb; ++kb) {
                mbar_wait(b.empty0 + 8 * stage, phase ^ 1);
                const uint32_t fb = b.full0 + 8 * stage;
                if constexpr (CTA2) {
                    if (crank == 0) mbar_expect_tx(fb, 2 * B_TILE);
                    tma_load_2d_2sm(smem_u32(bbase + (size_t)stage * B_TILE), map_xh, leader_addr(fb), kb * BK, row_b);
                } else {
                    mbar_expect_tx(fb, B_BYTES);
                    tma_load_2d_mc(smem_u32(bbase + (size_t)stage * B_BYTES) + crank * (B_BYTES / 2), map_xh, fb,
                                   kb * BK, row_b, 0x3);
                }
                if (++stage == KB) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    }
}
template <int KB, class Sched>
__device__ __forceinline__ void mma_loop_ares(uint8_t* abase, uint8_t* bbase, const Bars& b, uint32_t afull0,
                                              uint32_t aempty0, const Sched& sched, int num_kb, uint32_t tmem_base,
                                              int64_t cid, int64_t ncl) {
    int stage = 0;
    uint32_t phase = 0;
    int it = 0, ui = 0;
    for (auto cur = sched.first(cid); sched.valid(cur); sched.next(cur, ncl), ++ui) {
        const Unit w = sched.unit(cur);
        const int ab = ui & 1;
        mbar_wait(afull0 + 8 * ab, (ui >> 1) & 1);
        tc_fence_after();
        const uint32_t pa = smem_u32(abase + (size_t)ab * num_kb * A_BYTES);
        for (int64_t nb = w.nb0; nb < w.nb1; ++nb, ++it) {
            const int buf = it & 1;
            mbar_wait(b.tempty0 + 8 * buf, ((it >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t tmem_d = tmem_base + buf * BN;
            for (int kb = 0; kb < num_kb; ++kb) {
                mbar_wait(b.full0 + 8 * stage, phase);
                tc_fence_after();
                const uint32_t sa = pa + kb * A_BYTES;
                const uint32_t sb = smem_u32(bbase + (size_t)stage * B_TILE);
                #pragma unroll
                for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                    if constexpr (CTA2)
                        tc_mma2(tmem_d, sdesc(sa + kk * UMMA_K * 2), sdesc(sb + kk * UMMA_K * 2), (kb | kk) != 0);
                    else
                        tc_mma(tmem_d, sdesc(sa + kk * UMMA_K * 2), sdesc(sb + kk * UMMA_K * 2), (kb | kk) != 0);
                }
                if constexpr (CTA2)
                    tc_commit2_mc(b.empty0 + 8 * stage);
                else
                    tc_commit_mc(b.empty0 + 8 * stage, 0x3);  // stage free in both CTAs
                if (++stage == KB) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if constexpr (CTA2)
                tc_commit2_mc(b.tfull0 + 8 * buf);
            else
                tc_commit(b.tfull0 + 8 * buf);  // accumulator ready for the epilogue
        }
        if constexpr (CTA2)
            tc_commit2_mc(aempty0 + 8 * ab);  // the unit's MMAs done: both panel buffers free
        else
            tc_commit(aempty0 + 8 * ab);  // the unit's MMAs done: panel buffer free
    }
}

// Barrier init (one thread), TMEM allocation (warp 1), cluster-wide sync.
__device__ __forceinline__ uint32_t setup(uint64_t* bars, int stages, int epi_warps,
                                         uint32_t* tmem_slot, const CUtensorMap* maps, int nmaps) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + stages);
    const uint32_t tfull0 = smem_u32(bars + 2 * stages), tempty0 = smem_u32(bars + 2 * stages + 2);
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(full0 + 8 * s, 1);
            // CTA2: the leader's MMA commit releases the stage in both CTAs; else both CTAs'
            // own MMAs must release it (the B halves are multicast)
            mbar_init(empty0 + 8 * s, CTA2 ? 1 : CLUSTER);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull0 + 8 * b, 1);
            // one arrive per epilogue warp (CTA2: of both CTAs, on the leader's barrier)
            mbar_init(tempty0 + 8 * b, CTA2 ? 2 * epi_warps : epi_warps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < nmaps; ++i)
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(maps + i)));
    }
    if (warp == 1) {
        if constexpr (CTA2) {  // the same columns in both CTAs (warp 1 of each)
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    cluster_sync_all();  // barriers of both CTAs initialised before any multicast
    tc_fence_after();
    return *tmem_slot;
}

__device__ __forceinline__ void teardown(uint32_t tmem_base) {
    tc_fence_before();
    cluster_sync_all();  // no CTA leaves while its peer may still multicast into it
    if ((threadIdx.x >> 5) == 1) {
        tc_fence_after();
        if constexpr (CTA2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(TMEM_COLS));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(TMEM_COLS));
    }
}

}  // namespace tc

// host helpers (gemm_tc.cu)
bool tc_make_operand_map(CUtensorMap* m, const __half* base, int64_t rows, int32_t d_pad, int box_rows);
bool tc_make_output_map(CUtensorMap* m, float* D, int64_t rows, int64_t N, int64_t ldD);

}  // namespace knn
