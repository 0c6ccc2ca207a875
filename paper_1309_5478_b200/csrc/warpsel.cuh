// warpsel.cuh — warp-synchronous exact selection primitives shared by the select and
// fused kernels: radix passes on order-preserving key bits (then on the index among equal
// keys), exact k-selection with ballot/popc compaction, and a register bitonic sort.
#pragma once
#include "internal.cuh"

namespace knn {
namespace ws {

constexpr uint32_t FULL = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Warp radix pass: histogram of digit `shift` (of key, or of idx among key == key_eq)
// over cnt warp-private candidates; returns the bin holding the rank-th value and the
// counts below / in it (warp-uniform).
template <int STRIDE>
__device__ __forceinline__ void warp_radix_pass(const uint32_t* ckey, const uint32_t* cidx, int cnt,
                                                bool on_idx, uint32_t key_eq, uint32_t prefix,
                                                uint32_t mask, int shift, uint32_t rank,
                                                uint32_t* hist, uint32_t& bin, uint32_t& before,
                                                uint32_t& neq) {
    const int lane = threadIdx.x & 31;
    #pragma unroll
    for (int i = 0; i < 8; ++i) hist[lane + 32 * i] = 0;
    __syncwarp();
    for (int i = lane; i < cnt; i += 32) {
        const uint32_t key = ckey[i * STRIDE];
        const uint32_t v = on_idx ? cidx[i * STRIDE] : key;
        const bool ok = on_idx ? (key == key_eq) : true;
        if (ok && (v & mask) == prefix) atomicAdd(&hist[(v >> shift) & 255u], 1u);
    }
    __syncwarp();
    uint32_t c[8], sum = 0;
    #pragma unroll
    for (int j = 0; j < 8; ++j) {
        c[j] = hist[lane * 8 + j];
        sum += c[j];
    }
    uint32_t incl = sum;
    #pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += n;
    }
    const uint32_t excl = incl - sum;
    const uint32_t hit = __ballot_sync(FULL, excl < rank && rank <= incl);
    const int src = __ffs(hit) - 1;
    uint32_t b = 0, bef = 0, eq = 0;
    if (lane == src) {
        uint32_t run = excl;
        bool found = false;
        #pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (!found && run + c[j] >= rank) {
                b = lane * 8 + j;
                bef = run;
                eq = c[j];
                found = true;
            }
            if (!found) run += c[j];
        }
    }
    bin = __shfl_sync(FULL, b, src);
    before = __shfl_sync(FULL, bef, src);
    neq = __shfl_sync(FULL, eq, src);
    __syncwarp();
}

// Keep exactly the k best (key, idx) of cnt >= k warp-private candidates, compacted into
// okey/oidx[0, k); returns the key of the k-th best.  The radix passes start below the
// key bits all candidates share (warp AND/OR reduction), so the first digit is not the
// degenerate one of a narrow value range.
// Candidates are ckey[i*STRIDE], cidx[i*STRIDE]; the k kept go to okey/oidx[0, k).
template <int STRIDE>
__device__ __noinline__ uint32_t warp_select_k(const uint32_t* ckey, const uint32_t* cidx, int cnt,
                                               int k, uint32_t* okey, uint32_t* oidx,
                                               uint32_t* hist) {
    const int lane = threadIdx.x & 31;
    uint32_t andv = 0xFFFFFFFFu, orv = 0;
    for (int i = lane; i < cnt; i += 32) {
        const uint32_t v = ckey[i * STRIDE];
        andv &= v;
        orv |= v;
    }
    andv = __reduce_and_sync(FULL, andv);
    orv = __reduce_or_sync(FULL, orv);
    const uint32_t diff = andv ^ orv;
    uint32_t rank = (uint32_t)k, neq = (uint32_t)cnt, bin, before;
    uint32_t prefix = andv, mask = 0xFFFFFFFFu;
    if (diff) {
        const int hb = 31 - __clz(diff);
        mask = hb == 31 ? 0u : ~((2u << hb) - 1u);
        prefix = andv & mask;
        for (int hi = hb; hi >= 0; hi -= 8) {
            const int shift = hi >= 7 ? hi - 7 : 0;
            warp_radix_pass<STRIDE>(ckey, cidx, cnt, false, 0, prefix, mask, shift, rank, hist, bin, before, neq);
            rank -= before;
            const uint32_t wmask = ((2u << (hi - shift)) - 1u) << shift;  // digit bits
            prefix |= (bin << shift) & wmask;
            mask |= wmask;
        }
    }
    const uint32_t Tkey = prefix;
    uint32_t Tidx = 0xFFFFFFFFu;
    if (neq > rank) {
        uint32_t p2 = 0, m2 = 0;
        for (int shift = 24; shift >= 0; shift -= 8) {
            warp_radix_pass<STRIDE>(ckey, cidx, cnt, true, Tkey, p2, m2, shift, rank, hist, bin, before, neq);
            rank -= before;
            p2 |= bin << shift;
            m2 |= 0xFFu << shift;
        }
        Tidx = p2;
    }
    int base = 0;
    for (int b = 0; b < cnt; b += 32) {
        const int i = b + lane;
        bool p = false;
        uint32_t kk = 0, ii = 0;
        if (i < cnt) {
            kk = ckey[i * STRIDE];
            ii = cidx[i * STRIDE];
            p = kk < Tkey || (kk == Tkey && ii <= Tidx);
        }
        const uint32_t m = __ballot_sync(FULL, p);
        if (p) {
            const int pos = base + __popc(m & lanemask_lt());
            if (pos < k) {  // (only repeated (key, idx) pairs, never produced, could pass k)
                okey[pos] = kk;
                oidx[pos] = ii;
            }
        }
        base += __popc(m);
    }
    __syncwarp();
    return Tkey;
}

// Bitonic sort of R*32 (key, idx) pairs held as 64-bit words, element e = r*32 + lane.
template <int R>
__device__ __forceinline__ void warp_bitonic(uint64_t (&v)[R]) {
    const int lane = threadIdx.x & 31;
    #pragma unroll
    for (int size = 2; size <= 32 * R; size <<= 1) {
        #pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32) {
                const int rs = stride / 32;
                #pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int rp = r ^ rs;
                    if (rp > r) {
                        const int e = r * 32 + lane;
                        const bool asc = (e & size) == 0;
                        const uint64_t a = v[r], b = v[rp];
                        const bool sw = asc ? (a > b) : (a < b);
                        v[r] = sw ? b : a;
                        v[rp] = sw ? a : b;
                    }
                }
            } else {
                #pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int e = r * 32 + lane;
                    const uint64_t o = __shfl_xor_sync(FULL, v[r], stride);
                    const bool asc = (e & size) == 0;
                    const bool lower = (lane & stride) == 0;
                    const bool take_min = (lower == asc);
                    v[r] = take_min ? (o < v[r] ? o : v[r]) : (o > v[r] ? o : v[r]);
                }
            }
        }
    }
}

template <int R>
__device__ __forceinline__ void warp_sort_write(const uint32_t* key, const uint32_t* idx, int k,
                                                int64_t idx_offset, int32_t* out_idx,
                                                float* out_dist) {
    const int lane = threadIdx.x & 31;
    uint64_t v[R];
    #pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = r * 32 + lane;
        v[r] = e < k ? ((uint64_t)key[e] << 32 | idx[e]) : ~0ull;
    }
    warp_bitonic<R>(v);
    #pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = r * 32 + lane;
        if (e < k) {
            out_idx[e] = (int32_t)((int64_t)(uint32_t)v[r] + idx_offset);
            out_dist[e] = ukey_to_float((uint32_t)(v[r] >> 32));
        }
    }
}

// Fold up to 32 candidates into a sorted best-32 list.  L is this lane's entry of the
// list (64-bit key << 32 | idx, ascending over lanes; padding = ~0).  The candidates are
// ckey/cidx[i * STRIDE], i < n <= 32.  They are bitonic-sorted across the warp; the
// element-wise minimum of L and the reversed sorted candidates holds the 32 smallest of
// the union as a bitonic sequence, which a half-cleaner cascade sorts.  Returns the new
// entry of this lane.  ~25 warp-instructions per network stage, 21 stages.
template <int STRIDE>
__device__ __forceinline__ uint64_t warp_merge32(uint64_t L, const uint32_t* ckey, const uint32_t* cidx,
                                                 int n) {
    const int lane = threadIdx.x & 31;
    uint64_t b[1] = {lane < n ? ((uint64_t)ckey[lane * STRIDE] << 32 | cidx[lane * STRIDE]) : ~0ull};
    warp_bitonic<1>(b);
    const uint64_t br = __shfl_sync(FULL, b[0], 31 - lane);
    uint64_t c = L < br ? L : br;
    #pragma unroll
    for (int stride = 16; stride > 0; stride >>= 1) {
        const uint64_t o = __shfl_xor_sync(FULL, c, stride);
        c = (lane & stride) ? (o > c ? o : c) : (o < c ? o : c);
    }
    return c;
}

}  // namespace ws
}  // namespace knn
