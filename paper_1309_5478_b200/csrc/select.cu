// select.cu — a-S4 (per-row k-select on the materialised matrix) and a-S6 (k-way merge).
//
// Paper ("GPU-based quick multi-select"): each row is partitioned
// around a pivot; a warp reads 32 coalesced elements, `__ballot(p)` gives the vote word
// B, every lane finds its slot from `__popc` of the vote bits of the lanes before it,
// elements are staged in a shared-memory array and written out with coalesced writes;
// a block-per-row variant adds an inter-warp prefix; the partition recurses
// into the side that holds the k-th element.
//
// Blackwell redesign: the recursion's repeated global read/write
// passes are what bound the paper's kernel; on B200 the row is read from HBM ONCE.
//   * CTA per row streams the row with 128-bit loads, one chunk ahead in registers.
//   * Every element is compared with a running threshold T = the key of the current
//     k-th best; the "< pivot" side of the paper's partition is the accepted side.
//   * Survivors are compacted with the paper's primitive — ballot, popc of the lower
//     lanes' bits, one warp-aggregated shared counter — into a shared-memory candidate
//     buffer (the staging array that grows instead of flushing to global memory).
//   * When the buffer could overflow, an exact in-shared-memory radix select (8-bit
//     digits on order-preserving key bits, then on the index among equal keys) keeps
//     exactly the k best (key, index) pairs and lowers T: the "recurse into the side
//     holding the k-th element" of PAPER.md:56, done on the candidates only.
//   * Finally the k survivors are bitonic-sorted by (key, index) and written.
// Ties: the order is (value, index) (reading R1).  In a row, chunks arrive in index
// order, so an element equal to T has a larger index than the current k-th and is
// correctly rejected by the strict "< T" test.  The merge sees lists in arbitrary index
// order and uses the composite test (key, index) < (T, T_idx).
#include "internal.cuh"
#include "ptx.cuh"
#include "warpsel.cuh"

#include <climits>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cooperative_groups.h>
#include <cmath>

#define KNN_CUDA_TRY(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) return e_; } while (0)

namespace knn {
namespace {

constexpr uint32_t FULL = 0xFFFFFFFFu;

struct Scal {
    uint32_t bin, before, neq;
    int kept;
    uint32_t lo, hi;
};

// Barrier over the THREADS consumer threads 0..THREADS-1 of the CTA (named barrier 1), so
// that a producer warp outside them never takes part.
template <int THREADS>
__device__ __forceinline__ void csync() {
    named_bar(1, THREADS);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Warp 0 (threads 0..31) scans a 256-bin histogram and records the bin holding the
// rank-th (1-based) counted value in sc->{bin, before (count in lower bins), neq}.
__device__ __forceinline__ void hist_find(const uint32_t* hist, uint32_t rank, Scal* sc) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        uint32_t c[8], sum = 0;
        #pragma unroll
        for (int j = 0; j < 8; ++j) {
            c[j] = hist[lane * 8 + j];
            sum += c[j];
        }
        uint32_t incl = sum;
        #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t n = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += n;
        }
        uint32_t run = incl - sum;
        if (run < rank && rank <= incl) {
            #pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (run + c[j] >= rank) {
                    sc->bin = lane * 8 + j;
                    sc->before = run;
                    sc->neq = c[j];
                    break;
                }
                run += c[j];
            }
        }
    }
}

// Block-wide min and max of the keys ckey[0, cnt) (cnt >= 1), via sc->{lo, hi}.
template <int THREADS>
__device__ __forceinline__ void block_key_range(const uint32_t* ckey, int cnt, Scal* sc,
                                                uint32_t& mn, uint32_t& mx) {
    uint32_t a = 0xFFFFFFFFu, b = 0;
    for (int i = threadIdx.x; i < cnt; i += THREADS) {
        const uint32_t v = ckey[i];
        a = min(a, v);
        b = max(b, v);
    }
    a = __reduce_min_sync(FULL, a);
    b = __reduce_max_sync(FULL, b);
    if (threadIdx.x == 0) {
        sc->lo = 0xFFFFFFFFu;
        sc->hi = 0;
    }
    csync<THREADS>();
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&sc->lo, a);
        atomicMax(&sc->hi, b);
    }
    csync<THREADS>();
    mn = sc->lo;
    mx = sc->hi;
}

// The shift of the first 8-bit digit that can separate keys in [mn, mx]: the digit just
// below their common prefix (0 if they differ only in the low 8 bits or are equal).
__device__ __forceinline__ int top_digit_shift(uint32_t mn, uint32_t mx) {
    const uint32_t diff = mn ^ mx;
    const int msb = diff ? 31 - __clz(diff) : 0;
    return msb > 7 ? msb - 7 : 0;
}

// One 8-bit radix-histogram pass over the candidates.  Counts digit `shift` of the key
// (on_idx = false) or of the index among candidates whose key == key_eq (on_idx = true),
// restricted to values v with (v & mask) == prefix; finds the bin holding the rank-th
// (1-based) value.  Result in sc->{bin, before (count in lower bins), neq (count in bin)}.
template <int THREADS>
__device__ void radix_pass(const uint32_t* ckey, const uint32_t* cidx, int cnt, bool on_idx,
                           uint32_t key_eq, uint32_t prefix, uint32_t mask, int shift,
                           uint32_t rank, uint32_t* hist, Scal* sc) {
    const int tid = threadIdx.x;
    for (int i = tid; i < 256; i += THREADS) hist[i] = 0;
    csync<THREADS>();
    for (int i = tid; i < cnt; i += THREADS) {
        uint32_t key = ckey[i];
        uint32_t v = on_idx ? cidx[i] : key;
        bool ok = on_idx ? (key == key_eq) : true;
        if (ok && (v & mask) == prefix) atomicAdd(&hist[(v >> shift) & 255u], 1u);
    }
    csync<THREADS>();
    hist_find(hist, rank, sc);
    csync<THREADS>();
}

// Exact selection of the k best (key, idx) among cnt >= k candidates.  Writes them
// (unordered) to kkey/kidx[0, k) and returns the k-th best pair in (Tkey, Tidx).
// exact_idx: compute Tidx even when every candidate equal to Tkey is kept (needed by
// the composite threshold of the merge); otherwise Tidx = UINT_MAX in that case.
template <int THREADS>
__device__ void block_select_k(const uint32_t* ckey, const uint32_t* cidx, int cnt, int k,
                               uint32_t* kkey, uint32_t* kidx, uint32_t* hist, Scal* sc,
                               bool exact_idx, uint32_t& Tkey, uint32_t& Tidx) {
    // digits start just below the common prefix of the candidates' key range; a digit
    // may overlap bits already fixed by the prefix (their bins are then constant)
    uint32_t mn, mx;
    block_key_range<THREADS>(ckey, cnt, sc, mn, mx);
    const int top = top_digit_shift(mn, mx);
    uint32_t mask = top + 8 >= 32 ? 0u : ~((1u << (top + 8)) - 1u);
    uint32_t prefix = mn & mask, rank = (uint32_t)k, neq = 0;
    for (int shift = top;; shift = shift > 8 ? shift - 8 : 0) {
        radix_pass<THREADS>(ckey, cidx, cnt, false, 0, prefix, mask, shift, rank, hist, sc);
        rank -= sc->before;
        prefix = (prefix & ~(0xFFu << shift)) | (sc->bin << shift);
        mask |= 0xFFu << shift;
        neq = sc->neq;
        if (shift == 0) break;
    }
    Tkey = prefix;
    Tidx = 0xFFFFFFFFu;
    if (neq > rank || exact_idx) {
        uint32_t p2 = 0, m2 = 0;
        for (int shift = 24; shift >= 0; shift -= 8) {
            radix_pass<THREADS>(ckey, cidx, cnt, true, Tkey, p2, m2, shift, rank, hist, sc);
            rank -= sc->before;
            p2 |= sc->bin << shift;
            m2 |= 0xFFu << shift;
        }
        Tidx = p2;
    }
    // Compaction of the kept side with the paper's ballot/popc primitive.
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) sc->kept = 0;
    csync<THREADS>();
    for (int b = warp * 32; b < cnt; b += THREADS) {
        int i = b + lane;
        bool p = false;
        uint32_t kk = 0, ii = 0;
        if (i < cnt) {
            kk = ckey[i];
            ii = cidx[i];
            p = kk < Tkey || (kk == Tkey && ii <= Tidx);
        }
        uint32_t m = __ballot_sync(FULL, p);
        if (m) {
            int base = 0;
            if (lane == 0) base = atomicAdd(&sc->kept, __popc(m));
            base = __shfl_sync(FULL, base, 0);
            if (p) {
                int pos = base + __popc(m & lanemask_lt());
                kkey[pos] = kk;
                kidx[pos] = ii;
            }
        }
    }
    csync<THREADS>();
}

// Bitonic sort of KP (power of two) pairs by (key, idx) ascending.
template <int THREADS>
__device__ void block_bitonic(uint32_t* key, uint32_t* idx, int KP) {
    for (int size = 2; size <= KP; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < (KP >> 1); t += THREADS) {
                int i = 2 * t - (t & (stride - 1));
                int j = i + stride;
                uint32_t ki = key[i], kj = key[j], ii = idx[i], ij = idx[j];
                bool gt = ki > kj || (ki == kj && ii > ij);
                bool asc = (i & size) == 0;
                if (gt == asc) {
                    key[i] = kj; key[j] = ki;
                    idx[i] = ij; idx[j] = ii;
                }
            }
            csync<THREADS>();
        }
    }
}

// Register bitonic sort of KP = E * (KP / E threads) pairs by (key, idx), packed as
// u64 = key << 32 | idx (pairs are distinct), fully unrolled for the compile-time KP.
// Thread t holds positions t*E .. t*E+E-1: strides < E are exchanged in registers,
// strides < 32E with __shfl_xor across lanes, larger (cross-warp) strides through shared
// memory `tmp` (KP u64).  The first k positions are written to out_idx (idx + idx_offset)
// and out_dist (the key's float).
template <int THREADS, int KP, class Out>
__device__ void block_sort(const uint32_t* key, const uint32_t* idx, uint64_t* tmp, Out out) {
    constexpr int E = KP >= 4 * THREADS ? 4 : KP >= 2 * THREADS ? 2 : 1;
    static_assert(KP <= E * THREADS, "KP too large for the block");
    const int t = threadIdx.x;
    const bool act = t * E < KP;
    uint64_t v[E];
    #pragma unroll
    for (int e = 0; e < E; ++e)
        v[e] = act ? ((uint64_t)key[t * E + e] << 32 | idx[t * E + e]) : ~0ull;
    #pragma unroll
    for (int size = 2; size <= KP; size <<= 1) {
        #pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32 * E) {
                csync<THREADS>();
                if (act) {
                    #pragma unroll
                    for (int e = 0; e < E; ++e) tmp[t * E + e] = v[e];
                }
                csync<THREADS>();
                if (act) {
                    #pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const int p = t * E + e;
                        const uint64_t o = tmp[p ^ stride];
                        const bool up = ((p & size) == 0) == ((p & stride) == 0);  // keep min
                        v[e] = ((o < v[e]) == up) ? o : v[e];
                    }
                }
            } else if (stride >= E) {
                #pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int p = t * E + e;
                    const uint64_t o = __shfl_xor_sync(FULL, v[e], stride / E);
                    const bool up = ((p & size) == 0) == ((p & stride) == 0);
                    v[e] = ((o < v[e]) == up) ? o : v[e];
                }
            } else {
                #pragma unroll
                for (int e = 0; e < E; ++e) {
                    if (e & stride) continue;
                    const int f = e + stride;
                    const bool asc = ((t * E + e) & size) == 0;
                    const bool sw = (v[f] < v[e]) == asc;
                    const uint64_t x = v[e];
                    v[e] = sw ? v[f] : x;
                    v[f] = sw ? x : v[f];
                }
            }
        }
    }
    if (act) {
        #pragma unroll
        for (int e = 0; e < E; ++e) out(t * E + e, v[e]);
    }
}

// block_sort of KP (a power of two <= 4 THREADS) pairs; out(p, key << 32 | idx) per position.
template <int THREADS, class Out>
__device__ __forceinline__ void block_sort_kp(const uint32_t* key, const uint32_t* idx, int KP,
                                              uint64_t* tmp, Out out) {
    switch (KP) {
#define KNN_SORT_CASE(P) \
    case P: block_sort<THREADS, P>(key, idx, tmp, out); break;
        KNN_SORT_CASE(1) KNN_SORT_CASE(2) KNN_SORT_CASE(4) KNN_SORT_CASE(8) KNN_SORT_CASE(16)
        KNN_SORT_CASE(32) KNN_SORT_CASE(64) KNN_SORT_CASE(128) KNN_SORT_CASE(256)
        KNN_SORT_CASE(512) KNN_SORT_CASE(1024)
#undef KNN_SORT_CASE
        default: break;
    }
}

// The finishing steps shared by select and merge: exact k, sort, write.  `tmp` needs KP
// u64 of shared memory (the candidate buffer, free at this point, serves).
template <int THREADS>
__device__ void block_finish(uint32_t* ckey, uint32_t* cidx, int cnt, int k, int KP,
                             uint32_t* kkey, uint32_t* kidx, uint32_t* hist, Scal* sc,
                             int64_t idx_offset, int32_t* out_idx, float* out_dist) {
    if (cnt > k) {
        uint32_t tk, ti;
        block_select_k<THREADS>(ckey, cidx, cnt, k, kkey, kidx, hist, sc, false, tk, ti);
    } else {
        for (int i = threadIdx.x; i < cnt; i += THREADS) {
            kkey[i] = ckey[i];
            kidx[i] = cidx[i];
        }
    }
    for (int i = min(cnt, k) + threadIdx.x; i < KP; i += THREADS) {
        kkey[i] = 0xFFFFFFFFu;
        kidx[i] = 0xFFFFFFFFu;
    }
    csync<THREADS>();
    // ckey, cidx, kkey, kidx are contiguous (2 cap + 2 KP words, 8-byte aligned) and dead
    // once the sort holds its pairs in registers: KP u64 of scratch
    uint64_t* tmp = reinterpret_cast<uint64_t*>(ckey);
    block_sort_kp<THREADS>(kkey, kidx, KP, tmp, [&](int p, uint64_t v) {
        if (p < k) {
            out_idx[p] = (int32_t)((int64_t)(uint32_t)v + idx_offset);
            out_dist[p] = ukey_to_float((uint32_t)(v >> 32));
        }
    });
}

// Bucket finish for large k (the ring select, KP >= 64): instead of an exact radix select
// (3-4 histogram passes) plus a 55-stage bitonic sort, ONE BBINS-bucket histogram of the
// candidates' values over [min, max] gives, after an
// exclusive scan, every bucket's output offset (a counting sort: buckets are monotone in
// the key) and the bucket b* holding the k-th candidate.  Buckets are linear in the value.  Candidates of buckets < b* are
// scattered to their bucket's slots; b*'s few candidates are sorted by one warp and the
// first k - before of them appended; finally odd-even transposition passes order each
// bucket internally (pairs from different buckets are already in order, so plain passes
// over the whole array are correct; max-bucket-size passes suffice).  Returns false —
// before touching anything but `hist` and `sc` — when the buckets are too crowded (ties or
// a very concentrated key range): the caller then runs block_finish.
constexpr int BBITS = 10, BBINS = 1 << BBITS;
constexpr int BSTAR_MAX = 64;   // candidates in b* one warp sorts (2 per lane)
constexpr int BPASS_MAX = 16;   // odd-even passes (largest bucket below b*)
template <int THREADS, int NB = BBINS>
__device__ bool block_finish_bucket(const uint32_t* ckey, const uint32_t* cidx, int cnt, int k,
                                    uint32_t* kkey, uint32_t* kidx, uint32_t* hist, Scal* sc,
                                    int64_t idx_offset, int32_t* out_idx, float* out_dist) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = THREADS / 32;
    constexpr int BPT = NB / THREADS;  // bins per thread in the scan
    static_assert(BPT * THREADS == NB, "bins per thread");
    if (cnt <= k) return false;  // nothing to select: the plain finish is as cheap
    uint32_t mn, mx;
    block_key_range<THREADS>(ckey, cnt, sc, mn, mx);
    // buckets linear in the VALUE over [min, max] (monotone: a rounded subtraction, a
    // positive scale and floor are all monotone), so uniform keys and narrow distance
    // bands both spread; non-finite or degenerate ranges take the radix path
    const float fmn = ukey_to_float(mn), fmx = ukey_to_float(mx);
    const float span = fmx - fmn;
    const float scale = (float)NB / span;
    if (!(isfinite(fmn) && isfinite(fmx) && span > 0.0f && isfinite(span) && isfinite(scale))) return false;
    auto bucket = [&](uint32_t key) -> uint32_t {
        const float b = (ukey_to_float(key) - fmn) * scale;
        return min((uint32_t)b, (uint32_t)(NB - 1));
    };
    for (int i = tid; i < NB; i += THREADS) hist[i] = 0;
    csync<THREADS>();
    for (int i = tid; i < cnt; i += THREADS) atomicAdd(&hist[bucket(ckey[i])], 1u);
    csync<THREADS>();
    // exclusive scan of the bins; b* = bin holding rank k; largest bin below b*
    uint32_t c[BPT], tsum = 0;
    #pragma unroll
    for (int j = 0; j < BPT; ++j) {
        c[j] = hist[tid * BPT + j];
        tsum += c[j];
    }
    uint32_t incl = tsum;
    #pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    __shared__ uint32_t s_wsum[NW];
    if (lane == 31) s_wsum[warp] = incl;
    if (tid == 0) {
        sc->bin = 0xFFFFFFFFu;
        sc->kept = 0;
    }
    csync<THREADS>();
    uint32_t wbase = 0;
    #pragma unroll
    for (int w = 0; w < NW; ++w) wbase += w < warp ? s_wsum[w] : 0u;
    uint32_t run = wbase + incl - tsum;  // exclusive prefix of this thread's first bin
    uint32_t mymax = 0;
    #pragma unroll
    for (int j = 0; j < BPT; ++j) {
        const int b = tid * BPT + j;
        hist[b] = run;  // exclusive offset: the scatter's cursor
        if (run < (uint32_t)k && (uint32_t)k <= run + c[j]) {
            sc->bin = b;
            sc->before = run;
            sc->neq = c[j];
        }
        run += c[j];
    }
    csync<THREADS>();
    const uint32_t bstar = sc->bin, before = sc->before, nstar = sc->neq;
    #pragma unroll
    for (int j = 0; j < BPT; ++j)
        if ((uint32_t)(tid * BPT + j) < bstar) mymax = max(mymax, c[j]);
    mymax = __reduce_max_sync(FULL, mymax);
    if (lane == 0) atomicMax((uint32_t*)&sc->kept, mymax);
    csync<THREADS>();
    const uint32_t maxc = (uint32_t)sc->kept;
    if (nstar > BSTAR_MAX || maxc > BPASS_MAX) return false;  // crowded: exact radix path
    // scatter buckets < b* to their slots; b*'s candidates to a side list
    __shared__ uint64_t s_star[BSTAR_MAX];
    __shared__ int s_nstar;
    if (tid == 0) s_nstar = 0;
    csync<THREADS>();
    for (int i = tid; i < cnt; i += THREADS) {
        const uint32_t key = ckey[i];
        const uint32_t b = bucket(key);
        if (b < bstar) {
            const uint32_t pos = atomicAdd(&hist[b], 1u);
            kkey[pos] = key;
            kidx[pos] = cidx[i];
        } else if (b == bstar) {
            const int q = atomicAdd(&s_nstar, 1);
            s_star[q] = (uint64_t)key << 32 | cidx[i];
        }
    }
    csync<THREADS>();
    if (warp == 0) {
        // sort b*'s candidates (<= 64, 2 per lane) by (key, idx); append the first k - before
        uint64_t a0 = lane < (int)nstar ? s_star[lane] : ~0ull;
        uint64_t a1 = lane + 32 < (int)nstar ? s_star[lane + 32] : ~0ull;
        // bitonic over 64 = 2 x 32: element p = lane (a0) and 32 + lane (a1)
        #pragma unroll
        for (int size = 2; size <= 64; size <<= 1) {
            #pragma unroll
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                if (stride == 32) {
                    const bool sw = a1 < a0;  // size 64, ascending
                    const uint64_t x = a0;
                    a0 = sw ? a1 : a0;
                    a1 = sw ? x : a1;
                } else {
                    #pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint64_t& v = h ? a1 : a0;
                        const int p = lane + 32 * h;
                        const uint64_t o = __shfl_xor_sync(FULL, v, stride);
                        const bool up = ((p & size) == 0) == ((p & stride) == 0);
                        v = ((o < v) == up) ? o : v;
                    }
                }
            }
        }
        const uint32_t need = (uint32_t)k - before;
        if ((uint32_t)lane < need) {
            kkey[before + lane] = (uint32_t)(a0 >> 32);
            kidx[before + lane] = (uint32_t)a0;
        }
        if ((uint32_t)lane + 32 < need) {
            kkey[before + lane + 32] = (uint32_t)(a1 >> 32);
            kidx[before + lane + 32] = (uint32_t)a1;
        }
    }
    csync<THREADS>();
    // odd-even transposition inside the buckets below b* (positions [0, before))
    for (uint32_t pass = 0; pass < maxc; ++pass) {
        for (uint32_t p = 2 * tid + (pass & 1); p + 1 < before; p += 2 * THREADS) {
            const uint32_t k0 = kkey[p], k1 = kkey[p + 1], i0 = kidx[p], i1 = kidx[p + 1];
            if (k1 < k0 || (k1 == k0 && i1 < i0)) {
                kkey[p] = k1;
                kkey[p + 1] = k0;
                kidx[p] = i1;
                kidx[p + 1] = i0;
            }
        }
        csync<THREADS>();
    }
    if (out_idx == nullptr) return true;  // caller takes the sorted k from kkey / kidx
    for (int r = tid; r < k; r += THREADS) {
        out_idx[r] = (int32_t)((int64_t)kidx[r] + idx_offset);
        out_dist[r] = ukey_to_float(kkey[r]);
    }
    return true;
}

__device__ __forceinline__ float4 ld_stream4(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_stream1(const float* p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

// ------------------------------------------------------------------ select kernel ----
// One CTA per row.  VEC: rows are 16-byte aligned (ldD % 4 == 0) -> 128-bit loads.
// Element e = 4*j + c of a thread in the chunk at `base` sits at column
//   VEC:  base + 4*(j*THREADS + tid) + c        (one float4 per j)
//   else: base + (4*j + c)*THREADS + tid        (coalesced scalars)
// The next chunk is loaded into registers while the current one is filtered.  A warp
// first tests its 32*EPT elements against the float image tf of the threshold (exact for
// every non-NaN key once T is a finite/inf key); only warps holding a survivor run the
// key transform and the ballot/popc compaction.
template <int THREADS, int VPT, bool VEC>
__device__ __forceinline__ void load_chunk(float4 (&v)[VPT], const float* __restrict__ rp,
                                           int64_t N, int64_t base, int tid) {
    #pragma unroll
    for (int j = 0; j < VPT; ++j) {
        if (VEC) {
            const int64_t c0 = base + 4 * ((int64_t)j * THREADS + tid);
            v[j] = c0 < N ? ld_stream4(rp + c0) : make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            float t[4];
            #pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int64_t cc = base + (int64_t)(4 * j + c) * THREADS + tid;
                t[c] = cc < N ? ld_stream1(rp + cc) : 0.0f;
            }
            v[j] = make_float4(t[0], t[1], t[2], t[3]);
        }
    }
}

template <int THREADS, bool VEC>
__device__ __forceinline__ int64_t elem_col(int64_t base, int e, int tid) {
    return VEC ? base + 4 * ((int64_t)(e >> 2) * THREADS + tid) + (e & 3)
               : base + (int64_t)e * THREADS + tid;
}

template <int THREADS, int VPT, bool VEC>
__global__ void __maxnreg__(80)
select_rows_kernel(const float* __restrict__ D, int64_t N, int64_t ldD, int k, int cap, int KP,
                   int limit, int64_t idx_offset, int32_t* __restrict__ out_idx,
                   float* __restrict__ out_dist) {
    constexpr int EPT = VPT * 4;
    constexpr int CHUNK = THREADS * EPT;
    extern __shared__ uint32_t smem[];
    uint32_t* ckey = smem;
    uint32_t* cidx = ckey + cap;
    uint32_t* kkey = cidx + cap;
    uint32_t* kidx = kkey + KP;
    uint32_t* hist = kidx + KP;
    __shared__ Scal sc;
    __shared__ int s_count;

    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t row = blockIdx.x;
    const float* rp = D + row * ldD;
    if (tid == 0) s_count = 0;
    uint32_t T = kKeyMax;
    float tf = 0.0f;
    bool fast = false;  // T is the key of a non-NaN value: the float test is exact

    float4 cur[VPT], nxt[VPT];
    load_chunk<THREADS, VPT, VEC>(cur, rp, N, 0, tid);
    __syncthreads();
    for (int64_t base = 0; base < N; base += CHUNK) {
        if (base + CHUNK < N) load_chunk<THREADS, VPT, VEC>(nxt, rp, N, base + CHUNK, tid);
        const bool full = base + CHUNK <= N;
        bool any = !(fast && full);
        if (!any) {
            #pragma unroll
            for (int j = 0; j < VPT; ++j)
                any |= (cur[j].x < tf) | (cur[j].y < tf) | (cur[j].z < tf) | (cur[j].w < tf);
        }
        bool over = false;
        if (__any_sync(FULL, any)) {
            uint32_t pm = 0;
            #pragma unroll
            for (int j = 0; j < VPT; ++j) {
                const float c4[4] = {cur[j].x, cur[j].y, cur[j].z, cur[j].w};
                #pragma unroll
                for (int c = 0; c < 4; ++c) {
                    bool ok = ukey(c4[c]) < T;
                    if (!full) ok = ok && elem_col<THREADS, VEC>(base, 4 * j + c, tid) < N;
                    pm |= (uint32_t)ok << (4 * j + c);
                }
            }
            const int my = __popc(pm);
            // warp-inclusive scan of the per-thread survivor counts, one shared atomic
            // per warp (the paper's counters g_< kept in shared memory)
            int incl = my;
            #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int n = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += n;
            }
            const int wtot = __shfl_sync(FULL, incl, 31);
            if (wtot) {
                int wbase = 0;
                if (lane == 31) wbase = atomicAdd(&s_count, wtot);
                wbase = __shfl_sync(FULL, wbase, 31);
                over = wbase + wtot > limit;
                int off = wbase + incl - my;
                #pragma unroll
                for (int j = 0; j < VPT; ++j) {
                    const float c4[4] = {cur[j].x, cur[j].y, cur[j].z, cur[j].w};
                    #pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        if (pm & (1u << (4 * j + c))) {
                            ckey[off] = ukey(c4[c]);
                            cidx[off] = (uint32_t)elem_col<THREADS, VEC>(base, 4 * j + c, tid);
                            ++off;
                        }
                    }
                }
            }
        }
        if (named_bar_or(1, THREADS, over)) {
            uint32_t tk, ti;
            block_select_k<THREADS>(ckey, cidx, s_count, k, kkey, kidx, hist, &sc, false, tk, ti);
            for (int i = tid; i < k; i += THREADS) {
                ckey[i] = kkey[i];
                cidx[i] = kidx[i];
            }
            if (tid == 0) s_count = k;
            T = tk;
            fast = T <= 0xFF800000u;  // key of a non-NaN value (<= +inf)
            tf = ukey_to_float(T);
            csync<THREADS>();
        }
        #pragma unroll
        for (int j = 0; j < VPT; ++j) cur[j] = nxt[j];
    }
    __syncthreads();
    block_finish<THREADS>(ckey, cidx, s_count, k, KP, kkey, kidx, hist, &sc, idx_offset,
                          out_idx + row * k, out_dist + row * k);
}

// ------------------------------------------------------------------ ballot append ----
// The paper's partition primitive applied per 32-element segment: for
// element slot e of every lane, B = __ballot(x < T); a lane with its bit set stores its
// element at base + popc(B & lanemask_lt); the warp advances by popc(B).  Slots whose vote
// is empty are skipped warp-uniformly, so a chunk with a handful of survivors costs ~3
// instructions per slot.  In `fast` mode the test is the float compare x < tf, exact for
// every key once T is the key of a non-NaN value; otherwise the order-preserving key test.
// `col(e)` gives the column of slot e; positions >= N are rejected when !full.
// Returns the number appended (warp-uniform).
template <int J0, int NJ, int VPT, class ColF>
__device__ __forceinline__ int warp_append_generic(const float4 (&cur)[VPT], uint32_t Tlim, bool full,
                                                   int64_t N, ColF col, uint32_t* ckey,
                                                   uint32_t* cidx, int base) {
    const uint32_t lt = lanemask_lt();
    int added = 0;
    #pragma unroll
    for (int j = J0; j < J0 + NJ; ++j) {
        const float c4[4] = {cur[j].x, cur[j].y, cur[j].z, cur[j].w};
        #pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t u = ukey(c4[c]);
            bool ok = u < Tlim;
            if (!full) ok = ok && col(4 * j + c) < N;
            const uint32_t m = __ballot_sync(FULL, ok);
            if (m) {
                if (ok) {
                    const int pos = base + added + __popc(m & lt);
                    ckey[pos] = u;
                    cidx[pos] = (uint32_t)col(4 * j + c);
                }
                added += __popc(m);
            }
        }
    }
    return added;
}

// Steady state (full chunk, threshold the key of a non-NaN value): one vote per float4
// group on min(group) < tf, then per-element votes only inside groups holding a survivor.
template <int J0, int NJ, int VPT, class ColF>
__device__ __forceinline__ int warp_append_fast(const float4 (&cur)[VPT], float tf, ColF col,
                                                uint32_t* ckey, uint32_t* cidx, int base) {
    const uint32_t lt = lanemask_lt();
    int added = 0;
    #pragma unroll
    for (int j = J0; j < J0 + NJ; ++j) {
        const float mn = fminf(fminf(cur[j].x, cur[j].y), fminf(cur[j].z, cur[j].w));
        if (!__any_sync(FULL, mn < tf)) continue;
        const float c4[4] = {cur[j].x, cur[j].y, cur[j].z, cur[j].w};
        #pragma unroll
        for (int c = 0; c < 4; ++c) {
            const bool ok = c4[c] < tf;
            const uint32_t m = __ballot_sync(FULL, ok);
            if (m) {
                if (ok) {
                    const int pos = base + added + __popc(m & lt);
                    ckey[pos] = ukey(c4[c]);
                    cidx[pos] = (uint32_t)col(4 * j + c);
                }
                added += __popc(m);
            }
        }
    }
    return added;
}

// Block variant: slots with a non-empty vote reserve space in the CTA-shared buffer with
// one atomicAdd by the lowest voting lane.  Returns true if the buffer grew past `limit`.
template <int VPT, class ColF>
__device__ __forceinline__ bool block_append(const float4 (&cur)[VPT], uint32_t T, float tf, bool fast,
                                             bool full, int64_t N, ColF col, uint32_t* ckey,
                                             uint32_t* cidx, int* s_count, int limit) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = lanemask_lt();
    bool over = false;
    #pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const float c4[4] = {cur[j].x, cur[j].y, cur[j].z, cur[j].w};
        #pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float x = c4[c];
            bool ok = fast ? (x < tf) : (ukey(x) < T);
            if (!full) ok = ok && col(4 * j + c) < N;
            const uint32_t m = __ballot_sync(FULL, ok);
            if (m) {
                const int leader = __ffs(m) - 1;
                int wb = 0;
                if (lane == leader) wb = atomicAdd(s_count, __popc(m));
                wb = __shfl_sync(FULL, wb, leader);
                if (ok) {
                    const int pos = wb + __popc(m & lt);
                    ckey[pos] = ukey(x);
                    cidx[pos] = (uint32_t)col(4 * j + c);
                }
                over |= wb + __popc(m) > limit;
            }
        }
    }
    return over;
}

// Scan append for the ring select: each thread tests its EPT elements (held in registers)
// into a bit mask; a warp-inclusive scan of the per-thread counts gives every survivor its
// slot and one shared atomic per warp reserves the warp's range; survivors are re-read
// from the ring slot `buf` (still owned by the consumers) by dynamic index, so the store
// loop only visits set bits.  At low survival rates this costs ~2 instructions per element.
// Returns true if the buffer grew past `limit` (warp-uniform); `*any_out` = some survivor
// in the warp.
template <int CTHREADS, int VPT>
__device__ __forceinline__ bool ring_append(const float4 (&cur)[VPT], const float* buf, uint32_t T,
                                            float tf, bool fast, bool full, int64_t N, int64_t base,
                                            uint32_t* ckey, uint32_t* cidx, int* s_count, int limit) {
    static_assert(VPT * 4 <= 32, "mask width");
    const int lane = threadIdx.x & 31, tid = threadIdx.x;
    uint32_t pm = 0;
    if (full && fast) {  // steady state: float compares against the threshold's image
        #pragma unroll
        for (int j = 0; j < VPT; ++j) {
            pm |= (uint32_t)(cur[j].x < tf) << (4 * j) | (uint32_t)(cur[j].y < tf) << (4 * j + 1) |
                  (uint32_t)(cur[j].z < tf) << (4 * j + 2) | (uint32_t)(cur[j].w < tf) << (4 * j + 3);
        }
    } else if (full && T == kKeyMax) {  // no threshold yet: every key (NaN included) is < T
        pm = VPT * 4 == 32 ? 0xFFFFFFFFu : (1u << (VPT * 4)) - 1u;
    } else {
        #pragma unroll
        for (int j = 0; j < VPT; ++j) {
            const float c4[4] = {cur[j].x, cur[j].y, cur[j].z, cur[j].w};
            #pragma unroll
            for (int c = 0; c < 4; ++c) {
                bool ok = fast ? (c4[c] < tf) : (ukey(c4[c]) < T);
                if (!full) ok = ok && base + 4 * (j * CTHREADS + tid) + c < N;
                pm |= (uint32_t)ok << (4 * j + c);
            }
        }
    }
    if (!__any_sync(FULL, pm != 0)) return false;
    const int my = __popc(pm);
    int incl = my;
    #pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += n;
    }
    const int wtot = __shfl_sync(FULL, incl, 31);
    int wbase = 0;
    if (lane == 31) wbase = atomicAdd(s_count, wtot);
    wbase = __shfl_sync(FULL, wbase, 31);
    int off = wbase + incl - my;
    while (pm) {
        const int e = __ffs(pm) - 1;
        pm &= pm - 1;
        const int o = 4 * ((e >> 2) * CTHREADS + tid) + (e & 3);
        ckey[off] = ukey(buf[o]);
        cidx[off] = (uint32_t)(base + o);
        ++off;
    }
    return wbase + wtot > limit;
}

// ------------------------------------------------------------------ ring select ------
// Persistent CTAs, one row at a time: a producer warp streams the row in CHUNK-element
// slices through a STAGES-deep shared-memory ring with 1-D bulk async copies (the TMA
// engine; completion on mbarriers), prefetching across row boundaries, so the bytes in
// flight do not depend on registers; CTHREADS consumer threads filter each slice with the
// running threshold and compact survivors (warp scan + one shared atomic per warp).
// Requires 16-byte aligned rows (ldD % 4 == 0, aligned D).
//
// Rows: list == nullptr -> rows 0..M-1; else rows list[1 .. list[0]] (the redo pass).
//
// Sampled pivot (r_pivot > 0; the quick multi-select of PAPER.md:56 with its pivot drawn
// from a sample, reading R18): the first chunk is the sample; one histogram of its keys
// gives a pivot key P with at least r_pivot sample keys below it, and the candidates are
// all keys < P.  r_pivot < k is chosen so that ~1.4k elements of the row fall below P,
// which removes the repeated rebuilds of the plain running threshold (the k-th of the
// first chunk is far above the row's k-th when k/N is large).  Exactness: if at least k
// keys of the row are < P, the k smallest keys (ties included) are all < P, so the
// candidates hold the true top k; the count is checked at the end of the row.  A row with fewer (a sample unlike the rest of the row,
// e.g. a sorted row) is appended to redo[1..] (count redo[0]) and selected again by a
// second launch without the pivot; a buffer overflow instead rebuilds to the exact k
// best, after which the usual running-threshold invariant holds.
// Shared-memory state of one ring-select CTA.
struct RingSmem {
    float* ring;
    uint32_t full0, empty0;  // mbarrier arrays (shared addresses)
    uint32_t *ckey, *cidx, *kkey, *kidx, *hist;
    Scal* sc;
    int* s_count;
};

template <int CTHREADS, int CHUNK, int STAGES>
__device__ __forceinline__ RingSmem ring_smem(uint8_t* smem_raw, int cap, int KP, Scal* sc, int* s_count) {
    RingSmem r;
    r.ring = reinterpret_cast<float*>(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(r.ring + (size_t)STAGES * CHUNK);  // full, empty
    r.full0 = smem_u32(bars);
    r.empty0 = smem_u32(bars + STAGES);
    r.ckey = reinterpret_cast<uint32_t*>(bars + 2 * STAGES);
    r.cidx = r.ckey + cap;
    r.kkey = r.cidx + cap;
    r.kidx = r.kkey + KP;
    r.hist = r.kidx + KP;  // BBINS words (the bucket finish's histogram)
    r.sc = sc;
    r.s_count = s_count;
    if (threadIdx.x == 0) {
        for (int q = 0; q < STAGES; ++q) {
            mbar_init(r.full0 + 8 * q, 1);
            mbar_init(r.empty0 + 8 * q, CTHREADS / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    return r;
}

// Producer (one thread): stream the N-element row rp through the ring.
template <int CHUNK, int STAGES>
__device__ __forceinline__ void ring_produce_row(const RingSmem& r, const float* rp, int64_t N,
                                                 uint64_t pol, int& stage, uint32_t& phase) {
    const int64_t nchunk = ceil_div(N, CHUNK);
    for (int64_t c = 0; c < nchunk; ++c) {
        mbar_wait(r.empty0 + 8 * stage, phase ^ 1);
        const int64_t elems = (N - c * CHUNK) < CHUNK ? (N - c * CHUNK) : CHUNK;
        const uint32_t bytes = (uint32_t)round_up(elems * 4, 16);
        mbar_expect_tx(r.full0 + 8 * stage, bytes);
        bulk_load_evict_first(smem_u32(r.ring + (size_t)stage * CHUNK), rp + c * CHUNK, bytes,
                              r.full0 + 8 * stage, pol);
        if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
        }
    }
}

// Consumers (threads 0..CTHREADS-1): filter one N-element row arriving through the ring.
// On return the candidates are ckey/cidx[0, *s_count) (indices local to the row) and the
// result is the true top k of the row iff the function returned false; true means the
// sampled pivot kept fewer than k candidates (select the row again without it).
template <int CTHREADS, int CHUNK, int STAGES>
__device__ __forceinline__ bool ring_consume_row(const RingSmem& r, int64_t N, int k, int limit,
                                                 bool piv, int r_pivot, int& stage, uint32_t& phase) {
    constexpr int VPT = CHUNK / CTHREADS / 4;  // float4 per consumer thread per slice
    static_assert(VPT * 4 * CTHREADS == CHUNK, "CHUNK must be a multiple of 4*CTHREADS");
    const int lane = threadIdx.x & 31, tid = threadIdx.x;
    Scal& sc = *r.sc;
    if (tid == 0) {
        *r.s_count = 0;
        sc.lo = 0xFFFFFFFFu;
        sc.hi = 0;
    }
    if (piv)
        for (int q = tid; q < 256; q += CTHREADS) r.hist[q] = 0;
    uint32_t T = kKeyMax;
    float tf = 0.0f;
    bool fast = false;
    csync<CTHREADS>();
    const int64_t nchunk = ceil_div(N, CHUNK);
    for (int64_t c = 0; c < nchunk; ++c) {
        const int64_t base = c * CHUNK;
        mbar_wait(r.full0 + 8 * stage, phase);
        const float4* buf = reinterpret_cast<const float4*>(r.ring + (size_t)stage * CHUNK);
        float4 cur[VPT];
        #pragma unroll
        for (int j = 0; j < VPT; ++j) cur[j] = buf[j * CTHREADS + tid];
        const bool full = base + CHUNK <= N;
        if (piv && c == 0) {
            // The sample (the first chunk, still in registers): one 8-bit histogram of its
            // keys on the digit just below the common prefix of their range; the pivot P
            // is the upper edge of the bin holding the r_pivot-th key, so at least r_pivot
            // sample keys are < P.  Candidates: every key < P.
            uint32_t a = 0xFFFFFFFFu, b = 0;
            #pragma unroll
            for (int j = 0; j < VPT; ++j) {
                const uint32_t u0 = ukey(cur[j].x), u1 = ukey(cur[j].y), u2 = ukey(cur[j].z),
                               u3 = ukey(cur[j].w);
                a = min(a, min(min(u0, u1), min(u2, u3)));
                b = max(b, max(max(u0, u1), max(u2, u3)));
            }
            a = __reduce_min_sync(FULL, a);
            b = __reduce_max_sync(FULL, b);
            if (lane == 0) {
                atomicMin(&sc.lo, a);
                atomicMax(&sc.hi, b);
            }
            csync<CTHREADS>();
            const uint32_t mn = sc.lo, mx = sc.hi;
            const int sh = top_digit_shift(mn, mx);
            #pragma unroll
            for (int j = 0; j < VPT; ++j) {
                atomicAdd(&r.hist[(ukey(cur[j].x) >> sh) & 255u], 1u);
                atomicAdd(&r.hist[(ukey(cur[j].y) >> sh) & 255u], 1u);
                atomicAdd(&r.hist[(ukey(cur[j].z) >> sh) & 255u], 1u);
                atomicAdd(&r.hist[(ukey(cur[j].w) >> sh) & 255u], 1u);
            }
            csync<CTHREADS>();
            hist_find(r.hist, (uint32_t)r_pivot, &sc);
            csync<CTHREADS>();
            const uint64_t lowmask = (1ull << (sh + 8)) - 1ull;
            const uint64_t P = ((uint64_t)mn & ~lowmask) + ((uint64_t)(sc.bin + 1) << sh);
            T = P >= 0xFFFFFFFFull ? kKeyMax : (uint32_t)P;
            fast = T <= 0xFF800000u;
            tf = ukey_to_float(T);
        }
        const bool over = ring_append<CTHREADS, VPT>(cur, reinterpret_cast<const float*>(buf), T, tf,
                                                     fast, full, N, base, r.ckey, r.cidx, r.s_count,
                                                     limit);
        __syncwarp();
        if (lane == 0) mbar_arrive(r.empty0 + 8 * stage);  // slot may be refilled
        if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
        }
        if (named_bar_or(1, CTHREADS, over)) {
            uint32_t tk, ti;
            block_select_k<CTHREADS>(r.ckey, r.cidx, *r.s_count, k, r.kkey, r.kidx, r.hist, &sc, false,
                                     tk, ti);
            for (int q = tid; q < k; q += CTHREADS) {
                r.ckey[q] = r.kkey[q];
                r.cidx[q] = r.kidx[q];
            }
            if (tid == 0) *r.s_count = k;
            T = tk;
            fast = T <= 0xFF800000u;
            tf = ukey_to_float(T);
            piv = false;  // k exact best kept: the running-threshold invariant holds
            csync<CTHREADS>();
        }
    }
    csync<CTHREADS>();
    return piv && *r.s_count < k;
}

template <int CTHREADS, int CHUNK, int STAGES, int MINB = 2>
__global__ void __launch_bounds__(CTHREADS + 32, MINB)
select_ring_kernel(const float* __restrict__ D, int64_t M, int64_t N, int64_t ldD, int k, int cap,
                   int KP, int limit, int64_t idx_offset, int32_t* __restrict__ out_idx,
                   float* __restrict__ out_dist, const int32_t* __restrict__ list, int r_pivot,
                   int32_t* __restrict__ redo) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ Scal sc;
    __shared__ int s_count;
    const RingSmem r = ring_smem<CTHREADS, CHUNK, STAGES>(smem_raw, cap, KP, &sc, &s_count);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int64_t nrows = list ? (int64_t)list[0] : M;
    const bool use_pivot = r_pivot > 0 && r_pivot < k && N >= 2 * (int64_t)CHUNK;
    __syncthreads();
    int stage = 0;
    uint32_t phase = 0;
    if (warp == CTHREADS / 32) {
        // producer warp: streams the rows ahead of the consumers, across row boundaries
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int64_t i = blockIdx.x; i < nrows; i += gridDim.x) {
                const int64_t row = list ? (int64_t)list[1 + i] : i;
                ring_produce_row<CHUNK, STAGES>(r, D + row * ldD, N, pol, stage, phase);
            }
        }
        return;
    }
    for (int64_t i = blockIdx.x; i < nrows; i += gridDim.x) {
        const int64_t row = list ? (int64_t)list[1 + i] : i;
        if (ring_consume_row<CTHREADS, CHUNK, STAGES>(r, N, k, limit, use_pivot, r_pivot, stage, phase)) {
            // fewer than k elements beat the sampled pivot: select this row again later
            if (tid == 0) {
                const int slot = atomicAdd(redo, 1);
                redo[1 + slot] = (int32_t)row;
            }
            csync<CTHREADS>();
            continue;
        }
        if (KP < 64 || !block_finish_bucket<CTHREADS>(r.ckey, r.cidx, s_count, k, r.kkey, r.kidx, r.hist,
                                                        &sc, idx_offset, out_idx + row * k, out_dist + row * k))
            block_finish<CTHREADS>(r.ckey, r.cidx, s_count, k, KP, r.kkey, r.kidx, r.hist, &sc, idx_offset,
                                   out_idx + row * k, out_dist + row * k);
        csync<CTHREADS>();
    }
}

// ------------------------------------------------------------------ cluster select ---
// Few-row regime (NEXT-3; one block per query needs >= 128 queries to fill
// the GPU): a thread-block cluster of S CTAs per row.  CTA s of the cluster runs the ring
// select above on columns [s L, (s+1) L) (its own sampled pivot; a failed certificate
// re-streams the segment without it, the producer waiting on the consumers' decision) and
// leaves its sorted top-k as packed (key << 32 | column) in shared memory.  The S lists are
// then merged in log2 S rounds over distributed shared memory: in round l, CTA s (s a
// multiple of 2l) copies CTA s+l's list out of DSMEM and merges it with its own (each
// element's output slot = its rank in its own list + its rank in the other, a merge path
// without ties because the columns differ); CTA 0 writes the row.
template <int CTHREADS, int CHUNK, int STAGES>
__global__ void __launch_bounds__(CTHREADS + 32, 1)
select_cluster_kernel(const float* __restrict__ D, int64_t N, int64_t ldD, int k, int cap, int KP,
                      int limit, int64_t L, int64_t idx_offset, int32_t* __restrict__ out_idx,
                      float* __restrict__ out_dist, int r_pivot) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ Scal sc;
    __shared__ int s_count;
    __shared__ int s_redo;
    const RingSmem r = ring_smem<CTHREADS, CHUNK, STAGES>(smem_raw, cap, KP, &sc, &s_count);
    uint64_t* lst = reinterpret_cast<uint64_t*>(r.hist + BBINS);  // KP, 8-byte aligned
    uint64_t* bbuf = lst + KP;
    uint64_t* obuf = bbuf + KP;
    const int S = (int)cluster.num_blocks();
    const int seg = (int)cluster.block_rank();
    const int64_t row = blockIdx.x / S;
    const int64_t c0 = (int64_t)seg * L;
    const int64_t Ns = N - c0 < L ? N - c0 : L;  // may be <= 0 for trailing segments
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const bool use_pivot = r_pivot > 0 && r_pivot < k && Ns >= 2 * (int64_t)CHUNK;
    __syncthreads();
    int stage = 0;
    uint32_t phase = 0;
    if (warp == CTHREADS / 32) {
        const uint64_t pol = policy_evict_first();
        if (lane == 0 && Ns > 0) ring_produce_row<CHUNK, STAGES>(r, D + row * ldD + c0, Ns, pol, stage, phase);
        __syncwarp();
        named_bar(2, CTHREADS + 32);  // the consumers' verdict on the sampled pivot
        if (lane == 0 && s_redo) ring_produce_row<CHUNK, STAGES>(r, D + row * ldD + c0, Ns, pol, stage, phase);
        __syncwarp();
    } else {
        bool redo = false;
        if (Ns > 0) redo = ring_consume_row<CTHREADS, CHUNK, STAGES>(r, Ns, k, limit, use_pivot, r_pivot, stage, phase);
        if (tid == 0) s_redo = redo;
        named_bar(2, CTHREADS + 32);
        if (redo) ring_consume_row<CTHREADS, CHUNK, STAGES>(r, Ns, k, limit, false, 0, stage, phase);
        const int cnt = Ns > 0 ? s_count : 0;
        // exact min(k, cnt) best, sorted, as packed pairs with the row's column index
        if (cnt > k && KP >= 64 &&
            block_finish_bucket<CTHREADS>(r.ckey, r.cidx, cnt, k, r.kkey, r.kidx, r.hist, &sc, 0, nullptr, nullptr)) {
            for (int q = tid; q < KP; q += CTHREADS)
                lst[q] = q < k ? ((uint64_t)r.kkey[q] << 32 | r.kidx[q]) + (uint64_t)c0 : ~0ull;
        } else {
        if (cnt > k) {
            uint32_t tk, ti;
            block_select_k<CTHREADS>(r.ckey, r.cidx, cnt, k, r.kkey, r.kidx, r.hist, &sc, false, tk, ti);
        } else {
            for (int q = tid; q < cnt; q += CTHREADS) {
                r.kkey[q] = r.ckey[q];
                r.kidx[q] = r.cidx[q];
            }
        }
        for (int q = (cnt < k ? cnt : k) + tid; q < KP; q += CTHREADS) {
            r.kkey[q] = 0xFFFFFFFFu;
            r.kidx[q] = 0xFFFFFFFFu;
        }
        csync<CTHREADS>();
        block_sort_kp<CTHREADS>(r.kkey, r.kidx, KP, reinterpret_cast<uint64_t*>(r.ckey),
                                [&](int q, uint64_t v) { lst[q] = v == ~0ull ? v : v + (uint64_t)c0; });
        }
    }
    cluster.sync();
    for (int l = 1; l < S; l <<= 1) {
        if (seg % (2 * l) == 0) {
            const uint64_t* remote = cluster.map_shared_rank(lst, seg + l);
            for (int q = tid; q < KP; q += blockDim.x) bbuf[q] = remote[q];
            __syncthreads();
            for (int q = tid; q < KP; q += blockDim.x) {
                const uint64_t a = lst[q], b = bbuf[q];
                int lo = 0, hi = KP;  // #b' < a in bbuf
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (bbuf[mid] < a) lo = mid + 1; else hi = mid;
                }
                if (q + lo < KP) obuf[q + lo] = a;
                int lo2 = 0, hi2 = KP;  // #a' <= b in lst
                while (lo2 < hi2) {
                    const int mid = (lo2 + hi2) >> 1;
                    if (lst[mid] <= b) lo2 = mid + 1; else hi2 = mid;
                }
                if (q + lo2 < KP) obuf[q + lo2] = b;
            }
            __syncthreads();
            for (int q = tid; q < KP; q += blockDim.x) lst[q] = obuf[q];
        }
        cluster.sync();  // lists of this round final before the next round reads them
    }
    if (seg == 0) {
        for (int q = tid; q < k; q += blockDim.x) {
            const uint64_t v = lst[q];
            out_idx[row * k + q] = (int32_t)((int64_t)(uint32_t)v + idx_offset);
            out_dist[row * k + q] = ukey_to_float((uint32_t)(v >> 32));
        }
    }
}

// ------------------------------------------------------------------ warp select ------
// The paper's warp-per-query mode ("Each array is handled by a single
// thread warp ... synchronized by default"; >= 1024 queries saturate the
// GPU) made B200-native for k <= 128: one warp owns one row and runs the whole select —
// threshold filter, ballot/popc compaction into a warp-private shared buffer, exact radix
// rebuild, final register bitonic sort — with warp-synchronous code only, so no CTA
// barrier ever couples rows.  The row is streamed through a warp-private ring of 1-D
// bulk async copies (TMA engine) that lane 0 keeps WS stages ahead, across row
// boundaries, so one row's rebuild/sort tail overlaps the other warps' streaming.
constexpr int WSEL_K = 128;      // largest k of the warp path
#ifndef KNN_WSEL_C
#define KNN_WSEL_C 1024
#endif
#ifndef KNN_WSEL_S
#define KNN_WSEL_S 3
#endif
#ifndef KNN_WSEL_WARPS
#define KNN_WSEL_WARPS 4
#endif
constexpr int WSEL_C = KNN_WSEL_C;        // floats per ring stage (4 KB)
constexpr int WSEL_S = KNN_WSEL_S;        // ring stages per warp
constexpr int WSEL_WARPS = KNN_WSEL_WARPS;  // warps (rows in flight) per CTA
constexpr int WSEL_SUB = 256;    // elements appended between buffer checks

__host__ __device__ constexpr int64_t wsel_slab_bytes(int cap) {
    return round_up((int64_t)WSEL_S * WSEL_C * 4 + WSEL_S * 8 + (int64_t)(2 * cap + 2 * WSEL_K + 256) * 4,
                    128);
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Fold `count` buffered candidates into the sorted best-32 register list L (one entry per
// lane), 32 at a time.  Out of line to keep the streaming loop small in the I-cache.
__device__ __noinline__ uint64_t warp_fold32(uint64_t L, const uint32_t* ckey, const uint32_t* cidx,
                                             int count) {
    __syncwarp();  // the lanes' appends are visible to every lane (racecheck)
    for (int o = 0; o < count; o += 32)
        L = ws::warp_merge32<1>(L, ckey + o, cidx + o, count - o < 32 ? count - o : 32);
    __syncwarp();
    return L;
}

// Reduce the warp's candidate buffer to exactly its k best, in place; returns the
// k-th best key (the new strict threshold).  Out of line: it runs a few times per row.
__device__ __noinline__ uint32_t warp_rebuild(uint32_t* ckey, uint32_t* cidx, int count, int k,
                                              uint32_t* kkey, uint32_t* kidx, uint32_t* hist) {
    __syncwarp();  // the lanes' appends are visible to every lane
    const int lane = threadIdx.x & 31;
    const uint32_t t = ws::warp_select_k<1>(ckey, cidx, count, k, kkey, kidx, hist);
    for (int i = lane; i < k; i += 32) {
        ckey[i] = kkey[i];
        cidx[i] = kidx[i];
    }
    __syncwarp();
    return t;
}

template <int R>
__global__ void __maxnreg__(128)
select_warp_kernel(const float* __restrict__ D, int64_t M, int64_t N, int64_t ldD, int k, int cap,
                   int limit, int64_t idx_offset, int32_t* __restrict__ out_idx,
                   float* __restrict__ out_dist) {
    constexpr int VPT = WSEL_C / 128;      // float4 per lane per stage (8)
    constexpr int SUBJ = WSEL_SUB / 128;   // float4 per lane per append sub-group (2)
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per-warp slab: ring | full barriers | candidates key, idx | kept key, idx | hist
    uint8_t* my = smem_raw + wsel_slab_bytes(cap) * warp;
    float* ring = reinterpret_cast<float*>(my);
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + WSEL_S * WSEL_C);
    uint32_t* ckey = reinterpret_cast<uint32_t*>(bars + WSEL_S);
    uint32_t* cidx = ckey + cap;
    uint32_t* kkey = cidx + cap;
    uint32_t* kidx = kkey + WSEL_K;
    uint32_t* hist = kidx + WSEL_K;
    const uint32_t full0 = smem_u32(bars);
    const uint32_t ring0 = smem_u32(ring);

    const int64_t gw = (int64_t)blockIdx.x * WSEL_WARPS + warp;
    const int64_t nw = (int64_t)gridDim.x * WSEL_WARPS;
    const int64_t nchunk = ceil_div(N, WSEL_C);
    if (lane == 0) {
        for (int s = 0; s < WSEL_S; ++s) mbar_init(full0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // producer state (lane 0): next chunk to issue
    int64_t prow = gw, pc = 0;
    const float* psrc = D + gw * ldD;
    const uint32_t last_bytes = (uint32_t)round_up((N - (nchunk - 1) * WSEL_C) * 4, 16);
    auto issue = [&](int stage) {
        if (prow >= M) return;
        const uint32_t bytes = pc == nchunk - 1 ? last_bytes : (uint32_t)(WSEL_C * 4);
        mbar_expect_tx(full0 + 8 * stage, bytes);
        bulk_load(ring0 + stage * (WSEL_C * 4), psrc, bytes, full0 + 8 * stage);
        psrc += WSEL_C;
        if (++pc == nchunk) {
            pc = 0;
            prow += nw;
            psrc = D + prow * ldD;
        }
    };
    if (lane == 0)
        for (int st = 0; st < WSEL_S; ++st) issue(st);

    int stage = 0;
    uint32_t parity = 0;
    for (int64_t row = gw; row < M; row += nw) {
        uint32_t Tlim = kKeyMax;  // accept keys u < Tlim
        float tf = 0.0f;
        bool fast = false;
        int count = 0;
        // k <= 32 (R == 1): the row's best 32 live sorted in registers, one entry per lane
        // (key << 32 | idx); survivors are folded in 32 at a time (warp_merge32).  Larger
        // k: exact radix rebuild of the buffer to its k best.  Either way the threshold
        // only decreases and later elements (larger indices) are tested strictly.
        uint64_t L = ~0ull;
        auto rebuild = [&]() -> bool {
            if constexpr (R == 1) {
                L = warp_fold32(L, ckey, cidx, count);
                count = 0;
                const uint32_t tk = (uint32_t)(__shfl_sync(FULL, L, k - 1) >> 32);
                if (tk == 0xFFFFFFFFu) return false;  // fewer than k seen so far
                Tlim = tk;
                fast = tk <= 0xFF800000u;
                tf = ukey_to_float(tk);
                return true;
            } else {
                const uint32_t t = warp_rebuild(ckey, cidx, count, k, kkey, kidx, hist);
                count = k;
                Tlim = t;  // later elements have larger indices: strict
                fast = t <= 0xFF800000u;
                tf = ukey_to_float(t);
                return true;
            }
        };
        for (int64_t c = 0; c < nchunk; ++c) {
            mbar_wait(full0 + 8 * stage, parity);
            const float4* buf = reinterpret_cast<const float4*>(ring + stage * WSEL_C);
            float4 cur[VPT];
            #pragma unroll
            for (int j = 0; j < VPT; ++j) cur[j] = buf[j * 32 + lane];
            __syncwarp();
            if (lane == 0) {
                fence_proxy_async_smem();
                issue(stage);  // refill this slot (the reads above are complete)
            }
            if (++stage == WSEL_S) {
                stage = 0;
                parity ^= 1;
            }
            const int64_t base = c * WSEL_C;
            const bool full = base + WSEL_C <= N;
            const int lane_ = lane;
            auto col = [&](int e) -> int64_t { return base + 4 * ((e >> 2) * 32 + lane_) + (e & 3); };
            if (fast && full) {
                // steady state: tree minimum over the lane's 32 elements, one vote
                float m[VPT];
                #pragma unroll
                for (int j = 0; j < VPT; ++j)
                    m[j] = fminf(fminf(cur[j].x, cur[j].y), fminf(cur[j].z, cur[j].w));
                #pragma unroll
                for (int w = VPT / 2; w > 0; w >>= 1)
                    #pragma unroll
                    for (int j = 0; j < w; ++j) m[j] = fminf(m[j], m[j + w]);
                if (!__any_sync(FULL, m[0] < tf)) continue;
                // append in WSEL_SUB-element sub-groups (columns increase with the group),
                // rebuilding whenever the buffer passes `limit`
#define KNN_FAST_SG(J)                                                                  \
    count += warp_append_fast<J, SUBJ>(cur, tf, col, ckey, cidx, count);                \
    if (count > limit) rebuild();
                KNN_FAST_SG(0) KNN_FAST_SG(2) KNN_FAST_SG(4) KNN_FAST_SG(6)
#undef KNN_FAST_SG
                continue;
            }
            const bool first = (c == 0 && full);
            if (first) {
                // Initial threshold from the first chunk: split each lane's 32 elements into
                // R groups; t0 = the largest of the 32R group minima (keys).  At least
                // 32R >= k elements are <= t0, so every element > t0 is beaten by k others:
                // keep u <= t0 in this chunk and u < t0 afterwards (larger indices).
                constexpr int GS = (WSEL_C / 32) / R;  // elements per group
                uint32_t t0 = 0;
                #pragma unroll
                for (int g = 0; g < R; ++g) {
                    uint32_t mn = 0xFFFFFFFFu;
                    #pragma unroll
                    for (int e = g * GS; e < (g + 1) * GS; ++e) {
                        const float4& f = cur[e >> 2];
                        const float x = (e & 3) == 0 ? f.x : (e & 3) == 1 ? f.y : (e & 3) == 2 ? f.z : f.w;
                        mn = min(mn, ukey(x));
                    }
                    t0 = max(t0, mn);
                }
                t0 = __reduce_max_sync(FULL, t0);
                Tlim = t0 + 1;
            }
            // generic path: first / partial chunks, or a NaN / unset threshold
            bool rebuilt = false;
#define KNN_GEN_SG(J)                                                                   \
    count += warp_append_generic<J, SUBJ>(cur, Tlim, full, N, col, ckey, cidx, count);  \
    if (count > limit) rebuilt |= rebuild();
            KNN_GEN_SG(0) KNN_GEN_SG(2) KNN_GEN_SG(4) KNN_GEN_SG(6)
#undef KNN_GEN_SG
            if (first && !rebuilt) {  // later chunks: strict u < t0
                Tlim -= 1;
                fast = Tlim <= 0xFF800000u;
                tf = ukey_to_float(Tlim);
            }
        }
        if constexpr (R == 1) {
            if (count > 0) rebuild();
            if (lane < k) {
                out_idx[row * k + lane] = (int32_t)((int64_t)(uint32_t)L + idx_offset);
                out_dist[row * k + lane] = ukey_to_float((uint32_t)(L >> 32));
            }
        } else {
            const uint32_t* fk = ckey;
            const uint32_t* fi = cidx;
            if (count > k) {
                ws::warp_select_k<1>(ckey, cidx, count, k, kkey, kidx, hist);
                fk = kkey;
                fi = kidx;
            }
            ws::warp_sort_write<R>(fk, fi, k, idx_offset, out_idx + row * k, out_dist + row * k);
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ two-pass warp select --
// k <= 32, 32k <= N <= WS2_MAXN (materialised rows, warp per row).  The running-threshold
// select above admits ~k ln(N/1024) survivors per row (the threshold only tightens as the
// row streams by), and each survivor costs a ballot-compaction append and a share of a
// 32-wide bitonic fold: ~80 warp-instructions per survivor, most of the kernel's issue at
// N = 65536 and nearly all of it for short rows (ncu: 5.8 k warp-instructions per
// 4096-long row, 21.7 k per 65536-long row; latency-bound at 12 warps per SM).
// Here the paper's quick multi-select (partition around a pivot, keep the side
// holding the K-th) takes its pivot from the row itself, in two passes:
//   pass 1 (streamed from HBM through the warp's bulk-copy ring): every lane reduces its 32
//          elements of each 1024-element chunk to their minimum — a group minimum G_g, the
//          key of an actual element of group g — stores it, and keeps its 4 smallest;
//   pivot:  P = the k-th smallest group minimum (k pops off the 32 lanes' sorted heads;
//          a lane that runs out of heads only makes P larger).  At least k elements (one per
//          popped group) have key <= P, so every element of the row's true k nearest (ties
//          included) has key <= P: the partition is exact, no certificate needed;
//   pass 2: only the groups with G_g <= P (~k of N/32) are re-read — 8 float4 each, from
//          L2 — their elements with key <= P are compacted (warp scan + per-lane re-reads by
//          dynamic index, L1) and folded into the sorted best-32 register list.
// ~2.5 k warp-instructions per 65536-long row, ~1 k per 4096-long row.
constexpr int WS2_MAXN = 131072;
constexpr int WS2_CAP = 256;    // candidate buffer entries per warp
constexpr int WS2_MAXS = 16;    // ring stages per warp (runtime S <= this)
#ifndef KNN_WS2_PRE
#define KNN_WS2_PRE 1
#endif
constexpr int WS2_PRE = KNN_WS2_PRE;  // listed groups per lane loaded one row ahead (1 or 2)
// slab: ring | S full barriers | 16-bit group minima [nchunk][32] | 16-bit group list
// [nchunk * 32] | candidates key, idx [WS2_CAP]
__host__ __device__ constexpr int64_t ws2_cand_offset(int64_t N, int S) {
    return round_up((int64_t)S * WSEL_C * 4 + S * 8 + ceil_div(N, WSEL_C) * 32 * 2 * 2, 16);
}
__host__ __device__ constexpr int64_t ws2_slab_bytes(int64_t N, int S) {
    return round_up(ws2_cand_offset(N, S) + 2 * WS2_CAP * 4, 128);
}

// Fold `count` buffered candidates into the sorted best-32 list L (warp_fold32, inlined).
__device__ __forceinline__ uint64_t ws2_fold(uint64_t L, const uint32_t* ckey, const uint32_t* cidx, int count) {
    __syncwarp();  // the lanes' appends are visible to every lane
    for (int o = 0; o < count; o += 32)
        L = ws::warp_merge32<1>(L, ckey + o, cidx + o, count - o < 32 ? count - o : 32);
    __syncwarp();
    return L;
}

// Bitonic sort of 64 keys, 2 per lane (element e = r * 32 + lane), ascending.
__device__ __forceinline__ void warp_bitonic64_u32(uint32_t (&v)[2]) {
    const int lane = threadIdx.x & 31;
    #pragma unroll
    for (int size = 2; size <= 64; size <<= 1) {
        #pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride == 32) {
                const bool asc = (lane & size) == 0;  // e & 64 == 0 for both halves
                const uint32_t lo = min(v[0], v[1]), hi = max(v[0], v[1]);
                v[0] = asc ? lo : hi;
                v[1] = asc ? hi : lo;
            } else {
                #pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const int e = r * 32 + lane;
                    const uint32_t o = __shfl_xor_sync(FULL, v[r], stride);
                    const bool asc = (e & size) == 0;
                    const bool lower = (lane & stride) == 0;
                    v[r] = (lower == asc) ? min(o, v[r]) : max(o, v[r]);
                }
            }
        }
    }
}

// Group loads of pass 2, issued one row ahead: volatile so that the compiler keeps them
// where they are (before the next row's pass 1) instead of sinking them to their use.
__device__ __forceinline__ float4 ld_group4(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
// Element e (0..31) of a group held in registers (predicated selects, no local memory).
__device__ __forceinline__ float group_elem(const float4 (&v)[8], int e) {
    float x = 0.0f;
    #pragma unroll
    for (int j = 0; j < 8; ++j) {
        x = e == 4 * j + 0 ? v[j].x : x;
        x = e == 4 * j + 1 ? v[j].y : x;
        x = e == 4 * j + 2 ? v[j].z : x;
        x = e == 4 * j + 3 ? v[j].w : x;
    }
    return x;
}

// One warp per CTA (occupancy in whole warps), S ring stages of WSEL_C floats per warp.
// Software-pipelined over rows: the first 64 listed groups of row r are loaded into
// registers (two per lane) right after its pivot, and consumed only after pass 1 of the
// warp's next row, so their L2 / HBM round trip overlaps that streaming.
__global__ void __launch_bounds__(32)
select_warp2p_kernel(const float* __restrict__ D, int64_t M, int64_t N, int64_t ldD, int k, int S,
                     int64_t idx_offset, int32_t* __restrict__ out_idx, float* __restrict__ out_dist) {
    constexpr int VPT = WSEL_C / 128;  // float4 per lane per chunk (8)
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int lane = threadIdx.x & 31;
    const int64_t nchunk = ceil_div(N, WSEL_C);
    float* ring = reinterpret_cast<float*>(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + (size_t)S * WSEL_C);
    uint16_t* gmin = reinterpret_cast<uint16_t*>(bars + S);   // [nchunk][32] upper key halves
    uint16_t* glist = gmin + nchunk * 32;                      // [nchunk * 32] chunk << 5 | lane
    uint32_t* ckey = reinterpret_cast<uint32_t*>(smem_raw + ws2_cand_offset(N, S));
    uint32_t* cidx = ckey + WS2_CAP;
    const uint32_t full0 = smem_u32(bars);
    const uint32_t ring0 = smem_u32(ring);

    const int64_t gw = blockIdx.x;
    const int64_t nw = gridDim.x;
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(full0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // producer state (lane 0): the next chunk, prefetching across row boundaries
    int64_t prow = gw, pc = 0;
    const float* psrc = D + gw * ldD;
    const uint32_t last_bytes = (uint32_t)round_up((N - (nchunk - 1) * WSEL_C) * 4, 16);
    auto issue = [&](int stage) {
        if (prow >= M) return;
        const uint32_t bytes = pc == nchunk - 1 ? last_bytes : (uint32_t)(WSEL_C * 4);
        mbar_expect_tx(full0 + 8 * stage, bytes);
        bulk_load(ring0 + stage * (WSEL_C * 4), psrc, bytes, full0 + 8 * stage);
        psrc += WSEL_C;
        if (++pc == nchunk) {
            pc = 0;
            prow += nw;
            psrc = D + prow * ldD;
        }
    };
    if (lane == 0)
        for (int st = 0; st < S; ++st) issue(st);
    int stage = 0;
    uint32_t parity = 0;

    // ---- pass 1 of the next row of the FIFO: group minima (a group = one lane's 32
    // elements of a chunk), stored as their upper 16 key bits (the pass-2 test
    // hi16(G) <= hi16(P) keeps every group with G <= P, plus a few); the lane's two smallest
    // full keys in h0 <= h1
    auto pass1 = [&](uint32_t& h0, uint32_t& h1) {
        h0 = kKeyMax;
        h1 = kKeyMax;
        for (int64_t c = 0; c < nchunk; ++c) {
            mbar_wait(full0 + 8 * stage, parity);
            const float4* buf = reinterpret_cast<const float4*>(ring + (size_t)stage * WSEL_C);
            // the lane's group = its 32 CONTIGUOUS elements [32 lane, 32 lane + 32) of the chunk
            // (one 128-byte line to re-read in pass 2); float4 jj of the group is read as
            // cur[(jj - lane) & 7], a rotation that keeps the 16-byte accesses of the warp
            // conflict-free (4 wavefronts per load, the minimum)
            float4 cur[VPT];
            #pragma unroll
            for (int j = 0; j < VPT; ++j) cur[j] = buf[lane * VPT + ((j + lane) & (VPT - 1))];
            __syncwarp();
            if (lane == 0) {
                fence_proxy_async_smem();
                issue(stage);  // refill this slot (the reads above are complete)
            }
            if (++stage == S) {
                stage = 0;
                parity ^= 1;
            }
            const int64_t base = c * WSEL_C;
            if (base + WSEL_C > N) {  // ragged last chunk: columns >= N are NaN, which fminf ignores
                #pragma unroll
                for (int j = 0; j < VPT; ++j) {
                    const int64_t c0 = base + 32 * lane + 4 * ((j + lane) & (VPT - 1));
                    const float nan = __int_as_float(0x7FC00000);
                    if (c0 + 0 >= N) cur[j].x = nan;
                    if (c0 + 1 >= N) cur[j].y = nan;
                    if (c0 + 2 >= N) cur[j].z = nan;
                    if (c0 + 3 >= N) cur[j].w = nan;
                }
            }
            float m[VPT];
            #pragma unroll
            for (int j = 0; j < VPT; ++j) m[j] = fminf(fminf(cur[j].x, cur[j].y), fminf(cur[j].z, cur[j].w));
            #pragma unroll
            for (int w = VPT / 2; w > 0; w >>= 1)
                #pragma unroll
                for (int j = 0; j < w; ++j) m[j] = fminf(m[j], m[j + w]);
            // the key of an element of the group (all-NaN group: the NaN key); a group with
            // no column < N never counts
            const uint32_t g = base + 32 * lane < N ? ukey(m[0]) : kKeyMax;
            gmin[c * 32 + lane] = (uint16_t)(g >> 16);
            if (g < h1) {
                const uint32_t t = max(g, h0);
                h0 = min(g, h0);
                h1 = t;
            }
        }
    };

    // per-row pass-2 state, carried one row ahead
    uint32_t P = 0;
    float Pf = 0.0f;
    bool fastP = true;
    int ng = 0;                // groups listed
    float4 va[VPT], vb[VPT];   // this lane's listed groups lane and lane + 32 (when < ng)
    int64_t ga = 0, gb = 0;    // their element-0 columns
    // pivot, group list and the first round's loads of row r (after its pass 1)
    auto pivot_and_issue = [&](int64_t r, uint32_t h0, uint32_t h1) {
        // P = the k-th smallest of the lanes' two smallest group minima (>= the k-th
        // smallest group minimum; k of them, hence k elements of the row, are <= it)
        uint32_t hv[2] = {h0, h1};
        warp_bitonic64_u32(hv);
        P = __shfl_sync(FULL, hv[0], k - 1);  // element k - 1 (k <= 32)
        fastP = P <= 0xFF800000u;  // P is the key of a non-NaN value: x <= Pf is exact
        Pf = ukey_to_float(P);
        const uint32_t P16 = P >> 16;
        ng = 0;
        for (int64_t c = 0; c < nchunk; ++c) {
            const bool hit = (uint32_t)gmin[c * 32 + lane] <= P16;
            const uint32_t bm = __ballot_sync(FULL, hit);
            if (hit) glist[ng + __popc(bm & ws::lanemask_lt())] = (uint16_t)((uint32_t)c << 5 | lane);
            ng += __popc(bm);
        }
        __syncwarp();
        const float* rp = D + r * ldD;
        #pragma unroll
        for (int h = 0; h < WS2_PRE; ++h) {
            const int gi = lane + 32 * h;
            int64_t gbase = 0;
            float4* v = h ? vb : va;
            if (gi < ng) {
                const uint32_t ge = glist[gi];
                gbase = (int64_t)(ge >> 5) * WSEL_C + 32 * (ge & 31);
                #pragma unroll
                for (int j = 0; j < VPT; ++j)
                    v[j] = gbase + 4 * j < N ? ld_group4(rp + gbase + 4 * j)
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            if (h) gb = gbase; else ga = gbase;
        }
    };
    // survivors of one group held in registers: the keys <= P of columns < N.  Full chunk
    // and P non-NaN (the common case): one test per float4 on its minimum, element tests
    // only inside float4s holding a survivor.
    auto group_mask = [&](const float4 (&v)[VPT], int64_t gbase) -> uint32_t {
        uint32_t mask = 0;
        const bool full = (gbase / WSEL_C) * WSEL_C + WSEL_C <= N;  // the group's whole chunk is < N
        if (full && fastP) {
            #pragma unroll
            for (int j = 0; j < VPT; ++j) {
                if (fminf(fminf(v[j].x, v[j].y), fminf(v[j].z, v[j].w)) <= Pf) {
                    mask |= (uint32_t)(v[j].x <= Pf) << (4 * j);
                    mask |= (uint32_t)(v[j].y <= Pf) << (4 * j + 1);
                    mask |= (uint32_t)(v[j].z <= Pf) << (4 * j + 2);
                    mask |= (uint32_t)(v[j].w <= Pf) << (4 * j + 3);
                }
            }
            return mask;
        }
        #pragma unroll
        for (int j = 0; j < VPT; ++j) {
            const float x4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
            #pragma unroll
            for (int e = 0; e < 4; ++e) {
                const bool ok = (fastP ? x4[e] <= Pf : ukey(x4[e]) <= P) && gbase + 4 * j + e < N;
                mask |= (uint32_t)ok << (4 * j + e);
            }
        }
        return mask;
    };
    // write a group's survivors (register values, static indices) at ckey/cidx[pos...]
    auto put_group = [&](const float4 (&v)[VPT], int64_t gbase, uint32_t mask, int pos) {
        #pragma unroll
        for (int j = 0; j < VPT; ++j) {
            if ((mask >> (4 * j)) & 15u) {
                const float x4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
                #pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if ((mask >> (4 * j + e)) & 1u) {
                        ckey[pos] = ukey(x4[e]);
                        cidx[pos] = (uint32_t)(gbase + 4 * j + e);
                        ++pos;
                    }
                }
            }
        }
    };
    uint64_t L = ~0ull;
    int count = 0;
    // compact one round's survivors (mask per lane; element values re-read by dynamic index
    // from registers) into the buffer, folding as it fills; windows of WS2_CAP survivor
    // ranks when a round alone holds more (heavily tied rows)
    auto append = [&](uint32_t mask, const float4 (&v)[VPT], int64_t gbase) {
        const int n = __popc(mask);
        int incl = n;
        #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(FULL, incl, 31);
        const int excl = incl - n;
        if (count + total > WS2_CAP) {
            L = ws2_fold(L, ckey, cidx, count);
            count = 0;
        }
        if (total <= WS2_CAP) {
            put_group(v, gbase, mask, count + excl);
            count += total;
            return;
        }
        for (int w0 = 0; w0 < total; w0 += WS2_CAP) {
            uint32_t mm = mask;
            int r = excl;
            while (mm) {
                const int e = __ffs(mm) - 1;
                mm &= mm - 1;
                if (r >= w0 && r < w0 + WS2_CAP) {
                    ckey[r - w0] = ukey(group_elem(v, e));
                    cidx[r - w0] = (uint32_t)(gbase + e);
                }
                ++r;
            }
            L = ws2_fold(L, ckey, cidx, total - w0 < WS2_CAP ? total - w0 : WS2_CAP);
        }
    };
    // pass 2 of row r: the preloaded first 64 groups, then any further listed groups.  The
    // common case (<= 64 candidates in all) ends with one 64-wide sort instead of folds.
    auto complete = [&](int64_t r) {
        const float* rp = D + r * ldD;
        L = ~0ull;
        count = 0;
        {
            const uint32_t ma = lane < ng ? group_mask(va, ga) : 0u;
            const uint32_t mb = WS2_PRE > 1 && lane + 32 < ng ? group_mask(vb, gb) : 0u;
            const int n = __popc(ma) + __popc(mb);
            int incl = n;
            #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(FULL, incl, 31);
            if (total <= WS2_CAP) {
                put_group(va, ga, ma, incl - n);
                put_group(vb, gb, mb, incl - n + __popc(ma));
                count = total;
            } else {
                append(ma, va, ga);
                append(mb, vb, gb);
            }
        }
        for (int r0 = 32 * WS2_PRE; r0 < ng; r0 += 32) {  // (ties / loose pivots) synchronous rounds
            const int gi = r0 + lane;
            float4 v[VPT];
            int64_t gbase = 0;
            uint32_t mask = 0;
            if (gi < ng) {
                const uint32_t ge = glist[gi];
                gbase = (int64_t)(ge >> 5) * WSEL_C + 32 * (ge & 31);
                #pragma unroll
                for (int j = 0; j < VPT; ++j)
                    v[j] = gbase + 4 * j < N ? __ldg(reinterpret_cast<const float4*>(rp + gbase + 4 * j))
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
                mask = group_mask(v, gbase);
            }
            append(mask, v, gbase);
        }
        if (__all_sync(FULL, L == ~0ull) && count <= 64) {  // (no fold happened)
            // one sort of the (<= 64) candidates; the first k are the row's result
            __syncwarp();
            uint64_t sv[2];
            #pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = 32 * h + lane;
                sv[h] = i < count ? ((uint64_t)ckey[i] << 32 | cidx[i]) : ~0ull;
            }
            ws::warp_bitonic<2>(sv);
            L = sv[0];
        } else if (count > 0) {
            L = ws2_fold(L, ckey, cidx, count);
        }
        if (lane < k) {
            out_idx[r * k + lane] = (int32_t)((int64_t)(uint32_t)L + idx_offset);
            out_dist[r * k + lane] = ukey_to_float((uint32_t)(L >> 32));
        }
        __syncwarp();  // glist / buffer reads done before the next row's list
    };

    if (gw < M) {
        uint32_t h0, h1;
        pass1(h0, h1);
        pivot_and_issue(gw, h0, h1);
    }
    for (int64_t row = gw; row < M; row += nw) {
        const int64_t next = row + nw;
        uint32_t h0 = kKeyMax, h1 = kKeyMax;
        if (next < M) pass1(h0, h1);  // (gmin is free: row's list is built)
        complete(row);
        if (next < M) pivot_and_issue(next, h0, h1);
    }
}

// ------------------------------------------------------------------ merge kernel -----
struct Offsets {
    int64_t v[64];
};
// The G partial lists of a merge: list g of row (row0 + r) starts at d[g] + (row0 + r) * k.
// The pointers may be local or mapped from a peer GPU's memory (CUDA IPC over NVLink): the
// fused exchange + merge of the corpus-sharded k-NNG reads its peers' lists directly.
struct ListPtrs {
    const float* d[64];
    const int32_t* i[64];
};

template <int THREADS, int EPT>
__global__ void __launch_bounds__(THREADS)
merge_kernel(const ListPtrs lists, int64_t row0, int G, int k, int cap, int KP, int limit,
             Offsets offs, int32_t* __restrict__ out_idx, float* __restrict__ out_dist) {
    constexpr int CHUNK = THREADS * EPT;
    extern __shared__ uint32_t smem[];
    uint32_t* ckey = smem;
    uint32_t* cidx = ckey + cap;
    uint32_t* kkey = cidx + cap;
    uint32_t* kidx = kkey + KP;
    uint32_t* hist = kidx + KP;
    __shared__ Scal sc;
    __shared__ int s_count;

    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t row = blockIdx.x;
    const int64_t L = (int64_t)G * k;
    if (tid == 0) s_count = 0;
    uint32_t T = kKeyMax, Ti = 0xFFFFFFFFu;
    __syncthreads();
    for (int64_t base = 0; base < L; base += CHUNK) {
        uint32_t u[EPT], id[EPT];
        uint32_t pm = 0;
        #pragma unroll
        for (int e = 0; e < EPT; ++e) {
            int64_t p = base + (int64_t)e * THREADS + tid;
            bool ok = false;
            if (p < L) {
                int g = (int)(p / k), r = (int)(p - (int64_t)g * k);
                int64_t off = (row0 + row) * k + r;
                u[e] = ukey(__ldg(lists.d[g] + off));
                id[e] = (uint32_t)((int64_t)__ldg(lists.i[g] + off) + offs.v[g]);
                ok = u[e] < T || (u[e] == T && id[e] < Ti);
            }
            pm |= (uint32_t)ok << e;
        }
        int my = __popc(pm);
        bool over = false;
        if (__any_sync(FULL, my != 0)) {
            int incl = my;
            #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int n = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += n;
            }
            const int wtot = __shfl_sync(FULL, incl, 31);
            int wbase = 0;
            if (lane == 31) wbase = atomicAdd(&s_count, wtot);
            wbase = __shfl_sync(FULL, wbase, 31);
            over = wbase + wtot > limit;
            int off = wbase + incl - my;
            #pragma unroll
            for (int e = 0; e < EPT; ++e)
                if (pm & (1u << e)) {
                    ckey[off] = u[e];
                    cidx[off] = id[e];
                    ++off;
                }
        }
        if (named_bar_or(1, THREADS, over)) {
            uint32_t tk, ti;
            block_select_k<THREADS>(ckey, cidx, s_count, k, kkey, kidx, hist, &sc, true, tk, ti);
            for (int i = tid; i < k; i += THREADS) {
                ckey[i] = kkey[i];
                cidx[i] = kidx[i];
            }
            if (tid == 0) s_count = k;
            T = tk;
            Ti = ti;
            csync<THREADS>();
        }
    }
    __syncthreads();
    block_finish<THREADS>(ckey, cidx, s_count, k, KP, kkey, kidx, hist, &sc, 0,
                          out_idx + row * k, out_dist + row * k);
}


// Bitonic sort of one 32-bit key per lane (ascending across the warp).
__device__ __forceinline__ uint32_t warp_sort32(uint32_t v) {
    const int lane = threadIdx.x & 31;
    #pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
        #pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const uint32_t o = __shfl_xor_sync(FULL, v, stride);
            const bool asc = (lane & size) == 0 || size == 32;
            const bool lower = (lane & stride) == 0;
            v = (lower == asc) ? min(v, o) : max(v, o);
        }
    }
    return v;
}

// Pivot from chunk minima: the k-th smallest of the row's nchunk chunk minima (mins is
// [nchunk][M]).  At least k elements of the row are <= it (one per chunk), so it bounds the
// row's k-th distance from above: a quickselect pivot with L >= K.  A CTA takes 32 rows:
// the minima are staged [chunk][row] through shared memory (coalesced reads); lane l of a
// row's warp keeps the sorted 8 smallest of the chunks l, l+32, ...; the k-th smallest is
// then popped off the 32 lane heads with warp min-reductions.  (Beyond 256 chunks a lane
// may drop a minimum; the result is then the k-th of a subset: still a valid pivot, as at
// least k elements lie at or below it.)  One warp per row, 32 warps per CTA.
constexpr int PV_ROWS = 32, PV_SLAB = 256, PV_PER = PV_SLAB / 32;
__device__ __forceinline__ void cswap(uint32_t& a, uint32_t& b) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}
// sorted 8 smallest of a (sorted) and b (unsorted): sort b, then merge keeping 8
__device__ __forceinline__ void pv_fold(uint32_t (&a)[PV_PER], uint32_t (&b)[PV_PER], bool first) {
    // odd-even merge sort of 8 (19 compare-exchanges)
    cswap(b[0], b[1]); cswap(b[2], b[3]); cswap(b[4], b[5]); cswap(b[6], b[7]);
    cswap(b[0], b[2]); cswap(b[1], b[3]); cswap(b[4], b[6]); cswap(b[5], b[7]);
    cswap(b[1], b[2]); cswap(b[5], b[6]);
    cswap(b[0], b[4]); cswap(b[1], b[5]); cswap(b[2], b[6]); cswap(b[3], b[7]);
    cswap(b[2], b[4]); cswap(b[3], b[5]);
    cswap(b[1], b[2]); cswap(b[3], b[4]); cswap(b[5], b[6]);
    if (first) {
        #pragma unroll
        for (int i = 0; i < PV_PER; ++i) a[i] = b[i];
        return;
    }
    // the 8 smallest of two sorted 8-lists: min(a[i], b[7-i]) is a bitonic sequence
    #pragma unroll
    for (int i = 0; i < PV_PER; ++i) a[i] = min(a[i], b[PV_PER - 1 - i]);
    cswap(a[0], a[4]); cswap(a[1], a[5]); cswap(a[2], a[6]); cswap(a[3], a[7]);
    cswap(a[0], a[2]); cswap(a[1], a[3]); cswap(a[4], a[6]); cswap(a[5], a[7]);
    cswap(a[0], a[1]); cswap(a[2], a[3]); cswap(a[4], a[5]); cswap(a[6], a[7]);
}
__global__ void __launch_bounds__(32 * PV_ROWS, 2)
pivot_from_mins_kernel(const float* __restrict__ mins, int64_t nchunk, int64_t M, int64_t pad_end, int k,
                       int metric, float* __restrict__ thr, int32_t* __restrict__ cnt) {
    __shared__ uint32_t tile[PV_SLAB][PV_ROWS + 1];
    __shared__ uint32_t phist[PV_ROWS][32], pbuf[PV_ROWS][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;  // warp w owns row r0 + w
    const int64_t r0 = (int64_t)blockIdx.x * PV_ROWS;
    if (threadIdx.x < PV_ROWS) {  // zero padding of thr (read as whole tiles by the SYM partition)
        const int64_t row = r0 + threadIdx.x;
        if (row >= M && row < pad_end) thr[row] = 0.0f;
    }
    uint32_t a[PV_PER];  // this lane's sorted 8 smallest of the row's chunks lane, lane+32, ...
    for (int64_t s0 = 0; s0 < nchunk; s0 += PV_SLAB) {
        const int ns = (int)(nchunk - s0 < PV_SLAB ? nchunk - s0 : PV_SLAB);
        __syncthreads();
        {
            const int64_t row = r0 + lane;
            float x[PV_SLAB / PV_ROWS];  // all loads of this warp in flight at once
            #pragma unroll
            for (int t = 0; t < PV_SLAB / PV_ROWS; ++t) {
                const int i = w + PV_ROWS * t;
                x[t] = (i < ns && row < M) ? __ldg(mins + (s0 + i) * M + row) : 0.0f;
            }
            #pragma unroll
            for (int t = 0; t < PV_SLAB / PV_ROWS; ++t) {
                const int i = w + PV_ROWS * t;
                tile[i][lane] = (i < ns && row < M) ? ukey(x[t]) : 0xFFFFFFFFu;
            }
        }
        __syncthreads();
        uint32_t b[PV_PER];
        #pragma unroll
        for (int i = 0; i < PV_PER; ++i) b[i] = tile[lane + 32 * i][w];
        pv_fold(a, b, s0 == 0);
    }
    // k-th smallest of the 32 lanes' kept minima.  Common case: 32 value-linear buckets over
    // [min, max] of the keys; the bucket b* holding the k-th and the keys in it (usually a
    // handful) are sorted by one warp — ~4x fewer instructions than popping k heads.
    uint32_t T = 0;
    bool got = false;
    {
        uint32_t kmx = 0;
        #pragma unroll
        for (int i = 0; i < PV_PER; ++i)
            if (a[i] != 0xFFFFFFFFu) kmx = max(kmx, a[i]);
        const uint32_t gmn = __reduce_min_sync(FULL, a[0]);
        const uint32_t gmx = __reduce_max_sync(FULL, kmx);
        const float fmn = ukey_to_float(gmn), fmx = ukey_to_float(gmx);
        const float scale = 32.0f / (fmx - fmn);
        if (gmn != 0xFFFFFFFFu && fmn >= 0.0f && fmx > fmn && isfinite(fmx) && isfinite(scale)) {
            phist[w][lane] = 0;
            __syncwarp();
            auto bucket = [&](uint32_t u) -> uint32_t {
                return min((uint32_t)((ukey_to_float(u) - fmn) * scale), 31u);
            };
            #pragma unroll
            for (int i = 0; i < PV_PER; ++i)
                if (a[i] != 0xFFFFFFFFu) atomicAdd(&phist[w][bucket(a[i])], 1u);
            __syncwarp();
            const uint32_t c = phist[w][lane];
            uint32_t incl = c;
            #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            const uint32_t hit = __ballot_sync(FULL, incl >= (uint32_t)k);
            if (hit) {  // (else fewer than k finite keys: the pop path below)
                const int bs = __ffs(hit) - 1;
                const uint32_t before = __shfl_sync(FULL, incl - c, bs), nstar = __shfl_sync(FULL, c, bs);
                if (nstar <= 32) {
                    int base = 0;
                    #pragma unroll
                    for (int i = 0; i < PV_PER; ++i) {
                        const bool p2 = a[i] != 0xFFFFFFFFu && bucket(a[i]) == (uint32_t)bs;
                        const uint32_t bm = __ballot_sync(FULL, p2);
                        if (p2) pbuf[w][base + __popc(bm & ws::lanemask_lt())] = a[i];
                        base += __popc(bm);
                    }
                    __syncwarp();
                    const uint32_t v = warp_sort32(lane < base ? pbuf[w][lane] : 0xFFFFFFFFu);
                    T = __shfl_sync(FULL, v, k - 1 - (int)before);
                    got = true;
                }
            }
        }
    }
    // pop the k smallest off the lane heads (equal heads pop together)
    for (int c = 0; c < k && !got;) {
        const uint32_t mn = __reduce_min_sync(FULL, a[0]);
        const bool mine = a[0] == mn;
        c += __popc(__ballot_sync(FULL, mine));
        T = mn;
        if (mine) {
            #pragma unroll
            for (int i = 0; i < PV_PER - 1; ++i) a[i] = a[i + 1];
            a[PV_PER - 1] = 0xFFFFFFFFu;
        }
    }
    const int64_t row = r0 + w;
    if (lane == 0 && row < M) {
        const float t = T == 0xFFFFFFFFu ? __int_as_float(0x7F800000) : ukey_to_float(T);
        const float t1 = nextafterf(t, __int_as_float(0x7F800000));
        // stored as nextup(pivot): the partition keeps u < thr, i.e. u <= pivot
        thr[row] = nextafterf(metric == 1 ? __fmul_ru(t1, t1) : t, __int_as_float(0x7F800000));
        cnt[row] = 0;
    }
}

// Exact top-k (k <= 32) of each row's candidate list, warp per row.  Up to 512
// candidates: each lane sorts its <= 16 keys in registers and parks them in shared memory;
// the k-th smallest key T is popped off the 32 lane heads with warp min-reductions; the
// pairs with key < T, and those with key == T, are compacted and one 32-wide bitonic sort
// orders them (ties at T beyond 32 pairs, or more than 512 candidates: the radix select of
// warpsel.cuh over the list instead).
constexpr int CS_PER = 16;
__device__ __forceinline__ void sort16(uint32_t (&v)[CS_PER]) {
    #pragma unroll
    for (int size = 2; size <= CS_PER; size <<= 1)
        #pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1)
            #pragma unroll
            for (int i = 0; i < CS_PER; ++i) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool asc = (i & size) == 0;
                    const uint32_t lo = min(v[i], v[j]), hi = max(v[i], v[j]);
                    v[i] = asc ? lo : hi;
                    v[j] = asc ? hi : lo;
                }
            }
}
__device__ __forceinline__ void candidate_select_row(int64_t row, const int32_t* __restrict__ cnt,
                                                     const uint64_t* __restrict__ cent, int cap, int k,
                                                     int64_t idx_offset, int32_t* __restrict__ out_idx,
                                                     float* __restrict__ out_dist, int32_t* __restrict__ flag,
                                                     uint32_t (*heads_w)[33], uint32_t* hist_w, uint32_t* skey_w,
                                                     uint32_t* sidx_w) {
    const int lane = threadIdx.x & 31;
    int n = cnt[row];
    // certificate of the partition: k elements at or below the pivot means every element of
    // the true k nearest (ties included) is a candidate; otherwise redo (flag bit 2)
    if (n < k && lane == 0) atomicOr(flag, 2);
    n = n < cap ? n : cap;
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(flag + 2), (unsigned long long)n);
    // the row's entries (ukey << 32 | col): keys are the odd words, columns the even ones
    const uint32_t* ri = reinterpret_cast<const uint32_t*>(cent + row * cap);
    const uint32_t* rk = ri + 1;
    const uint32_t* fk = rk;  // the kept pairs: the list itself (stride 2 words) when n <= k,
    const uint32_t* fi = ri;  // else the compacted shared-memory copy (stride 1)
    int fs = 2;
    int m = n;
    if (n > k) {
        bool done = false;
        if (n <= 32 * CS_PER) {
            uint32_t uk[CS_PER], v[CS_PER];  // this lane's keys (list order), sorted copy
            #pragma unroll
            for (int i = 0; i < CS_PER; ++i) uk[i] = lane + 32 * i < n ? __ldg(rk + 2 * (lane + 32 * i)) : 0xFFFFFFFFu;
            // Bucket select (the common case): 32 value-linear buckets over [min, max] of the
            // keys (the candidates of a row are spread over [0, pivot]); the bucket b* holding
            // the k-th key and every bucket below it hold every key of the k nearest, ties at
            // the k-th included (the bucket map is monotone in the value).  When those are at
            // most 64 they are compacted and sorted once (64-wide bitonic); crowded buckets
            // take the exact path below.  ~4x fewer instructions than sorting and popping.
            {
                uint32_t kmn = 0xFFFFFFFFu, kmx = 0;
                #pragma unroll
                for (int i = 0; i < CS_PER; ++i)
                    if (lane + 32 * i < n) {
                        kmn = min(kmn, uk[i]);
                        kmx = max(kmx, uk[i]);
                    }
                kmn = __reduce_min_sync(FULL, kmn);
                kmx = __reduce_max_sync(FULL, kmx);
                const float fmn = ukey_to_float(kmn), fmx = ukey_to_float(kmx);
                const float scale = 32.0f / (fmx - fmn);
                if (fmn >= 0.0f && fmx > fmn && isfinite(fmx) && isfinite(scale)) {
                    hist_w[lane] = 0;
                    __syncwarp();
                    auto bucket = [&](uint32_t u) -> uint32_t {
                        return min((uint32_t)((ukey_to_float(u) - fmn) * scale), 31u);
                    };
                    #pragma unroll
                    for (int i = 0; i < CS_PER; ++i)
                        if (lane + 32 * i < n) atomicAdd(&hist_w[bucket(uk[i])], 1u);
                    __syncwarp();
                    const uint32_t c = hist_w[lane];
                    uint32_t incl = c;
                    #pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(FULL, incl, o);
                        if (lane >= o) incl += y;
                    }
                    const int bs = __ffs(__ballot_sync(FULL, incl >= (uint32_t)k)) - 1;  // b*
                    const uint32_t upto = __shfl_sync(FULL, incl, bs);  // keys in buckets <= b*
                    if (upto <= 64) {
                        int base = 0;
                        #pragma unroll
                        for (int i = 0; i < CS_PER; ++i) {
                            const bool p2 = lane + 32 * i < n && bucket(uk[i]) <= (uint32_t)bs;
                            const uint32_t bm = __ballot_sync(FULL, p2);
                            if (p2) {
                                const int pos = base + __popc(bm & ws::lanemask_lt());
                                skey_w[pos] = uk[i];
                                sidx_w[pos] = __ldg(ri + 2 * (lane + 32 * i));
                            }
                            base += __popc(bm);
                        }
                        __syncwarp();
                        uint64_t b2[2];
                        #pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int e = h * 32 + lane;
                            b2[h] = e < base ? ((uint64_t)skey_w[e] << 32 | sidx_w[e]) : ~0ull;
                        }
                        ws::warp_bitonic<2>(b2);
                        if (lane < k) {
                            out_idx[row * k + lane] = (int32_t)((int64_t)(uint32_t)b2[0] + idx_offset);
                            out_dist[row * k + lane] = ukey_to_float((uint32_t)(b2[0] >> 32));
                        }
                        return;
                    }
                }
            }
            #pragma unroll
            for (int i = 0; i < CS_PER; ++i) v[i] = uk[i];
            sort16(v);
            #pragma unroll
            for (int i = 0; i < CS_PER; ++i) heads_w[i][lane] = v[i];
            __syncwarp();
            uint32_t h = v[0], T = 0;
            int p = 0;
            for (int c = 0; c < k;) {
                const uint32_t mn = __reduce_min_sync(FULL, h);
                const bool mine = h == mn;
                c += __popc(__ballot_sync(FULL, mine));
                T = mn;
                if (mine) h = ++p < CS_PER ? heads_w[p][lane] : 0xFFFFFFFFu;
            }
            // compact the pairs with key < T (fewer than k), then those with key == T
            int base = 0;
            #pragma unroll
            for (int i = 0; i < CS_PER; ++i) {
                const bool p2 = uk[i] < T;
                const uint32_t bm = __ballot_sync(FULL, p2);
                if (p2) {
                    const int pos = base + __popc(bm & ws::lanemask_lt());
                    skey_w[pos] = uk[i];
                    sidx_w[pos] = __ldg(ri + 2 * (lane + 32 * i));
                }
                base += __popc(bm);
            }
            int eq = 0;
            #pragma unroll
            for (int i = 0; i < CS_PER; ++i) {
                const bool p2 = uk[i] == T && lane + 32 * i < n;
                const uint32_t bm = __ballot_sync(FULL, p2);
                const int pos = base + eq + __popc(bm & ws::lanemask_lt());
                if (p2 && pos < 32) {
                    skey_w[pos] = T;
                    sidx_w[pos] = __ldg(ri + 2 * (lane + 32 * i));
                }
                eq += __popc(bm);
            }
            __syncwarp();
            if (base + eq <= 32) {  // every tie at T kept: the k best are among them
                fk = skey_w;
                fi = sidx_w;
                fs = 1;
                m = base + eq;
                done = true;
            }
        }
        if (!done) {
            ws::warp_select_k<2>(rk, ri, n, k, skey_w, sidx_w, hist_w);
            fk = skey_w;
            fi = sidx_w;
            fs = 1;
            m = k;
        }
    }
    // sort the m <= 32 kept pairs; slots past m are empty (-1, +inf).  (n <= k reads the list's
    // interleaved entries directly: stride 2 — a stride-1 read here returned garbage for rows
    // with exactly k candidates, reachable since the per-point bound's tighter pivots.)
    uint64_t v[1] = {lane < m ? ((uint64_t)fk[fs * lane] << 32 | fi[fs * lane]) : ~0ull};
    ws::warp_bitonic<1>(v);
    if (lane < k) {
        const uint32_t key = (uint32_t)(v[0] >> 32);
        out_idx[row * k + lane] = key == 0xFFFFFFFFu ? -1 : (int32_t)((int64_t)(uint32_t)v[0] + idx_offset);
        out_dist[row * k + lane] = key == 0xFFFFFFFFu ? __int_as_float(0x7F800000) : ukey_to_float(key);
    }
}


__global__ void __launch_bounds__(256)
candidate_select_kernel(const int32_t* __restrict__ cnt, const uint64_t* __restrict__ cent,
                        int cap, int64_t M, int k,
                        int64_t idx_offset, int32_t* __restrict__ out_idx,
                        float* __restrict__ out_dist, int32_t* __restrict__ flag, int gate) {
    if (gate >= 0 && flag[1] != gate) return;  // the other partition ran (device plan choice)
    __shared__ uint32_t heads[8][CS_PER][33];  // [warp][position][lane]
    __shared__ uint32_t hist[8][256], skey[8][64], sidx[8][64];
    const int w = threadIdx.x >> 5;
    // rows strided over a grid of a few CTAs per SM (a gated-off launch costs little)
    for (int64_t row = (int64_t)blockIdx.x * 8 + w; row < M; row += (int64_t)gridDim.x * 8) {
        candidate_select_row(row, cnt, cent, cap, k, idx_offset, out_idx, out_dist, flag, heads[w], hist[w], skey[w],
                             sidx[w]);
        __syncwarp();
    }
}

// Exact top-k (k <= 32) of the single-product partition (gemm_tc.cu MODE_PIVOT1, L2
// metrics), warp per row.  The list holds lower bounds L = u_hh - (F1_q ||q||^2 + F1_x
// ||x||^2) <= D (per-point terms, prep.cu launch_bound_norms), so U = L + 2 (bq + bx) >= D
// with b = RU(F1 ||.||^2):
//  1. T = the k-th smallest U over the first <= 512 candidates: k candidates have D <= T,
//     so the row's k nearest candidates (and their fp32 ties) all have L <= T;
//  2. R = {L <= T (1 + 4 e) + slack} (e = the re-evaluation's error bound): typically k
//     plus the few whose bounds straddle T (51 per row at the headline);
//  3. D of every member of R from the fp32 inputs as the sum of squared differences, in
//     fp32 (relative error <= e = (d/32 + 8) 2^-24: ~1e-6 at d = 256, 1e-7 typical, vs
//     ~1e-5 for the split-fp16 GEMM value), 8 candidates per step so that their L2
//     loads overlap; the k smallest (value, index) pairs kept by a warp merge;
//  4. certificate: the k-th D (1 + 2 e + 2^-20) <= the pivot, i.e. every element that can
//     rank among the k, had L <= pivot and is a candidate; else flag bit 2 and the caller
//     redoes the call on the full matrix.
constexpr int CR_PER = 16;
constexpr int CR_RCAP = 256;
constexpr int CR_G = 8;
#ifndef KNN_CR_ONEHALF
#define KNN_CR_ONEHALF 1  // one 128-float slice of the candidates at a time (no spills)
#endif
#ifndef KNN_CR_T
#define KNN_CR_T 8  // candidates per lane that the k-th upper bound T is taken from
#endif
#ifndef KNN_CR_MINB
#define KNN_CR_MINB 4  // CTAs per SM of the re-evaluation (4: 64 registers)
#endif
// Step 1 of the re-evaluation: an upper bound T >= the k-th smallest U of the warp's
// values v (ukey order, padding 0xFFFFFFFF; at least k valid).  32 buckets of power-of-two
// width over [min, max] in the key domain (exact integer arithmetic), shared-memory counts,
// a warp scan for the bucket b* holding the k-th; b*'s values (<= 32) sorted by a warp
// bitonic network give the k-th exactly; a crowded b* gives its largest value (at least k
// values are at or below it: still a valid T, one bucket looser).
template <int PER>
__device__ __forceinline__ uint32_t kth_upper(const uint32_t (&v)[PER], int k, uint32_t* hist, uint32_t* sbuf) {
    const int lane = threadIdx.x & 31;
    uint32_t mn = 0xFFFFFFFFu, mx = 0u;
    #pragma unroll
    for (int i = 0; i < PER; ++i)
        if (v[i] != 0xFFFFFFFFu) {
            mn = min(mn, v[i]);
            mx = max(mx, v[i]);
        }
    mn = __reduce_min_sync(FULL, mn);
    mx = __reduce_max_sync(FULL, mx);
    const uint32_t span = mx - mn;
    if (span == 0) return mx;
    const int sh = max(0, 27 - __clz(span));  // span >> sh <= 31
    hist[lane] = 0u;
    __syncwarp();
    #pragma unroll
    for (int i = 0; i < PER; ++i)
        if (v[i] != 0xFFFFFFFFu) atomicAdd(hist + ((v[i] - mn) >> sh), 1u);
    __syncwarp();
    const uint32_t c = hist[lane];
    uint32_t incl = c;
    #pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    const int bs = __ffs(__ballot_sync(FULL, incl >= (uint32_t)k)) - 1;
    const uint32_t cb = __shfl_sync(FULL, c, bs);
    const int need = k - (int)__shfl_sync(FULL, incl - c, bs);  // rank in b*, 1..cb
    if (cb > 32) {
        uint32_t bm = 0u;
        #pragma unroll
        for (int i = 0; i < PER; ++i)
            if (v[i] != 0xFFFFFFFFu && (int)((v[i] - mn) >> sh) <= bs) bm = max(bm, v[i]);
        return __reduce_max_sync(FULL, bm);
    }
    int base = 0;
    #pragma unroll
    for (int i = 0; i < PER; ++i) {
        const bool p = v[i] != 0xFFFFFFFFu && (int)((v[i] - mn) >> sh) == bs;
        const uint32_t m = __ballot_sync(FULL, p);
        if (p) sbuf[base + __popc(m & ws::lanemask_lt())] = v[i];
        base += __popc(m);
    }
    __syncwarp();
    uint32_t x = lane < (int)cb ? sbuf[lane] : 0xFFFFFFFFu;
    #pragma unroll
    for (int size = 2; size <= 32; size <<= 1)
        #pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const uint32_t o = __shfl_xor_sync(FULL, x, stride);
            const bool take_min = ((lane & stride) == 0) == ((lane & size) == 0);
            x = take_min ? min(x, o) : max(x, o);
        }
    return __shfl_sync(FULL, x, need - 1);
}

template <int PER>
__device__ __forceinline__ void recompute_row(int64_t row, int n, const uint64_t* __restrict__ cent, int cap,
                                              int k, int64_t idx_offset, const float* __restrict__ Q,
                                              const float* __restrict__ X, int d, const float* __restrict__ qn,
                                              const float* __restrict__ bq, const float* __restrict__ bx,
                                              const float* __restrict__ thr, float rerr, int metric, int vec,
                                              int32_t* __restrict__ out_idx, float* __restrict__ out_dist,
                                              int32_t* __restrict__ flag, uint32_t* hist, uint32_t* sbuf,
                                              uint32_t* rl) {
    const int lane = threadIdx.x & 31;
    const uint32_t* ri = reinterpret_cast<const uint32_t*>(cent + row * cap);  // (key << 32 | col)
    const uint32_t* rk = ri + 1;
    const float qnr = __ldg(qn + row), bqr = __ldg(bq + row);
    // 1. T from the first <= 32 PER candidates (a subset's k-th U bounds the list's from above)
    const int n1 = n < 32 * PER ? n : 32 * PER;
    uint32_t v[PER], lk[PER], li[PER];
    #pragma unroll
    for (int i = 0; i < PER; ++i) {  // one 8-byte load per entry: x = column, y = key
        const int pos = lane + 32 * i;
        const uint2 e = pos < n1 ? __ldg(reinterpret_cast<const uint2*>(ri) + pos) : make_uint2(0u, 0xFFFFFFFFu);
        lk[i] = e.y;
        li[i] = e.x;
    }
    #pragma unroll
    for (int i = 0; i < PER; ++i) {
        const float bj = lane + 32 * i < n1 ? __ldg(bx + li[i]) : 0.0f;
        v[i] = lk[i] == 0xFFFFFFFFu ? 0xFFFFFFFFu : ukey(__fmaf_ru(2.0f, __fadd_ru(bqr, bj), ukey_to_float(lk[i])));
    }
    const float T = ukey_to_float(kth_upper<PER>(v, k, hist, sbuf));
    // every candidate whose re-evaluated value can reach the k-th re-evaluated value
    const uint32_t Tf = ukey(T + (4.0f * rerr + 0x1p-20f) * (fabsf(T) + qnr));
    // 2. R (the first 512 from registers)
    int nr = 0;
    #pragma unroll
    for (int i = 0; i < PER; ++i) {
        const bool keep = lk[i] <= Tf;  // padding is 0xFFFFFFFF
        const uint32_t bm = __ballot_sync(FULL, keep);
        const int slot = nr + __popc(bm & ws::lanemask_lt());
        if (keep && slot < CR_RCAP) rl[slot] = li[i];
        nr += __popc(bm);
    }
    for (int base = n1; base < n; base += 32) {
        const int pos = base + lane;
        const bool keep = pos < n && __ldg(rk + 2 * pos) <= Tf;
        const uint32_t bm = __ballot_sync(FULL, keep);
        const int slot = nr + __popc(bm & ws::lanemask_lt());
        if (keep && slot < CR_RCAP) rl[slot] = __ldg(ri + 2 * pos);
        nr += __popc(bm);
    }
    if (lane == 0 && (vec & 2))  // diagnostic (KNN_RECOMP_STATS): count |R| instead
        atomicAdd(reinterpret_cast<unsigned long long*>(flag + 2), (unsigned long long)nr);
    const int nr_total = nr;
    __syncwarp();
    // 3. exact values, k smallest (CR_G candidates per step, all their loads in flight);
    //    more than CR_RCAP members (wide bounds: data far from the origin) are processed in
    //    windows of CR_RCAP, each re-collected by a scan of the list
    const float* q = Q + row * (int64_t)d;
    uint64_t best = ~0ull;  // this lane's entry of the sorted best-32 (key << 32 | idx)
    for (int win = 0; win * CR_RCAP < nr_total; ++win) {
    if (win > 0) {
        __syncwarp();
        int ridx = 0;
        for (int base = 0; base < n; base += 32) {
            const int pos = base + lane;
            const bool keep = pos < n && __ldg(rk + 2 * pos) <= Tf;
            const uint32_t bm = __ballot_sync(FULL, keep);
            const int slot = ridx + __popc(bm & ws::lanemask_lt()) - win * CR_RCAP;
            if (keep && slot >= 0 && slot < CR_RCAP) rl[slot] = __ldg(ri + 2 * pos);
            ridx += __popc(bm);
        }
        __syncwarp();
    }
    const int nr = nr_total - win * CR_RCAP < CR_RCAP ? nr_total - win * CR_RCAP : CR_RCAP;
    for (int g = 0; g < nr; g += 32) {
        uint64_t mine = ~0ull;
        for (int t0 = 0; t0 < 32 && g + t0 < nr; t0 += CR_G) {
            const float* xr[CR_G];
            uint32_t id[CR_G];
            #pragma unroll
            for (int u = 0; u < CR_G; ++u) {
                const int c = g + t0 + u;
                id[u] = rl[c < nr ? c : g + t0];
                xr[u] = X + (int64_t)id[u] * d;
            }
            float acc[CR_G];
            uint64_t acc2[CR_G];
            #pragma unroll
            for (int u = 0; u < CR_G; ++u) {
                acc[u] = 0.0f;
                acc2[u] = 0ull;
            }
            if (vec & 1) {
#if KNN_CR_ONEHALF
                // one 128-float slice at a time: CR_G float4 loads in flight per lane (32
                // registers), no spills at 64 registers; the other warps supply the MLP
                #pragma unroll 1
                for (int t = 4 * lane; t < d; t += 128) {
                    const float4 qv = __ldg(reinterpret_cast<const float4*>(q + t));
                    float4 xv[CR_G];
                    #pragma unroll
                    for (int u = 0; u < CR_G; ++u) xv[u] = __ldg(reinterpret_cast<const float4*>(xr[u] + t));
                    // two components per FADD2 / FFMA2 (even / odd partial sums per lane)
                    #pragma unroll
                    for (int u = 0; u < CR_G; ++u) {
                        const uint64_t e01 = f2_sub(f2_pack(qv.x, qv.y), f2_pack(xv[u].x, xv[u].y));
                        const uint64_t e23 = f2_sub(f2_pack(qv.z, qv.w), f2_pack(xv[u].z, xv[u].w));
                        acc2[u] = f2_fma(e01, e01, acc2[u]);
                        acc2[u] = f2_fma(e23, e23, acc2[u]);
                    }
                }
                #pragma unroll
                for (int u = 0; u < CR_G; ++u) {
                    float lo, hi;
                    f2_unpack(acc2[u], lo, hi);
                    acc[u] = lo + hi;
                }
#else
                for (int t = 4 * lane; t < d; t += 256) {
                    const bool two = t + 128 < d;
                    const float4 qv = __ldg(reinterpret_cast<const float4*>(q + t));
                    const float4 qv2 = two ? __ldg(reinterpret_cast<const float4*>(q + t + 128)) : qv;
                    float4 xv[CR_G], xv2[CR_G];
                    #pragma unroll
                    for (int u = 0; u < CR_G; ++u) {
                        xv[u] = __ldg(reinterpret_cast<const float4*>(xr[u] + t));
                        xv2[u] = two ? __ldg(reinterpret_cast<const float4*>(xr[u] + t + 128)) : qv2;
                    }
                    #pragma unroll
                    for (int u = 0; u < CR_G; ++u) {
                        const float e0 = qv.x - xv[u].x, e1 = qv.y - xv[u].y;
                        const float e2 = qv.z - xv[u].z, e3 = qv.w - xv[u].w;
                        const float f0 = qv2.x - xv2[u].x, f1 = qv2.y - xv2[u].y;
                        const float f2_ = qv2.z - xv2[u].z, f3 = qv2.w - xv2[u].w;
                        acc[u] = fmaf(e0, e0, acc[u]);
                        acc[u] = fmaf(e1, e1, acc[u]);
                        acc[u] = fmaf(e2, e2, acc[u]);
                        acc[u] = fmaf(e3, e3, acc[u]);
                        acc[u] = fmaf(f0, f0, acc[u]);
                        acc[u] = fmaf(f1, f1, acc[u]);
                        acc[u] = fmaf(f2_, f2_, acc[u]);
                        acc[u] = fmaf(f3, f3, acc[u]);
                    }
                }
#endif
            } else {
                for (int t = lane; t < d; t += 32) {
                    const float qv = __ldg(q + t);
                    float xv[CR_G];
                    #pragma unroll
                    for (int u = 0; u < CR_G; ++u) xv[u] = __ldg(xr[u] + t);
                    #pragma unroll
                    for (int u = 0; u < CR_G; ++u) {
                        const float e = qv - xv[u];
                        acc[u] = fmaf(e, e, acc[u]);
                    }
                }
            }
            // butterfly reduce-scatter of the 8 sums (9 shuffles): lanes 4u..4u+3 end with
            // candidate u's total
            static_assert(CR_G == 8, "reduce-scatter is written for 8 candidates");
            float a4[4], a2[2];
            {
                const bool b = lane & 16;
                #pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float send = b ? acc[i] : acc[i + 4], keep = b ? acc[i + 4] : acc[i];
                    a4[i] = keep + __shfl_xor_sync(FULL, send, 16);
                }
            }
            {
                const bool b = lane & 8;
                #pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const float send = b ? a4[i] : a4[i + 2], keep = b ? a4[i + 2] : a4[i];
                    a2[i] = keep + __shfl_xor_sync(FULL, send, 8);
                }
            }
            float tot;
            {
                const bool b = lane & 4;
                const float send = b ? a2[0] : a2[1], keep = b ? a2[1] : a2[0];
                tot = keep + __shfl_xor_sync(FULL, send, 4);
            }
            tot += __shfl_xor_sync(FULL, tot, 2);
            tot += __shfl_xor_sync(FULL, tot, 1);
            const float su = __shfl_sync(FULL, tot, ((lane - t0) & 7) * 4);
            if (lane >= t0 && lane < t0 + CR_G && g + lane < nr) {
                const float val = metric == 1 ? sqrtf(su) : su;
                mine = (uint64_t)ukey(val) << 32 | rl[g + lane];
            }
        }
        uint64_t b[1] = {mine};
        ws::warp_bitonic<1>(b);
        const uint64_t br = __shfl_sync(FULL, b[0], 31 - lane);
        uint64_t c = best < br ? best : br;
        #pragma unroll
        for (int stride = 16; stride > 0; stride >>= 1) {
            const uint64_t o = __shfl_xor_sync(FULL, c, stride);
            c = (lane & stride) ? (o > c ? o : c) : (o < c ? o : c);
        }
        best = c;
    }
    }
    // 4. certificate, output
    const float vk = ukey_to_float((uint32_t)(__shfl_sync(FULL, best, k - 1) >> 32));
    const double dk = metric == 1 ? (double)vk * vk : (double)vk;
    if (!(dk * (1.0 + 2.0 * rerr + 0x1p-20) <= (double)__ldg(thr + row))) {
        if (lane == 0) atomicOr(flag, 2);
        return;
    }
    if (lane < k) {
        out_idx[row * k + lane] = (int32_t)((int64_t)(uint32_t)best + idx_offset);
        out_dist[row * k + lane] = ukey_to_float((uint32_t)(best >> 32));
    }
}


__global__ void __launch_bounds__(256, KNN_CR_MINB)
candidate_recompute_kernel(const int32_t* __restrict__ cnt, const uint64_t* __restrict__ cent,
                           int cap, int64_t M, int k, int64_t idx_offset,
                           const float* __restrict__ Q, const float* __restrict__ X, int d,
                           const float* __restrict__ qn, const float* __restrict__ bq,
                           const float* __restrict__ bx, const float* __restrict__ thr, float rerr,
                           int metric, int vec,
                           int32_t* __restrict__ out_idx, float* __restrict__ out_dist,
                           int32_t* __restrict__ flag, int gate) {
    if (gate >= 0 && flag[1] != gate) return;  // the other partition ran (device plan choice)
    __shared__ uint32_t hist[8][32], sbuf[8][32];
    __shared__ uint32_t rlist[8][CR_RCAP];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // rows strided over a grid of a few CTAs per SM (a gated-off launch costs little)
    for (int64_t row = (int64_t)blockIdx.x * 8 + w; row < M; row += (int64_t)gridDim.x * 8) {
        int n = cnt[row];
        if (n < k) {  // fewer than k lower bounds at or below the pivot: the partition is not exact
            if (lane == 0) atomicOr(flag, 2);
            continue;
        }
        n = n < cap ? n : cap;
        if (lane == 0 && !(vec & 2)) atomicAdd(reinterpret_cast<unsigned long long*>(flag + 2), (unsigned long long)n);
        // (T from the first <= 256 candidates: longer lists get a slightly looser T, their
        // remaining candidates join R through the scan of step 2)
        recompute_row<KNN_CR_T>(row, n, cent, cap, k, idx_offset, Q, X, d, qn, bq, bx, thr, rerr, metric, vec, out_idx,
                            out_dist, flag, hist[w], sbuf[w], rlist[w]);
        __syncwarp();
    }
}

int next_pow2(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

bool getenv_flag(const char* name) {
    const char* v = getenv(name);
    return v && v[0] && v[0] != '0';
}

template <class K>
cudaError_t set_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// ------------------------------------------------------------ quantile pivot (k > 32) --
// The pivot plan for k > 32: per row, a pivot P with at least r of the
// row's S sampled upper bounds v <= P, from value-linear buckets: min/max of the finite
// samples, one 1024-bucket histogram, the bucket b* holding the r-th sample, and P = the
// largest sample in buckets <= b* (exact, so the r-th sample is <= P).  Fewer than r
// finite samples: P = +inf (every element becomes a candidate; the list overflow then
// sends the call to the materialised plan).  One CTA per row, rows re-read from L2.
constexpr int QP_THREADS = 256;
// EPT > 0: the row (S <= EPT * QP_THREADS) is held in registers and read from memory once;
// EPT == 0: three passes over the row (L2-resident after the first).
template <int EPT>
__global__ void __launch_bounds__(QP_THREADS)
pivot_from_sample_kernel(const float* __restrict__ Ds, int64_t M, int64_t S, int64_t ldS, int r,
                         float* __restrict__ thr) {
    __shared__ uint32_t hist[BBINS];
    __shared__ Scal sc;
    __shared__ int s_nfin;
    const int tid = threadIdx.x, lane = tid & 31;
    constexpr int NR = EPT > 0 ? EPT : 1;
    for (int64_t row = blockIdx.x; row < M; row += gridDim.x) {
        const float* rp = Ds + row * ldS;
        float xr[NR];
        auto elem = [&](int e, int64_t j) -> float { return EPT > 0 ? xr[e] : rp[j]; };
        if (EPT > 0) {
            #pragma unroll
            for (int e = 0; e < NR; ++e) {
                const int64_t j = (int64_t)e * QP_THREADS + tid;
                xr[e] = j < S ? __ldg(rp + j) : __int_as_float(0x7F800000);
            }
        }
        if (tid == 0) {
            sc.lo = 0xFFFFFFFFu;
            sc.hi = 0;
            sc.kept = 0;
            sc.bin = BBINS - 1;
            s_nfin = 0;
        }
        for (int i = tid; i < BBINS; i += QP_THREADS) hist[i] = 0;
        __syncthreads();
        float lo = __int_as_float(0x7F800000), hi = -__int_as_float(0x7F800000);
        int nfin = 0;
        auto for_each = [&](auto f) {
            if (EPT > 0) {
                #pragma unroll
                for (int e = 0; e < NR; ++e) f(elem(e, 0));
            } else {
                for (int64_t j = tid; j < S; j += QP_THREADS) f(elem(0, j));
            }
        };
        for_each([&](float x) {
            if (isfinite(x)) {
                lo = fminf(lo, x);
                hi = fmaxf(hi, x);
                ++nfin;
            }
        });
        for (int o = 16; o > 0; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(FULL, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(FULL, hi, o));
            nfin += __shfl_xor_sync(FULL, nfin, o);
        }
        if (lane == 0) {
            atomicAdd(&s_nfin, nfin);
            atomicMin(&sc.lo, ukey(lo));  // float min / max through the order-preserving keys
            atomicMax(&sc.hi, ukey(hi));
        }
        __syncthreads();
        if (s_nfin < r) {  // not reached for finite inputs (S - 1 >= r finite samples)
            if (tid == 0) thr[row] = nextafterf(s_nfin ? ukey_to_float(sc.hi) : -__int_as_float(0x7F800000), __int_as_float(0x7F800000));
            __syncthreads();
            continue;
        }
        const float fmn = ukey_to_float(sc.lo), fmx = ukey_to_float(sc.hi);
        const float span = fmx - fmn;
        const float scale = span > 0.0f && isfinite(span) && isfinite((float)BBINS / span) ? (float)BBINS / span : 0.0f;
        auto bucket = [&](float x) -> uint32_t {
            return min((uint32_t)((x - fmn) * scale), (uint32_t)(BBINS - 1));
        };
        for_each([&](float x) {
            if (isfinite(x)) atomicAdd(&hist[bucket(x)], 1u);
        });
        __syncthreads();
        // bucket holding the r-th finite sample (warp 0 scans 1024 bins, 32 per lane)
        if (tid < 32) {
            uint32_t c[32], sum = 0;
            #pragma unroll
            for (int j = 0; j < 32; ++j) {
                c[j] = hist[lane * 32 + j];
                sum += c[j];
            }
            uint32_t incl = sum;
            #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            uint32_t run = incl - sum;
            if (run < (uint32_t)r && (uint32_t)r <= incl) {
                #pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (run + c[j] >= (uint32_t)r) {
                        sc.bin = lane * 32 + j;
                        break;
                    }
                    run += c[j];
                }
            }
        }
        __syncthreads();
        const uint32_t bstar = sc.bin;
        float p = -__int_as_float(0x7F800000);
        for_each([&](float x) {
            if (isfinite(x) && bucket(x) <= bstar) p = fmaxf(p, x);
        });
        for (int o = 16; o > 0; o >>= 1) p = fmaxf(p, __shfl_xor_sync(FULL, p, o));
        if (lane == 0) atomicMax(reinterpret_cast<uint32_t*>(&sc.kept), ukey(p));
        __syncthreads();
        if (tid == 0) thr[row] = nextafterf(ukey_to_float((uint32_t)sc.kept), __int_as_float(0x7F800000));
        __syncthreads();
    }
}

// Warp-per-row form of the same pivot (no CTA barriers; rows re-read from L2): pass 1 the
// row's finite min / max, pass 2 a warp-private 1024-bucket histogram, a warp scan for the
// bucket b* holding the r-th sample, pass 3 the largest sample in buckets <= b*.
constexpr int QPW_WARPS = 8;
__global__ void __launch_bounds__(32 * QPW_WARPS)
pivot_from_sample_warp_kernel(const float* __restrict__ Ds, int64_t M, int64_t S, int64_t ldS, int r,
                              float* __restrict__ thr) {
    __shared__ uint32_t hist_all[QPW_WARPS][BBINS];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t* hist = hist_all[w];
    const int64_t gw = (int64_t)blockIdx.x * QPW_WARPS + w, nw = (int64_t)gridDim.x * QPW_WARPS;
    const bool vec = (S % 4 == 0) && (ldS % 4 == 0) && ((reinterpret_cast<uintptr_t>(Ds) & 15) == 0);
    for (int64_t row = gw; row < M; row += nw) {
        const float* rp = Ds + row * ldS;
        auto for_each = [&](auto f) {
            if (vec) {
                const float4* r4 = reinterpret_cast<const float4*>(rp);
                for (int64_t j = lane; j < S / 4; j += 32) {
                    const float4 x = __ldg(r4 + j);
                    f(x.x); f(x.y); f(x.z); f(x.w);
                }
            } else {
                for (int64_t j = lane; j < S; j += 32) f(__ldg(rp + j));
            }
        };
        for (int i = lane; i < BBINS; i += 32) hist[i] = 0;
        float lo = __int_as_float(0x7F800000), hi = -__int_as_float(0x7F800000);
        int nfin = 0;
        for_each([&](float x) {
            if (isfinite(x)) {
                lo = fminf(lo, x);
                hi = fmaxf(hi, x);
                ++nfin;
            }
        });
        for (int o = 16; o > 0; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(FULL, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(FULL, hi, o));
            nfin += __shfl_xor_sync(FULL, nfin, o);
        }
        if (nfin < r) {  // not reached for finite inputs (S - 1 >= r finite samples)
            if (lane == 0) thr[row] = nextafterf(nfin ? hi : -__int_as_float(0x7F800000), __int_as_float(0x7F800000));
            __syncwarp();
            continue;
        }
        const float span = hi - lo;
        const float scale = span > 0.0f && isfinite(span) && isfinite((float)BBINS / span) ? (float)BBINS / span : 0.0f;
        auto bucket = [&](float x) -> uint32_t { return min((uint32_t)((x - lo) * scale), (uint32_t)(BBINS - 1)); };
        __syncwarp();
        for_each([&](float x) {
            if (isfinite(x)) atomicAdd(&hist[bucket(x)], 1u);
        });
        __syncwarp();
        uint32_t c[BBINS / 32], sum = 0;
        #pragma unroll
        for (int j = 0; j < BBINS / 32; ++j) {
            c[j] = hist[lane * (BBINS / 32) + j];
            sum += c[j];
        }
        uint32_t incl = sum;
        #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        uint32_t run = incl - sum, mybin = 0xFFFFFFFFu;
        if (run < (uint32_t)r && (uint32_t)r <= incl) {
            #pragma unroll
            for (int j = 0; j < BBINS / 32; ++j) {
                if (mybin == 0xFFFFFFFFu && run + c[j] >= (uint32_t)r) mybin = lane * (BBINS / 32) + j;
                run += c[j];
            }
        }
        const uint32_t bstar = __reduce_min_sync(FULL, mybin);
        float p = -__int_as_float(0x7F800000);
        for_each([&](float x) {
            if (isfinite(x) && bucket(x) <= bstar) p = fmaxf(p, x);
        });
        for (int o = 16; o > 0; o >>= 1) p = fmaxf(p, __shfl_xor_sync(FULL, p, o));
        if (lane == 0) thr[row] = nextafterf(p, __int_as_float(0x7F800000));  // nextup: u < thr <=> u <= P
        __syncwarp();
    }
}

// Exact select over the partition's candidate lists for k > 32: one CTA per row loads the
// row's candidates (ukeys of the distances + column) into shared memory and runs the
// bucket finish (or the exact radix + bitonic finish).  Certificate: fewer than k
// candidates (or an overflowed list) sets flag bit 2, and the caller redoes the call.
constexpr int CS_THREADS = 256;
constexpr int CS_BINS = 4096;
__global__ void __launch_bounds__(CS_THREADS, 4)
candidate_select_large_kernel(const int32_t* __restrict__ cnt, const uint64_t* __restrict__ cent,
                              int32_t cap, int64_t M, int k,
                              int KP, int64_t idx_offset, int32_t* __restrict__ out_idx,
                              float* __restrict__ out_dist, int32_t* __restrict__ flag,
                              const int32_t* __restrict__ list) {
    extern __shared__ uint32_t smem[];
    uint32_t* ckey = smem;
    uint32_t* cidx = ckey + cap;
    uint32_t* kkey = cidx + cap;
    uint32_t* kidx = kkey + KP;
    uint32_t* hist = kidx + KP;  // CS_BINS
    __shared__ Scal sc;
    const int64_t nrows = list ? (int64_t)list[0] : M;
    for (int64_t i_row = blockIdx.x; i_row < nrows; i_row += gridDim.x) {
        const int64_t row = list ? (int64_t)list[1 + i_row] : i_row;
        const int n = cnt[row];
        if (threadIdx.x == 0 && !list)  // diagnostic: candidates kept (knn_last_candidates)
            atomicAdd(reinterpret_cast<unsigned long long*>(flag + 2), (unsigned long long)n);
        if (n > cap || n < k) {
            if (threadIdx.x == 0) atomicOr(flag, 2);
            continue;
        }
        // all of this thread's loads in flight before the shared-memory stores
        const unsigned long long* ge = reinterpret_cast<const unsigned long long*>(cent + row * cap);
        for (int i0 = 0; i0 < n; i0 += 8 * CS_THREADS) {
            uint64_t ev[8];
            #pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * CS_THREADS + threadIdx.x;
                ev[u] = i < n ? __ldcs(ge + i) : 0ull;
            }
            #pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * CS_THREADS + threadIdx.x;
                if (i < n) {
                    ckey[i] = (uint32_t)(ev[u] >> 32);
                    cidx[i] = (uint32_t)ev[u];
                }
            }
        }
        __syncthreads();
        if (!block_finish_bucket<CS_THREADS, CS_BINS>(ckey, cidx, n, k, kkey, kidx, hist, &sc, idx_offset,
                                                       out_idx + row * k, out_dist + row * k))
            block_finish<CS_THREADS>(ckey, cidx, n, k, KP, kkey, kidx, hist, &sc, idx_offset,
                                     out_idx + row * k, out_dist + row * k);
        __syncthreads();
    }
}

// Warp-per-row form (the default for k > 32): the bucket finish of block_finish_bucket done
// by one warp with warp-private buckets and output, the candidates re-read from global
// memory (L2) in three passes (key range; 1024-bucket histogram; scatter), no CTA
// barriers.  Rows whose buckets are crowded, or whose keys are non-finite, are appended
// to redo[1..] for the CTA kernel above.
constexpr int CSW_WARPS = 4;  // 4-warp CTAs, 5 per SM (20 warps) with the 10.8 KB slabs
constexpr int CSW_BINS = 1024;  // 16-bit counters, two per word (n <= cap < 2^16); 2048 measured
                                // slower at C4 (0.58 -> 0.67 ms: the per-lane bin scan doubles)
constexpr int CSW_STAR = 64;
constexpr int CSW_PASS = 16;
constexpr int CSW_EPT = 8;
__host__ __device__ constexpr size_t csw_slab_bytes(int KP) {
    return (size_t)CSW_BINS * 2 + (size_t)KP * 8 + (size_t)CSW_STAR * 8 + 16;
}
__global__ void __launch_bounds__(32 * CSW_WARPS)
candidate_select_warp_kernel(const int32_t* __restrict__ cnt, const uint64_t* __restrict__ cent,
                             int32_t cap, int64_t M, int k, int KP,
                             int64_t idx_offset, int32_t* __restrict__ out_idx, float* __restrict__ out_dist,
                             int32_t* __restrict__ flag, int32_t* __restrict__ redo) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint8_t* slab = smem_raw + csw_slab_bytes(KP) * w;
    uint64_t* star = reinterpret_cast<uint64_t*>(slab);
    uint32_t* hist = reinterpret_cast<uint32_t*>(star + CSW_STAR);
    uint32_t* okey = hist + CSW_BINS / 2;
    uint32_t* oidx = okey + KP;
    int* nst = reinterpret_cast<int*>(oidx + KP);
    const int64_t gw = (int64_t)blockIdx.x * CSW_WARPS + w, nw = (int64_t)gridDim.x * CSW_WARPS;
    for (int64_t row = gw; row < M; row += nw) {
        const int n = cnt[row];
        if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(flag + 2), (unsigned long long)n);
        if (n > cap || n < k) {  // overflow or failed certificate: the caller redoes the call
            if (lane == 0) atomicOr(flag, 2);
            continue;
        }
        // the row's entries (ukey << 32 | col): keys are the odd words, columns the even ones
        const uint32_t* gi = reinterpret_cast<const uint32_t*>(cent + row * cap);
        const uint32_t* gk = gi + 1;
        auto to_redo = [&]() {
            if (lane == 0) {
                const int slot = atomicAdd(redo, 1);
                redo[1 + slot] = (int32_t)row;
            }
            __syncwarp();
        };
        // pass 1: key range
        // (every pass loads CSW_EPT elements per lane before using them: the loads are
        // L2 latency bound, one outstanding load per lane would stall each iteration)
        uint32_t kmin = 0xFFFFFFFFu, kmax = 0;
        for (int base = 0; base < n; base += 32 * CSW_EPT) {
            uint32_t kv[CSW_EPT];
            #pragma unroll
            for (int j = 0; j < CSW_EPT; ++j) {
                const int i = base + 32 * j + lane;
                kv[j] = i < n ? __ldcg(gk + 2 * i) : 0xFFFFFFFFu;
            }
            #pragma unroll
            for (int j = 0; j < CSW_EPT; ++j) {
                kmin = min(kmin, kv[j]);
                if (base + 32 * j + lane < n) kmax = max(kmax, kv[j]);
            }
        }
        kmin = __reduce_min_sync(FULL, kmin);
        kmax = __reduce_max_sync(FULL, kmax);
        const float fmn = ukey_to_float(kmin), fmx = ukey_to_float(kmax);
        const float span = fmx - fmn;
        const float scale = (float)CSW_BINS / span;
        if (!(isfinite(fmn) && isfinite(fmx) && span > 0.0f && isfinite(span) && isfinite(scale))) {
            to_redo();
            continue;
        }
        auto bucket = [&](uint32_t key) -> uint32_t {
            return min((uint32_t)((ukey_to_float(key) - fmn) * scale), (uint32_t)(CSW_BINS - 1));
        };
        for (int i = lane; i < CSW_BINS / 2; i += 32) hist[i] = 0;
        if (lane == 0) *nst = 0;
        __syncwarp();
        // pass 2: histogram
        for (int base = 0; base < n; base += 32 * CSW_EPT) {
            uint32_t kv[CSW_EPT];
            #pragma unroll
            for (int j = 0; j < CSW_EPT; ++j) {
                const int i = base + 32 * j + lane;
                kv[j] = i < n ? __ldcg(gk + 2 * i) : 0u;
            }
            #pragma unroll
            for (int j = 0; j < CSW_EPT; ++j)
                if (base + 32 * j + lane < n) {
                    const uint32_t b = bucket(kv[j]);
                    atomicAdd(&hist[b >> 1], 1u << ((b & 1) * 16));
                }
        }
        __syncwarp();
        // exclusive offsets; b* = bucket of rank k; the largest bucket below b*
        constexpr int BPL = CSW_BINS / 32;
        uint32_t c[BPL], sum = 0;
        #pragma unroll
        for (int j = 0; j < BPL; j += 2) {
            const uint32_t wd = hist[(lane * BPL + j) >> 1];
            c[j] = wd & 0xFFFFu;
            c[j + 1] = wd >> 16;
            sum += c[j] + c[j + 1];
        }
        uint32_t incl = sum;
        #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        uint32_t run = incl - sum, mybin = 0xFFFFFFFFu, mybefore = 0, myn = 0;
        #pragma unroll
        for (int j = 0; j < BPL; ++j) {
            if (j & 1) hist[(lane * BPL + j) >> 1] = (run << 16) | (run - c[j - 1]);
            if (mybin == 0xFFFFFFFFu && run < (uint32_t)k && (uint32_t)k <= run + c[j]) {
                mybin = lane * BPL + j;
                mybefore = run;
                myn = c[j];
            }
            run += c[j];
        }
        const uint32_t bstar = __reduce_min_sync(FULL, mybin);
        const int owner = (int)(bstar / BPL);
        const uint32_t before = __shfl_sync(FULL, mybefore, owner);
        const uint32_t nstar = __shfl_sync(FULL, myn, owner);
        uint32_t mymax = 0;
        #pragma unroll
        for (int j = 0; j < BPL; ++j)
            if ((uint32_t)(lane * BPL + j) < bstar) mymax = max(mymax, c[j]);
        const uint32_t maxc = __reduce_max_sync(FULL, mymax);
        if (nstar > CSW_STAR || maxc > CSW_PASS) {
            to_redo();
            continue;
        }
        __syncwarp();
        // pass 3: scatter below b*, collect b*
        for (int base = 0; base < n; base += 32 * CSW_EPT) {
            uint32_t kv[CSW_EPT], iv[CSW_EPT];
            #pragma unroll
            for (int j = 0; j < CSW_EPT; ++j) {
                const int i = base + 32 * j + lane;
                kv[j] = i < n ? __ldcs(gk + 2 * i) : 0xFFFFFFFFu;
                iv[j] = i < n ? __ldcs(gi + 2 * i) : 0u;
            }
            #pragma unroll
            for (int j = 0; j < CSW_EPT; ++j) {
                if (base + 32 * j + lane >= n) continue;
                const uint32_t b = bucket(kv[j]);
                if (b < bstar) {
                    const uint32_t sh = (b & 1) * 16;
                    const uint32_t pos = (atomicAdd(&hist[b >> 1], 1u << sh) >> sh) & 0xFFFFu;
                    okey[pos] = kv[j];
                    oidx[pos] = iv[j];
                } else if (b == bstar) {
                    const int q = atomicAdd(nst, 1);
                    star[q] = (uint64_t)kv[j] << 32 | iv[j];
                }
            }
        }
        __syncwarp();
        {   // b*'s candidates sorted (<= 64, two per lane); the first k - before appended
            uint64_t a0 = lane < (int)nstar ? star[lane] : ~0ull;
            uint64_t a1 = lane + 32 < (int)nstar ? star[lane + 32] : ~0ull;
            #pragma unroll
            for (int size = 2; size <= 64; size <<= 1) {
                #pragma unroll
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    if (stride == 32) {
                        const bool sw = a1 < a0;
                        const uint64_t x = a0;
                        a0 = sw ? a1 : a0;
                        a1 = sw ? x : a1;
                    } else {
                        #pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            uint64_t& v = h ? a1 : a0;
                            const int p = lane + 32 * h;
                            const uint64_t o = __shfl_xor_sync(FULL, v, stride);
                            const bool up = ((p & size) == 0) == ((p & stride) == 0);
                            v = ((o < v) == up) ? o : v;
                        }
                    }
                }
            }
            const uint32_t need = (uint32_t)k - before;
            if ((uint32_t)lane < need) {
                okey[before + lane] = (uint32_t)(a0 >> 32);
                oidx[before + lane] = (uint32_t)a0;
            }
            if ((uint32_t)lane + 32 < need) {
                okey[before + lane + 32] = (uint32_t)(a1 >> 32);
                oidx[before + lane + 32] = (uint32_t)a1;
            }
        }
        __syncwarp();
        // odd-even transposition inside the buckets below b* (maxc passes); a lane per
        // bucket (insertion sort) measured slower: the counts are skewed toward b*, so the
        // few lanes holding the dense buckets serialise the warp
        for (uint32_t pass = 0; pass < maxc; ++pass) {
            for (uint32_t p = 2 * lane + (pass & 1); p + 1 < before; p += 64) {
                const uint32_t k0 = okey[p], k1 = okey[p + 1], i0 = oidx[p], i1 = oidx[p + 1];
                if (k1 < k0 || (k1 == k0 && i1 < i0)) {
                    okey[p] = k1;
                    okey[p + 1] = k0;
                    oidx[p] = i1;
                    oidx[p + 1] = i0;
                }
            }
            __syncwarp();
        }
        for (int q = lane; q < k; q += 32) {
            out_idx[row * k + q] = (int32_t)((int64_t)oidx[q] + idx_offset);
            out_dist[row * k + q] = ukey_to_float(okey[q]);
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------ multi-GPU gather -------
// Symmetric multi-GPU k-NNG: the G ranks' partial candidate lists of rows [row0, row0+rows)
// (list g may live in a peer GPU's memory, mapped with CUDA IPC: the reads cross NVLink)
// are concatenated into one local list per row.  Warp per row.  A source list that
// overflowed (cnt > cap_src) or a row whose concatenation exceeds cap_dst sets flag bit 2.
struct SrcLists {
    const int32_t* cnt[64];
    const uint64_t* ent[64];
};
__global__ void __launch_bounds__(256)
gather_lists_kernel(const SrcLists src, int G, int cap_src, int64_t row0, int64_t rows, int cap_dst,
                    int32_t* __restrict__ cnt_dst, uint64_t* __restrict__ ent_dst, int32_t* __restrict__ flag) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (r >= rows) return;
    const int64_t row = row0 + r;
    int total = 0;
    bool bad = false;
    for (int g = 0; g < G; ++g) {
        int n = src.cnt[g][row];
        if (n > cap_src) {
            bad = true;
            n = cap_src;
        }
        const uint64_t* se = src.ent[g] + row * cap_src;
        for (int i = lane; i < n; i += 32) {
            const int o = total + i;
            if (o < cap_dst) ent_dst[r * cap_dst + o] = se[i];
        }
        total += n;
    }
    if (total > cap_dst) bad = true;
    if (lane == 0) {
        cnt_dst[r] = total < cap_dst ? total : cap_dst;
        if (bad) atomicOr(flag, 2);
    }
}

}  // namespace

int g_last_select_kind = -1, g_last_select_splits = 1;

cudaError_t launch_select(const float* D, int64_t M, int64_t N, int64_t ldD, int32_t k,
                          int64_t idx_offset, int32_t* out_idx, float* out_dist, int32_t* redo,
                          cudaStream_t s) {
    if (M == 0) return cudaSuccess;
    const int KP = next_pow2(k);
    const bool aligned = (ldD % 4 == 0) && ((reinterpret_cast<uintptr_t>(D) & 15) == 0);
    cudaError_t e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static const int warp_maxk = [] {
        const char* v = getenv("KNN_WARP_MAXK");  // tuning knob: largest k of the warp path
        const int x = v ? atoi(v) : WSEL_K;
        return x < 0 ? 0 : x > WSEL_K ? WSEL_K : x;
    }();
    // two-pass warp per row (pivot = k-th smallest group minimum) for k <= 32 on rows of
    // 1024..131072 elements; measured against the running-threshold warp select below:
    //
    static const bool two_pass = !getenv_flag("KNN_SELECT_ONEPASS");
    if (two_pass && aligned && k <= 32 && N >= 32 * (int64_t)k && N >= WSEL_C && N <= WS2_MAXN &&
        M >= 4 * (int64_t)sms) {
        int S = 3;
        if (const char* v = getenv("KNN_WS2_STAGES")) S = atoi(v);  // tuning knob
        S = S < 2 ? 2 : S > WS2_MAXS ? WS2_MAXS : S;
        const size_t smem = (size_t)ws2_slab_bytes(N, S);
        if ((e = set_smem(select_warp2p_kernel, smem)) != cudaSuccess) return e;
        int per_sm = 0;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_warp2p_kernel, 32, smem)) !=
            cudaSuccess)
            return e;
        int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
        if (grid > M) grid = M;
        select_warp2p_kernel<<<(unsigned)grid, 32, smem, s>>>(D, M, N, ldD, k, S, idx_offset, out_idx, out_dist);
        g_last_select_kind = 4;
        g_last_select_splits = 1;
        return cudaGetLastError();
    }
    // warp per row for k <= 32; k > 32 goes to the CTA ring (sampled pivot, bucket finish):
    // measured 8192-long rows k = 64: 0.15 vs 0.30 ms, 65536-long rows k = 64: 3.6 vs
    // 6.5 ms (scripts/select_short.sh, select_mini.sh)
    if (aligned && k <= warp_maxk && k <= 32 && M >= 4 * (int64_t)sms) {
        // warp per row: enough rows to give every SM >= 4 warps
        // k <= 32 folds every 32 survivors into the sorted register list; larger k
        // rebuilds the buffer once it passes max(2k, k + 64)
        const int limit = k <= 32 ? 31 : (int)round_up(k + 64 > 2 * k ? k + 64 : 2 * k, 32);
        const int cap = WSEL_SUB + limit + 1;
        const size_t smem = (size_t)wsel_slab_bytes(cap) * WSEL_WARPS;
        auto pick = [&](auto kern) -> cudaError_t {
            cudaError_t e2;
            if ((e2 = set_smem(kern, smem)) != cudaSuccess) return e2;
            int per_sm = 0;
            if ((e2 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * WSEL_WARPS, smem)) != cudaSuccess)
                return e2;
            int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
            const int64_t need = ceil_div(M, WSEL_WARPS);
            if (grid > need) grid = need;
            kern<<<(unsigned)grid, 32 * WSEL_WARPS, smem, s>>>(D, M, N, ldD, k, cap, limit, idx_offset,
                                                               out_idx, out_dist);
            return cudaGetLastError();
        };
        g_last_select_kind = 0;
        g_last_select_splits = 1;
        if (k <= 32) return pick(select_warp_kernel<1>);
        if (k <= 64) return pick(select_warp_kernel<2>);
        return pick(select_warp_kernel<4>);
    }
    if (aligned && M < sms && N >= 2 * 4096 && !getenv_flag("KNN_NO_CLUSTER_SELECT")) {
        // few rows: a cluster of S CTAs per row (select_cluster_kernel)
        constexpr int CT = 256, CHUNK = 4096, STAGES = 4;
        int S = 1;
        while (S < 16 && (int64_t)S * M < sms && (int64_t)(2 * S) * CHUNK <= N) S <<= 1;
        if (S > 1) {
            const int64_t L = round_up(ceil_div(N, S), CHUNK);
            int cap, limit;
            if (L <= CHUNK) {
                cap = (int)round_up(L, 32);
                limit = INT_MAX;
            } else {
                limit = (int)round_up(k + 256 > 2 * k ? k + 256 : 2 * k, 32);
                cap = CHUNK + limit;
            }
            int r_pivot = 0;
            if (L >= 2 * CHUNK) {
                const double mean = (double)CHUNK * k / (double)L;
                const double r = std::ceil(mean + 4.0 * std::sqrt(mean) + 2.0);
                if (r < 0.75 * k) r_pivot = (int)r;
            }
            const size_t smem = (size_t)STAGES * CHUNK * 4 + 2 * STAGES * 8 +
                                (size_t)(2 * cap + 2 * KP + BBINS) * sizeof(uint32_t) + 3 * (size_t)KP * 8;
            auto kern = select_cluster_kernel<CT, CHUNK, STAGES>;
            if ((e = set_smem(kern, smem)) != cudaSuccess) return e;
            if (S > 8 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
                return e;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(M * S), 1, 1);
            cfg.blockDim = dim3(CT + 32, 1, 1);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = S;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, (void*)kern, &cfg) == cudaSuccess && nclusters > 0) {
                g_last_select_kind = 3;
                g_last_select_splits = S;
                e = cudaLaunchKernelEx(&cfg, kern, D, N, ldD, k, cap, KP, limit, L, idx_offset, out_idx,
                                       out_dist, r_pivot);
                return e != cudaSuccess ? e : cudaGetLastError();
            }
            cudaGetLastError();  // cluster shape not schedulable: fall through to one CTA per row
        }
    }
    if (aligned) {
        static const int ring_chunk = [] {  // tuning knob (A/B): 4096 (default) or 2048
            const char* v = getenv("KNN_RING_CHUNK");
            return v && atoi(v) == 2048 ? 2048 : 4096;
        }();
        auto ring = [&](auto chunk_c, auto k4, auto k3) -> cudaError_t {
        constexpr int CT = 256, CHUNK = decltype(chunk_c)::value;
        int cap, limit;
        if (N <= CHUNK) {
            cap = (int)round_up(N, 32);
            limit = INT_MAX;
        } else {
            limit = (int)round_up(k + 256 > 2 * k ? k + 256 : 2 * k, 32);
            cap = CHUNK + limit;
        }
        // sampled pivot (see select_ring_kernel): r = the rank in the first chunk whose
        // expected share of the row is ~k plus four standard deviations
        int r_pivot = 0;
        if (redo && N >= 2 * CHUNK) {
            const double mean = (double)CHUNK * k / (double)N;
            const double r = std::ceil(mean + 4.0 * std::sqrt(mean) + 2.0);
            if (r < 0.75 * k) r_pivot = (int)r;
        }
        if (r_pivot) KNN_CUDA_TRY(cudaMemsetAsync(redo, 0, sizeof(int32_t), s));
        auto run = [&](auto kern, int stages, const int32_t* list, int rp, int64_t grid_rows) -> cudaError_t {
            const size_t smem = (size_t)stages * CHUNK * 4 + 2 * stages * 8 +
                                (size_t)(2 * cap + 2 * KP + BBINS) * sizeof(uint32_t);
            cudaError_t e2;
            if ((e2 = set_smem(kern, smem)) != cudaSuccess) return e2;
            int per_sm = 0;
            if ((e2 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, CT + 32, smem)) != cudaSuccess)
                return e2;
            int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
            if (grid > grid_rows) grid = grid_rows;
            kern<<<(unsigned)grid, CT + 32, smem, s>>>(D, M, N, ldD, k, cap, KP, limit, idx_offset,
                                                      out_idx, out_dist, list, rp, redo);
            return cudaGetLastError();
        };
        g_last_select_kind = 1;
        g_last_select_splits = 1;
        // 4 ring stages when two CTAs still fit on an SM, else 3
        const size_t base_smem = (size_t)(2 * cap + 2 * KP + BBINS) * sizeof(uint32_t);
        const bool four = CHUNK < 4096 || base_smem + 4 * (size_t)CHUNK * 4 + 64 <= 112 * 1024;
        cudaError_t e3 = four ? run(k4, 4, nullptr, r_pivot, M) : run(k3, 3, nullptr, r_pivot, M);
        if (e3 != cudaSuccess || !r_pivot) return e3;
        // redo pass: rows whose sampled pivot kept fewer than k candidates (grid covers
        // any count; CTAs beyond it exit at once)
        return four ? run(k4, 4, redo, 0, M) : run(k3, 3, redo, 0, M);
        };
        // short rows: 2048-element slices, 3 CTAs per SM (n = 4096, k = 512: 1.85 -> 0.89 ms);
        // longer rows keep 4096 (a better sample for the pivot, fewer slices per row)
        if (ring_chunk == 2048 || N <= 8192)
            return ring(std::integral_constant<int, 2048>{}, select_ring_kernel<256, 2048, 4, 3>,
                        select_ring_kernel<256, 2048, 4, 3>);
        return ring(std::integral_constant<int, 4096>{}, select_ring_kernel<256, 4096, 4>,
                    select_ring_kernel<256, 4096, 3>);
    }
    constexpr int THREADS = 256, VPT = 4, CHUNK = THREADS * VPT * 4;
    int cap, limit;
    if (N <= CHUNK) {  // whole row fits: no rebuild during the stream
        cap = (int)round_up(N, 32);
        limit = INT_MAX;
    } else {
        // Rebuild as soon as more than max(2k, k + 256) candidates are buffered: the
        // first chunk (accepted whole) sets the threshold right away, after which a
        // random-order row adds ~k ln(N/CHUNK) survivors in total.
        limit = (int)round_up(k + 256 > 2 * k ? k + 256 : 2 * k, 32);
        cap = CHUNK + limit;
    }
    const size_t smem = (size_t)(2 * cap + 2 * KP + 256) * sizeof(uint32_t);
    auto kern = select_rows_kernel<THREADS, VPT, false>;
    g_last_select_kind = 2;
    g_last_select_splits = 1;
    if ((e = set_smem(kern, smem)) != cudaSuccess) return e;
    kern<<<(unsigned)M, THREADS, smem, s>>>(D, N, ldD, k, cap, KP, limit, idx_offset, out_idx,
                                           out_dist);
    return cudaGetLastError();
}

cudaError_t launch_pivot_from_mins(const float* mins, int64_t nchunk, int64_t M, int64_t pad_end, int32_t k,
                                   int32_t metric, float* thr, int32_t* cnt, cudaStream_t s) {
    if (M == 0) return cudaSuccess;
    if (k > 64 || nchunk < k) return cudaErrorInvalidValue;  // k: the pivot rank (<= 32 + self)
    if (pad_end < M) pad_end = M;
    pivot_from_mins_kernel<<<(unsigned)ceil_div(pad_end, PV_ROWS), 32 * PV_ROWS, 0, s>>>(mins, nchunk, M, pad_end,
                                                                                        k, metric, thr, cnt);
    return cudaGetLastError();
}

cudaError_t launch_candidate_select(const int32_t* cnt, const uint64_t* cent,
                                    int32_t cap, int64_t M, int32_t k, int64_t idx_offset,
                                    int32_t* out_idx, float* out_dist, int32_t* flag, cudaStream_t s,
                                    int32_t gate) {
    if (M == 0) return cudaSuccess;
    if (k > 32) return cudaErrorInvalidValue;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t blocks = std::min<int64_t>(ceil_div(M, 8), (int64_t)sms * 4);
    candidate_select_kernel<<<(unsigned)blocks, 256, 0, s>>>(cnt, cent, cap, M, k, idx_offset,
                                                                    out_idx, out_dist, flag, gate);
    return cudaGetLastError();
}

cudaError_t launch_merge_lists(const float* const* dist_lists, const int32_t* const* idx_lists, int32_t G,
                               int64_t row0, int64_t M, int32_t k, const int64_t* offsets_host,
                               int32_t* out_idx, float* out_dist, cudaStream_t s) {
    if (M == 0) return cudaSuccess;
    if (G < 1 || G > 64) return cudaErrorInvalidValue;
    constexpr int THREADS = 256, EPT = 4, CHUNK = THREADS * EPT;
    Offsets offs{};
    ListPtrs lists{};
    for (int g = 0; g < G; ++g) {
        offs.v[g] = offsets_host[g];
        lists.d[g] = dist_lists[g];
        lists.i[g] = idx_lists[g];
    }
    const int KP = next_pow2(k);
    const int64_t L = (int64_t)G * k;
    int cap, limit;
    if (L <= 2 * CHUNK + 2048) {
        cap = (int)round_up(L, 32);
        limit = INT_MAX;
    } else {
        cap = CHUNK + (int)round_up(k > CHUNK ? k : CHUNK, 32);
        limit = cap - CHUNK;
    }
    const size_t smem = (size_t)(2 * cap + 2 * KP + 256) * sizeof(uint32_t);
    auto kern = merge_kernel<THREADS, EPT>;
    cudaError_t e;
    if ((e = set_smem(kern, smem)) != cudaSuccess) return e;
    kern<<<(unsigned)M, THREADS, smem, s>>>(lists, row0, G, k, cap, KP, limit, offs, out_idx, out_dist);
    return cudaGetLastError();
}

cudaError_t launch_merge(const float* part_dist, const int32_t* part_idx, int32_t G, int64_t M,
                         int32_t k, const int64_t* offsets_host, int32_t* out_idx,
                         float* out_dist, cudaStream_t s) {
    if (G < 1 || G > 64) return cudaErrorInvalidValue;
    const float* dl[64];
    const int32_t* il[64];
    for (int g = 0; g < G; ++g) {  // contiguous [G][M][k]
        dl[g] = part_dist + (size_t)g * M * k;
        il[g] = part_idx + (size_t)g * M * k;
    }
    return launch_merge_lists(dl, il, G, 0, M, k, offsets_host, out_idx, out_dist, s);
}

cudaError_t launch_pivot_from_sample(const float* Ds, int64_t M, int64_t S, int64_t ldS, int32_t r,
                                     float* thr, cudaStream_t s) {
    if (M == 0) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (!getenv_flag("KNN_PIVOT_CTA")) {  // warp per row (default); env: the CTA-per-row form
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pivot_from_sample_warp_kernel, 32 * QPW_WARPS, 0);
        int64_t g = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
        if (g > ceil_div(M, QPW_WARPS)) g = ceil_div(M, QPW_WARPS);
        pivot_from_sample_warp_kernel<<<(unsigned)g, 32 * QPW_WARPS, 0, s>>>(Ds, M, S, ldS, r, thr);
        return cudaGetLastError();
    }
    int64_t grid = (int64_t)sms * 8;
    if (grid > M) grid = M;
    if (S <= 16 * QP_THREADS)
        pivot_from_sample_kernel<16><<<(unsigned)grid, QP_THREADS, 0, s>>>(Ds, M, S, ldS, r, thr);
    else if (S <= 32 * QP_THREADS)
        pivot_from_sample_kernel<32><<<(unsigned)grid, QP_THREADS, 0, s>>>(Ds, M, S, ldS, r, thr);
    else
        pivot_from_sample_kernel<0><<<(unsigned)grid, QP_THREADS, 0, s>>>(Ds, M, S, ldS, r, thr);
    return cudaGetLastError();
}

cudaError_t launch_candidate_select_large(const int32_t* cnt, const uint64_t* cent,
                                          int32_t cap, int64_t M, int32_t k, int64_t idx_offset,
                                          int32_t* out_idx, float* out_dist, int32_t* flag, int32_t* redo,
                                          cudaStream_t s) {
    if (M == 0) return cudaSuccess;
    const int KP = next_pow2(k);
    cudaError_t e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // warp per row while its slab fits and the 16-bit counters hold the list (always for
    // the API's k <= 1024)
    const bool warp = redo != nullptr && KP <= 2048 && cap < 65536 && !getenv_flag("KNN_CANDSEL_CTA");
    if (warp) {
        if ((e = cudaMemsetAsync(redo, 0, sizeof(int32_t), s)) != cudaSuccess) return e;
        const size_t wsm = csw_slab_bytes(KP) * CSW_WARPS;
        if ((e = set_smem(candidate_select_warp_kernel, wsm)) != cudaSuccess) return e;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, candidate_select_warp_kernel, 32 * CSW_WARPS, wsm);
        int64_t g = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
        if (g > ceil_div(M, CSW_WARPS)) g = ceil_div(M, CSW_WARPS);
        candidate_select_warp_kernel<<<(unsigned)g, 32 * CSW_WARPS, wsm, s>>>(cnt, cent, cap, M, k, KP,
                                                                            idx_offset, out_idx, out_dist, flag,
                                                                            redo);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (getenv_flag("KNN_CANDSEL_STATS")) {  // diagnostic: rows handed to the CTA kernel
            int32_t nr = 0;
            cudaMemcpyAsync(&nr, redo, sizeof(nr), cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            fprintf(stderr, "candidate_select_warp: %d of %lld rows redone\n", nr, (long long)M);
        }
    }
    // CTA per row: every row, or (after the warp kernel) the rows it could not bucket
    const size_t smem = (size_t)(2 * cap + 2 * KP + CS_BINS) * sizeof(uint32_t);
    if ((e = set_smem(candidate_select_large_kernel, smem)) != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, candidate_select_large_kernel, CS_THREADS, smem);
    int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (grid > M) grid = M;
    candidate_select_large_kernel<<<(unsigned)grid, CS_THREADS, smem, s>>>(cnt, cent, cap, M, k, KP,
                                                                          idx_offset, out_idx, out_dist, flag,
                                                                          warp ? redo : nullptr);
    return cudaGetLastError();
}

cudaError_t launch_candidate_recompute(const int32_t* cnt, const uint64_t* cent,
                                       int32_t cap, int64_t M, int32_t k, int64_t idx_offset, const float* Q,
                                       const float* X, int32_t d, const float* qn, const float* bq,
                                       const float* bx, const float* thr, int32_t metric, int32_t* out_idx,
                                       float* out_dist, int32_t* flag, cudaStream_t s, int32_t gate) {
    if (M == 0) return cudaSuccess;
    if (k < 1 || k > 32 || metric < 0 || metric > 1) return cudaErrorInvalidValue;
    // relative error bound of the fp32 re-evaluation: d/32 sequential fmas per lane, a
    // 5-level shuffle tree, the difference and (L2) the sqrt, each 2^-24 relative
    const float rerr = (float)(((d + 31) / 32 + 8) * std::ldexp(1.0, -24));
    const int vec = ((d % 4 == 0) && ((reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(X)) & 15) == 0) |
                    (getenv_flag("KNN_RECOMP_STATS") ? 2 : 0);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t blocks = std::min<int64_t>(ceil_div(M, 8), (int64_t)sms * KNN_CR_MINB);
    candidate_recompute_kernel<<<(unsigned)blocks, 256, 0, s>>>(cnt, cent, cap, M, k, idx_offset, Q,
                                                                       X, d, qn, bq, bx, thr, rerr, metric, vec,
                                                                       out_idx, out_dist, flag, gate);
    return cudaGetLastError();
}

cudaError_t launch_gather_lists(const int32_t* const* cnts, const uint64_t* const* ents,
                                int32_t G, int32_t cap_src, int64_t row0, int64_t rows, int32_t cap_dst,
                                int32_t* cnt_dst, uint64_t* ent_dst, int32_t* flag, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    if (G < 1 || G > 64) return cudaErrorInvalidValue;
    SrcLists src{};
    for (int g = 0; g < G; ++g) {
        src.cnt[g] = cnts[g];
        src.ent[g] = ents[g];
    }
    gather_lists_kernel<<<(unsigned)ceil_div(rows, 8), 256, 0, s>>>(src, G, cap_src, row0, rows, cap_dst, cnt_dst,
                                                                    ent_dst, flag);
    return cudaGetLastError();
}

}  // namespace knn
