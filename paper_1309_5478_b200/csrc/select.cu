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

#include <climits>

namespace knn {
namespace {

constexpr uint32_t FULL = 0xFFFFFFFFu;

struct Scal {
    uint32_t bin, before, neq;
    int kept;
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
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
    __syncthreads();
    for (int i = tid; i < cnt; i += THREADS) {
        uint32_t key = ckey[i];
        uint32_t v = on_idx ? cidx[i] : key;
        bool ok = on_idx ? (key == key_eq) : true;
        if (ok && (v & mask) == prefix) atomicAdd(&hist[(v >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
        const int lane = tid;
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
    __syncthreads();
}

// Exact selection of the k best (key, idx) among cnt >= k candidates.  Writes them
// (unordered) to kkey/kidx[0, k) and returns the k-th best pair in (Tkey, Tidx).
// exact_idx: compute Tidx even when every candidate equal to Tkey is kept (needed by
// the composite threshold of the merge); otherwise Tidx = UINT_MAX in that case.
template <int THREADS>
__device__ void block_select_k(const uint32_t* ckey, const uint32_t* cidx, int cnt, int k,
                               uint32_t* kkey, uint32_t* kidx, uint32_t* hist, Scal* sc,
                               bool exact_idx, uint32_t& Tkey, uint32_t& Tidx) {
    uint32_t prefix = 0, mask = 0, rank = (uint32_t)k, neq = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        radix_pass<THREADS>(ckey, cidx, cnt, false, 0, prefix, mask, shift, rank, hist, sc);
        rank -= sc->before;
        prefix |= sc->bin << shift;
        mask |= 0xFFu << shift;
        neq = sc->neq;
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
    __syncthreads();
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
    __syncthreads();
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
            __syncthreads();
        }
    }
}

// The finishing steps shared by select and merge: exact k, sort, write.
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
    __syncthreads();
    block_bitonic<THREADS>(kkey, kidx, KP);
    for (int r = threadIdx.x; r < k; r += THREADS) {
        out_idx[r] = (int32_t)((int64_t)kidx[r] + idx_offset);
        out_dist[r] = ukey_to_float(kkey[r]);
    }
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

__device__ __forceinline__ float f4get(const float4& v, int c) {
    return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}

// ------------------------------------------------------------------ select kernel ----
// One CTA per row.  VEC: rows are 16-byte aligned (ldD % 4 == 0) -> 128-bit loads.
// Element e = 4*j + c of a thread in the chunk at `base` sits at column
//   VEC:  base + 4*(j*THREADS + tid) + c        (one float4 per j)
//   else: base + (4*j + c)*THREADS + tid        (coalesced scalars)
template <int THREADS, int VPT, bool VEC>
__global__ void __launch_bounds__(THREADS)
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

    auto col = [&](int64_t base, int e) -> int64_t {
        return VEC ? base + 4 * ((int64_t)(e >> 2) * THREADS + tid) + (e & 3)
                   : base + (int64_t)e * THREADS + tid;
    };
    auto load = [&](float4* v, int64_t base) {
        #pragma unroll
        for (int j = 0; j < VPT; ++j) {
            if (VEC) {
                int64_t c0 = col(base, 4 * j);
                v[j] = c0 < N ? ld_stream4(rp + c0) : make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
                float t[4];
                #pragma unroll
                for (int c = 0; c < 4; ++c) {
                    int64_t cc = col(base, 4 * j + c);
                    t[c] = cc < N ? ld_stream1(rp + cc) : 0.0f;
                }
                v[j] = make_float4(t[0], t[1], t[2], t[3]);
            }
        }
    };

    float4 cur[VPT], nxt[VPT];
    load(cur, 0);
    __syncthreads();
    for (int64_t base = 0; base < N; base += CHUNK) {
        if (base + CHUNK < N) load(nxt, base + CHUNK);
        const bool full = base + CHUNK <= N;
        uint32_t pm = 0;
        #pragma unroll
        for (int e = 0; e < EPT; ++e) {
            bool ok = ukey(f4get(cur[e >> 2], e & 3)) < T;
            if (!full) ok = ok && col(base, e) < N;
            pm |= (uint32_t)ok << e;
        }
        int my = __popc(pm);
        bool over = false;
        if (__any_sync(FULL, my != 0)) {
            // warp-inclusive scan of the per-thread survivor counts, one shared atomic
            // per warp (the paper's counters g_< kept in shared memory)
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
            for (int e = 0; e < EPT; ++e) {
                if (pm & (1u << e)) {
                    ckey[off] = ukey(f4get(cur[e >> 2], e & 3));
                    cidx[off] = (uint32_t)col(base, e);
                    ++off;
                }
            }
        }
        if (__syncthreads_or(over)) {
            uint32_t tk, ti;
            block_select_k<THREADS>(ckey, cidx, s_count, k, kkey, kidx, hist, &sc, false, tk, ti);
            for (int i = tid; i < k; i += THREADS) {
                ckey[i] = kkey[i];
                cidx[i] = kidx[i];
            }
            if (tid == 0) s_count = k;
            T = tk;
            __syncthreads();
        }
        #pragma unroll
        for (int j = 0; j < VPT; ++j) cur[j] = nxt[j];
    }
    __syncthreads();
    block_finish<THREADS>(ckey, cidx, s_count, k, KP, kkey, kidx, hist, &sc, idx_offset,
                          out_idx + row * k, out_dist + row * k);
}

// ------------------------------------------------------------------ merge kernel -----
struct Offsets {
    int64_t v[64];
};

template <int THREADS, int EPT>
__global__ void __launch_bounds__(THREADS)
merge_kernel(const float* __restrict__ part_dist, const int32_t* __restrict__ part_idx, int G,
             int64_t M, int k, int cap, int KP, int limit, Offsets offs,
             int32_t* __restrict__ out_idx, float* __restrict__ out_dist) {
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
                int64_t off = ((int64_t)g * M + row) * k + r;
                u[e] = ukey(__ldg(part_dist + off));
                id[e] = (uint32_t)((int64_t)__ldg(part_idx + off) + offs.v[g]);
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
        if (__syncthreads_or(over)) {
            uint32_t tk, ti;
            block_select_k<THREADS>(ckey, cidx, s_count, k, kkey, kidx, hist, &sc, true, tk, ti);
            for (int i = tid; i < k; i += THREADS) {
                ckey[i] = kkey[i];
                cidx[i] = kidx[i];
            }
            if (tid == 0) s_count = k;
            T = tk;
            Ti = ti;
            __syncthreads();
        }
    }
    __syncthreads();
    block_finish<THREADS>(ckey, cidx, s_count, k, KP, kkey, kidx, hist, &sc, 0,
                          out_idx + row * k, out_dist + row * k);
}

int next_pow2(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

template <class K>
cudaError_t set_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

cudaError_t launch_select(const float* D, int64_t M, int64_t N, int64_t ldD, int32_t k,
                          int64_t idx_offset, int32_t* out_idx, float* out_dist, cudaStream_t s) {
    if (M == 0) return cudaSuccess;
    constexpr int THREADS = 256, VPT = 2, CHUNK = THREADS * VPT * 4;
    const int KP = next_pow2(k);
    int cap, limit;
    if (N <= CHUNK) {  // whole row fits: no rebuild during the stream
        cap = (int)round_up(N, 32);
        limit = INT_MAX;
    } else {
        cap = CHUNK + (int)round_up(k > CHUNK ? k : CHUNK, 32);
        limit = cap - CHUNK;
    }
    const size_t smem = (size_t)(2 * cap + 2 * KP + 256) * sizeof(uint32_t);
    const bool vec = (ldD % 4 == 0) && ((reinterpret_cast<uintptr_t>(D) & 15) == 0);
    cudaError_t e;
    if (vec) {
        auto kern = select_rows_kernel<THREADS, VPT, true>;
        if ((e = set_smem(kern, smem)) != cudaSuccess) return e;
        kern<<<(unsigned)M, THREADS, smem, s>>>(D, N, ldD, k, cap, KP, limit, idx_offset, out_idx,
                                               out_dist);
    } else {
        auto kern = select_rows_kernel<THREADS, VPT, false>;
        if ((e = set_smem(kern, smem)) != cudaSuccess) return e;
        kern<<<(unsigned)M, THREADS, smem, s>>>(D, N, ldD, k, cap, KP, limit, idx_offset, out_idx,
                                               out_dist);
    }
    return cudaGetLastError();
}

cudaError_t launch_merge(const float* part_dist, const int32_t* part_idx, int32_t G, int64_t M,
                         int32_t k, const int64_t* offsets_host, int32_t* out_idx,
                         float* out_dist, cudaStream_t s) {
    if (M == 0) return cudaSuccess;
    if (G < 1 || G > 64) return cudaErrorInvalidValue;
    constexpr int THREADS = 256, EPT = 4, CHUNK = THREADS * EPT;
    Offsets offs{};
    for (int g = 0; g < G; ++g) offs.v[g] = offsets_host[g];
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
    kern<<<(unsigned)M, THREADS, smem, s>>>(part_dist, part_idx, G, M, k, cap, KP, limit, offs,
                                           out_idx, out_dist);
    return cudaGetLastError();
}

}  // namespace knn
