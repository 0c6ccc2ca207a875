// select_paper.cu — ablation: the paper's own quick multi-select, as written (NEXT-3).
//
// PAPER.md:49-56 ("GPU-based quick multi-select"), one warp per query (PAPER.md:50,
// "Each array is handled by a single thread warp"):
//   * a pivot is chosen and the row is partitioned into an auxiliary array in global
//     memory, 32 elements at a time: every lane holds one element in a register, the vote
//     B = __ballot(x >= pivot) tells each lane its slot in a 32-wide shared-memory array
//     (elements < pivot packed from the left end, >= pivot from the right end, slot =
//     popc of the lower lanes' votes; Fig 1-2), and the warp writes the
//     array out with two coalesced writes, the left part at the running counter g_< and
//     the right part at g_>= counted from the end of the range (Fig 3);
//   * with L elements left of the pivot: K < L -> continue on the left side only; K > L
//     -> keep the left side as it is (a reference, not a copy: the "stack of references"
//     of PAPER.md:56), K -= L, continue on the right side; K = L -> done (reading R11).
//     Input and auxiliary arrays swap roles after each pass;
//   * once the live range is small (<= 1024) it is sorted directly in shared memory
//     (the bitonic finish of PAPER.md:47) and its first K elements are taken.
// Differences from the paper, needed for exact results (readings R1, R2, R12): elements are
// (key, index) pairs ordered by the composite order, so every partition is strict and
// ties are broken by index; the pivot is the element at a position drawn from a
// counter-based hash of (row, pass) (the Cederman recap's random pivot, PAPER.md:47,
// made reproducible); the k results are sorted at the end.
//
// This kernel is NOT on the product path: it exists to measure the paper's algorithm on
// B200 next to the single-pass select (scripts/select_sweep.py).
#include "internal.cuh"

namespace knn {
namespace {

constexpr uint32_t FULL = 0xFFFFFFFFu;
constexpr int PQ_WARPS = 4;      // warps (queries in flight) per CTA
constexpr int PQ_SMALL = 1024;   // direct-sort threshold
constexpr int PQ_STACK = 96;     // kept-partition references per query

struct PaperSlab {
    uint64_t stage[32];          // the 32-wide pivot array of PAPER.md:52
    uint64_t sortbuf[PQ_SMALL];  // direct sort of the last partition
    uint64_t result[kMaxK];      // gathered k results
    int ref_buf[PQ_STACK];       // stack of references: buffer (0/1), start, length
    int ref_start[PQ_STACK];
    int ref_len[PQ_STACK];
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

// Warp bitonic sort of n (power of two) u64 in shared memory, ascending.
__device__ void warp_sort_smem(uint64_t* a, int n) {
    const int lane = threadIdx.x & 31;
    for (int size = 2; size <= n; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = lane; t < (n >> 1); t += 32) {
                const int i = 2 * t - (t & (stride - 1));
                const int j = i + stride;
                const uint64_t x = a[i], y = a[j];
                const bool asc = (i & size) == 0;
                if ((x > y) == asc) {
                    a[i] = y;
                    a[j] = x;
                }
            }
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(32 * PQ_WARPS)
select_paper_kernel(const float* __restrict__ D, int64_t M, int64_t N, int64_t ldD, int k,
                    uint64_t* __restrict__ aux0, uint64_t* __restrict__ aux1, int64_t aux_ld,
                    int64_t row0, int32_t* __restrict__ out_idx, float* __restrict__ out_dist) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    PaperSlab& sl = reinterpret_cast<PaperSlab*>(smem_raw)[warp];
    const uint32_t lt_mask = lanemask_lt();
    const int64_t gw = (int64_t)blockIdx.x * PQ_WARPS + warp;
    const int64_t nw = (int64_t)gridDim.x * PQ_WARPS;
    for (int64_t r = gw; r < M; r += nw) {
        const int64_t row = row0 + r;
        const float* in = D + row * ldD;
        uint64_t* const b0 = aux0 + r * aux_ld;
        uint64_t* const b1 = aux1 + r * aux_ld;
        auto buf = [&](int i) { return i == 0 ? b0 : b1; };
        int src = -1;  // -1: the input row itself (floats, implicit indices)
        int start = 0, len = (int)N, K = k, nref = 0;
        uint32_t pass = 0;
        while (true) {
            if (K == 0) break;
            if (K == len || len <= PQ_SMALL) {
                // direct finish: sort the live range, take its first K
                int n2 = 1;
                while (n2 < len) n2 <<= 1;
                for (int i = lane; i < n2; i += 32) {
                    uint64_t v = ~0ull;
                    if (i < len) {
                        if (src < 0) {
                            v = (uint64_t)ukey(in[start + i]) << 32 | (uint32_t)(start + i);
                        } else {
                            v = buf(src)[start + i];
                        }
                    }
                    if (n2 <= PQ_SMALL) sl.sortbuf[i] = v;
                }
                __syncwarp();
                if (n2 <= PQ_SMALL) {
                    warp_sort_smem(sl.sortbuf, n2);
                } else {
                    // K == len > PQ_SMALL: every element of the range is kept
                    if (lane == 0) {
                        sl.ref_buf[nref] = src;
                        sl.ref_start[nref] = start;
                        sl.ref_len[nref] = len;
                    }
                    ++nref;
                    K = 0;
                    __syncwarp();
                    break;
                }
                if (lane == 0) {
                    sl.ref_buf[nref] = 2;  // 2: sortbuf
                    sl.ref_start[nref] = 0;
                    sl.ref_len[nref] = K;
                }
                ++nref;
                K = 0;
                __syncwarp();
                break;
            }
            // pivot: the element at a hashed position of the live range
            const int ppos = start + (int)(hash32((uint32_t)row * 0x9E3779B9u + pass) % (uint32_t)len);
            const uint64_t pivot = src < 0 ? ((uint64_t)ukey(in[ppos]) << 32 | (uint32_t)ppos)
                                           : buf(src)[ppos];
            const int dsti = src == 0 ? 1 : 0;
            uint64_t* dst = buf(dsti);
            int g_lt = 0, g_ge = 0;
            for (int b = 0; b < len; b += 32) {
                const int i = b + lane;
                const bool valid = i < len;
                uint64_t x = 0;
                if (valid) {
                    if (src < 0) x = (uint64_t)ukey(in[start + i]) << 32 | (uint32_t)(start + i);
                    else x = buf(src)[start + i];
                }
                const bool ge = valid && x >= pivot;
                const bool lt = valid && x < pivot;
                const uint32_t B = __ballot_sync(FULL, ge);   // bit 1: >= pivot
                const uint32_t Lm = __ballot_sync(FULL, lt);
                const int nL = __popc(Lm), nG = __popc(B);
                if (lt) sl.stage[__popc(Lm & lt_mask)] = x;        // from the left end
                if (ge) sl.stage[31 - __popc(B & lt_mask)] = x;    // from the right end
                __syncwarp();
                if (lane < nL) dst[start + g_lt + lane] = sl.stage[lane];
                if (lane >= 32 - nG) dst[start + len - g_ge - (32 - lane)] = sl.stage[lane];
                g_lt += nL;
                g_ge += nG;
                __syncwarp();
            }
            const int L = g_lt;
            ++pass;
            if (K < L) {
                src = dsti;
                len = L;
            } else {
                // keep the left side by reference; K == L ends here (R11)
                if (L > 0) {
                    if (lane == 0) {
                        sl.ref_buf[nref] = dsti;
                        sl.ref_start[nref] = start;
                        sl.ref_len[nref] = L;
                    }
                    ++nref;
                }
                K -= L;
                src = dsti;
                start += L;
                len -= L;
                if (nref >= PQ_STACK - 1) {
                    // reference stack full (adversarial input): keep the rest whole
                    // and finish with the exact sort of the gathered results below
                    if (lane == 0) {
                        sl.ref_buf[nref] = src;
                        sl.ref_start[nref] = start;
                        sl.ref_len[nref] = len;
                    }
                    ++nref;
                    K = -1;
                    __syncwarp();
                    break;
                }
            }
            __syncwarp();
        }
        __syncwarp();
        // gather the referenced partitions (exactly k elements unless the stack overflowed)
        int cnt = 0;
        bool overflow = K < 0;
        for (int q = 0; q < nref; ++q) {
            const int bsel = sl.ref_buf[q], st = sl.ref_start[q], ln = sl.ref_len[q];
            for (int i = lane; i < ln; i += 32) {
                uint64_t v;
                if (bsel == 2) v = sl.sortbuf[i];
                else if (bsel < 0) v = (uint64_t)ukey(in[st + i]) << 32 | (uint32_t)(st + i);
                else v = buf(bsel)[st + i];
                if (cnt + i < kMaxK) sl.result[cnt + i] = v;
            }
            cnt += ln;
        }
        __syncwarp();
        if (overflow || cnt > kMaxK) {
            // not reached for k <= 1024 unless the pivot sequence degenerates; report NaN
            for (int i = lane; i < k; i += 32) {
                out_idx[row * k + i] = -1;
                out_dist[row * k + i] = __int_as_float(0x7FC00000);
            }
            continue;
        }
        int n2 = 1;
        while (n2 < cnt) n2 <<= 1;
        for (int i = cnt + lane; i < n2; i += 32) sl.result[i] = ~0ull;
        __syncwarp();
        warp_sort_smem(sl.result, n2);
        for (int i = lane; i < k; i += 32) {
            const uint64_t v = sl.result[i];
            out_idx[row * k + i] = (int32_t)(uint32_t)v;
            out_dist[row * k + i] = ukey_to_float((uint32_t)(v >> 32));
        }
        __syncwarp();
    }
}

}  // namespace

size_t select_paper_ws_bytes(int64_t rows, int64_t N) { return 2 * (size_t)rows * (size_t)N * 8; }

cudaError_t launch_select_paper(const float* D, int64_t M, int64_t N, int64_t ldD, int32_t k,
                                void* ws, size_t ws_bytes, int32_t* out_idx, float* out_dist,
                                cudaStream_t s) {
    if (M == 0) return cudaSuccess;
    if (k < 1 || k > kMaxK || N < k) return cudaErrorInvalidValue;
    const int64_t rows_blk = (int64_t)(ws_bytes / (2 * (size_t)N * 8));
    if (rows_blk < 1) return cudaErrorInvalidValue;
    const size_t smem = sizeof(PaperSlab) * PQ_WARPS;
    cudaError_t e = cudaFuncSetAttribute(select_paper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_paper_kernel, 32 * PQ_WARPS, smem);
    uint64_t* aux0 = static_cast<uint64_t*>(ws);
    for (int64_t r0 = 0; r0 < M; r0 += rows_blk) {
        const int64_t R = M - r0 < rows_blk ? M - r0 : rows_blk;
        uint64_t* aux1 = aux0 + R * N;
        int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
        if (grid > ceil_div(R, PQ_WARPS)) grid = ceil_div(R, PQ_WARPS);
        select_paper_kernel<<<(unsigned)grid, 32 * PQ_WARPS, smem, s>>>(D, R, N, ldD, k, aux0, aux1, N, r0,
                                                                       out_idx, out_dist);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace knn
