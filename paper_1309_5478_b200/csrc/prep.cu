// prep.cu — a-S2: row norms + input validation + split of the operands for the
// FP32-accurate tensor-core GEMM.
//
// Paper: "we compute the vector norms of the vectors in X,Y using a combination of a
// transform iterator and reduction_by_key ... The transform iterator generates the
// square of individual elements and feeds the result into the reduction_by_key function
// which in turn computes the square of the vector norms".  Here one warp
// reduces one vector: squares accumulated in fp64 (reading R15), rounded to fp32.
//
// In the same pass (one HBM read of X) it writes, for the GEMM of gemm_tc.cu, each
// vector scaled by a power of two s = 2^sh chosen so that max|x|*s lies in [2^14, 2^15),
// split into two fp16 halves:  hi = fp16(x*s),  lo = fp16(x*s - hi).
// x*s = hi + lo + r with |r| <= 2^-22 |x*s|, so hi.hi + hi.lo + lo.hi reproduces every
// product to ~3*2^-22 relative, and rscale = 2^-sh undoes the scale
// exactly in the epilogue.  Rows are zero-padded to d_pad (a multiple of 64) so TMA
// boxes of 64 fp16 (= one 128-byte swizzle atom) tile K exactly.
//
// Validation (reading R8): flag = 1 if any x is NaN/inf or
// ||x||^2 >= FLT_MAX/4 (which bounds every distance below FLT_MAX).
//
// Cosine / Pearson (NEXT-2): the same GEMM computes 1 - cos.  Pearson
// first centres the vector (fp64 mean, PAPER.md:69-71 / 85 "we center each vector"; the
// centred value is rounded to fp32 once).  The per-vector terms become sqn = 1/2 (5/2 for
// a zero-norm vector: the epilogue's clamp at 3 gives SPEC.md:143's sentinel) and
// rscale = 2^-sh / (sqrt(2) ||x||), so the epilogue's fma(acc * (-2 rs_q), rs_x, 1/2 + 1/2)
// is 1 - x.y / (||x|| ||y||).
#include "internal.cuh"

#include <cfloat>
#include <cmath>

namespace knn {
namespace {

constexpr int kWarpsPerBlock = 8;

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
prep_kernel(const float* __restrict__ X, int64_t N, int32_t d, int32_t d_pad,
            float* __restrict__ sqn, float* __restrict__ rscale, __half* __restrict__ hi,
            __half* __restrict__ lo, int32_t* __restrict__ flag, int32_t metric,
            float* __restrict__ eps2, float* __restrict__ tmax2) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (row >= N) {
        // tensor-core path: the column arrays are padded to a multiple of 256 entries (the
        // GEMM bulk-copies whole tiles of them); the padding is zero
        if (hi != nullptr && lane == 0 && row < round_up(N, (int64_t)kColPad)) {
            sqn[row] = 0.0f;
            rscale[row] = 0.0f;
            if (eps2) eps2[row] = 0.0f;
        }
        return;
    }
    const float* x = X + row * (int64_t)d;
    const bool angular = hi != nullptr && (metric == 2 || metric == 3);

    // Pearson: the vector mean, fp64; the operands are x - mean
    double mean = 0.0;
    bool finite = true;
    if (angular && metric == 3) {
        double s1 = 0.0;
        for (int t = lane; t < d; t += 32) {
            const float v = __ldg(x + t);
            finite &= isfinite(v);
            s1 += (double)v;
        }
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) s1 += __shfl_xor_sync(0xFFFFFFFFu, s1, o);
        mean = s1 / (double)d;
    }
    double s = 0.0;
    float amax = 0.0f;
    // 16-byte loads when the rows allow (d % 4 == 0, X 16-byte aligned); same sums per lane
    // order is not required: s is fp64 and rounded once (reading R15)
    const bool vec4 = (d & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
    if (vec4) {
        const float4* x4 = reinterpret_cast<const float4*>(x);
        for (int t = lane; t < d / 4; t += 32) {
            const float4 q = __ldg(x4 + t);
            const float vv[4] = {q.x, q.y, q.z, q.w};
            #pragma unroll
            for (int e = 0; e < 4; ++e) {
                finite &= isfinite(vv[e]);
                const double c = (double)vv[e] - mean;
                amax = fmaxf(amax, fabsf((float)c));
                s = fma(c, c, s);
            }
        }
    } else {
        for (int t = lane; t < d; t += 32) {
            float v = __ldg(x + t);
            finite &= isfinite(v);
            const double c = (double)v - mean;
            amax = fmaxf(amax, fabsf((float)c));
            s += c * c;
        }
    }
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
        amax = fmaxf(amax, __shfl_xor_sync(0xFFFFFFFFu, amax, o));
    }
    finite = __all_sync(0xFFFFFFFFu, finite);
    if (lane == 0) {
        // L2: ||x||^2.  Cosine / Pearson: the GEMM epilogue's "norm" term is 1/2 per
        // vector, so ||q||^2 + ||x||^2 = 1 and the epilogue yields 1 - cos; a zero-norm
        // vector gets 5/2, which the cosine clamp turns into the sentinel 3
        sqn[row] = angular ? (s > 0.0 ? 0.5f : 2.5f) : (float)s;
        if (flag && (!finite || !(s < (double)(FLT_MAX / 4)))) *flag = 1;
    }
    if (hi == nullptr) return;

    // sh such that amax * 2^sh in [2^14, 2^15); frexp: amax = m 2^e, m in [0.5, 1).
    int e = 0;
    int sh = 0;
    if (amax > 0.0f && finite) {
        frexpf(amax, &e);
        sh = 15 - e;
    }
    // 2^sh may exceed the fp32 range for subnormal-only rows: apply it in two exact steps.
    const int sh1 = sh > 120 ? 120 : sh;
    const float s1 = ldexpf(1.0f, sh1), s2 = ldexpf(1.0f, sh - sh1);
    if (lane == 0) {
        // L2: 2^-sh (the epilogue multiplies -2 rs_q rs_x).  Cosine / Pearson:
        // 2^-sh / (sqrt(2) ||x||), so that -2 rs_q rs_x = -2^-(shq+shx) / (||q|| ||x||)
        rscale[row] = !angular ? ldexpf(1.0f, -sh)
                               : (s > 0.0 ? (float)(ldexp(1.0, -sh) / (sqrt(2.0) * sqrt(s))) : 0.0f);
    }
    __half* h = hi + row * (int64_t)d_pad;
    __half* l = lo + row * (int64_t)d_pad;
    // eps2 (L2 metrics): the row's split residual ratio ||s x - hi||^2 / ||s x||^2 in fp64
    // from the exact scaled input (per-point bound of the single product)
    const double sd = ldexp(1.0, sh);
    double rr = 0.0, vv = 0.0;
    if ((d & 7) == 0 && vec4 && !(metric == 3 && angular)) {
        // 8 elements per lane per step: two 16-byte loads, one 16-byte store per half
        const float4* x4 = reinterpret_cast<const float4*>(x);
        for (int g = lane; g < d_pad / 8; g += 32) {
            float xv[8];
            if (8 * g < d && finite) {
                const float4 a = __ldg(x4 + 2 * g), b = __ldg(x4 + 2 * g + 1);
                xv[0] = a.x; xv[1] = a.y; xv[2] = a.z; xv[3] = a.w;
                xv[4] = b.x; xv[5] = b.y; xv[6] = b.z; xv[7] = b.w;
            } else {
                #pragma unroll
                for (int e = 0; e < 8; ++e) xv[e] = 0.0f;
            }
            __align__(16) __half hh[8], ll[8];
            #pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float v = xv[e] * s1 * s2;  // exact power-of-two scaling
                hh[e] = __float2half_rn(v);
                ll[e] = __float2half_rn(v - __half2float(hh[e]));
                if (eps2) {
                    const double vx = (double)xv[e] * sd, r = vx - (double)__half2float(hh[e]);
                    rr = fma(r, r, rr);
                    vv = fma(vx, vx, vv);
                }
            }
            *reinterpret_cast<uint4*>(h + 8 * g) = *reinterpret_cast<const uint4*>(hh);
            *reinterpret_cast<uint4*>(l + 8 * g) = *reinterpret_cast<const uint4*>(ll);
        }
    } else
    for (int t = lane; t < d_pad; t += 32) {
        float v = 0.0f;
        float xv = 0.0f;
        if (t < d && finite) {
            // exact power-of-two scaling of x (or of the fp32-rounded centred value)
            xv = metric == 3 && angular ? (float)((double)__ldg(x + t) - mean) : __ldg(x + t);
            v = xv * s1 * s2;
        }
        __half vh = __float2half_rn(v);
        h[t] = vh;
        l[t] = __float2half_rn(v - __half2float(vh));
        if (eps2) {
            const double vx = (double)xv * sd, r = vx - (double)__half2float(vh);
            rr = fma(r, r, rr);
            vv = fma(vx, vx, vv);
        }
    }
    if (eps2) {
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            rr += __shfl_xor_sync(0xFFFFFFFFu, rr, o);
            vv += __shfl_xor_sync(0xFFFFFFFFu, vv, o);
        }
        if (lane == 0) {
            // rounded up, with room for the fp64 sums' own rounding (d 2^-53 each)
            const float e2 = vv > 0.0 ? __double2float_ru(rr / vv * (1.0 + 0x1p-30)) : 0.0f;
            eps2[row] = e2;
            // the call's t^2 = max eps2 (>= 0: int order); the read skips most atomics
            if (tmax2 && e2 > *reinterpret_cast<volatile float*>(tmax2))
                atomicMax(reinterpret_cast<int*>(tmax2), __float_as_int(e2));
        }
    }
}

}  // namespace

cudaError_t launch_prep(const float* X, int64_t N, int32_t d, int32_t d_pad, float* sqn,
                        float* rscale, __half* hi, __half* lo, int32_t* flag, int32_t metric,
                        cudaStream_t s, float* eps2, float* tmax2) {
    if (N == 0) return cudaSuccess;
    if (eps2 && (hi == nullptr || metric > 1)) return cudaErrorInvalidValue;  // split, L2 metrics only
    dim3 grid((unsigned)ceil_div(hi != nullptr ? round_up(N, (int64_t)kColPad) : N, kWarpsPerBlock));
    prep_kernel<<<grid, kWarpsPerBlock * 32, 0, s>>>(X, N, d, d_pad, sqn, rscale, hi, lo, flag, metric, eps2,
                                                     tmax2);
    return cudaGetLastError();
}

namespace {
// Per-point terms of the single-product bound (reading R21).  With v = s x
// the exact scaled point, hi its fp16 split and e = ||v - hi|| / ||v|| (prep's eps2), for
// any t > 0 (the same for every point of the call: t = sqrt(max eps2), at least 2^-13)
//   2 |q||x| (e_q + e_x) <= (t + e_q^2 / t) ||q||^2 + (t + e_x^2 / t) ||x||^2     (AM-GM),
//   2 |q||x| e_q e_x    <= 2^-11' (e_q ||q||^2 + e_x ||x||^2)         (every e <= 2^-11'),
// so |2 q.x - 2 qh.xh / (s_q s_x)| <= B_q ||q||^2 + B_x ||x||^2 with the per-point
// B = (t + e^2 / t)(1 + 2^-10) + 2^-11 (1 + 2^-9) e (the 1 + 2^-10 also covers the
// 3-product value's rounded lo halves), and the accumulation / rounding terms of the
// constant bound (gemm_tc.cu launch_dist_tc_mins) follow per point:
//   Fs = B + gs (sample values: upper bounds),  F1 = B + g1 (partition lower bounds),
//   gs = gamma (1 + 2^-9) + 2^-20,  g1 = 2 gamma (1 + 2^-9) + 2^-19,  gamma = d_pad 2^-23.
// Outputs (fp64 arithmetic, directed roundings):  nsc = RD(sqn (1 - F1)) (the partition's
// lower-bound norms), ninf = RU(sqn (1 + Fs)) (the sample's upper-bound norms),
// bnd = RU(sqn F1) (half the width of the re-evaluation window, per point).
__global__ void bound_norms_kernel(const float* __restrict__ sqn, const float* __restrict__ eps2, int64_t n,
                                   const float* __restrict__ tmax2, double gs, double g1,
                                   float* __restrict__ nsc, float* __restrict__ ninf, float* __restrict__ bnd) {
    // (floor 2^-13: a call whose t-defining points happen to be fp16-exact, e.g. the
    // pipelined k-NNG's sample, keeps every other point's F within ~2x the constant bound)
    const double t = fmax(sqrt((double)__ldg(tmax2)), 0x1p-13);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double e2 = (double)eps2[i], q = (double)sqn[i];
        const double B = (t + e2 / t) * (1.0 + 0x1p-10) + 0x1p-11 * (1.0 + 0x1p-9) * sqrt(e2);
        const double F1 = B + g1;
        if (nsc) nsc[i] = __double2float_rd(q * (1.0 - F1));
        if (ninf) ninf[i] = __double2float_ru(q * (1.0 + B + gs));
        if (bnd) bnd[i] = __double2float_ru(q * F1);
    }
}
}  // namespace

cudaError_t launch_bound_norms(const float* sqn, const float* eps2, int64_t n, const float* tmax2, int32_t d_pad,
                               float* nsc, float* ninf, float* bnd, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const double gamma = d_pad * std::ldexp(1.0, -23);
    const double gs = gamma * (1.0 + std::ldexp(1.0, -9)) + std::ldexp(1.0, -20);
    const double g1 = 2.0 * gamma * (1.0 + std::ldexp(1.0, -9)) + std::ldexp(1.0, -19);
    const int64_t blocks = ceil_div(n, (int64_t)256);
    bound_norms_kernel<<<(unsigned)(blocks < 1184 ? blocks : 1184), 256, 0, s>>>(sqn, eps2, n, tmax2, gs, g1, nsc,
                                                                               ninf, bnd);
    return cudaGetLastError();
}

// Column sample of the pivot plans: sample column j < S is point
// perm(j) = (j * a) mod N (a coprime to N), a deterministic permutation that spreads the
// sample over the whole index range one point at a time, so that ordered inputs (e.g.
// points sorted along a coordinate or by cluster) still give every row a representative
// sample.  Copies the split operands and the per-point epilogue terms of those points;
// the column arrays are padded to kColPad with zeros.  One warp per sample column.
namespace {
__global__ void __launch_bounds__(256)
gather_sample_kernel(const __half* __restrict__ hi, const __half* __restrict__ lo,
                     const float* __restrict__ sqn, const float* __restrict__ rs, int64_t N,
                     int64_t S, int64_t Spad, int64_t a, int32_t d_pad, __half* __restrict__ shi,
                     __half* __restrict__ slo, float* __restrict__ ssqn, float* __restrict__ srs,
                     float* __restrict__ smax) {
    const int lane = threadIdx.x & 31;
    const int64_t j = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (j >= Spad) return;
    if (j >= S) {
        if (lane == 0) {
            ssqn[j] = 0.0f;
            srs[j] = 0.0f;
        }
        return;
    }
    const int64_t src = (int64_t)(((uint64_t)j * (uint64_t)a) % (uint64_t)N);
    const uint4* h4 = reinterpret_cast<const uint4*>(hi + src * d_pad);
    const uint4* l4 = reinterpret_cast<const uint4*>(lo + src * d_pad);
    uint4* sh4 = reinterpret_cast<uint4*>(shi + j * d_pad);
    uint4* sl4 = reinterpret_cast<uint4*>(slo + j * d_pad);
    for (int t = lane; t < d_pad / 8; t += 32) {
        sh4[t] = h4[t];
        sl4[t] = l4[t];
    }
    if (lane == 0) {
        ssqn[j] = sqn[src];
        srs[j] = rs[src];
        // max of the sample's epilogue terms (>= 0: ordered as ints), for the sample pass's
        // per-chunk error bound
        if (smax) atomicMax(reinterpret_cast<int*>(smax), __float_as_int(fmaxf(sqn[src], 0.0f)));
    }
}
}  // namespace

int64_t sample_stride(int64_t N) {
    // odd, coprime to N, near N * (sqrt(5) - 1) / 2
    int64_t a = (int64_t)((double)N * 0.6180339887498949) | 1;
    auto gcd = [](int64_t x, int64_t y) { while (y) { const int64_t t = x % y; x = y; y = t; } return x; };
    while (a > 1 && gcd(a, N) != 1) a -= 2;
    return a < 1 ? 1 : a;
}

cudaError_t launch_gather_sample(const __half* hi, const __half* lo, const float* sqn, const float* rs,
                                 int64_t N, int64_t S, int32_t d_pad, __half* shi, __half* slo, float* ssqn,
                                 float* srs, float* smax, cudaStream_t s) {
    if (S == 0) return cudaSuccess;
    const int64_t Spad = round_up(S, kColPad);
    if (smax) {
        const cudaError_t e = cudaMemsetAsync(smax, 0, sizeof(float), s);
        if (e != cudaSuccess) return e;
    }
    gather_sample_kernel<<<(unsigned)ceil_div(Spad, 8), 256, 0, s>>>(hi, lo, sqn, rs, N, S, Spad,
                                                                     sample_stride(N), d_pad, shi, slo,
                                                                     ssqn, srs, smax);
    return cudaGetLastError();
}

namespace {
__global__ void max_nonneg_kernel(const float* __restrict__ v, int64_t n, float* __restrict__ out) {
    float m = 0.0f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = fmaxf(m, v[i]);
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(m));  // >= 0: int order
}
}  // namespace

// *out = max(0, v[0..n)) (the sample pass's bound of the columns' sqn terms for a sample
// that was prepared in place rather than gathered)
cudaError_t launch_max_nonneg(const float* v, int64_t n, float* out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(float), s);
    if (e != cudaSuccess || n == 0) return e;
    const int64_t blocks = ceil_div(n, (int64_t)256);
    max_nonneg_kernel<<<(unsigned)(blocks < 592 ? blocks : 592), 256, 0, s>>>(v, n, out);
    return cudaGetLastError();
}



namespace {
// Sums of the row terms, the column terms and the finite pivots, then the decision.
// kDecBlocks CTAs each reduce a strided slice (fp32 partials per thread, <= M / 32768 terms
// each, then fp64) into part[block]; the last CTA to finish (counter, zeroed by the
// caller) adds the partials in block order (deterministic) and writes flag[1].
constexpr int kDecBlocks = 128;
__global__ void __launch_bounds__(256) pivot1_decide_kernel(const float* __restrict__ thr,
                                                           const float* __restrict__ qn, int64_t M,
                                                           const float* __restrict__ xn, int64_t N, float F,
                                                           float ratio, int32_t* __restrict__ flag,
                                                           double* __restrict__ part, unsigned* counter) {
    __shared__ double red[4][8];
    __shared__ bool last;
    float sq = 0.0f, sx = 0.0f, st = 0.0f;
    int nt = 0;
    const int64_t M4 = M / 4, N4 = N / 4;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    const float4* qn4 = reinterpret_cast<const float4*>(qn);
    const float4* th4 = reinterpret_cast<const float4*>(thr);
    const float4* xn4 = reinterpret_cast<const float4*>(xn);
    for (int64_t i = t0; i < M4; i += nth) {
        const float4 a = qn4[i], t = th4[i];
        sq += (a.x + a.y) + (a.z + a.w);
        const float tv[4] = {t.x, t.y, t.z, t.w};
        #pragma unroll
        for (int e = 0; e < 4; ++e)
            if (isfinite(tv[e])) {
                st += tv[e];
                ++nt;
            }
    }
    for (int64_t j = t0; j < N4; j += nth) {
        const float4 b = xn4[j];
        sx += (b.x + b.y) + (b.z + b.w);
    }
    for (int64_t i = 4 * M4 + t0; i < M; i += nth) {
        sq += qn[i];
        if (isfinite(thr[i])) {
            st += thr[i];
            ++nt;
        }
    }
    for (int64_t j = 4 * N4 + t0; j < N; j += nth) sx += xn[j];
    double v[4] = {(double)sq, (double)sx, (double)st, (double)nt};
    #pragma unroll
    for (int a = 0; a < 4; ++a) {
        for (int o = 16; o > 0; o >>= 1) v[a] += __shfl_xor_sync(0xFFFFFFFFu, v[a], o);
        if ((threadIdx.x & 31) == 0) red[a][threadIdx.x >> 5] = v[a];
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double acc = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) acc += red[threadIdx.x][w];
        part[blockIdx.x * 4 + threadIdx.x] = acc;
        __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x < 32) {  // one warp adds the partials in a fixed order (deterministic)
        __threadfence();
        const int lane = threadIdx.x;
        double v4[4] = {0, 0, 0, 0};
        for (int k = lane; k < (int)gridDim.x; k += 32)
            #pragma unroll
            for (int a = 0; a < 4; ++a) v4[a] += __ldcg(part + 4 * k + a);
        #pragma unroll
        for (int a = 0; a < 4; ++a)
            for (int o = 16; o > 0; o >>= 1) v4[a] += __shfl_xor_sync(0xFFFFFFFFu, v4[a], o);
        if (lane == 0) {
            const double width = 2.0 * (double)F * (v4[0] / (double)M + v4[1] / (double)N);
            flag[1] = (v4[3] > 0 && width <= (double)ratio * (v4[2] / v4[3])) ? 1 : 0;
        }
    }
}
}  // namespace

size_t pivot1_decide_ws_bytes() { return kDecBlocks * 4 * sizeof(double); }

cudaError_t launch_pivot1_decide(const float* thr, const float* qn, int64_t M, const float* xn, int64_t N,
                                 float F, float ratio, int32_t* flag, double* part, unsigned* counter,
                                 cudaStream_t s) {
    if (M == 0 || N == 0) return cudaSuccess;
    pivot1_decide_kernel<<<kDecBlocks, 256, 0, s>>>(thr, qn, M, xn, N, F, ratio, flag, part, counter);
    return cudaGetLastError();
}



}  // namespace knn
