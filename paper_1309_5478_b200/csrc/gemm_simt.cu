// gemm_simt.cu — a-S3 on the FP32 FFMA (SIMT) pipe: the "FFMA path" of the north star.
//
// D[i,j] = max(||q_i||^2 + ||x_j||^2 - 2 q_i.x_j, 0), sqrt for L2
// (PAPER.md:61), +inf on the excluded self pair.  The dot products are the matrix
// product of PAPER.md:73-77 computed in plain fp32 FMA from the unsplit inputs.
//
// This path is the plan for tiny problems (fewer rows/columns than one tensor-core
// tile) and the independent cross-check of the tensor-core path (KNN_GEMM=simt); the
// split tensor-core GEMM of gemm_tc.cu is the hot path.
#include "internal.cuh"

namespace knn {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, THREADS = 256;

__global__ void __launch_bounds__(THREADS)
dist_simt_kernel(const float* __restrict__ Q, const float* __restrict__ qn, int64_t M,
                 const float* __restrict__ X, const float* __restrict__ xn, int64_t N,
                 int32_t d, int32_t metric, int64_t self_shift, float* __restrict__ D,
                 int64_t ldD) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t row0 = (int64_t)blockIdx.y * BM, col0 = (int64_t)blockIdx.x * BN;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < d; k0 += BK) {
        #pragma unroll
        for (int it = 0; it < (BM * BK) / THREADS; ++it) {
            int e = tid + it * THREADS;
            int r = e / BK, kk = e % BK;
            int64_t gr = row0 + r, gc = col0 + r;
            As[kk][r] = (gr < M && k0 + kk < d) ? __ldg(Q + gr * d + k0 + kk) : 0.0f;
            Bs[kk][r] = (gc < N && k0 + kk < d) ? __ldg(X + gc * d + k0 + kk) : 0.0f;
        }
        __syncthreads();
        #pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[4], b[4];
            #pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
            #pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
            #pragma unroll
            for (int i = 0; i < 4; ++i)
                #pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    #pragma unroll
    for (int i = 0; i < 4; ++i) {
        int64_t r = row0 + ty + 16 * i;
        if (r >= M) continue;
        const float nq = qn[r];
        #pragma unroll
        for (int j = 0; j < 4; ++j) {
            int64_t c = col0 + tx + 16 * j;
            if (c >= N) continue;
            float v = fmaxf(fmaf(-2.0f, acc[i][j], nq + xn[c]), 0.0f) + 0.0f;
            if (metric == 1) v = sqrtf(v);
            if (c == r + self_shift) v = __int_as_float(0x7F800000);
            D[r * ldD + c] = v;
        }
    }
}

}  // namespace

cudaError_t launch_dist_simt(const float* Q, const float* qn, int64_t M, const float* X,
                             const float* xn, int64_t N, int32_t d, int32_t metric,
                             int64_t self_shift, float* D, int64_t ldD, cudaStream_t s) {
    if (M == 0 || N == 0) return cudaSuccess;
    dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM));
    if (grid.y > 65535) return cudaErrorInvalidValue;
    dist_simt_kernel<<<grid, THREADS, 0, s>>>(Q, qn, M, X, xn, N, d, metric, self_shift, D, ldD);
    return cudaGetLastError();
}

}  // namespace knn
