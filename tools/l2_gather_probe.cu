// l2_gather_probe.cu — measured peak of the re-evaluation's memory pattern on B200: warps
// gathering random 1 KB rows (d = 256 fp32) of a 64 MB L2-resident matrix with float4
// loads, G rows in flight per warp, the bytes reduced in registers (no output traffic).
// The best rate over the launch shapes is the `peak` bench.py reports for
// candidate_recompute_kernel ("bound": "l2").
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o l2_gather_probe tools/l2_gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

constexpr int D = 256;  // floats per row (1 KB)

__global__ void fill(float* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = (float)((i * 2654435761u) & 0xFFFF) * 1.0e-5f;
}
__global__ void fill_idx(uint32_t* idx, size_t n, uint32_t rows) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint64_t h = (i + 1) * 0x9E3779B97F4A7C15ull;
        h ^= h >> 31;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 29;
        idx[i] = (uint32_t)(h % rows);
    }
}

// each warp: groups of G rows, every lane loads float4 t = lane + 32 s of every row
template <int G>
__global__ void gather(const float* __restrict__ X, const uint32_t* __restrict__ idx, size_t n_rows, float* out) {
    const int lane = threadIdx.x & 31;
    const size_t gw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
    float acc = 0.0f;
    for (size_t r0 = gw * G; r0 + G <= n_rows; r0 += nw * G) {
        const float* xr[G];
#pragma unroll
        for (int u = 0; u < G; ++u) xr[u] = X + (size_t)__ldg(idx + r0 + u) * D;
#pragma unroll 1
        for (int t = 4 * lane; t < D; t += 128) {
            float4 v[G];
#pragma unroll
            for (int u = 0; u < G; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(xr[u] + t));
#pragma unroll
            for (int u = 0; u < G; ++u) acc += (v[u].x + v[u].y) + (v[u].z + v[u].w);
        }
    }
    if (acc == 1234.5f) out[0] = acc;  // keep the loads
}

template <int G>
float run(const float* X, const uint32_t* idx, size_t n, float* out, int blocks, int threads) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather<G><<<blocks, threads>>>(X, idx, n, out);  // warm: X into L2
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) gather<G><<<blocks, threads>>>(X, idx, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return (float)(n * D * 4.0 * 10 / (ms * 1e-3) / 1e9);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint32_t rows = 65536;             // 64 MB: L2-resident (126 MB)
    const size_t n = (size_t)rows * 40;      // 2.6 M gathers (the headline's ~39 per row)
    float *X, *out;
    uint32_t* idx;
    cudaMalloc(&X, (size_t)rows * D * 4);
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&out, 4);
    fill<<<1024, 256>>>(X, (size_t)rows * D);
    fill_idx<<<1024, 256>>>(idx, n, rows);
    cudaDeviceSynchronize();
    float best = 0;
    for (int per_sm : {4, 8, 16}) {
        for (int threads : {256, 512}) {
            const int blocks = sms * per_sm * 256 / threads;
            const float g4 = run<4>(X, idx, n, out, blocks, threads);
            const float g8 = run<8>(X, idx, n, out, blocks, threads);
            printf("warps/SM %2d (%3d-thread CTAs): G=4 %7.1f GB/s  G=8 %7.1f GB/s\n", per_sm * 8, threads, g4, g8);
            best = g4 > best ? g4 : best;
            best = g8 > best ? g8 : best;
        }
    }
    printf("{\"l2_gather_gbs\": %.1f, \"row_bytes\": %d, \"rows_resident_mb\": %d}\n", best, D * 4,
           (int)((size_t)rows * D * 4 >> 20));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
