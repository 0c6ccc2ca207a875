// stream_probe.cu — measure HBM read bandwidth of streaming schemes on B200:
// plain 128-bit loads vs 1-D bulk async copies into per-warp / per-CTA smem rings.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o stream_probe tools/stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c)); }
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(bar), "r"(ph) : "memory");
}
__device__ int g_policy_mode = 0;
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    if (g_policy_mode) {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
    } else
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__global__ void fill(float* p, size_t n) { for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = (float)((i * 2654435761u) & 0xFFFFFF) * 5.9604645e-08f; }

__global__ void ldg_kernel(const float4* __restrict__ p, size_t n4, float* out) {
    float acc = 0.f;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
    for (; i + 7 * st < n4; i += 8 * st) {
        float4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v[j].x), "=f"(v[j].y), "=f"(v[j].z), "=f"(v[j].w) : "l"(p + i + j * st));
#pragma unroll
        for (int j = 0; j < 8; ++j) acc += v[j].x + v[j].y + v[j].z + v[j].w;
    }
    if (acc == 12345.f) out[0] = acc;
}

// each warp streams its own rows (row = rowlen floats) through a private ring
template <int C, int S>
__global__ void warp_ring(const float* __restrict__ D, int64_t rows, int64_t rowlen, float* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
    float* ring = (float*)(sm + (size_t)warp * (S * C * 4 + 64));
    uint64_t* bars = (uint64_t*)(ring + S * C);
    uint32_t b0 = smem_u32(bars);
    if (lane == 0) { for (int s = 0; s < S; ++s) mbar_init(b0 + 8 * s, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncwarp();
    int64_t gw = (int64_t)blockIdx.x * W + warp, nw = (int64_t)gridDim.x * W;
    int64_t nch = rowlen / C;
    int64_t prow = gw, pc = 0;
    auto issue = [&](int s) { if (prow >= rows) return; mbar_expect_tx(b0 + 8 * s, C * 4); bulk(smem_u32(ring + s * C), D + prow * rowlen + pc * C, C * 4, b0 + 8 * s); if (++pc == nch) { pc = 0; prow += nw; } };
    if (lane == 0) for (int s = 0; s < S; ++s) issue(s);
    float acc = 0.f; uint32_t q = 0;
    for (int64_t r = gw; r < rows; r += nw)
        for (int64_t c = 0; c < nch; ++c, ++q) {
            int s = q % S; mbar_wait(b0 + 8 * s, (q / S) & 1);
            const float4* b = (const float4*)(ring + s * C);
            for (int j = lane; j < C / 4; j += 32) { float4 v = b[j]; acc += v.x + v.y + v.z + v.w; }
            __syncwarp();
            if (lane == 0) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(s); }
        }
    if (acc == 12345.f) out[0] = acc;
}

__global__ void stg_kernel(float4* __restrict__ p, size_t n4) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
    const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
    for (; i + 7 * st < n4; i += 8 * st) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p + i + j * st), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    }
}

template <class F>
float timeit(F f) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); cudaDeviceSynchronize();
    cudaEventRecord(a); for (int i = 0; i < 5; ++i) f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5;
}

int main() {
    const size_t bytes = (size_t)4 << 30;
    float* D; cudaMalloc(&D, bytes); cudaMemset(D, 0, bytes);
    float* out; cudaMalloc(&out, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t n4 = bytes / 16;
    for (int bpsm : {2, 4, 8}) {
        float ms = timeit([&] { stg_kernel<<<sms * bpsm, 256>>>((float4*)D, n4); });
        printf("stg128 (write only) 256thr x %d CTA/SM: %.0f GB/s\n", bpsm, bytes / ms / 1e6);
    }
    {
        float ms = timeit([&] { cudaMemsetAsync(D, 1, bytes); });
        printf("cudaMemset (write only): %.0f GB/s\n", bytes / ms / 1e6);
        float* E; cudaMalloc(&E, bytes);
        ms = timeit([&] { cudaMemcpyAsync(E, D, bytes, cudaMemcpyDeviceToDevice); });
        printf("cudaMemcpy D2D (read+write counted): %.0f GB/s\n", 2.0 * bytes / ms / 1e6);
        cudaFree(E);
    }
  for (int pass = 0; pass < 1; ++pass) {
    if (pass == 1) { fill<<<sms * 8, 256>>>(D, bytes / 4); cudaDeviceSynchronize(); printf("--- random data\n"); }
    if (pass == 2) { int one = 1; cudaMemcpyToSymbol(g_policy_mode, &one, sizeof(int)); printf("--- random data + evict_first policy\n"); }
    for (int bpsm : {2, 4, 8}) {
        float ms = timeit([&] { ldg_kernel<<<sms * bpsm, 256>>>((const float4*)D, n4, out); });
        printf("ldg128 unroll8 256thr x %d CTA/SM: %.0f GB/s\n", bpsm, bytes / ms / 1e6);
    }
    auto run_ring = [&](auto kern, int C, int S, int W, int64_t rowlen, const char* name) {
        size_t smem = (size_t)W * (S * C * 4 + 64);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 32 * W, smem);
        int64_t rows = bytes / 4 / rowlen;
        float ms = timeit([&] { kern<<<sms * per, 32 * W, smem>>>(D, rows, rowlen, out); });
        printf("%s C=%dKB S=%d W=%d CTA/SM=%d rowlen=%lld: %.0f GB/s\n", name, C * 4 / 1024, S, W, per, (long long)rowlen, bytes / ms / 1e6);
    };
    run_ring(warp_ring<1024, 4>, 1024, 4, 4, 65536, "warp_ring");
    run_ring(warp_ring<2048, 4>, 2048, 4, 4, 65536, "warp_ring");
    run_ring(warp_ring<4096, 3>, 4096, 3, 4, 65536, "warp_ring");
    run_ring(warp_ring<1024, 4>, 1024, 4, 8, 65536, "warp_ring");
  }
    return 0;
}
