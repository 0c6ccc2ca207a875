// Probe (diagnostic, not part of the library): does compute-sanitizer racecheck model the
// textbook producer/consumer ring in which a bulk async copy (cp.async.bulk, TMA engine)
// fills a shared-memory slot, completion is signalled on a "full" mbarrier (complete_tx),
// consumer warps wait on it, read, and release the slot on an "empty" mbarrier that the
// producer thread waits on (then fence.proxy.async) before the next copy?  This is the
// column-data ring of gemm_tc.cu.  If racecheck reports hazards here, they are the tool's.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t par) {
    asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(b), "r"(par) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}

constexpr int SLOTS = 2, ITEMS = 16, BYTES = 1024, CONSUMERS = 4;
__global__ void ring(const float* src, float* out) {
    __shared__ __align__(128) float buf[SLOTS][BYTES / 4];
    __shared__ __align__(8) uint64_t full[SLOTS], empty[SLOTS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < SLOTS; ++s) { mbar_init(su32(&full[s]), 1); mbar_init(su32(&empty[s]), CONSUMERS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == CONSUMERS) {  // producer
        if (lane == 0)
            for (int it = 0; it < ITEMS; ++it) {
                const int s = it % SLOTS;
                mbar_wait(su32(&empty[s]), ((it / SLOTS) & 1) ^ 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(BYTES) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su32(buf[s])), "l"(src + it * (BYTES / 4)), "r"(BYTES), "r"(su32(&full[s])) : "memory");
            }
        __syncwarp();
    } else {  // consumers
        float acc = 0.f;
        for (int it = 0; it < ITEMS; ++it) {
            const int s = it % SLOTS;
            mbar_wait(su32(&full[s]), (it / SLOTS) & 1);
            for (int i = lane; i < BYTES / 4; i += 32) acc += buf[s][i];
            __syncwarp();
            if (lane == 0) mbar_arrive(su32(&empty[s]));
        }
        out[threadIdx.x] = acc;
    }
}

int main() {
    float *src, *out;
    cudaMalloc(&src, ITEMS * BYTES);
    cudaMalloc(&out, 1024 * 4);
    cudaMemset(src, 0, ITEMS * BYTES);
    ring<<<1, 32 * (CONSUMERS + 1)>>>(src, out);
    printf("probe: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
