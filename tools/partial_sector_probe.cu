// Probe (diagnostic, not part of the library): does the B200 L2 fetch a 32-byte sector
// from HBM when a store covers only part of it?  Each kernel writes the same 256 MiB
// (every byte once); only the store granularity / timing differs.  Run under ncu with
// dram__bytes_read.sum: full-sector stores need no reads; partial stores completed within
// a short time either need none (merge in L2) or one fill per sector (fill on first touch).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// A: each thread writes one 16-byte vector; a warp covers 512 contiguous bytes (full sectors)
__global__ void full_sectors(uint4* p, size_t n16) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i < n16; i += (size_t)gridDim.x * blockDim.x) p[i] = make_uint4(1, 2, 3, 4);
}
// B: 4-byte stores, sector completed by 8 consecutive stores of the same thread
__global__ void partial_quick(uint32_t* p, size_t n4) {
    size_t s = blockIdx.x * (size_t)blockDim.x + threadIdx.x;  // sector index
    for (; s * 8 < n4; s += (size_t)gridDim.x * blockDim.x)
        #pragma unroll
        for (int j = 0; j < 8; ++j) p[s * 8 + j] = j;
}
// C: 8-byte stores, sector completed by 4 stores spread over the whole kernel (pass j writes
// word j of every sector), the pattern of per-row candidate lists
__global__ void partial_slow(uint2* p, size_t n8, int j) {
    size_t s = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; s * 4 < n8; s += (size_t)gridDim.x * blockDim.x) p[s * 4 + j] = make_uint2(j, j);
}

int main() {
    const size_t bytes = (size_t)256 << 20;
    void* p = nullptr;
    cudaMalloc(&p, bytes);
    cudaMemset(p, 0, bytes);
    cudaDeviceSynchronize();
    full_sectors<<<148 * 8, 256>>>(static_cast<uint4*>(p), bytes / 16);
    partial_quick<<<148 * 8, 256>>>(static_cast<uint32_t*>(p), bytes / 4);
    for (int j = 0; j < 4; ++j) partial_slow<<<148 * 8, 256>>>(static_cast<uint2*>(p), bytes / 8, j);
    cudaDeviceSynchronize();
    printf("probe done: %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaFree(p);
    return 0;
}
