/* knn_demo.c — the C ABI of libknn.so used from plain C (no Python, no PyTorch).
 *
 *   gcc -std=c11 -Iinclude -I/usr/local/cuda/include examples/knn_demo.c \
 *       -Lpaper_1309_5478_b200 -lknn -L/usr/local/cuda/lib64 -lcudart -o knn_demo
 *   LD_LIBRARY_PATH=paper_1309_5478_b200 ./knn_demo [N d k]
 *
 * Builds the k-NN graph of N random points (knn_graph, device buffers) and prints the
 * neighbours of the first point; then the same through the host-buffer entry point. */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "knn.h"

#define CHECK(x)                                                                  \
    do {                                                                          \
        knn_status st_ = (x);                                                     \
        if (st_ != KNN_OK) {                                                      \
            fprintf(stderr, "%s failed: %d (%s)\n", #x, (int)st_, knn_last_error(ctx)); \
            return 1;                                                             \
        }                                                                         \
    } while (0)

int main(int argc, char** argv) {
    const int64_t N = argc > 1 ? atoll(argv[1]) : 4096;
    const int32_t d = argc > 2 ? atoi(argv[2]) : 64, k = argc > 3 ? atoi(argv[3]) : 8;
    float* X = (float*)malloc((size_t)N * d * sizeof(float));
    int32_t* idx = (int32_t*)malloc((size_t)N * k * sizeof(int32_t));
    float* dist = (float*)malloc((size_t)N * k * sizeof(float));
    uint64_t s = 1309;
    for (int64_t i = 0; i < N * d; ++i) {  /* xorshift, uniform [0, 1) */
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        X[i] = (float)((s >> 40) * (1.0 / 16777216.0));
    }
    knn_ctx_t ctx = NULL;
    if (knn_ctx_create(0, &ctx) != KNN_OK) {
        fprintf(stderr, "no usable CUDA device\n");
        return 1;
    }
    float *dX = NULL, *dD = NULL;
    int32_t* dI = NULL;
    cudaMalloc((void**)&dX, (size_t)N * d * sizeof(float));
    cudaMalloc((void**)&dI, (size_t)N * k * sizeof(int32_t));
    cudaMalloc((void**)&dD, (size_t)N * k * sizeof(float));
    cudaMemcpy(dX, X, (size_t)N * d * sizeof(float), cudaMemcpyHostToDevice);
    CHECK(knn_graph(ctx, dX, N, d, k, KNN_L2SQ, dI, dD, NULL));
    cudaMemcpy(idx, dI, (size_t)N * k * sizeof(int32_t), cudaMemcpyDeviceToHost);
    cudaMemcpy(dist, dD, (size_t)N * k * sizeof(float), cudaMemcpyDeviceToHost);
    printf("k-NNG N=%lld d=%d k=%d, plan %d; point 0:", (long long)N, d, k, knn_last_plan(ctx));
    for (int r = 0; r < k; ++r) printf(" %d(%.4f)", idx[r], dist[r]);
    printf("\n");
    /* the same graph through the host-buffer entry point (copies inside the call) */
    CHECK(knn_search_block_host(ctx, X, N, X, N, d, k, KNN_L2SQ, 0, 0, idx, dist, NULL));
    printf("host-buffer API, point 0 nearest: %d (%.4f)\n", idx[0], dist[0]);
    /* the multi-GPU boundary from C: an NCCL communicator (one rank here; with one process
       per GPU, rank 0 makes the id and the caller ships it to the others) and the sharded
       k-NNG (the triangle split over the ranks; every rank gets the full graph) */
    uint8_t uid[128];
    if (knn_comm_unique_id(uid) == KNN_OK) {
        CHECK(knn_comm_init(ctx, 0, 1, uid));
        CHECK(knn_graph_sharded(ctx, KNN_SHARD_SYM, dX, N, d, k, KNN_L2SQ, dI, dD, NULL));
        cudaMemcpy(idx, dI, (size_t)k * sizeof(int32_t), cudaMemcpyDeviceToHost);
        int32_t backend = 0, rank = 0, nranks = 0;
        knn_comm_info(ctx, &backend, &rank, &nranks);
        printf("sharded (backend %d, %d rank): point 0 nearest: %d\n", backend, nranks, idx[0]);
        CHECK(knn_comm_destroy(ctx));
    } else {
        printf("NCCL not loadable: sharded call skipped\n");
    }
    cudaFree(dX);
    cudaFree(dI);
    cudaFree(dD);
    knn_ctx_destroy(ctx);
    free(X);
    free(idx);
    free(dist);
    return 0;
}
