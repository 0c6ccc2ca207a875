// runtime.h — host runtime internals shared by the C-ABI translation units (api.cu:
// single-GPU entry points, shard.cu: multi-GPU entry points).  Host code only.
#pragma once
#include "../../include/knn.h"
#include "internal.cuh"

#include <cuda_fp16.h>
#include <string>
#include <utility>
#include <vector>

namespace knn_rt {
struct Comm;  // shard.cu: the multi-GPU communicator (NCCL or host-callback transport)
}  // namespace knn_rt

struct knn_ctx {
    int device = 0;
    int num_sms = 148;
    bool tc_ok = false;
    int gemm_mode = 0;  // 0 = tensor-core split GEMM, 1 = SIMT FFMA (KNN_GEMM=simt)
    std::string err;
    void* ws = nullptr;  // compute workspace
    size_t ws_size = 0;
    void* io = nullptr;  // device copies for the host-buffer entry point
    size_t io_size = 0;
    int32_t* flag_host = nullptr;  // pinned copy of the workspace's flag slice (int32 x 4)
    int64_t last_candidates = 0;   // pivot plans: candidates kept by the last call
    int64_t launches = 0;
    size_t d_budget = (size_t)4 << 30;  // bytes of distance-matrix block per launch pair
    // per-kernel event timing (knn_profile_*)
    bool prof_on = false;
    std::vector<cudaEvent_t> ev_pool;
    struct Pending { int kind; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    int plan = KNN_PLAN_AUTO;  // knn_set_plan / env KNN_FUSED
    bool sym_ok = true;        // env KNN_SYM=0 disables the symmetric k-NNG GEMM
    bool pivot_ok = true;      // env KNN_PIVOT=0 disables the pivot (partition) plan
    int32_t pivot_cap = 2048;  // candidates per row kept by the partition GEMM
    int32_t pivot_div = 0;     // k <= 32 sample = N / pivot_div corpus points; 0: by N (sample_div)
    // k <= 32, L2 metrics: single-product partition + re-evaluation: -1 chosen
    // on the device per call (default), 1 always (env KNN_PIVOT1=1), 0 never (KNN_PIVOT1=0)
    int pivot1 = -1;
    bool last_plan_auto1 = false;
    float pivot1_ratio = 0.02f;  // pivot1_decide: largest bound width / mean pivot (env KNN_PIVOT1_RATIO)  // the last pivot-plan call let the device choose (finish_blocking reads it)
    float pivot_margin = __builtin_nanf("");  // KNN_PIVOT_MARGIN: override of the sample's error margin
    int64_t pivot_redos = 0;   // calls redone with the full matrix after an overflow
    int last_plan = -1;
    size_t sym_budget = (size_t)96 << 30;  // largest full N x N matrix for the symmetric plan
    double prof_ms[6] = {0, 0, 0, 0, 0, 0};
    int64_t prof_n[6] = {0, 0, 0, 0, 0, 0};
    // out-of-core streaming (knn_search_streamed): staging + running lists, copy stream
    void* st_buf = nullptr;
    size_t st_size = 0;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> ev_chunk;  // the host-pipelined k-NNG's chunk arrivals
    double last_stream_copy_ms = 0, last_stream_total_ms = 0;
    // knn_graph_pivots leaves the prepared operands of X at the start of ws (after the flag);
    // knn_graph_partition on the same (X, N, d, metric) reuses them while ws is untouched
    const float* prep_X = nullptr;
    int64_t prep_N = 0;
    int32_t prep_d = 0, prep_metric = -1;
    // Par-3 phases: the input-validation flag of the prep passes run by knn_graph_pivots /
    // knn_graph_partition (a dedicated slice: the workspace flag is reset by every call),
    // reported by knn_graph_gather_select as KNN_ERR_NONFINITE
    int32_t* pv_flag = nullptr;
    // Par-3 phases with the single-product partition (L2, k <= 32): knn_graph_partition
    // queues the device-chosen pair (p3_state 1) or the single-product one alone (2);
    // knn_graph_gather_select then re-evaluates from p3_X with the prep norms and bound terms
    // kept in p3_buf ([sqn | bnd], roundup(N, 256) floats each) and the pivots p3_thr
    int32_t p3_state = 0;
    const float* p3_X = nullptr;
    const float* p3_thr = nullptr;
    int64_t p3_N = 0;
    int32_t p3_d = 0, p3_metric = -1;
    void* p3_buf = nullptr;
    size_t p3_size = 0;
    // CUDA IPC mappings opened by knn_ipc_open: handle bytes -> mapped base
    std::vector<std::pair<std::string, void*>> ipc_open;
    // multi-GPU (shard.cu): communicator + the sharded calls' own buffers
    knn_rt::Comm* comm = nullptr;
};

namespace knn_rt {

using knn::ceil_div;
using knn::round_up;

knn_status fail(knn_ctx* c, knn_status st, const char* fmt, ...);
void comm_release(knn_ctx* ctx);  // shard.cu: frees ctx->comm (knn_ctx_destroy)

#define KNN_CUDA(call)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(ctx, KNN_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

#define KNN_TRY(call)                  \
    do {                               \
        knn_status s_ = (call);        \
        if (s_ != KNN_OK) return s_;   \
    } while (0)

knn_status ensure(knn_ctx* ctx, void** buf, size_t* size, size_t need);
cudaEvent_t take_event(knn_ctx* ctx);
void drain_profile(knn_ctx* ctx);
knn_status set_device(knn_ctx* ctx);
bool metric_ok(knn_ctx* ctx, int32_t metric, knn_status* st);

// Bump allocator over a workspace region (256-byte aligned slices).
struct Carve {
    char* base;
    size_t off = 0;
    template <class T>
    T* take(size_t count) {
        off = round_up((int64_t)off, 256);
        T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
        off += count * sizeof(T);
        return p;
    }
};

// Bracket one launch with events when profiling; usage:
//   Timed t(ctx, KIND, s); launch...; t.done();
struct Timed {
    knn_ctx* ctx; int kind; cudaStream_t s; cudaEvent_t a = nullptr;
    Timed(knn_ctx* c, int k, cudaStream_t st) : ctx(c), kind(k), s(st) {
        if (ctx->prof_on) {
            a = take_event(ctx);
            cudaEventRecord(a, s);
        }
    }
    void done() {
        ctx->launches++;
        if (!a) return;
        cudaEvent_t b = take_event(ctx);
        cudaEventRecord(b, s);
        ctx->pending.push_back({kind, a, b});
        a = nullptr;
    }
};

// Split operands of one point set, produced by prep.
struct Prepared {
    float* sqn;
    float* rs;
    __half* hi;
    __half* lo;
};

// The k <= 32 pivot sample's divisor for N corpus points (api.cu).
int32_t sample_div(const knn_ctx* ctx, int64_t N);
// Queue the whole hot path for one block problem (knn_search_block semantics); asynchronous.
knn_status run_block(knn_ctx* ctx, const float* Q, int64_t M, const float* X, int64_t N,
                     int32_t d, int32_t k, int32_t metric, int64_t self_shift, int64_t idx_offset,
                     int32_t* out_idx, float* out_dist, cudaStream_t s, bool allow_pivot = true);
// Wait for `s`, read the workspace flag: NONFINITE / INTERNAL (pivot-plan redo) / OK.
knn_status finish_blocking(knn_ctx* ctx, cudaStream_t s);
knn_status check_block_args(knn_ctx* ctx, const float* Q, int64_t M, const float* X, int64_t N,
                            int32_t d, int32_t k, int32_t metric, int64_t self_shift,
                            int64_t idx_offset, const void* out_idx, const void* out_dist);

}  // namespace knn_rt
