// shard.cu — multi-GPU entry points of the C ABI (include/knn.h, "multi-GPU"): one process
// per GPU, a communicator per ctx (NCCL over NVLink / NVSwitch, loaded at run time, or a
// caller-supplied host transport), and the three shardings of the brute-force k-NN
// (PAPER.md:102 names batch execution with data partitioning and the
// merging of results as the way past one GPU).  Host code only: every step of the hot path
// is one of the single-GPU phases of api.cu (run_block, the Par-3 phases) or a kernel of
// select.cu (the k-way merge); the collectives are issued on the caller's stream.
#include "runtime.h"

#include <dlfcn.h>
#include <nccl.h>  // types and enum values only: the library is dlopen'ed

#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#ifndef KNN_NCCL_LIB
#define KNN_NCCL_LIB ""
#endif

namespace knn_rt {

// ----------------------------------------------------------------------- NCCL loader --
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string err;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = nullptr;
        const char* env = getenv("KNN_NCCL_LIB");
        // torch (or any earlier user) has usually loaded libnccl.so.2 already: same instance
        const char* names[] = {env, "libnccl.so.2", KNN_NCCL_LIB};
        for (const char* n : names) {
            if (!n || !n[0]) continue;
            h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            a.err = "cannot load libnccl.so.2 (set KNN_NCCL_LIB)";
            return a;
        }
        bool all = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) all = false;
        };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.AllGather, "ncclAllGather");
        sym(a.Broadcast, "ncclBroadcast");
        sym(a.AllReduce, "ncclAllReduce");
        sym(a.Send, "ncclSend");
        sym(a.Recv, "ncclRecv");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        sym(a.GetErrorString, "ncclGetErrorString");
        a.ok = all;
        if (!all) a.err = "libnccl.so.2 lacks an expected symbol";
        return a;
    }();
    return api;
}

// ----------------------------------------------------------------------- communicator --
struct Comm {
    int backend = 0;  // 1 NCCL, 2 host callbacks
    int rank = 0, nranks = 1;
    ncclComm_t nc = nullptr;
    knn_comm_ops ops{};
    // device scratch of the sharded calls (thr, staged outputs, partial lists); apart from
    // ctx->ws, which the single-GPU phases they call reuse
    void* buf = nullptr;
    size_t buf_size = 0;
    int32_t* dflag = nullptr;  // device int32 x 4: agreement / barrier all-reduces
    void* hbuf = nullptr;      // pinned host staging of the callback transport
    size_t hbuf_size = 0;
    // Par-3 candidate lists: one cudaMalloc (cnt | cent) so that one IPC handle maps it;
    // peers' lists mapped once per allocation
    void* lists = nullptr;
    int64_t lists_N = 0;
    int32_t lists_cap = 0;
    std::vector<void*> peer;  // per rank: base of its lists in this process (own = lists)
    int peer_state = 0;       // 0 not exchanged, 1 mapped, -1 unavailable (fallback)
    int last_mode = -1;
};

namespace {

#define KNN_NCCL(call)                                                                        \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return fail(ctx, KNN_ERR_NCCL, "%s failed: %s", #call, nccl().GetErrorString(r_)); \
    } while (0)

void release_lists(knn_ctx* ctx, Comm* c) {
    for (int g = 0; g < (int)c->peer.size(); ++g)
        if (c->peer[g] && g != c->rank) cudaIpcCloseMemHandle(c->peer[g]);
    c->peer.clear();
    c->peer_state = 0;
    if (c->lists) cudaFree(c->lists);
    c->lists = nullptr;
    c->lists_N = 0;
    c->lists_cap = 0;
    (void)ctx;
}

knn_status host_stage(knn_ctx* ctx, Comm* c, size_t bytes) {
    if (bytes <= c->hbuf_size) return KNN_OK;
    if (c->hbuf) cudaFreeHost(c->hbuf);
    c->hbuf = nullptr;
    c->hbuf_size = 0;
    if (cudaHostAlloc(&c->hbuf, bytes, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        c->hbuf = nullptr;
        return fail(ctx, KNN_ERR_OOM, "cannot pin %zu bytes of host staging", bytes);
    }
    c->hbuf_size = bytes;
    return KNN_OK;
}

// --- collectives (device buffers, stream-ordered for NCCL; blocking for callbacks) -------
knn_status c_bcast(knn_ctx* ctx, void* buf, size_t bytes, cudaStream_t s) {
    Comm* c = ctx->comm;
    if (!c || c->nranks == 1 || bytes == 0) return KNN_OK;
    if (c->backend == 1) {
        KNN_NCCL(nccl().Broadcast(buf, buf, bytes, ncclUint8, 0, c->nc, s));
        return KNN_OK;
    }
    KNN_TRY(host_stage(ctx, c, bytes));
    if (c->rank == 0) KNN_CUDA(cudaMemcpyAsync(c->hbuf, buf, bytes, cudaMemcpyDeviceToHost, s));
    KNN_CUDA(cudaStreamSynchronize(s));
    if (c->ops.broadcast(c->ops.user, c->hbuf, (int64_t)bytes, 0) != 0)
        return fail(ctx, KNN_ERR_NCCL, "broadcast callback failed");
    if (c->rank != 0) KNN_CUDA(cudaMemcpyAsync(buf, c->hbuf, bytes, cudaMemcpyHostToDevice, s));
    KNN_CUDA(cudaStreamSynchronize(s));
    return KNN_OK;
}

// recv holds nranks blocks of `bytes`; send may be recv + rank * bytes (in place)
knn_status c_allgather(knn_ctx* ctx, const void* send, void* recv, size_t bytes, cudaStream_t s) {
    Comm* c = ctx->comm;
    const int G = c ? c->nranks : 1;
    if (G == 1) {
        if (send != recv) KNN_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
        return KNN_OK;
    }
    if (c->backend == 1) {
        KNN_NCCL(nccl().AllGather(send, recv, bytes, ncclUint8, c->nc, s));
        return KNN_OK;
    }
    KNN_TRY(host_stage(ctx, c, bytes * (G + 1)));
    char* hsend = static_cast<char*>(c->hbuf) + bytes * G;
    KNN_CUDA(cudaMemcpyAsync(hsend, send, bytes, cudaMemcpyDeviceToHost, s));
    KNN_CUDA(cudaStreamSynchronize(s));
    if (c->ops.allgather(c->ops.user, hsend, c->hbuf, (int64_t)bytes) != 0)
        return fail(ctx, KNN_ERR_NCCL, "allgather callback failed");
    KNN_CUDA(cudaMemcpyAsync(recv, c->hbuf, bytes * G, cudaMemcpyHostToDevice, s));
    KNN_CUDA(cudaStreamSynchronize(s));
    return KNN_OK;
}

// block g of send (bytes each) goes to rank g; block g of recv comes from rank g
knn_status c_alltoall(knn_ctx* ctx, const void* send, void* recv, size_t bytes, cudaStream_t s) {
    Comm* c = ctx->comm;
    const int G = c ? c->nranks : 1;
    if (G == 1) {
        KNN_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
        return KNN_OK;
    }
    if (c->backend == 1) {
        const char* sp = static_cast<const char*>(send);
        char* rp = static_cast<char*>(recv);
        KNN_NCCL(nccl().GroupStart());
        for (int g = 0; g < G; ++g) {
            KNN_NCCL(nccl().Send(sp + g * bytes, bytes, ncclUint8, g, c->nc, s));
            KNN_NCCL(nccl().Recv(rp + g * bytes, bytes, ncclUint8, g, c->nc, s));
        }
        KNN_NCCL(nccl().GroupEnd());
        return KNN_OK;
    }
    KNN_TRY(host_stage(ctx, c, 2 * bytes * G));
    char* hs = static_cast<char*>(c->hbuf);
    char* hr = hs + bytes * G;
    KNN_CUDA(cudaMemcpyAsync(hs, send, bytes * G, cudaMemcpyDeviceToHost, s));
    KNN_CUDA(cudaStreamSynchronize(s));
    if (c->ops.alltoall(c->ops.user, hs, hr, (int64_t)bytes) != 0)
        return fail(ctx, KNN_ERR_NCCL, "alltoall callback failed");
    KNN_CUDA(cudaMemcpyAsync(recv, hr, bytes * G, cudaMemcpyHostToDevice, s));
    KNN_CUDA(cudaStreamSynchronize(s));
    return KNN_OK;
}

// The largest `code` over the ranks (0 = all fine).  Blocking.  Also a full barrier: it
// returns on a rank only after every rank has reached it.
knn_status c_agree(knn_ctx* ctx, int32_t code, int32_t* out, cudaStream_t s) {
    Comm* c = ctx->comm;
    *out = code;
    if (!c || c->nranks == 1) return KNN_OK;
    if (c->backend == 1) {
        KNN_CUDA(cudaMemcpyAsync(c->dflag, &code, sizeof code, cudaMemcpyHostToDevice, s));
        KNN_NCCL(nccl().AllReduce(c->dflag, c->dflag, 1, ncclInt32, ncclMax, c->nc, s));
        KNN_CUDA(cudaMemcpyAsync(ctx->flag_host, c->dflag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        KNN_CUDA(cudaStreamSynchronize(s));
        *out = ctx->flag_host[0];
        return KNN_OK;
    }
    KNN_CUDA(cudaStreamSynchronize(s));
    int32_t v = code;
    if (c->ops.allreduce_max_i32(c->ops.user, &v, 1) != 0)
        return fail(ctx, KNN_ERR_NCCL, "allreduce callback failed");
    *out = v;
    return KNN_OK;
}

// Stream-ordered barrier: work queued on `s` after it runs only when every rank's work
// queued before it has completed (an all-reduce cannot finish before every rank joined).
knn_status c_stream_barrier(knn_ctx* ctx, cudaStream_t s) {
    Comm* c = ctx->comm;
    if (!c || c->nranks == 1) return KNN_OK;
    if (c->backend == 1) {
        KNN_NCCL(nccl().AllReduce(c->dflag + 1, c->dflag + 1, 1, ncclInt32, ncclMax, c->nc, s));
        return KNN_OK;
    }
    int32_t v;
    return c_agree(ctx, 0, &v, s);
}

// ----------------------------------------------------------------------- helpers ------
struct Range {
    int64_t lo, hi;
};
Range shard_range(int64_t n, int parts, int r) {
    const int64_t per = ceil_div(n, (int64_t)parts);
    int64_t lo = (int64_t)r * per;
    if (lo > n) lo = n;
    const int64_t hi = lo + per < n ? lo + per : n;
    return {lo, hi};
}

// Status agreement: 0 ok, 1 fall back (certificate / no peer mappings), 2 local error.
// Returns the agreed code; `local` keeps the rank's own failure message.
knn_status agree_status(knn_ctx* ctx, knn_status local, int fallback, int32_t* agreed, cudaStream_t s) {
    const int32_t code = local != KNN_OK ? 2 : fallback ? 1 : 0;
    const std::string msg = ctx->err;
    KNN_TRY(c_agree(ctx, code, agreed, s));
    if (local != KNN_OK) {
        ctx->err = msg;
        return local;
    }
    if (*agreed == 2) return fail(ctx, KNN_ERR_INTERNAL, "a peer rank failed in the sharded call");
    return KNN_OK;
}

// Gather every rank's block of `per` rows (k entries each) into the rows×k outputs.  When
// the blocks tile the output exactly the gather runs in place on it; else through a staged
// [G*per][k] copy.  `own_*` is where this rank wrote its block.
knn_status gather_rows(knn_ctx* ctx, int32_t* own_i, float* own_d, int32_t* stage_i, float* stage_d,
                       int64_t per, int64_t rows, int32_t k, int32_t* out_idx, float* out_dist,
                       cudaStream_t s) {
    const int G = ctx->comm ? ctx->comm->nranks : 1;
    const bool inplace = per * G == rows;
    int32_t* ri = inplace ? out_idx : stage_i;
    float* rd = inplace ? out_dist : stage_d;
    KNN_TRY(c_allgather(ctx, own_i, ri, (size_t)per * k * sizeof(int32_t), s));
    KNN_TRY(c_allgather(ctx, own_d, rd, (size_t)per * k * sizeof(float), s));
    if (!inplace) {
        KNN_CUDA(cudaMemcpyAsync(out_idx, stage_i, (size_t)rows * k * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        KNN_CUDA(cudaMemcpyAsync(out_dist, stage_d, (size_t)rows * k * sizeof(float), cudaMemcpyDeviceToDevice, s));
    }
    KNN_CUDA(cudaStreamSynchronize(s));
    return KNN_OK;
}

// Par-1: query rows.  graph: Q == X (k-NNG, self excluded by global position).
knn_status run_query_sharded(knn_ctx* ctx, const float* Q, int64_t M, const float* X, int64_t N, int32_t d,
                             int32_t k, int32_t metric, bool graph, int32_t* out_idx, float* out_dist,
                             cudaStream_t s) {
    const int G = ctx->comm ? ctx->comm->nranks : 1, r = ctx->comm ? ctx->comm->rank : 0;
    const int64_t per = ceil_div(M, (int64_t)G);
    const Range rr = shard_range(M, G, r);
    const bool inplace = per * G == M;
    int32_t *stage_i = nullptr, *own_i;
    float *stage_d = nullptr, *own_d;
    if (inplace) {
        own_i = out_idx + rr.lo * k;
        own_d = out_dist + rr.lo * k;
    } else {
        Comm* c = ctx->comm;
        Carve probe{nullptr};
        probe.take<int32_t>((size_t)G * per * k);
        probe.take<float>((size_t)G * per * k);
        KNN_TRY(ensure(ctx, &c->buf, &c->buf_size, probe.off + 256));
        Carve cv{static_cast<char*>(c->buf)};
        stage_i = cv.take<int32_t>((size_t)G * per * k);
        stage_d = cv.take<float>((size_t)G * per * k);
        own_i = stage_i + (size_t)r * per * k;
        own_d = stage_d + (size_t)r * per * k;
    }
    knn_status st = KNN_OK;
    if (rr.hi > rr.lo)
        st = knn_search_block(ctx, Q + rr.lo * d, rr.hi - rr.lo, X, N, d, k, metric, graph ? rr.lo : KNN_NO_SELF,
                              0, own_i, own_d, s);
    int32_t agreed;
    KNN_TRY(agree_status(ctx, st, 0, &agreed, s));
    if (ctx->comm) ctx->comm->last_mode = KNN_SHARD_QUERY;
    return gather_rows(ctx, own_i, own_d, stage_i, stage_d, per, M, k, out_idx, out_dist, s);
}

// Par-2: corpus columns.  Every rank: partial top-k of all M rows against its columns,
// all-to-all of the row blocks, k-way merge (a-S6) of the rank's rows, all-gather.
knn_status run_corpus_sharded(knn_ctx* ctx, const float* Q, int64_t M, const float* X, int64_t N, int32_t d,
                              int32_t k, int32_t metric, bool graph, int32_t* out_idx, float* out_dist,
                              cudaStream_t s) {
    Comm* c = ctx->comm;
    const int G = c ? c->nranks : 1, r = c ? c->rank : 0;
    for (int g = 0; g < G; ++g) {
        const Range cg = shard_range(N, G, g);
        if (cg.hi - cg.lo < k)
            return fail(ctx, KNN_ERR_ARG, "corpus sharding needs k <= every column block (k=%d, block %lld)", k,
                        (long long)(cg.hi - cg.lo));
    }
    const int64_t per = ceil_div(M, (int64_t)G);
    const Range cr = shard_range(N, G, r), rr = shard_range(M, G, r);
    const size_t ent = (size_t)G * per * k;
    int32_t *part_i, *recv_i, *stage_i, *own_i;
    float *part_d, *recv_d, *stage_d, *own_d;
    auto layout = [&](Carve& cv) {
        part_i = cv.take<int32_t>(ent);
        part_d = cv.take<float>(ent);
        recv_i = cv.take<int32_t>(ent);
        recv_d = cv.take<float>(ent);
        stage_i = cv.take<int32_t>(ent);
        stage_d = cv.take<float>(ent);
    };
    if (!c) return fail(ctx, KNN_ERR_INTERNAL, "no communicator");
    Carve probe{nullptr};
    layout(probe);
    KNN_TRY(ensure(ctx, &c->buf, &c->buf_size, probe.off + 256));
    Carve cv{static_cast<char*>(c->buf)};
    layout(cv);
    const bool inplace = per * G == M;
    own_i = inplace ? out_idx + rr.lo * k : stage_i + (size_t)r * per * k;
    own_d = inplace ? out_dist + rr.lo * k : stage_d + (size_t)r * per * k;
    // rows M .. G*per of the partial lists are padding: never merged
    knn_status st = knn_search_block(ctx, Q, M, X + cr.lo * d, cr.hi - cr.lo, d, k, metric,
                                     graph ? -cr.lo : KNN_NO_SELF, cr.lo, part_i, part_d, s);
    int32_t agreed;
    KNN_TRY(agree_status(ctx, st, 0, &agreed, s));
    KNN_TRY(c_alltoall(ctx, part_i, recv_i, (size_t)per * k * sizeof(int32_t), s));
    KNN_TRY(c_alltoall(ctx, part_d, recv_d, (size_t)per * k * sizeof(float), s));
    if (rr.hi > rr.lo) {
        // recv block g = rank g's lists of this rank's rows ([G][per][k]; global indices)
        std::vector<const float*> dl(G);
        std::vector<const int32_t*> il(G);
        std::vector<int64_t> zeros(G, 0);
        for (int g = 0; g < G; ++g) {
            dl[g] = recv_d + (size_t)g * per * k;
            il[g] = recv_i + (size_t)g * per * k;
        }
        Timed tm(ctx, KNN_KERNEL_SHARD_MERGE, s);
        KNN_CUDA(knn::launch_merge_lists(dl.data(), il.data(), G, 0, rr.hi - rr.lo, k, zeros.data(), own_i, own_d,
                                         s));
        tm.done();
    }
    c->last_mode = KNN_SHARD_CORPUS;
    return gather_rows(ctx, own_i, own_d, stage_i, stage_d, per, M, k, out_idx, out_dist, s);
}

// Par-3 lists: (re)allocate for (N, cap); a new allocation needs a new peer exchange.
knn_status ensure_lists(knn_ctx* ctx, Comm* c, int64_t N, int32_t cap) {
    if (c->lists && c->lists_N == N && c->lists_cap == cap) return KNN_OK;
    KNN_CUDA(cudaDeviceSynchronize());
    release_lists(ctx, c);
    const size_t bytes = (size_t)round_up(N, knn::kColPad) * 4 + (size_t)N * cap * 8;
    if (cudaMalloc(&c->lists, bytes) != cudaSuccess) {
        cudaGetLastError();
        c->lists = nullptr;
        return fail(ctx, KNN_ERR_OOM, "cannot allocate %zu bytes of Par-3 candidate lists", bytes);
    }
    c->lists_N = N;
    c->lists_cap = cap;
    return KNN_OK;
}

// Exchange IPC handles of the lists allocation and map every peer's (once per allocation).
// Every rank ends with the same verdict (agreement all-reduce).
knn_status exchange_peers(knn_ctx* ctx, Comm* c, cudaStream_t s) {
    if (c->peer_state != 0) return KNN_OK;
    const int G = c->nranks;
    struct Entry {
        uint8_t handle[64];
        int32_t ok;
        int32_t pad;
    };
    static_assert(sizeof(Entry) == 72, "entry");
    Entry mine{};
    cudaIpcMemHandle_t h;
    const bool no_ipc = getenv("KNN_SHARD_NO_IPC") && strcmp(getenv("KNN_SHARD_NO_IPC"), "1") == 0;
    if (!no_ipc && cudaIpcGetMemHandle(&h, c->lists) == cudaSuccess) {
        memcpy(mine.handle, &h, 64);
        mine.ok = 1;
    }
    cudaGetLastError();
    // device staging: [G+1] entries at the start of the scratch buffer
    KNN_TRY(ensure(ctx, &c->buf, &c->buf_size, sizeof(Entry) * (G + 1) + 256));
    Entry* dall = static_cast<Entry*>(c->buf);
    Entry* dmine = dall + G;
    KNN_CUDA(cudaMemcpyAsync(dmine, &mine, sizeof mine, cudaMemcpyHostToDevice, s));
    KNN_TRY(c_allgather(ctx, dmine, dall, sizeof(Entry), s));
    std::vector<Entry> all(G);
    KNN_CUDA(cudaMemcpyAsync(all.data(), dall, sizeof(Entry) * G, cudaMemcpyDeviceToHost, s));
    KNN_CUDA(cudaStreamSynchronize(s));
    bool ok = true;
    c->peer.assign(G, nullptr);
    for (int g = 0; g < G && ok; ++g) {
        if (!all[g].ok) {
            ok = false;
            break;
        }
        if (g == c->rank) {
            c->peer[g] = c->lists;
            continue;
        }
        cudaIpcMemHandle_t hg;
        memcpy(&hg, all[g].handle, 64);
        void* base = nullptr;
        if (cudaIpcOpenMemHandle(&base, hg, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            ok = false;
            break;
        }
        c->peer[g] = base;
    }
    int32_t agreed;
    KNN_TRY(c_agree(ctx, ok ? 0 : 1, &agreed, s));
    if (agreed != 0) {
        for (int g = 0; g < G; ++g)
            if (c->peer[g] && g != c->rank) cudaIpcCloseMemHandle(c->peer[g]);
        c->peer.clear();
        c->peer_state = -1;
    } else {
        c->peer_state = 1;
    }
    return KNN_OK;
}

// Par-3: the symmetric k-NNG with the upper triangle split over the ranks.
// Returns KNN_OK with *fallback = true when the caller must run Par-1 instead (all ranks
// alike).
knn_status run_sym_sharded(knn_ctx* ctx, const float* X, int64_t N, int32_t d, int32_t k, int32_t metric,
                           int32_t* out_idx, float* out_dist, cudaStream_t s, bool* fallback) {
    Comm* c = ctx->comm;
    const int G = c->nranks, r = c->rank;
    *fallback = false;
    const int64_t per = ceil_div(N, (int64_t)G);
    const Range rr = shard_range(N, G, r);
    const int64_t npad = round_up(N, knn::kColPad);
    const int64_t T = npad > G * per ? npad : G * per;
    const int32_t cap = knn_graph_list_cap(k);
    KNN_TRY(ensure_lists(ctx, c, N, cap));
    if (G > 1) KNN_TRY(exchange_peers(ctx, c, s));
    if (G > 1 && c->peer_state != 1) {
        *fallback = true;
        return KNN_OK;
    }
    const bool inplace = per * G == N;
    float* thr;
    int32_t *stage_i = nullptr, *own_i;
    float *stage_d = nullptr, *own_d;
    auto layout = [&](Carve& cv) {
        cv.take<uint8_t>(72 * (G + 1));  // exchange_peers' staging (kept)
        thr = cv.take<float>(T);
        if (!inplace) {
            stage_i = cv.take<int32_t>((size_t)G * per * k);
            stage_d = cv.take<float>((size_t)G * per * k);
        }
    };
    Carve probe{nullptr};
    layout(probe);
    KNN_TRY(ensure(ctx, &c->buf, &c->buf_size, probe.off + 256));
    Carve cv{static_cast<char*>(c->buf)};
    layout(cv);
    own_i = inplace ? out_idx + rr.lo * k : stage_i + (size_t)r * per * k;
    own_d = inplace ? out_dist + rr.lo * k : stage_d + (size_t)r * per * k;
    // 1. pivots of this rank's rows, all-gathered (thr past N: NaN, keeps nothing)
    KNN_CUDA(cudaMemsetAsync(thr, 0xFF, (size_t)T * sizeof(float), s));
    knn_status st = KNN_OK;
    if (rr.hi > rr.lo) st = knn_graph_pivots(ctx, X, N, d, k, metric, rr.lo, rr.hi - rr.lo, thr, s);
    int32_t agreed;
    KNN_TRY(agree_status(ctx, st, 0, &agreed, s));
    KNN_TRY(c_allgather(ctx, thr + (size_t)r * per, thr, (size_t)per * sizeof(float), s));
    KNN_CUDA(cudaMemsetAsync(thr + N, 0xFF, (size_t)(T - N) * sizeof(float), s));
    // 2. partition GEMM over this rank's units of the triangle -> own lists (any row)
    int32_t* cnt = static_cast<int32_t*>(c->lists);
    uint64_t* cent = reinterpret_cast<uint64_t*>(static_cast<char*>(c->lists) + npad * 4);
    const Range ur = shard_range(knn_graph_units(N), G, r);
    st = knn_graph_partition(ctx, X, N, d, k, metric, thr, ur.lo, ur.hi, cnt, cent, cap, s);
    KNN_TRY(agree_status(ctx, st, 0, &agreed, s));  // also: every rank's partition was queued
    // every rank's partition must be complete before any rank reads its lists
    KNN_TRY(c_stream_barrier(ctx, s));
    // 3. exact select of this rank's rows from the G ranks' lists (peer memory over NVLink)
    std::vector<const int32_t*> cnts(G);
    std::vector<const uint64_t*> cents(G);
    for (int g = 0; g < G; ++g) {
        char* base = static_cast<char*>(G > 1 ? c->peer[g] : c->lists);
        cnts[g] = reinterpret_cast<const int32_t*>(base);
        cents[g] = reinterpret_cast<const uint64_t*>(base + npad * 4);
    }
    st = KNN_OK;
    if (rr.hi > rr.lo)
        st = knn_graph_gather_select(ctx, G, cnts.data(), cents.data(), cap, N, k, rr.lo, rr.hi - rr.lo, own_i,
                                     own_d, s);
    const bool cert_failed = st == KNN_ERR_INTERNAL;
    // after this agreement no rank reads another's lists any more (each contributes after
    // its blocking select), so the next call may overwrite them
    KNN_TRY(agree_status(ctx, cert_failed ? KNN_OK : st, cert_failed, &agreed, s));
    if (agreed == 1) {
        *fallback = true;
        return KNN_OK;
    }
    c->last_mode = KNN_SHARD_SYM;
    return gather_rows(ctx, own_i, own_d, stage_i, stage_d, per, N, k, out_idx, out_dist, s);
}

// One rank runs the single-GPU call directly (the decompositions only add exchanges);
// env KNN_SHARD_G1_PHASES=1 (tests) runs the sharded phases anyway.
bool g1_phases() {
    const char* v = getenv("KNN_SHARD_G1_PHASES");
    return v && strcmp(v, "1") == 0;
}

// One-rank communicator used when the caller never initialised one.
Comm* comm_or_single(knn_ctx* ctx) {
    if (!ctx->comm) {
        ctx->comm = new Comm();
        ctx->comm->backend = 0;
    }
    return ctx->comm;
}

knn_status comm_common_init(knn_ctx* ctx, int32_t rank, int32_t nranks) {
    if (rank < 0 || nranks < 1 || rank >= nranks) return fail(ctx, KNN_ERR_ARG, "bad rank %d / nranks %d", rank, nranks);
    KNN_TRY(set_device(ctx));
    comm_release(ctx);
    Comm* c = new Comm();
    c->rank = rank;
    c->nranks = nranks;
    if (cudaMalloc(&c->dflag, 4 * sizeof(int32_t)) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return fail(ctx, KNN_ERR_OOM, "cannot allocate the communicator flag");
    }
    cudaMemset(c->dflag, 0, 4 * sizeof(int32_t));
    ctx->comm = c;
    return KNN_OK;
}

}  // namespace

void comm_release(knn_ctx* ctx) {
    Comm* c = ctx->comm;
    if (!c) return;
    cudaDeviceSynchronize();
    release_lists(ctx, c);
    if (c->nc && nccl().ok) nccl().CommDestroy(c->nc);
    if (c->buf) cudaFree(c->buf);
    if (c->dflag) cudaFree(c->dflag);
    if (c->hbuf) cudaFreeHost(c->hbuf);
    delete c;
    ctx->comm = nullptr;
}

}  // namespace knn_rt

using namespace knn_rt;

extern "C" {

void knn_shard_range(int64_t n, int32_t parts, int32_t r, int64_t* lo, int64_t* hi) {
    if (!lo || !hi) return;
    if (n < 0 || parts < 1 || r < 0 || r >= parts) {
        *lo = *hi = 0;
        return;
    }
    const Range rg = shard_range(n, parts, r);
    *lo = rg.lo;
    *hi = rg.hi;
}

knn_status knn_comm_unique_id(uint8_t id[128]) {
    if (!id) return KNN_ERR_ARG;
    if (!nccl().ok) return KNN_ERR_NCCL;
    ncclUniqueId u;
    if (nccl().GetUniqueId(&u) != ncclSuccess) return KNN_ERR_NCCL;
    static_assert(sizeof(u) == 128, "NCCL unique id size");
    memcpy(id, &u, 128);
    return KNN_OK;
}

knn_status knn_comm_init(knn_ctx_t ctx, int32_t rank, int32_t nranks, const uint8_t id[128]) {
    if (!ctx || !id) return KNN_ERR_ARG;
    if (!nccl().ok) return fail(ctx, KNN_ERR_NCCL, "%s", nccl().err.c_str());
    KNN_TRY(comm_common_init(ctx, rank, nranks));
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclComm_t nc = nullptr;
    const ncclResult_t r = nccl().CommInitRank(&nc, nranks, u, rank);
    if (r != ncclSuccess) {
        comm_release(ctx);
        return fail(ctx, KNN_ERR_NCCL, "ncclCommInitRank: %s", nccl().GetErrorString(r));
    }
    ctx->comm->nc = nc;
    ctx->comm->backend = 1;
    return KNN_OK;
}

knn_status knn_comm_init_ops(knn_ctx_t ctx, int32_t rank, int32_t nranks, const knn_comm_ops* ops) {
    if (!ctx || !ops || !ops->allgather || !ops->broadcast || !ops->alltoall || !ops->allreduce_max_i32)
        return KNN_ERR_ARG;
    KNN_TRY(comm_common_init(ctx, rank, nranks));
    ctx->comm->ops = *ops;
    ctx->comm->backend = 2;
    return KNN_OK;
}

knn_status knn_comm_destroy(knn_ctx_t ctx) {
    if (!ctx) return KNN_ERR_ARG;
    cudaSetDevice(ctx->device);
    comm_release(ctx);
    return KNN_OK;
}

knn_status knn_comm_info(knn_ctx_t ctx, int32_t* backend, int32_t* rank, int32_t* nranks) {
    if (!ctx || !backend || !rank || !nranks) return KNN_ERR_ARG;
    const Comm* c = ctx->comm;
    *backend = c ? c->backend : 0;
    *rank = c ? c->rank : 0;
    *nranks = c ? c->nranks : 1;
    return KNN_OK;
}

int knn_last_shard_mode(knn_ctx_t ctx) { return ctx && ctx->comm ? ctx->comm->last_mode : -1; }

knn_status knn_graph_sharded(knn_ctx_t ctx, int32_t shard_mode, float* X, int64_t N, int32_t d, int32_t k,
                             int32_t metric, int32_t* out_idx, float* out_dist, void* stream) {
    if (!ctx) return KNN_ERR_ARG;
    if (shard_mode < KNN_SHARD_QUERY || shard_mode > KNN_SHARD_SYM)
        return fail(ctx, KNN_ERR_ARG, "unknown shard mode %d", shard_mode);
    if (N >= 1 && k > N - 1)
        return fail(ctx, KNN_ERR_ARG, "knn_graph needs k <= N-1 (k=%d, N=%lld)", k, (long long)N);
    KNN_TRY(check_block_args(ctx, X, N, X, N, d, k, metric, 0, 0, out_idx, out_dist));
    KNN_TRY(set_device(ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Comm* c = comm_or_single(ctx);
    if (c->nranks == 1 && !g1_phases()) {  // one rank: every mode is the single-GPU k-NNG
        c->last_mode = shard_mode;
        return knn_search_block(ctx, X, N, X, N, d, k, metric, 0, 0, out_idx, out_dist, stream);
    }
    KNN_TRY(c_bcast(ctx, X, (size_t)N * d * sizeof(float), s));
    if (shard_mode == KNN_SHARD_SYM) {
        const bool able = N >= 16384 && k <= KNN_MAX_K && ctx->gemm_mode == 0 && ctx->tc_ok;
        if (able) {
            bool fallback = false;
            KNN_TRY(run_sym_sharded(ctx, X, N, d, k, metric, out_idx, out_dist, s, &fallback));
            if (!fallback) return KNN_OK;
        }
        shard_mode = KNN_SHARD_QUERY;
    }
    (void)c;
    if (shard_mode == KNN_SHARD_CORPUS)
        return run_corpus_sharded(ctx, X, N, X, N, d, k, metric, true, out_idx, out_dist, s);
    return run_query_sharded(ctx, X, N, X, N, d, k, metric, true, out_idx, out_dist, s);
}

knn_status knn_search_sharded(knn_ctx_t ctx, int32_t shard_mode, float* Q, int64_t M, float* X, int64_t N,
                              int32_t d, int32_t k, int32_t* out_idx, float* out_dist, void* stream) {
    if (!ctx) return KNN_ERR_ARG;
    if (shard_mode != KNN_SHARD_QUERY && shard_mode != KNN_SHARD_CORPUS)
        return fail(ctx, KNN_ERR_ARG, "knn_search_sharded: mode must be QUERY or CORPUS (got %d)", shard_mode);
    KNN_TRY(check_block_args(ctx, Q, M, X, N, d, k, KNN_L2SQ, KNN_NO_SELF, 0, out_idx, out_dist));
    if (M == 0) return KNN_OK;
    KNN_TRY(set_device(ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Comm* c = comm_or_single(ctx);
    if (c->nranks == 1 && !g1_phases()) {
        c->last_mode = shard_mode;
        return knn_search_block(ctx, Q, M, X, N, d, k, KNN_L2SQ, KNN_NO_SELF, 0, out_idx, out_dist, stream);
    }
    KNN_TRY(c_bcast(ctx, X, (size_t)N * d * sizeof(float), s));
    if (Q != X) KNN_TRY(c_bcast(ctx, Q, (size_t)M * d * sizeof(float), s));
    if (shard_mode == KNN_SHARD_CORPUS)
        return run_corpus_sharded(ctx, Q, M, X, N, d, k, KNN_L2SQ, false, out_idx, out_dist, s);
    return run_query_sharded(ctx, Q, M, X, N, d, k, KNN_L2SQ, false, out_idx, out_dist, s);
}

}  // extern "C"
