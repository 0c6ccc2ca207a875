// api.cu — host runtime behind the C ABI of include/knn.h: argument validation,
// workspace management, plan choice and the orchestration of the hot path
//   a-S2 prep (norms + split)  ->  a-S3 distance GEMM  ->  a-S4 per-row select
// over bounded row blocks of the distance matrix.  No kernels live here.
#include "runtime.h"

#include <cuda.h>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>


namespace knn_rt {

knn_status fail(knn_ctx* c, knn_status st, const char* fmt, ...) {
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->err = buf;
    }
    return st;
}

knn_status ensure(knn_ctx* ctx, void** buf, size_t* size, size_t need) {
    if (buf == &ctx->ws) ctx->prep_X = nullptr;  // any new use of ws invalidates the kept operands
    if (need <= *size) return KNN_OK;
    if (*buf) {
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return fail(ctx, KNN_ERR_CUDA, "sync: %s", cudaGetErrorString(e));
        cudaFree(*buf);
        *buf = nullptr;
        *size = 0;
    }
    size_t sz = need + (need >> 3);
    if (cudaMalloc(buf, sz) != cudaSuccess) {
        cudaGetLastError();
        if (cudaMalloc(buf, need) != cudaSuccess) {
            cudaGetLastError();
            *buf = nullptr;
            return fail(ctx, KNN_ERR_OOM, "cannot allocate %zu bytes of workspace", need);
        }
        sz = need;
    }
    *size = sz;
    return KNN_OK;
}

cudaEvent_t take_event(knn_ctx* ctx) {
    if (!ctx->ev_pool.empty()) {
        cudaEvent_t e = ctx->ev_pool.back();
        ctx->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

void drain_profile(knn_ctx* ctx) {
    for (auto& p : ctx->pending) {
        float ms = 0.f;
        cudaEventSynchronize(p.b);
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            ctx->prof_ms[p.kind] += ms;
            ctx->prof_n[p.kind] += 1;
        }
        cudaGetLastError();
        ctx->ev_pool.push_back(p.a);
        ctx->ev_pool.push_back(p.b);
    }
    ctx->pending.clear();
}

knn_status set_device(knn_ctx* ctx) {
    KNN_CUDA(cudaSetDevice(ctx->device));
    return KNN_OK;
}

bool metric_ok(knn_ctx* ctx, int32_t metric, knn_status* st) {
    if (metric == KNN_L2SQ || metric == KNN_L2) return true;
    if (metric == KNN_COSINE || metric == KNN_PEARSON) {
        // NEXT-2: the tensor-core GEMM only (the FFMA cross-check path is L2)
        if (ctx->gemm_mode == 0 && ctx->tc_ok) return true;
        *st = fail(ctx, KNN_ERR_UNSUPPORTED, "metric %d (cosine/pearson) needs the tensor-core path",
                   metric);
        return false;
    }
    *st = fail(ctx, KNN_ERR_ARG, "unknown metric %d", metric);
    return false;
}

// Rank of the chunk-minimum pivot.  Rank kk (the k-th smallest non-self
// element guaranteed at or below the pivot: kk distinct chunk minima are) certifies the
// partition by construction, at ~kk N/S candidates per row.  A smaller rank r keeps ~r N/S
// and fails — fewer than k candidates, which the candidate select detects (the call is then
// redone on the full matrix) — only if r or more of the S sampled columns fall among the
// row's kk - 1 nearest points: probability <= P(Bin(kk - 1, S/N) >= r) per row (the r-th
// chunk minimum is >= the r-th smallest sampled value; the sample's error margin only raises
// the pivot).  r = the smallest rank with that tail below 1e-3 / M: a call is redone with
// probability < 1e-3 on data the column sample represents (headline: 18 instead of 33,
// ~150 instead of ~330 candidates per row).  KNN_PIVOT_RANK: 0 = certified, r > 0 = fixed.
int32_t pivot_rank(int32_t kk, int64_t S, int64_t N, int64_t M) {
    static const int env = [] {
        const char* v = getenv("KNN_PIVOT_RANK");
        return v ? atoi(v) : -1;
    }();
    if (env == 0) return kk;
    if (env > 0) return env < kk ? env : kk;
    const double p = (double)S / (double)N, eps = 1e-3 / (double)(M > 1 ? M : 1);
    const int n = kk - 1;
    if (n < 1 || p >= 1.0) return kk;
    double tail = 0.0;  // P(Bin(n, p) >= r), accumulated from r = n down
    int best = kk;
    for (int r = n; r >= 1; --r) {
        tail += std::exp(std::lgamma(n + 1.0) - std::lgamma(r + 1.0) - std::lgamma(n - r + 1.0) +
                         r * std::log(p) + (n - r) * std::log1p(-p));
        if (tail > eps) break;
        best = r;
    }
    return best;
}

// The chunk-minimum sample's divisor (k <= 32): S = N / div sampled columns.  The sample
// pass costs ~N^2 / div, the partition's survivors grow as div / (sample rank) (DESIGN.md
// §6.5); measured optimum (one B200, k = 32, d = 256): 8 at N = 16384, 12 at 65536 (2.24
// -> 2.20 ms), 16 at 131072 (7.7 -> 7.4 ms).  KNN_PIVOT_DIV overrides.
int32_t sample_div(const knn_ctx* ctx, int64_t N) {
    if (ctx->pivot_div > 0) return ctx->pivot_div;
    return N < 49152 ? 8 : N < 98304 ? 12 : 16;
}

// Queue the whole hot path for one block problem; asynchronous on `s`.
knn_status run_block(knn_ctx* ctx, const float* Q, int64_t M, const float* X, int64_t N,
                     int32_t d, int32_t k, int32_t metric, int64_t self_shift, int64_t idx_offset,
                     int32_t* out_idx, float* out_dist, cudaStream_t s, bool allow_pivot) {
    const bool same = (Q == X) && (M == N);
    const bool tc = ctx->gemm_mode == 0 && ctx->tc_ok;
    // Pivot plan (PAPER.md:56 quickselect at matrix scale): per-row pivot = k-th smallest of
    // the minima of the 32-column chunks of a column sample (>= the row's k-th distance),
    // then the GEMM keeps only elements <= pivot.
    const int64_t Ssamp = round_up(N / sample_div(ctx, N), 256);
    // the sample is a permuted column subset that may contain the row's own point: one
    // more rank keeps k non-self elements at or below the pivot
    const int32_t kk = self_shift != KNN_NO_SELF ? k + 1 : k;
    // (fewer than 256 query rows fill less than one 2-CTA row-block pair: the sample pass
    // then costs as much as it saves; measured M = 8 vs N = 2^20: 0.66 vs 0.82 ms)
    const bool pivot = allow_pivot && tc && ctx->pivot_ok && k <= 32 && N >= 16384 && M >= 256 &&
                       ctx->plan != KNN_PLAN_MATERIALISED && Ssamp / 32 >= kk + 1;
    // Quantile pivot for k > 32 (the same quickselect partition; the pivot is a bucketed
    // order statistic of a single-product sample of Sq columns)
    const int32_t qdiv = ctx->pivot_div > 0 ? ctx->pivot_div : 8;  // (k > 32: N / 8, at least 4096)
    const int64_t Sq = round_up(N / qdiv > 4096 ? N / qdiv : 4096, 256);
    const bool pivotq = allow_pivot && tc && ctx->pivot_ok && k > 32 && N >= 16384 && M >= 256 &&
                        ctx->plan != KNN_PLAN_MATERIALISED && Sq <= (N / 256) * 256;
    int32_t rq = 0;
    if (pivotq) {
        const double mu = (double)Sq * k / (double)N;
        // five standard deviations: a row below its k-th (certificate failure) redoes the
        // whole call, so the per-row failure rate must be ~1e-7
        rq = (int32_t)std::ceil(mu + 5.0 * std::sqrt(mu) + 4.0) + (self_shift != KNN_NO_SELF ? 1 : 0);
    }
    const int32_t capq = (int32_t)round_up(3 * (int64_t)k > 2048 ? 3 * (int64_t)k : 2048, 256);
    const bool pivot_sym = (pivot || pivotq) && same && self_shift == 0 && ctx->sym_ok;
    const int32_t cap = ctx->pivot_cap;
    const int32_t d_pad = (int32_t)round_up(d, knn::kSplitKAlign);
    const int64_t ldD = round_up(N, 4);
    int64_t rows_blk = (int64_t)(ctx->d_budget / ((size_t)ldD * sizeof(float)));
    rows_blk = rows_blk < 128 ? 128 : (rows_blk / 128) * 128;
    if (rows_blk > M) rows_blk = M;
    // k-NNG with the transpose reuse of PAPER.md:83: only the upper triangle is multiplied
    // (bit-identical to the other plans thanks to the canonical orientation)
    const bool sym = !pivot && !pivotq && tc && ctx->sym_ok && same && self_shift == 0 &&
                     (size_t)N * ldD * sizeof(float) <= ctx->sym_budget;
    if (sym) rows_blk = M;
    ctx->last_plan = pivot_sym ? 3 : (pivot || pivotq) ? 4 : sym ? 2 : 0;
    // the pivot plans' sample storage is processed in row blocks of at most d_budget bytes
    const int64_t samp_row_bytes = pivot ? (Ssamp / 32) * 4 : pivotq ? Sq * 4 : 1;
    int64_t samp_blk = (int64_t)(ctx->d_budget / (size_t)samp_row_bytes);
    samp_blk = samp_blk < 256 ? 256 : (samp_blk / 256) * 256;
    if (samp_blk > M) samp_blk = M;

    // L2 pivot plans: per-point single-product bound terms (prep's split residuals, reading
    // R21) instead of the constant worst-case bound
    const bool bnd_ok = (pivot || pivotq) && metric <= KNN_L2;
    auto layout = [&](Carve& c, Prepared& pq, Prepared& px, float*& D, int32_t*& flag) {
        flag = c.take<int32_t>(8);  // [0] flags, [1] plan, [2..3] candidates, [4] max eps2, [5] decide counter
        auto prep = [&](Prepared& p, int64_t n) {
            p.sqn = c.take<float>(round_up(n, knn::kColPad));
            p.rs = c.take<float>(round_up(n, knn::kColPad));
            p.hi = tc ? c.take<__half>((size_t)n * d_pad) : nullptr;
            p.lo = tc ? c.take<__half>((size_t)n * d_pad) : nullptr;
        };
        prep(px, N);
        if (same) pq = px; else prep(pq, M);
        D = c.take<float>(pivot ? (size_t)(Ssamp / 32) * samp_blk : pivotq ? (size_t)Sq * samp_blk
                                                                        : (size_t)rows_blk * ldD);
    };
    Carve probe{nullptr};
    Prepared pq{}, px{};
    float* D = nullptr;
    int32_t* flag = nullptr;
    float* thr = nullptr;
    int32_t* cnt = nullptr;
    uint64_t* cent = nullptr;  // per-row candidate lists (ukey << 32 | col)
    int32_t* redo = nullptr;
    Prepared smp{};  // the pivot plans' column sample (gathered points)
    float *nsc_x = nullptr, *nsc_q = nullptr;  // single-product partition: scaled norms
    float *eps_x = nullptr, *eps_q = nullptr, *ninf_x = nullptr, *ninf_q = nullptr;  // bound terms
    float *bnd_x = nullptr, *bnd_q = nullptr;
    double* dec_part = nullptr;  // the plan decision's partial sums
    float* smax = nullptr;  // max of the sample's sqn terms
    auto layout_all = [&](Carve& c) {
        layout(c, pq, px, D, flag);
        if (bnd_ok) {
            const int64_t np = round_up(N, knn::kColPad), mp = round_up(M, knn::kColPad);
            dec_part = c.take<double>(knn::pivot1_decide_ws_bytes() / sizeof(double));
            eps_x = c.take<float>(np);
            ninf_x = c.take<float>(np);
            bnd_x = c.take<float>(np);
            nsc_x = c.take<float>(np);
            eps_q = same ? eps_x : c.take<float>(mp);
            ninf_q = same ? ninf_x : c.take<float>(mp);
            bnd_q = same ? bnd_x : c.take<float>(mp);
            nsc_q = same ? nsc_x : c.take<float>(mp);
        }
        if (!pivot) redo = c.take<int32_t>((size_t)(rows_blk > 0 && !pivotq ? rows_blk : M) + 1);
        if (pivot || pivotq) {
            const int64_t Sx = pivot ? Ssamp : Sq;
            smax = c.take<float>(1);
            smp.hi = c.take<__half>((size_t)Sx * d_pad);
            smp.lo = c.take<__half>((size_t)Sx * d_pad);
            smp.sqn = c.take<float>(round_up(Sx, knn::kColPad));
            smp.rs = c.take<float>(round_up(Sx, knn::kColPad));
            const int32_t cp = pivot ? cap : capq;
            thr = c.take<float>(round_up(M, knn::kColPad));
            cnt = c.take<int32_t>(M);
            cent = c.take<uint64_t>((size_t)M * cp);
        }
    };
    layout_all(probe);
    KNN_TRY(ensure(ctx, &ctx->ws, &ctx->ws_size, probe.off + 256));
    Carve carve{static_cast<char*>(ctx->ws)};
    layout_all(carve);

    KNN_CUDA(cudaMemsetAsync(flag, 0, 8 * sizeof(int32_t), s));
    float* tmax2 = bnd_ok ? reinterpret_cast<float*>(flag + 4) : nullptr;
    {
        Timed t(ctx, KNN_KERNEL_PREP, s);
        KNN_CUDA(knn::launch_prep(X, N, d, d_pad, px.sqn, px.rs, px.hi, px.lo, flag, metric, s, eps_x, tmax2));
        t.done();
    }
    if (!same) {
        Timed t(ctx, KNN_KERNEL_PREP, s);
        KNN_CUDA(knn::launch_prep(Q, M, d, d_pad, pq.sqn, pq.rs, pq.hi, pq.lo, flag, metric, s, eps_q, tmax2));
        t.done();
    }
    if (bnd_ok) {  // nsc / ninf / bnd of every point, one t for the call
        KNN_CUDA(knn::launch_bound_norms(px.sqn, eps_x, round_up(N, knn::kColPad), tmax2, d_pad, nsc_x, ninf_x,
                                         bnd_x, s));
        if (!same)
            KNN_CUDA(knn::launch_bound_norms(pq.sqn, eps_q, round_up(M, knn::kColPad), tmax2, d_pad, nsc_q,
                                             ninf_q, bnd_q, s));
        ctx->launches += same ? 1 : 2;
    }
    if (pivot) {
        // 1. sample pass: per-row minima of 32-column chunks over the first Ssamp corpus
        //    points (written by the GEMM epilogue; no sample matrix), 2. pivots
        {
            ctx->launches++;  // (not timed separately)
            // (L2: the sample's epilogue terms are the upper-bound norms ninf)
            KNN_CUDA(knn::launch_gather_sample(px.hi, px.lo, bnd_ok ? ninf_x : px.sqn, px.rs, N, Ssamp, d_pad,
                                               smp.hi, smp.lo, smp.sqn, smp.rs, smax, s));
            for (int64_t r0 = 0; r0 < M; r0 += samp_blk) {
                const int64_t R = M - r0 < samp_blk ? M - r0 : samp_blk;
                knn::TcOperands op{pq.hi + r0 * d_pad, pq.lo + r0 * d_pad, (bnd_ok ? ninf_q : pq.sqn) + r0,
                                   pq.rs + r0, R, smp.hi, smp.lo, smp.sqn, smp.rs, Ssamp, d_pad};
                Timed tg(ctx, KNN_KERNEL_GEMM, s);
                KNN_CUDA(knn::launch_dist_tc_mins(op, Ssamp, metric, KNN_NO_SELF, D, ctx->pivot_margin,
                                                  ctx->num_sms, s, smax, bnd_ok));
                tg.done();
                Timed tp(ctx, KNN_KERNEL_SELECT, s);  // the pivot select (a-S4 on the chunk minima)
                KNN_CUDA(knn::launch_pivot_from_mins(D, Ssamp / 32, R, round_up(r0 + R, knn::kColPad) - r0,
                                                     pivot_rank(kk, Ssamp, N, M), metric,
                                                         thr + r0, cnt + r0, s));
                tp.done();
            }
        }
        // 3. partition GEMM over the whole matrix, 4. exact select of the candidates
        knn::TcOperands op{pq.hi, pq.lo, pq.sqn, pq.rs, M, px.hi, px.lo, px.sqn, px.rs, N, d_pad};
        // L2 metrics: the partition from the single hi.hi product with its error bound (a
        // third of the MMA work) and the survivors near the k-th re-evaluated exactly from the
        // fp32 inputs.  Chosen on the device (pivot1_decide: the bound must be narrow against
        // the pivots — data far from the origin widens it), forced by KNN_PIVOT1=1, never
        // with KNN_PIVOT1=0 or KNN_PLAN_PIVOT_EXACT (the FP32-accurate 3-product partition,
        // bit-identical to the materialised plan).
        const bool p1_ok = metric <= KNN_L2 && ctx->plan != KNN_PLAN_PIVOT_EXACT && ctx->pivot1 != 0;
        const bool p1_auto = p1_ok && ctx->pivot1 < 0;
        const bool one = p1_ok && ctx->pivot1 > 0;
        knn::TcOperands op1 = op;
        if (p1_ok) {  // the lower bound u_hh - F1_q ||q||^2 - F1_x ||x||^2: the u of the nsc norms
            op1.qn = nsc_q;
            op1.xn = nsc_x;
        }
        if (p1_auto) {  // window 2 (mean bq + mean bx) against the mean pivot
            KNN_CUDA(knn::launch_pivot1_decide(thr, bnd_q, M, bnd_x, N, 1.0f, ctx->pivot1_ratio, flag, dec_part,
                                               reinterpret_cast<unsigned*>(flag + 5), s));
            ctx->launches++;
        }
        ctx->last_plan_auto1 = p1_auto;
        if (one) ctx->last_plan += 2;  // 5 / 6: the single-product partition
        Timed tg(ctx, KNN_KERNEL_FUSED, s);
        if (one || p1_auto)
            KNN_CUDA(knn::launch_dist_tc_pivot1(op1, metric, self_shift, pivot_sym, thr, cnt, cent, cap,
                                                flag, ctx->num_sms, s, p1_auto ? 1 : -1));
        if (!one)
            KNN_CUDA(knn::launch_dist_tc_pivot(op, metric, self_shift, pivot_sym, thr, cnt, cent, cap,
                                               flag, ctx->num_sms, s, -1, -1, false, p1_auto ? 0 : -1));
        ctx->launches += p1_auto ? 1 : 0;
        tg.done();
        Timed tc2(ctx, KNN_KERNEL_MERGE, s);
        if (one || p1_auto)
            KNN_CUDA(knn::launch_candidate_recompute(cnt, cent, cap, M, k, idx_offset, Q, X, d, pq.sqn,
                                                     bnd_q, bnd_x, thr, metric, out_idx, out_dist, flag, s,
                                                     p1_auto ? 1 : -1));
        if (!one)
            KNN_CUDA(knn::launch_candidate_select(cnt, cent, cap, M, k, idx_offset, out_idx, out_dist, flag,
                                                  s, p1_auto ? 0 : -1));
        ctx->launches += p1_auto ? 1 : 0;
        tc2.done();
        return KNN_OK;
    }
    if (pivotq) {
        // 1. sample: single-product upper bounds of the rows against the first Sq columns
        //    (the self pair +inf), 2. pivots, 3. partition GEMM, 4. exact select (k > 32)
        {
            ctx->launches++;  // (not timed separately)
            KNN_CUDA(knn::launch_gather_sample(px.hi, px.lo, bnd_ok ? ninf_x : px.sqn, px.rs, N, Sq, d_pad,
                                               smp.hi, smp.lo, smp.sqn, smp.rs, nullptr, s));
            KNN_CUDA(cudaMemsetAsync(thr, 0xFF, round_up(M, knn::kColPad) * sizeof(float), s));  // pad: NaN
            KNN_CUDA(cudaMemsetAsync(cnt, 0, (size_t)M * sizeof(int32_t), s));
            for (int64_t r0 = 0; r0 < M; r0 += samp_blk) {
                const int64_t R = M - r0 < samp_blk ? M - r0 : samp_blk;
                knn::TcOperands op{pq.hi + r0 * d_pad, pq.lo + r0 * d_pad, (bnd_ok ? ninf_q : pq.sqn) + r0,
                                   pq.rs + r0, R, smp.hi, smp.lo, smp.sqn, smp.rs, Sq, d_pad};
                Timed tg(ctx, KNN_KERNEL_GEMM, s);
                KNN_CUDA(knn::launch_dist_tc_sample(op, Sq, metric, KNN_NO_SELF, D, Sq, ctx->pivot_margin,
                                                    ctx->num_sms, s, bnd_ok));
                tg.done();
                Timed tp(ctx, KNN_KERNEL_SELECT, s);
                KNN_CUDA(knn::launch_pivot_from_sample(D, R, Sq, Sq, rq, thr + r0, s));
                tp.done();
            }
        }
        knn::TcOperands op{pq.hi, pq.lo, pq.sqn, pq.rs, M, px.hi, px.lo, px.sqn, px.rs, N, d_pad};
        Timed tg(ctx, KNN_KERNEL_FUSED, s);
        KNN_CUDA(knn::launch_dist_tc_pivot(op, metric, self_shift, pivot_sym, thr, cnt, cent, capq,
                                           flag, ctx->num_sms, s));
        tg.done();
        Timed tc2(ctx, KNN_KERNEL_MERGE, s);
        ctx->launches++;  // warp-per-row select + the CTA kernel for its redo rows
        KNN_CUDA(knn::launch_candidate_select_large(cnt, cent, capq, M, k, idx_offset, out_idx, out_dist,
                                                    flag, redo, s));
        tc2.done();
        return KNN_OK;
    }
    if (sym) {
        knn::TcOperands op{px.hi, px.lo, px.sqn, px.rs, N, px.hi, px.lo, px.sqn, px.rs, N, d_pad};
        Timed tg(ctx, KNN_KERNEL_GEMM, s);
        KNN_CUDA(knn::launch_dist_tc_sym(op, metric, D, ldD, ctx->num_sms, s));
        tg.done();
        Timed ts(ctx, KNN_KERNEL_SELECT, s);
        KNN_CUDA(knn::launch_select(D, M, N, ldD, k, idx_offset, out_idx, out_dist, redo, s));
        ts.done();
        return KNN_OK;
    }
    for (int64_t r0 = 0; r0 < M; r0 += rows_blk) {
        const int64_t R = (M - r0) < rows_blk ? (M - r0) : rows_blk;
        const int64_t shift = self_shift == KNN_NO_SELF ? KNN_NO_SELF : self_shift + r0;
        Timed tg(ctx, KNN_KERNEL_GEMM, s);
        if (tc) {
            knn::TcOperands op{pq.hi + r0 * d_pad, pq.lo + r0 * d_pad, pq.sqn + r0, pq.rs + r0, R,
                               px.hi, px.lo, px.sqn, px.rs, N, d_pad};
            KNN_CUDA(knn::launch_dist_tc(op, metric, shift, D, ldD, ctx->num_sms, s));
        } else {
            KNN_CUDA(knn::launch_dist_simt(Q + r0 * d, pq.sqn + r0, R, X, px.sqn, N, d, metric,
                                           shift, D, ldD, s));
        }
        tg.done();
        Timed ts(ctx, KNN_KERNEL_SELECT, s);
        KNN_CUDA(knn::launch_select(D, R, N, ldD, k, idx_offset, out_idx + r0 * k,
                                    out_dist + r0 * k, redo, s));
        ts.done();
    }
    return KNN_OK;
}

knn_status finish_blocking(knn_ctx* ctx, cudaStream_t s) {
    // The flag is the first slice of the workspace (see run_block's layout).
    int32_t* flag = static_cast<int32_t*>(ctx->ws);
    // [0] = flags, [2..3] = int64 candidate count of the pivot plan
    KNN_CUDA(cudaMemcpyAsync(ctx->flag_host, flag, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    KNN_CUDA(cudaStreamSynchronize(s));
    memcpy(&ctx->last_candidates, ctx->flag_host + 2, sizeof(int64_t));
    // the device chose the single-product partition: plans 3 / 4 -> 5 / 6
    if (ctx->last_plan_auto1 && ctx->flag_host[1] == 1 && (ctx->last_plan == 3 || ctx->last_plan == 4))
        ctx->last_plan += 2;
    ctx->last_plan_auto1 = false;
    if (*ctx->flag_host & 1)
        return fail(ctx, KNN_ERR_NONFINITE,
                    "input contains NaN/inf or a vector with ||x||^2 >= FLT_MAX/4");
    if (*ctx->flag_host & 2) return KNN_ERR_INTERNAL;  // pivot candidates overflowed: redo
    return KNN_OK;
}

knn_status check_block_args(knn_ctx* ctx, const float* Q, int64_t M, const float* X, int64_t N,
                            int32_t d, int32_t k, int32_t metric, int64_t self_shift,
                            int64_t idx_offset, const void* out_idx, const void* out_dist) {
    knn_status st = KNN_OK;
    if (!metric_ok(ctx, metric, &st)) return st;
    if (N < 1 || M < 0 || d < 1) return fail(ctx, KNN_ERR_ARG, "bad sizes M=%lld N=%lld d=%d",
                                             (long long)M, (long long)N, d);
    if (N > INT32_MAX || M > INT32_MAX) return fail(ctx, KNN_ERR_ARG, "M and N must be < 2^31");
    if (idx_offset < 0 || idx_offset + N - 1 > INT32_MAX)
        return fail(ctx, KNN_ERR_ARG, "idx_offset + N must fit int32");
    if (k < 1 || k > N) return fail(ctx, KNN_ERR_ARG, "k=%d outside [1, N=%lld]", k, (long long)N);
    if (k > KNN_MAX_K) return fail(ctx, KNN_ERR_UNSUPPORTED, "k=%d > %d", k, KNN_MAX_K);
    if (M > 0 && (!Q || !X || !out_idx || !out_dist)) return fail(ctx, KNN_ERR_ARG, "null pointer");
    (void)self_shift;
    return KNN_OK;
}

}  // namespace knn_rt

using namespace knn_rt;

extern "C" {

int knn_abi_version(void) { return KNN_ABI_VERSION; }

knn_status knn_ctx_create(int device, knn_ctx_t* out) {
    if (!out) return KNN_ERR_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        return KNN_ERR_CUDA;
    }
    knn_ctx* c = new knn_ctx();
    c->device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete c;
        return KNN_ERR_CUDA;
    }
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    c->tc_ok = knn::tc_supported();
    const char* g = getenv("KNN_GEMM");
    if (g && strcmp(g, "simt") == 0) c->gemm_mode = 1;
    const char* fz = getenv("KNN_FUSED");
    if (fz && strcmp(fz, "0") == 0) c->plan = KNN_PLAN_MATERIALISED;
    const char* pv = getenv("KNN_PIVOT");
    if (pv && strcmp(pv, "0") == 0) c->pivot_ok = false;
    const char* pd = getenv("KNN_PIVOT_DIV");
    if (pd && atoi(pd) >= 2) c->pivot_div = atoi(pd);
    const char* p1 = getenv("KNN_PIVOT1");
    if (p1 && p1[0]) c->pivot1 = strcmp(p1, "0") != 0 ? 1 : 0;
    const char* pr = getenv("KNN_PIVOT1_RATIO");
    if (pr) c->pivot1_ratio = strtof(pr, nullptr);
    const char* pm = getenv("KNN_PIVOT_MARGIN");
    if (pm) c->pivot_margin = strtof(pm, nullptr);
    const char* pc = getenv("KNN_PIVOT_CAP");
    if (pc) c->pivot_cap = atoi(pc) > 32 ? atoi(pc) : 32;
    const char* sy = getenv("KNN_SYM");
    if (sy && strcmp(sy, "0") == 0) c->sym_ok = false;
    const char* b = getenv("KNN_D_BUDGET_MB");
    if (b) c->d_budget = (size_t)atoll(b) << 20;
    if (cudaMallocHost(&c->flag_host, 4 * sizeof(int32_t)) != cudaSuccess) {
        delete c;
        return KNN_ERR_CUDA;
    }
    *out = c;
    return KNN_OK;
}

knn_status knn_ctx_destroy(knn_ctx_t ctx) {
    if (!ctx) return KNN_ERR_ARG;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    drain_profile(ctx);
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->ws) cudaFree(ctx->ws);
    if (ctx->io) cudaFree(ctx->io);
    if (ctx->st_buf) cudaFree(ctx->st_buf);
    for (auto& m : ctx->ipc_open) cudaIpcCloseMemHandle(m.second);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    for (int b = 0; b < 2; ++b) {
        if (ctx->ev_copied[b]) cudaEventDestroy(ctx->ev_copied[b]);
        if (ctx->ev_free[b]) cudaEventDestroy(ctx->ev_free[b]);
    }
    for (auto e : ctx->ev_chunk) cudaEventDestroy(e);
    if (ctx->flag_host) cudaFreeHost(ctx->flag_host);
    if (ctx->pv_flag) cudaFree(ctx->pv_flag);
    if (ctx->p3_buf) cudaFree(ctx->p3_buf);
    comm_release(ctx);
    delete ctx;
    return KNN_OK;
}

const char* knn_last_error(knn_ctx_t ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

int64_t knn_launch_count(knn_ctx_t ctx) { return ctx ? ctx->launches : -1; }

knn_status knn_set_plan(knn_ctx_t ctx, int32_t plan) {
    if (!ctx) return KNN_ERR_ARG;
    if (plan < KNN_PLAN_AUTO || plan > KNN_PLAN_PIVOT_EXACT)
        return fail(ctx, KNN_ERR_ARG, "unknown plan %d", plan);
    if (plan == KNN_PLAN_FUSED)  // the per-row-list fused kernel was retired
        return fail(ctx, KNN_ERR_UNSUPPORTED, "KNN_PLAN_FUSED was retired; the pivot plan is the fused path");
    ctx->plan = plan;
    return KNN_OK;
}

int knn_last_plan(knn_ctx_t ctx) { return ctx ? ctx->last_plan : -1; }

int64_t knn_last_candidates(knn_ctx_t ctx) { return ctx ? ctx->last_candidates : -1; }

int knn_gemm_path(knn_ctx_t ctx) {
    if (!ctx) return -1;
    return (ctx->gemm_mode == 0 && ctx->tc_ok) ? 0 : 1;
}

knn_status knn_profile_enable(knn_ctx_t ctx, int32_t on) {
    if (!ctx) return KNN_ERR_ARG;
    cudaSetDevice(ctx->device);
    drain_profile(ctx);
    for (int i = 0; i < 6; ++i) {
        ctx->prof_ms[i] = 0;
        ctx->prof_n[i] = 0;
    }
    ctx->prof_on = on != 0;
    return KNN_OK;
}

knn_status knn_profile_read(knn_ctx_t ctx, int32_t kernel, double* total_ms, int64_t* launches) {
    if (!ctx || kernel < 0 || kernel > 5 || !total_ms || !launches) return KNN_ERR_ARG;
    cudaSetDevice(ctx->device);
    drain_profile(ctx);
    *total_ms = ctx->prof_ms[kernel];
    *launches = ctx->prof_n[kernel];
    return KNN_OK;
}

knn_status knn_search_block(knn_ctx_t ctx, const float* Q, int64_t M, const float* X, int64_t N,
                            int32_t d, int32_t k, int32_t metric, int64_t self_shift,
                            int64_t idx_offset, int32_t* out_idx, float* out_dist, void* stream) {
    if (!ctx) return KNN_ERR_ARG;
    KNN_TRY(check_block_args(ctx, Q, M, X, N, d, k, metric, self_shift, idx_offset, out_idx,
                             out_dist));
    if (M == 0) return KNN_OK;
    KNN_TRY(set_device(ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    KNN_TRY(run_block(ctx, Q, M, X, N, d, k, metric, self_shift, idx_offset, out_idx, out_dist, s));
    knn_status st = finish_blocking(ctx, s);
    if (st == KNN_ERR_INTERNAL) {  // pivot plan overflowed (heavy ties): full matrix instead
        ctx->pivot_redos++;
        KNN_TRY(run_block(ctx, Q, M, X, N, d, k, metric, self_shift, idx_offset, out_idx, out_dist, s,
                          false));
        st = finish_blocking(ctx, s);
    }
    return st;
}

knn_status knn_graph(knn_ctx_t ctx, const float* X, int64_t N, int32_t d, int32_t k,
                     int32_t metric, int32_t* out_idx, float* out_dist, void* stream) {
    if (!ctx) return KNN_ERR_ARG;
    if (N >= 1 && k > N - 1)
        return fail(ctx, KNN_ERR_ARG, "knn_graph needs k <= N-1 (k=%d, N=%lld)", k, (long long)N);
    return knn_search_block(ctx, X, N, X, N, d, k, metric, 0, 0, out_idx, out_dist, stream);
}

knn_status knn_search(knn_ctx_t ctx, const float* Q, int64_t M, const float* X, int64_t N,
                      int32_t d, int32_t k, int32_t* out_idx, float* out_dist, void* stream) {
    return knn_search_block(ctx, Q, M, X, N, d, k, KNN_L2SQ, KNN_NO_SELF, 0, out_idx, out_dist,
                            stream);
}

namespace {
// Page-locks a host range for the duration of a call unless it is already pinned.
struct HostPin {
    void* p = nullptr;
    bool mine = false;
    void pin(const void* ptr, size_t bytes) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, ptr) == cudaSuccess && a.type == cudaMemoryTypeHost) return;
        cudaGetLastError();
        const cudaError_t e = cudaHostRegister(const_cast<void*>(ptr), bytes, cudaHostRegisterDefault);
        if (e == cudaSuccess) {
            p = const_cast<void*>(ptr);
            mine = true;
        } else {
            cudaGetLastError();  // stays pageable: copies are correct, just not overlapped
        }
    }
    ~HostPin() {
        if (mine) cudaHostUnregister(p);
    }
};
}  // namespace

// End-to-end k-NNG from HOST points with the host->device copy overlapped by the hot path
// ("overlap computation with data transfer").  The pivot
// plan over the symmetric GEMM, reorganised by arrival: the copy stream sends a sample of
// every 8th point (one strided 2-D copy) and then the points in chunks; the compute stream
// prepares the sample, and per chunk: its rows' split operands, their sample pass and
// pivots, and the partition of the triangle's units whose column block lies in the chunk
// (column-major unit order: those units only touch rows and columns that have arrived).
// After the last chunk: the candidate select and the device->host copy of the lists.
// Results are those of the device-resident call: the pivots (sample) differ, but every
// plan's result is the exact select of the same per-pair values (certificates redo).
// Returns KNN_ERR_UNSUPPORTED (nothing queued) when the shape does not fit the scheme.
knn_status host_graph_pipelined(knn_ctx* ctx, const float* X_host, int64_t N, int32_t d, int32_t k,
                                int32_t metric, int32_t* out_idx_host, float* out_dist_host, cudaStream_t s) {
    const char* env = getenv("KNN_HOST_PIPE");
    const bool tc = ctx->gemm_mode == 0 && ctx->tc_ok;
    if ((env && strcmp(env, "0") == 0) || !tc || !ctx->pivot_ok || !ctx->sym_ok ||
        ctx->plan == KNN_PLAN_MATERIALISED || k > 32 || N < 16384 || N % 2048 != 0 ||
        (ctx->pivot_div > 0 && ctx->pivot_div != 8))
        return KNN_ERR_UNSUPPORTED;
    const int64_t S = N / 8;                    // sample: points 8j, j < S (a multiple of 256)
    // chunk rows (a multiple of 256): N / 8, at least 8192.  (The last chunk's partition
    // covers its columns against every row, ~2/n of the triangle after the last copy, but
    // N / 16 measured slower: e2e 3.06 -> 3.38 ms at the headline; env KNN_PIPE_DIV.)
    const char* pdv = getenv("KNN_PIPE_DIV");
    const int64_t pdiv = pdv && atoi(pdv) >= 1 ? atoi(pdv) : 8;
    const int64_t CH = round_up(N / pdiv >= 8192 ? N / pdiv : 8192, 256);
    const int nch = (int)ceil_div(N, CH);
    const int32_t d_pad = (int32_t)round_up(d, knn::kSplitKAlign);
    const int32_t cap = ctx->pivot_cap;
    const int32_t kk = k + 1;  // the sample may hold the row's own point
    if (S / 32 < kk + 1) return KNN_ERR_UNSUPPORTED;
    // device buffers: io = points | sample staging | outputs; ws = operands, sample, lists
    float *x, *xs, *od;
    int32_t* oi;
    auto io_layout = [&](Carve& c) {
        x = c.take<float>((size_t)N * d);
        xs = c.take<float>((size_t)S * d);
        oi = c.take<int32_t>((size_t)N * k);
        od = c.take<float>((size_t)N * k);
    };
    // the single-product partition (chosen on the device after the first chunk's pivots, or
    // forced by KNN_PIVOT1=1; L2 metrics, not under KNN_PLAN_PIVOT_EXACT), as in run_block
    const bool p1_ok = metric <= KNN_L2 && ctx->plan != KNN_PLAN_PIVOT_EXACT && ctx->pivot1 != 0;
    const bool p1_auto = p1_ok && ctx->pivot1 < 0;
    const bool one = p1_ok && ctx->pivot1 > 0;
    // L2: per-point single-product bound terms (as in run_block; t from the sample, which is
    // prepared first: any t > 0 gives a valid bound, the same t for every point of the call)
    const bool bnd_ok = metric <= KNN_L2;
    Prepared px{}, smp{};
    float *D, *smax, *thr, *nsc = nullptr;
    float *eps = nullptr, *ninf = nullptr, *bnd = nullptr, *s_eps = nullptr, *s_ninf = nullptr, *s_bnd = nullptr;
    double* dec_part = nullptr;
    int32_t *flag, *cnt;
    uint64_t* cent;
    auto ws_layout = [&](Carve& c) {
        flag = c.take<int32_t>(8);  // [4]: max eps2 of the sample, [5]: decide counter
        if (bnd_ok) {
            nsc = c.take<float>(round_up(N, knn::kColPad));
            eps = c.take<float>(N);
            ninf = c.take<float>(N);
            bnd = c.take<float>(N);
            s_eps = c.take<float>(S);
            s_ninf = c.take<float>(S);
            s_bnd = c.take<float>(S);
            dec_part = c.take<double>(knn::pivot1_decide_ws_bytes() / sizeof(double));
        }
        px.sqn = c.take<float>(N);
        px.rs = c.take<float>(N);
        px.hi = c.take<__half>((size_t)N * d_pad);
        px.lo = c.take<__half>((size_t)N * d_pad);
        smp.sqn = c.take<float>(S);
        smp.rs = c.take<float>(S);
        smp.hi = c.take<__half>((size_t)S * d_pad);
        smp.lo = c.take<__half>((size_t)S * d_pad);
        smax = c.take<float>(1);
        D = c.take<float>((size_t)(S / 32) * CH);
        thr = c.take<float>(N);
        cnt = c.take<int32_t>(N);
        cent = c.take<uint64_t>((size_t)N * cap);
    };
    Carve p1{nullptr}, p2{nullptr};
    io_layout(p1);
    ws_layout(p2);
    KNN_TRY(ensure(ctx, &ctx->io, &ctx->io_size, p1.off + 256));
    KNN_TRY(ensure(ctx, &ctx->ws, &ctx->ws_size, p2.off + 256));
    Carve c1{static_cast<char*>(ctx->io)}, c2{static_cast<char*>(ctx->ws)};
    io_layout(c1);
    ws_layout(c2);
    if (!ctx->copy_stream) {
        KNN_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            KNN_CUDA(cudaEventCreateWithFlags(&ctx->ev_copied[b], cudaEventDisableTiming));
            KNN_CUDA(cudaEventCreateWithFlags(&ctx->ev_free[b], cudaEventDisableTiming));
        }
    }
    constexpr int kOutChunks = 4;  // re-evaluation row chunks, each copied back as it ends
    while ((int)ctx->ev_chunk.size() < nch + 3 + kOutChunks) {
        cudaEvent_t e = nullptr;
        KNN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->ev_chunk.push_back(e);
    }
    cudaStream_t cs = ctx->copy_stream;
    HostPin pin;
    pin.pin(X_host, (size_t)N * d * sizeof(float));
    // the copies overwrite x / xs only after the work queued before this call on s
    KNN_CUDA(cudaEventRecord(ctx->ev_chunk[nch + 1], s));
    KNN_CUDA(cudaStreamWaitEvent(cs, ctx->ev_chunk[nch + 1], 0));
    KNN_CUDA(cudaMemcpy2DAsync(xs, (size_t)d * sizeof(float), X_host, (size_t)8 * d * sizeof(float),
                               (size_t)d * sizeof(float), (size_t)S, cudaMemcpyHostToDevice, cs));
    KNN_CUDA(cudaEventRecord(ctx->ev_chunk[nch], cs));
    for (int c = 0; c < nch; ++c) {
        const int64_t c0 = c * CH, R = N - c0 < CH ? N - c0 : CH;
        KNN_CUDA(cudaMemcpyAsync(x + c0 * d, X_host + c0 * d, (size_t)R * d * sizeof(float), cudaMemcpyHostToDevice,
                                 cs));
        KNN_CUDA(cudaEventRecord(ctx->ev_chunk[c], cs));
    }
    struct CopyGuard {  // errors below: the copies drain before the pin is released
        cudaStream_t cs;
        ~CopyGuard() { cudaStreamSynchronize(cs); }
    } cg{cs};
    KNN_CUDA(cudaMemsetAsync(flag, 0, 8 * sizeof(int32_t), s));
    KNN_CUDA(cudaStreamWaitEvent(s, ctx->ev_chunk[nch], 0));
    float* tmax2 = reinterpret_cast<float*>(flag + 4);
    {
        Timed t(ctx, KNN_KERNEL_PREP, s);
        KNN_CUDA(knn::launch_prep(xs, S, d, d_pad, smp.sqn, smp.rs, smp.hi, smp.lo, flag, metric, s, s_eps,
                                  bnd_ok ? tmax2 : nullptr));
        t.done();
    }
    if (bnd_ok) {  // the sample's upper-bound norms replace its sqn terms in the sample pass
        KNN_CUDA(knn::launch_bound_norms(smp.sqn, s_eps, S, tmax2, d_pad, nullptr, s_ninf, s_bnd, s));
        KNN_CUDA(cudaMemcpyAsync(smp.sqn, s_ninf, (size_t)S * sizeof(float), cudaMemcpyDeviceToDevice, s));
        ctx->launches++;
    }
    KNN_CUDA(knn::launch_max_nonneg(smp.sqn, S, smax, s));
    ctx->launches++;
    knn::TcOperands full{px.hi, px.lo, px.sqn, px.rs, N, px.hi, px.lo, px.sqn, px.rs, N, d_pad};
    knn::TcOperands full1 = full;  // the single-product partition: norms scaled by 1 - F
    full1.qn = nsc;
    full1.xn = nsc;
    for (int c = 0; c < nch; ++c) {
        const int64_t c0 = c * CH, R = N - c0 < CH ? N - c0 : CH;
        KNN_CUDA(cudaStreamWaitEvent(s, ctx->ev_chunk[c], 0));
        {
            Timed t(ctx, KNN_KERNEL_PREP, s);
            KNN_CUDA(knn::launch_prep(x + c0 * d, R, d, d_pad, px.sqn + c0, px.rs + c0, px.hi + c0 * d_pad,
                                      px.lo + c0 * d_pad, flag, metric, s, bnd_ok ? eps + c0 : nullptr));
            t.done();
        }
        if (bnd_ok) {  // with the sample's t (tmax2 is not raised by the chunks)
            KNN_CUDA(knn::launch_bound_norms(px.sqn + c0, eps + c0, R, tmax2, d_pad, nsc + c0, ninf + c0, bnd + c0,
                                             s));
            ctx->launches++;
        }
        knn::TcOperands op{px.hi + c0 * d_pad, px.lo + c0 * d_pad, (bnd_ok ? ninf : px.sqn) + c0, px.rs + c0, R,
                           smp.hi, smp.lo, smp.sqn, smp.rs, S, d_pad};
        {
            Timed tg(ctx, KNN_KERNEL_GEMM, s);
            KNN_CUDA(knn::launch_dist_tc_mins(op, S, metric, KNN_NO_SELF, D, ctx->pivot_margin, ctx->num_sms, s,
                                              smax, bnd_ok));
            tg.done();
        }
        {
            Timed tp(ctx, KNN_KERNEL_SELECT, s);
            KNN_CUDA(knn::launch_pivot_from_mins(D, S / 32, R, R, knn_rt::pivot_rank(kk, S, N, N), metric,
                                                 thr + c0, cnt + c0, s));
            tp.done();
        }
        if (c == 0 && p1_auto) {  // the device's choice, from the first chunk's rows and the sample
            KNN_CUDA(knn::launch_pivot1_decide(thr, bnd, R, s_bnd, S, 1.0f, ctx->pivot1_ratio, flag, dec_part,
                                               reinterpret_cast<unsigned*>(flag + 5), s));
            ctx->launches++;
        }
        // the triangle's units whose column block lies in this chunk (rows and columns < c0 + R)
        const int64_t b0 = c0 / knn::kColPad, b1 = (c0 + R) / knn::kColPad;  // 256-column blocks
        Timed tf(ctx, KNN_KERNEL_FUSED, s);
        if (one || p1_auto)
            KNN_CUDA(knn::launch_dist_tc_pivot1(full1, metric, 0, true, thr, cnt, cent, cap, flag, ctx->num_sms, s,
                                                p1_auto ? 1 : -1, b0 * (b0 + 1) / 2, b1 * (b1 + 1) / 2, true));
        if (!one)
            KNN_CUDA(knn::launch_dist_tc_pivot(full, metric, 0, true, thr, cnt, cent, cap, flag, ctx->num_sms, s,
                                               b0 * (b0 + 1) / 2, b1 * (b1 + 1) / 2, true, p1_auto ? 0 : -1));
        ctx->launches += p1_auto ? 1 : 0;
        tf.done();
    }
    // the exact select / re-evaluation in row chunks, each chunk's results copied back on the
    // copy stream while the next chunk computes (a failed certificate redoes the whole call
    // below and copies again)
    const int64_t RC = round_up(ceil_div(N, (int64_t)kOutChunks), (int64_t)256);
    for (int oc = 0; oc * RC < N; ++oc) {
        const int64_t r0 = oc * RC, R = N - r0 < RC ? N - r0 : RC;
        Timed tc2(ctx, KNN_KERNEL_MERGE, s);
        if (one || p1_auto)
            KNN_CUDA(knn::launch_candidate_recompute(cnt + r0, cent + r0 * cap, cap, R, k, 0, x + r0 * d, x, d,
                                                     px.sqn + r0, bnd + r0, bnd, thr + r0, metric, oi + r0 * k,
                                                     od + r0 * k, flag, s, p1_auto ? 1 : -1));
        if (!one)
            KNN_CUDA(knn::launch_candidate_select(cnt + r0, cent + r0 * cap, cap, R, k, 0, oi + r0 * k, od + r0 * k,
                                                  flag, s, p1_auto ? 0 : -1));
        ctx->launches += p1_auto ? 1 : 0;
        tc2.done();
        cudaEvent_t ev = ctx->ev_chunk[nch + 2 + oc];
        KNN_CUDA(cudaEventRecord(ev, s));
        KNN_CUDA(cudaStreamWaitEvent(cs, ev, 0));
        KNN_CUDA(cudaMemcpyAsync(out_idx_host + r0 * k, oi + r0 * k, (size_t)R * k * sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, cs));
        KNN_CUDA(cudaMemcpyAsync(out_dist_host + r0 * k, od + r0 * k, (size_t)R * k * sizeof(float),
                                 cudaMemcpyDeviceToHost, cs));
    }
    KNN_CUDA(cudaEventRecord(ctx->ev_chunk[nch + 2 + kOutChunks], cs));
    KNN_CUDA(cudaStreamWaitEvent(s, ctx->ev_chunk[nch + 2 + kOutChunks], 0));
    ctx->last_plan = one ? 5 : 3;
    ctx->last_plan_auto1 = p1_auto;
    knn_status st = finish_blocking(ctx, s);
    if (st == KNN_ERR_INTERNAL) {  // a certificate failed / a list overflowed: the full matrix
        ctx->pivot_redos++;
        KNN_TRY(run_block(ctx, x, N, x, N, d, k, metric, 0, 0, oi, od, s, false));
        st = finish_blocking(ctx, s);
        if (st != KNN_OK) return st;
        KNN_CUDA(cudaMemcpyAsync(out_idx_host, oi, (size_t)N * k * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        KNN_CUDA(cudaMemcpyAsync(out_dist_host, od, (size_t)N * k * sizeof(float), cudaMemcpyDeviceToHost, s));
        return finish_blocking(ctx, s);
    }
    return st;
}

knn_status knn_search_block_host(knn_ctx_t ctx, const float* Q_host, int64_t M,
                                 const float* X_host, int64_t N, int32_t d, int32_t k,
                                 int32_t metric, int64_t self_shift, int64_t idx_offset,
                                 int32_t* out_idx_host, float* out_dist_host, void* stream) {
    if (!ctx) return KNN_ERR_ARG;
    KNN_TRY(check_block_args(ctx, Q_host, M, X_host, N, d, k, metric, self_shift, idx_offset,
                             out_idx_host, out_dist_host));
    if (M == 0) return KNN_OK;
    KNN_TRY(set_device(ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool same = Q_host == X_host && M == N;
    if (same && self_shift == 0 && idx_offset == 0) {
        const knn_status sp = host_graph_pipelined(ctx, X_host, N, d, k, metric, out_idx_host, out_dist_host, s);
        if (sp != KNN_ERR_UNSUPPORTED) return sp;
    }
    auto layout = [&](Carve& c, float*& q, float*& x, int32_t*& oi, float*& od) {
        x = c.take<float>((size_t)N * d);
        q = same ? x : c.take<float>((size_t)M * d);
        oi = c.take<int32_t>((size_t)M * k);
        od = c.take<float>((size_t)M * k);
    };
    Carve probe{nullptr};
    float *q, *x, *od;
    int32_t* oi;
    layout(probe, q, x, oi, od);
    KNN_TRY(ensure(ctx, &ctx->io, &ctx->io_size, probe.off + 256));
    Carve carve{static_cast<char*>(ctx->io)};
    layout(carve, q, x, oi, od);
    KNN_CUDA(cudaMemcpyAsync(x, X_host, (size_t)N * d * sizeof(float), cudaMemcpyHostToDevice, s));
    if (!same)
        KNN_CUDA(cudaMemcpyAsync(q, Q_host, (size_t)M * d * sizeof(float), cudaMemcpyHostToDevice, s));
    KNN_TRY(run_block(ctx, q, M, x, N, d, k, metric, self_shift, idx_offset, oi, od, s));
    {
        knn_status st0 = finish_blocking(ctx, s);
        if (st0 == KNN_ERR_INTERNAL) {
            ctx->pivot_redos++;
            KNN_TRY(run_block(ctx, q, M, x, N, d, k, metric, self_shift, idx_offset, oi, od, s, false));
        } else if (st0 != KNN_OK) {
            return st0;
        }
    }
    KNN_CUDA(cudaMemcpyAsync(out_idx_host, oi, (size_t)M * k * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, s));
    KNN_CUDA(cudaMemcpyAsync(out_dist_host, od, (size_t)M * k * sizeof(float),
                             cudaMemcpyDeviceToHost, s));
    return finish_blocking(ctx, s);
}


knn_status knn_search_streamed(knn_ctx_t ctx, const float* Q_host, int64_t M, const float* X_host,
                               int64_t N, int32_t d, int32_t k, int32_t metric, int32_t graph,
                               int64_t chunk_points, int64_t query_block, int32_t* out_idx_host,
                               float* out_dist_host) {
    if (!ctx) return KNN_ERR_ARG;
    if (graph && (Q_host != X_host || M != N))
        return fail(ctx, KNN_ERR_ARG, "graph mode needs Q_host == X_host and M == N");
    const int64_t kmin = graph ? (int64_t)k + 1 : (int64_t)k;
    if (N < kmin) return fail(ctx, KNN_ERR_ARG, "k=%d too large for N=%lld", k, (long long)N);
    KNN_TRY(check_block_args(ctx, Q_host, M, X_host, N, d, k, metric, graph ? 0 : KNN_NO_SELF, 0,
                             out_idx_host, out_dist_host));
    if (M == 0) return KNN_OK;
    KNN_TRY(set_device(ctx));
    cudaEvent_t t0 = take_event(ctx), t1 = take_event(ctx);
    int64_t C = chunk_points > 0 ? chunk_points : 131072;
    if (C < kmin) C = kmin;
    if (C > N) C = N;
    const int64_t Cmax = C + kmin;  // a trailing chunk shorter than kmin joins its predecessor
    int64_t QB = query_block > 0 ? query_block : M;
    const int64_t qb_cap = (int64_t)(((size_t)2 << 30) / ((size_t)d * sizeof(float)));
    if (QB > qb_cap) QB = qb_cap;
    if (QB > M) QB = M;
    // device layout: staging x2 | query block | lists [2][QB][k] (running, chunk) | merged
    auto layout = [&](Carve& c, float** xs, float*& q, int32_t*& li, float*& ld, int32_t*& mi, float*& md) {
        xs[0] = c.take<float>((size_t)Cmax * d);
        xs[1] = c.take<float>((size_t)Cmax * d);
        q = c.take<float>((size_t)QB * d);
        li = c.take<int32_t>((size_t)2 * QB * k);
        ld = c.take<float>((size_t)2 * QB * k);
        mi = c.take<int32_t>((size_t)QB * k);
        md = c.take<float>((size_t)QB * k);
    };
    float* xs[2];
    float *q, *ld, *md;
    int32_t *li, *mi;
    Carve probe{nullptr};
    layout(probe, xs, q, li, ld, mi, md);
    KNN_TRY(ensure(ctx, &ctx->st_buf, &ctx->st_size, probe.off + 256));
    Carve carve{static_cast<char*>(ctx->st_buf)};
    layout(carve, xs, q, li, ld, mi, md);
    if (!ctx->copy_stream) {
        KNN_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            KNN_CUDA(cudaEventCreateWithFlags(&ctx->ev_copied[b], cudaEventDisableTiming));
            KNN_CUDA(cudaEventCreateWithFlags(&ctx->ev_free[b], cudaEventDisableTiming));
        }
    }
    HostPin pin_x, pin_q;
    pin_x.pin(X_host, (size_t)N * d * sizeof(float));
    if (!graph) pin_q.pin(Q_host, (size_t)M * d * sizeof(float));
    cudaStream_t s = nullptr;
    KNN_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaStream_t cs = ctx->copy_stream;
    // on every exit (errors included) both streams drain before the host pins (declared
    // above, destroyed after this guard) are released and st_buf can be reused
    struct StreamGuard {
        cudaStream_t s, cs;
        ~StreamGuard() {
            cudaStreamSynchronize(cs);
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    } sg{s, cs};
    // chunk boundaries
    std::vector<int64_t> cb;
    for (int64_t c0 = 0; c0 < N; c0 += C) cb.push_back(c0);
    if (cb.size() > 1 && N - cb.back() < kmin) cb.pop_back();
    cb.push_back(N);
    const int nch = (int)cb.size() - 1;
    const int64_t offsets[2] = {0, 0};
    KNN_CUDA(cudaEventRecord(t0, s));
    for (int b = 0; b < 2; ++b) KNN_CUDA(cudaEventRecord(ctx->ev_free[b], s));
    for (int64_t q0 = 0; q0 < M; q0 += QB) {
        const int64_t R = M - q0 < QB ? M - q0 : QB;
        KNN_CUDA(cudaMemcpyAsync(q, Q_host + q0 * d, (size_t)R * d * sizeof(float), cudaMemcpyHostToDevice, s));
        auto issue_copy = [&](int c) -> knn_status {
            const int b = c & 1;
            KNN_CUDA(cudaStreamWaitEvent(cs, ctx->ev_free[b], 0));
            KNN_CUDA(cudaMemcpyAsync(xs[b], X_host + cb[c] * d, (size_t)(cb[c + 1] - cb[c]) * d * sizeof(float),
                                     cudaMemcpyHostToDevice, cs));
            KNN_CUDA(cudaEventRecord(ctx->ev_copied[b], cs));
            return KNN_OK;
        };
        KNN_TRY(issue_copy(0));
        for (int c = 0; c < nch; ++c) {
            if (c + 1 < nch) KNN_TRY(issue_copy(c + 1));
            const int b = c & 1;
            const int64_t c0 = cb[c], Cc = cb[c + 1] - cb[c];
            KNN_CUDA(cudaStreamWaitEvent(s, ctx->ev_copied[b], 0));
            // chunk partial lists: list 0 (running) for the first chunk, else list 1
            int32_t* pi = c == 0 ? li : li + (size_t)R * k;
            float* pd = c == 0 ? ld : ld + (size_t)R * k;
            const int64_t shift = graph ? q0 - c0 : KNN_NO_SELF;
            KNN_TRY(run_block(ctx, q, R, xs[b], Cc, d, k, metric, shift, c0, pi, pd, s));
            KNN_CUDA(cudaEventRecord(ctx->ev_free[b], s));
            knn_status st0 = finish_blocking(ctx, s);
            if (st0 == KNN_ERR_INTERNAL) {
                ctx->pivot_redos++;
                KNN_TRY(run_block(ctx, q, R, xs[b], Cc, d, k, metric, shift, c0, pi, pd, s, false));
                KNN_CUDA(cudaEventRecord(ctx->ev_free[b], s));
            } else if (st0 != KNN_OK) {
                return st0;
            }
            if (c > 0) {
                // running top-k <- merge(running, chunk) (a-S6); the lists are [2][R][k]
                Timed tm(ctx, KNN_KERNEL_MERGE, s);
                KNN_CUDA(knn::launch_merge(ld, li, 2, R, k, offsets, mi, md, s));
                tm.done();
                KNN_CUDA(cudaMemcpyAsync(li, mi, (size_t)R * k * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
                KNN_CUDA(cudaMemcpyAsync(ld, md, (size_t)R * k * sizeof(float), cudaMemcpyDeviceToDevice, s));
            }
        }
        KNN_CUDA(cudaMemcpyAsync(out_idx_host + q0 * k, li, (size_t)R * k * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        KNN_CUDA(cudaMemcpyAsync(out_dist_host + q0 * k, ld, (size_t)R * k * sizeof(float), cudaMemcpyDeviceToHost, s));
    }
    KNN_CUDA(cudaEventRecord(t1, s));
    KNN_TRY(finish_blocking(ctx, s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    ctx->last_stream_total_ms = ms;
    ctx->ev_pool.push_back(t0);
    ctx->ev_pool.push_back(t1);
    drain_profile(ctx);
    return KNN_OK;
}

knn_status knn_rownorms(knn_ctx_t ctx, const float* X, int64_t N, int32_t d, float* out_sqn,
                        int32_t* out_flag, void* stream) {
    if (!ctx) return KNN_ERR_ARG;
    if (N < 0 || d < 1) return fail(ctx, KNN_ERR_ARG, "bad sizes");
    if (N > 0 && (!X || !out_sqn)) return fail(ctx, KNN_ERR_ARG, "null pointer");
    if (N == 0) return KNN_OK;
    KNN_TRY(set_device(ctx));
    Timed t(ctx, KNN_KERNEL_PREP, static_cast<cudaStream_t>(stream));
    KNN_CUDA(knn::launch_prep(X, N, d, 0, out_sqn, nullptr, nullptr, nullptr, out_flag, 0,
                              static_cast<cudaStream_t>(stream)));
    t.done();
    return KNN_OK;
}

knn_status knn_distances(knn_ctx_t ctx, const float* Q, int64_t M, const float* X, int64_t N,
                         int32_t d, int32_t metric, int64_t self_shift, float* D, int64_t ldD,
                         void* stream) {
    if (!ctx) return KNN_ERR_ARG;
    knn_status st = KNN_OK;
    if (!metric_ok(ctx, metric, &st)) return st;
    if (M < 0 || N < 1 || d < 1 || ldD < N) return fail(ctx, KNN_ERR_ARG, "bad sizes");
    if (M > INT32_MAX || N > INT32_MAX) return fail(ctx, KNN_ERR_ARG, "M and N must be < 2^31");
    if (M > 0 && (!Q || !X || !D)) return fail(ctx, KNN_ERR_ARG, "null pointer");
    if (M == 0) return KNN_OK;
    KNN_TRY(set_device(ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool same = (Q == X) && (M == N);
    const bool tc = ctx->gemm_mode == 0 && ctx->tc_ok;
    const int32_t d_pad = (int32_t)round_up(d, knn::kSplitKAlign);
    auto layout = [&](Carve& c, Prepared& pq, Prepared& px, int32_t*& flag) {
        flag = c.take<int32_t>(4);
        auto prep = [&](Prepared& p, int64_t n) {
            p.sqn = c.take<float>(round_up(n, knn::kColPad));
            p.rs = c.take<float>(round_up(n, knn::kColPad));
            p.hi = tc ? c.take<__half>((size_t)n * d_pad) : nullptr;
            p.lo = tc ? c.take<__half>((size_t)n * d_pad) : nullptr;
        };
        prep(px, N);
        if (same) pq = px; else prep(pq, M);
    };
    Carve probe{nullptr};
    Prepared pq{}, px{};
    int32_t* flag;
    layout(probe, pq, px, flag);
    KNN_TRY(ensure(ctx, &ctx->ws, &ctx->ws_size, probe.off + 256));
    Carve carve{static_cast<char*>(ctx->ws)};
    layout(carve, pq, px, flag);
    {
        Timed t(ctx, KNN_KERNEL_PREP, s);
        KNN_CUDA(knn::launch_prep(X, N, d, d_pad, px.sqn, px.rs, px.hi, px.lo, flag, metric, s));
        t.done();
    }
    if (!same) {
        Timed t(ctx, KNN_KERNEL_PREP, s);
        KNN_CUDA(knn::launch_prep(Q, M, d, d_pad, pq.sqn, pq.rs, pq.hi, pq.lo, flag, metric, s));
        t.done();
    }
    Timed tg(ctx, KNN_KERNEL_GEMM, s);
    if (tc) {
        knn::TcOperands op{pq.hi, pq.lo, pq.sqn, pq.rs, M, px.hi, px.lo, px.sqn, px.rs, N, d_pad};
        KNN_CUDA(knn::launch_dist_tc(op, metric, self_shift, D, ldD, ctx->num_sms, s));
    } else {
        KNN_CUDA(knn::launch_dist_simt(Q, pq.sqn, M, X, px.sqn, N, d, metric, self_shift, D, ldD, s));
    }
    tg.done();
    return KNN_OK;
}

knn_status knn_select(knn_ctx_t ctx, const float* D, int64_t M, int64_t N, int64_t ldD, int32_t k,
                      int32_t* out_idx, float* out_dist, void* stream) {
    if (!ctx) return KNN_ERR_ARG;
    if (M < 0 || N < 1 || ldD < N) return fail(ctx, KNN_ERR_ARG, "bad sizes");
    if (N > INT32_MAX || M > INT32_MAX) return fail(ctx, KNN_ERR_ARG, "M and N must be < 2^31");
    if (k < 1 || k > N) return fail(ctx, KNN_ERR_ARG, "k=%d outside [1, N]", k);
    if (k > KNN_MAX_K) return fail(ctx, KNN_ERR_UNSUPPORTED, "k=%d > %d", k, KNN_MAX_K);
    if (M > 0 && (!D || !out_idx || !out_dist)) return fail(ctx, KNN_ERR_ARG, "null pointer");
    if (M == 0) return KNN_OK;
    KNN_TRY(set_device(ctx));
    // workspace: the redo row list of the sampled-pivot select (M + 1 int32)
    KNN_TRY(ensure(ctx, &ctx->ws, &ctx->ws_size, (size_t)(M + 1) * sizeof(int32_t) + 256));
    Timed t(ctx, KNN_KERNEL_SELECT, static_cast<cudaStream_t>(stream));
    KNN_CUDA(knn::launch_select(D, M, N, ldD, k, 0, out_idx, out_dist,
                                static_cast<int32_t*>(ctx->ws), static_cast<cudaStream_t>(stream)));
    t.done();
    return KNN_OK;
}

knn_status knn_last_select_kernel(int32_t* kind, int32_t* splits) {
    if (!kind || !splits) return KNN_ERR_ARG;
    *kind = knn::g_last_select_kind;
    *splits = knn::g_last_select_splits;
    return KNN_OK;
}

knn_status knn_select_paper(knn_ctx_t ctx, const float* D, int64_t M, int64_t N, int64_t ldD,
                            int32_t k, int32_t* out_idx, float* out_dist, void* stream) {
    if (!ctx) return KNN_ERR_ARG;
    if (M < 0 || N < 1 || ldD < N) return fail(ctx, KNN_ERR_ARG, "bad sizes");
    if (N > INT32_MAX || M > INT32_MAX) return fail(ctx, KNN_ERR_ARG, "M and N must be < 2^31");
    if (k < 1 || k > N) return fail(ctx, KNN_ERR_ARG, "k=%d outside [1, N]", k);
    if (k > KNN_MAX_K) return fail(ctx, KNN_ERR_UNSUPPORTED, "k=%d > %d", k, KNN_MAX_K);
    if (M > 0 && (!D || !out_idx || !out_dist)) return fail(ctx, KNN_ERR_ARG, "null pointer");
    if (M == 0) return KNN_OK;
    KNN_TRY(set_device(ctx));
    // aux arrays for a block of rows, at most 4 GiB (at least one row)
    int64_t rows = (int64_t)(((size_t)4 << 30) / knn::select_paper_ws_bytes(1, N));
    if (rows < 1) rows = 1;
    if (rows > M) rows = M;
    const size_t bytes = knn::select_paper_ws_bytes(rows, N);
    KNN_TRY(ensure(ctx, &ctx->ws, &ctx->ws_size, bytes + 256));
    Timed t(ctx, KNN_KERNEL_SELECT, static_cast<cudaStream_t>(stream));
    KNN_CUDA(knn::launch_select_paper(D, M, N, ldD, k, ctx->ws, bytes, out_idx, out_dist,
                                      static_cast<cudaStream_t>(stream)));
    t.done();
    return KNN_OK;
}

knn_status knn_merge_lists(knn_ctx_t ctx, const float* const* dist_lists,
                           const int32_t* const* idx_lists, int32_t G, int64_t row0, int64_t M,
                           int32_t k, const int64_t* offsets_host, int32_t* out_idx,
                           float* out_dist, void* stream) {
    if (!ctx) return KNN_ERR_ARG;
    if (G < 1 || G > 64 || M < 0 || row0 < 0) return fail(ctx, KNN_ERR_ARG, "bad G=%d, M or row0", G);
    if (M > INT32_MAX) return fail(ctx, KNN_ERR_ARG, "M must be < 2^31");
    if (k < 1) return fail(ctx, KNN_ERR_ARG, "k=%d < 1", k);
    if (k > KNN_MAX_K) return fail(ctx, KNN_ERR_UNSUPPORTED, "k=%d > %d", k, KNN_MAX_K);
    if (M == 0) return KNN_OK;
    if (!dist_lists || !idx_lists || !offsets_host || !out_idx || !out_dist)
        return fail(ctx, KNN_ERR_ARG, "null pointer");
    for (int g = 0; g < G; ++g) {
        if (!dist_lists[g] || !idx_lists[g]) return fail(ctx, KNN_ERR_ARG, "null list %d", g);
        if (offsets_host[g] < 0 || offsets_host[g] > INT32_MAX)
            return fail(ctx, KNN_ERR_ARG, "offset %d out of range", g);
    }
    KNN_TRY(set_device(ctx));
    Timed t(ctx, KNN_KERNEL_MERGE, static_cast<cudaStream_t>(stream));
    KNN_CUDA(knn::launch_merge_lists(dist_lists, idx_lists, G, row0, M, k, offsets_host, out_idx,
                                     out_dist, static_cast<cudaStream_t>(stream)));
    t.done();
    return KNN_OK;
}

int64_t knn_graph_units(int64_t N) {
    const int64_t n = knn::ceil_div(N, 256);
    return n * (n + 1) / 2;
}

int64_t knn_pivot_sample_size(knn_ctx_t ctx, int64_t N, int32_t k) {
    if (!ctx || N < 1) return 0;
    if (k <= 32) return round_up(N / sample_div(ctx, N), 256);
    const int32_t qdiv = ctx->pivot_div > 0 ? ctx->pivot_div : 8;
    return round_up(N / qdiv > 4096 ? N / qdiv : 4096, 256);
}

int32_t knn_graph_list_cap(int32_t k) {
    return k <= 32 ? 2048 : (int32_t)round_up(3 * (int64_t)k > 2048 ? 3 * (int64_t)k : 2048, 256);
}

namespace {
knn_status ensure_pv_flag(knn_ctx* ctx) {
    if (ctx->pv_flag) return KNN_OK;
    if (cudaMalloc(&ctx->pv_flag, 4 * sizeof(int32_t)) != cudaSuccess) {
        cudaGetLastError();
        ctx->pv_flag = nullptr;
        return fail(ctx, KNN_ERR_OOM, "cannot allocate the Par-3 flag");
    }
    return KNN_OK;
}

knn_status graph_shard_check(knn_ctx_t ctx, const float* X, int64_t N, int32_t d, int32_t k, int32_t metric) {
    if (!ctx || !X) return KNN_ERR_ARG;
    if (N < 2 || d < 1 || k < 1 || k > N - 1) return fail(ctx, KNN_ERR_ARG, "bad N, d or k");
    if (N > INT32_MAX) return fail(ctx, KNN_ERR_ARG, "N must be < 2^31");
    if (k > KNN_MAX_K || N < 16384) return fail(ctx, KNN_ERR_UNSUPPORTED, "needs N >= 16384, k <= 1024");
    if (!(ctx->gemm_mode == 0 && ctx->tc_ok)) return fail(ctx, KNN_ERR_UNSUPPORTED, "needs the tensor-core path");
    knn_status st;
    if (!metric_ok(ctx, metric, &st)) return st;
    return KNN_OK;
}

// The workspace prefix of knn_graph_pivots and knn_graph_partition (same offsets, so the
// partition reuses what the pivots call prepared): flag, split operands and, L2, the
// per-point bound terms (prep.cu launch_bound_norms; bnd goes to ctx->p3_buf).
struct ShardPrep {
    int32_t* flag = nullptr;
    Prepared px{};
    float *eps = nullptr, *nsc = nullptr, *ninf = nullptr;
    double* dec = nullptr;
};
void shard_prefix(Carve& c, ShardPrep& p, int64_t N, int32_t d_pad, bool l2) {
    p.flag = c.take<int32_t>(8);  // [0] flags, [1] plan, [2..3] candidates, [4] max eps2, [5] decide counter
    p.px.sqn = c.take<float>(round_up(N, knn::kColPad));
    p.px.rs = c.take<float>(round_up(N, knn::kColPad));
    p.px.hi = c.take<__half>((size_t)N * d_pad);
    p.px.lo = c.take<__half>((size_t)N * d_pad);
    if (l2) {
        p.eps = c.take<float>(round_up(N, knn::kColPad));
        p.nsc = c.take<float>(round_up(N, knn::kColPad));
        p.ninf = c.take<float>(round_up(N, knn::kColPad));
        p.dec = c.take<double>(knn::pivot1_decide_ws_bytes() / sizeof(double));
    }
}

// prep of all N points (+ L2: the bound terms, one t for the call; sqn and bnd copied to
// ctx->p3_buf for knn_graph_gather_select)
knn_status shard_prep(knn_ctx* ctx, const ShardPrep& p, const float* X, int64_t N, int32_t d, int32_t d_pad,
                      int32_t metric, cudaStream_t s) {
    const bool l2 = metric <= KNN_L2;
    KNN_CUDA(cudaMemsetAsync(p.flag, 0, 8 * sizeof(int32_t), s));
    KNN_TRY(ensure_pv_flag(ctx));
    {
        Timed t(ctx, KNN_KERNEL_PREP, s);
        KNN_CUDA(knn::launch_prep(X, N, d, d_pad, p.px.sqn, p.px.rs, p.px.hi, p.px.lo, ctx->pv_flag, metric, s,
                                  l2 ? p.eps : nullptr, l2 ? reinterpret_cast<float*>(p.flag + 4) : nullptr));
        t.done();
    }
    if (l2) {
        const int64_t np = round_up(N, knn::kColPad);
        KNN_TRY(ensure(ctx, &ctx->p3_buf, &ctx->p3_size, 2 * np * sizeof(float)));
        float* bnd = static_cast<float*>(ctx->p3_buf) + np;
        KNN_CUDA(knn::launch_bound_norms(p.px.sqn, p.eps, np, reinterpret_cast<float*>(p.flag + 4), d_pad, p.nsc,
                                         p.ninf, bnd, s));
        KNN_CUDA(cudaMemcpyAsync(ctx->p3_buf, p.px.sqn, np * sizeof(float), cudaMemcpyDeviceToDevice, s));
        ctx->launches++;
    }
    return KNN_OK;
}
}  // namespace

knn_status knn_graph_pivots(knn_ctx_t ctx, const float* X, int64_t N, int32_t d, int32_t k, int32_t metric,
                            int64_t row0, int64_t rows, float* thr, void* stream) {
    KNN_TRY(graph_shard_check(ctx, X, N, d, k, metric));
    if (row0 < 0 || rows < 0 || row0 + rows > N || !thr) return fail(ctx, KNN_ERR_ARG, "bad row range");
    if (rows == 0) return KNN_OK;
    KNN_TRY(set_device(ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int32_t d_pad = (int32_t)round_up(d, knn::kSplitKAlign);
    const int32_t kk = k + 1;  // the sample may hold the row's own point
    const bool small = k <= 32;
    const int32_t qdiv = ctx->pivot_div > 0 ? ctx->pivot_div : 8;
    const int64_t S = small ? round_up(N / sample_div(ctx, N), 256)
                            : round_up(N / qdiv > 4096 ? N / qdiv : 4096, 256);
    if (small && S / 32 < kk + 1) return fail(ctx, KNN_ERR_UNSUPPORTED, "sample too small for k");
    const bool l2 = metric <= KNN_L2;
    ShardPrep sp;
    Prepared smp{};
    float *D = nullptr, *smax = nullptr;
    int32_t* cnt = nullptr;
    auto layout = [&](Carve& c) {
        shard_prefix(c, sp, N, d_pad, l2);
        smp.sqn = c.take<float>(round_up(S, knn::kColPad));
        smp.rs = c.take<float>(round_up(S, knn::kColPad));
        smp.hi = c.take<__half>((size_t)S * d_pad);
        smp.lo = c.take<__half>((size_t)S * d_pad);
        D = c.take<float>(small ? (size_t)(S / 32) * rows : (size_t)S * rows);
        cnt = c.take<int32_t>(rows);
        smax = c.take<float>(1);
    };
    Carve probe{nullptr};
    layout(probe);
    KNN_TRY(ensure(ctx, &ctx->ws, &ctx->ws_size, probe.off + 256));
    Carve carve{static_cast<char*>(ctx->ws)};
    layout(carve);
    const Prepared& px = sp.px;
    KNN_TRY(ensure_pv_flag(ctx));
    KNN_CUDA(cudaMemsetAsync(ctx->pv_flag, 0, 4 * sizeof(int32_t), s));
    KNN_TRY(shard_prep(ctx, sp, X, N, d, d_pad, metric, s));
    ctx->prep_X = X;  // knn_graph_partition may reuse px (same carve offsets, ws untouched)
    ctx->prep_N = N;
    ctx->prep_d = d;
    ctx->prep_metric = metric;
    ctx->launches++;
    // (L2: the sample pass on the per-point upper-bound norms ninf)
    KNN_CUDA(knn::launch_gather_sample(px.hi, px.lo, l2 ? sp.ninf : px.sqn, px.rs, N, S, d_pad, smp.hi, smp.lo,
                                       smp.sqn, smp.rs, small ? smax : nullptr, s));
    knn::TcOperands op{px.hi + row0 * d_pad, px.lo + row0 * d_pad, (l2 ? sp.ninf : px.sqn) + row0, px.rs + row0,
                       rows, smp.hi, smp.lo, smp.sqn, smp.rs, S, d_pad};
    Timed tg(ctx, KNN_KERNEL_GEMM, s);
    if (small)
        KNN_CUDA(knn::launch_dist_tc_mins(op, S, metric, KNN_NO_SELF, D, ctx->pivot_margin, ctx->num_sms, s, smax,
                                          l2));
    else
        KNN_CUDA(knn::launch_dist_tc_sample(op, S, metric, KNN_NO_SELF, D, S, ctx->pivot_margin, ctx->num_sms, s,
                                            l2));
    tg.done();
    Timed tp(ctx, KNN_KERNEL_SELECT, s);
    if (small) {
        KNN_CUDA(knn::launch_pivot_from_mins(D, S / 32, rows,
                                                     // pad only to the absolute 256-row boundary
                                                     round_up(row0 + rows, knn::kColPad) - row0,
                                                     knn_rt::pivot_rank(kk, S, N, N), metric, thr + row0, cnt, s));
    } else {
        const double mu = (double)S * k / (double)N;
        const int32_t rq = (int32_t)std::ceil(mu + 5.0 * std::sqrt(mu) + 4.0) + 1;
        KNN_CUDA(knn::launch_pivot_from_sample(D, rows, S, S, rq, thr + row0, s));
    }
    tp.done();
    return KNN_OK;
}

knn_status knn_graph_partition(knn_ctx_t ctx, const float* X, int64_t N, int32_t d, int32_t k,
                               int32_t metric, const float* thr, int64_t unit_lo, int64_t unit_hi,
                               int32_t* cnt, uint64_t* cent, int32_t cap, void* stream) {
    KNN_TRY(graph_shard_check(ctx, X, N, d, k, metric));
    if (!thr || !cnt || !cent || cap < k) return fail(ctx, KNN_ERR_ARG, "bad lists");
    KNN_TRY(set_device(ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int32_t d_pad = (int32_t)round_up(d, knn::kSplitKAlign);
    const bool l2 = metric <= KNN_L2;
    ShardPrep sp;
    auto layout = [&](Carve& c) { shard_prefix(c, sp, N, d_pad, l2); };
    Carve probe{nullptr};
    layout(probe);
    // the operands knn_graph_pivots prepared are still at the same offsets of ws if the
    // last ws user was that call on the same points (ensure() does not reallocate: this
    // call needs less workspace)
    const bool reuse = ctx->prep_X == X && ctx->prep_N == N && ctx->prep_d == d && ctx->prep_metric == metric &&
                       probe.off + 256 <= ctx->ws_size && (!l2 || (ctx->p3_buf && ctx->p3_size >= 2 * round_up(N, knn::kColPad) * sizeof(float)));
    KNN_TRY(ensure(ctx, &ctx->ws, &ctx->ws_size, probe.off + 256));
    Carve carve{static_cast<char*>(ctx->ws)};
    layout(carve);
    const Prepared& px = sp.px;
    int32_t* flag = sp.flag;
    KNN_CUDA(cudaMemsetAsync(cnt, 0, (size_t)N * sizeof(int32_t), s));
    if (!reuse) {
        KNN_TRY(shard_prep(ctx, sp, X, N, d, d_pad, metric, s));
    } else {
        KNN_CUDA(cudaMemsetAsync(flag, 0, 8 * sizeof(int32_t), s));
    }
    ctx->prep_X = X;  // (ensure() above cleared it; the operands are those of X)
    ctx->prep_N = N;
    ctx->prep_d = d;
    ctx->prep_metric = metric;
    knn::TcOperands op{px.hi, px.lo, px.sqn, px.rs, N, px.hi, px.lo, px.sqn, px.rs, N, d_pad};
    // k <= 32, L2: the single-product partition as in the one-GPU call,
    // chosen on the device from ALL N pivots (every rank takes the same decision: the same
    // all-gathered pivots and bound terms) unless KNN_PLAN_PIVOT_EXACT / KNN_PIVOT1=0
    const bool p1_ok = l2 && k <= 32 && ctx->plan != KNN_PLAN_PIVOT_EXACT && ctx->pivot1 != 0;
    const bool p1_auto = p1_ok && ctx->pivot1 < 0, one = p1_ok && ctx->pivot1 > 0;
    if (p1_auto) {
        const float* bnd = static_cast<const float*>(ctx->p3_buf) + round_up(N, knn::kColPad);
        // (the decision lives in ctx->pv_flag[1]: knn_graph_gather_select's workspace may
        // be reallocated, pv_flag is not)
        KNN_CUDA(knn::launch_pivot1_decide(thr, bnd, N, bnd, N, 1.0f, ctx->pivot1_ratio, ctx->pv_flag, sp.dec,
                                           reinterpret_cast<unsigned*>(flag + 5), s));
        ctx->launches++;
    }
    int32_t* pflag = p1_auto ? ctx->pv_flag : flag;  // the gated pair reads pv_flag[1]
    Timed tg(ctx, KNN_KERNEL_FUSED, s);
    if (p1_ok) {
        knn::TcOperands op1 = op;
        op1.qn = sp.nsc;
        op1.xn = sp.nsc;
        KNN_CUDA(knn::launch_dist_tc_pivot1(op1, metric, 0, true, thr, cnt, cent, cap, pflag, ctx->num_sms, s,
                                            p1_auto ? 1 : -1, unit_lo, unit_hi));
    }
    if (!one)
        KNN_CUDA(knn::launch_dist_tc_pivot(op, metric, 0, true, thr, cnt, cent, cap, pflag, ctx->num_sms, s,
                                           unit_lo, unit_hi, false, p1_auto ? 0 : -1));
    ctx->launches += p1_auto ? 1 : 0;
    tg.done();
    ctx->p3_state = p1_auto ? 1 : one ? 2 : 0;
    ctx->p3_X = X;
    ctx->p3_thr = thr;
    ctx->p3_N = N;
    ctx->p3_d = d;
    ctx->p3_metric = metric;
    ctx->last_plan = one ? 5 : 3;
    return KNN_OK;
}

knn_status knn_graph_gather_select(knn_ctx_t ctx, int32_t G, const int32_t* const* cnts,
                                   const uint64_t* const* cents, int32_t cap, int64_t N, int32_t k,
                                   int64_t row0, int64_t rows, int32_t* out_idx, float* out_dist, void* stream) {
    if (!ctx) return KNN_ERR_ARG;
    if (G < 1 || G > 64 || !cnts || !cents || cap < k || k < 1 || k > KNN_MAX_K)
        return fail(ctx, KNN_ERR_ARG, "bad G, lists or k");
    if (row0 < 0 || rows < 0 || row0 + rows > N) return fail(ctx, KNN_ERR_ARG, "bad row range");
    if (rows == 0) return KNN_OK;
    if (!out_idx || !out_dist) return fail(ctx, KNN_ERR_ARG, "null output");
    KNN_TRY(set_device(ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int32_t *flag = nullptr, *cnt = nullptr;
    uint64_t* cent = nullptr;
    int32_t* redo = nullptr;
    auto layout = [&](Carve& c) {
        flag = c.take<int32_t>(4);
        redo = c.take<int32_t>(rows + 1);
        cnt = c.take<int32_t>(rows);
        cent = c.take<uint64_t>((size_t)rows * cap);
    };
    Carve probe{nullptr};
    layout(probe);
    KNN_TRY(ensure(ctx, &ctx->ws, &ctx->ws_size, probe.off + 256));
    Carve carve{static_cast<char*>(ctx->ws)};
    layout(carve);
    KNN_CUDA(cudaMemsetAsync(flag, 0, 4 * sizeof(int32_t), s));
    // the single-product partition's lists (lower bounds): re-evaluation from the points
    const int p1 = ctx->p3_state != 0 && k <= 32 && ctx->p3_N == N && ctx->p3_X && ctx->p3_thr && ctx->p3_buf &&
                           ctx->pv_flag
                       ? ctx->p3_state : 0;
    if (p1 == 1)  // the device's partition choice (knn_graph_partition) into flag[1]
        KNN_CUDA(cudaMemcpyAsync(flag + 1, ctx->pv_flag + 1, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    Timed tm(ctx, KNN_KERNEL_MERGE, s);
    KNN_CUDA(knn::launch_gather_lists(cnts, cents, G, cap, row0, rows, cap, cnt, cent, flag, s));
    if (p1) {
        const int64_t np = round_up(N, knn::kColPad);
        const float* sqn = static_cast<const float*>(ctx->p3_buf);
        const float* bnd = sqn + np;
        const int32_t d = ctx->p3_d;
        KNN_CUDA(knn::launch_candidate_recompute(cnt, cent, cap, rows, k, 0, ctx->p3_X + row0 * d, ctx->p3_X, d,
                                                 sqn + row0, bnd + row0, bnd, ctx->p3_thr + row0, ctx->p3_metric,
                                                 out_idx, out_dist, flag, s, p1 == 1 ? 1 : -1));
        if (p1 == 1)
            KNN_CUDA(knn::launch_candidate_select(cnt, cent, cap, rows, k, 0, out_idx, out_dist, flag, s, 0));
        ctx->last_plan = p1 == 1 ? 3 : 5;
        ctx->last_plan_auto1 = p1 == 1;
    } else if (k <= 32) {
        KNN_CUDA(knn::launch_candidate_select(cnt, cent, cap, rows, k, 0, out_idx, out_dist, flag, s));
    } else {
        KNN_CUDA(knn::launch_candidate_select_large(cnt, cent, cap, rows, k, 0, out_idx, out_dist, flag, redo, s));
    }
    tm.done();
    knn_status st = finish_blocking(ctx, s);
    drain_profile(ctx);
    if (st == KNN_OK && ctx->pv_flag) {  // the prep flag of this rank's pivots / partition
        int32_t f = 0;
        KNN_CUDA(cudaMemcpy(&f, ctx->pv_flag, sizeof f, cudaMemcpyDeviceToHost));
        if (f & 1)
            return fail(ctx, KNN_ERR_NONFINITE, "input contains NaN/inf or a vector with ||x||^2 >= FLT_MAX/4");
    }
    return st;
}

knn_status knn_diag_mainloop(knn_ctx_t ctx, const float* X, int64_t N, int32_t d, int32_t sym,
                             int32_t reps, double* ms) {
    if (!ctx || !X || !ms || N < 1 || d < 1 || reps < 1) return KNN_ERR_ARG;
    if (!(ctx->gemm_mode == 0 && ctx->tc_ok)) return fail(ctx, KNN_ERR_UNSUPPORTED, "needs the tensor-core path");
    KNN_TRY(set_device(ctx));
    const int32_t d_pad = (int32_t)round_up(d, knn::kSplitKAlign);
    Prepared px{};
    int32_t* flag = nullptr;
    auto layout = [&](Carve& c) {
        flag = c.take<int32_t>(4);
        px.sqn = c.take<float>(round_up(N, knn::kColPad));
        px.rs = c.take<float>(round_up(N, knn::kColPad));
        px.hi = c.take<__half>((size_t)N * d_pad);
        px.lo = c.take<__half>((size_t)N * d_pad);
    };
    Carve probe{nullptr};
    layout(probe);
    KNN_TRY(ensure(ctx, &ctx->ws, &ctx->ws_size, probe.off + 256));
    Carve carve{static_cast<char*>(ctx->ws)};
    layout(carve);
    cudaStream_t s = nullptr;
    KNN_CUDA(cudaMemsetAsync(flag, 0, 4 * sizeof(int32_t), s));
    KNN_CUDA(knn::launch_prep(X, N, d, d_pad, px.sqn, px.rs, px.hi, px.lo, flag, 0, s));
    knn::TcOperands op{px.hi, px.lo, px.sqn, px.rs, N, px.hi, px.lo, px.sqn, px.rs, N, d_pad};
    KNN_CUDA(knn::launch_dist_tc_null(op, sym != 0, ctx->num_sms, s));
    cudaEvent_t a = take_event(ctx), b = take_event(ctx);
    KNN_CUDA(cudaEventRecord(a, s));
    for (int i = 0; i < reps; ++i) KNN_CUDA(knn::launch_dist_tc_null(op, sym != 0, ctx->num_sms, s));
    KNN_CUDA(cudaEventRecord(b, s));
    KNN_CUDA(cudaEventSynchronize(b));
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    ctx->ev_pool.push_back(a);
    ctx->ev_pool.push_back(b);
    *ms = t / reps;
    return KNN_OK;
}

knn_status knn_ipc_export(knn_ctx_t ctx, const void* dev_ptr, uint8_t handle[64], int64_t* offset) {
    if (!ctx || !dev_ptr || !handle || !offset) return KNN_ERR_ARG;
    KNN_TRY(set_device(ctx));
    // the IPC handle names a whole cudaMalloc allocation: find its base (driver API)
    static CUresult (*get_range)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
    if (!get_range) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return fail(ctx, KNN_ERR_CUDA, "cuMemGetAddressRange unavailable");
        get_range = reinterpret_cast<CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr)>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
        return fail(ctx, KNN_ERR_ARG, "pointer is not device memory");
    cudaIpcMemHandle_t h;
    KNN_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    static_assert(sizeof(h) == 64, "IPC handle size");
    memcpy(handle, &h, 64);
    *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
    return KNN_OK;
}

knn_status knn_ipc_open(knn_ctx_t ctx, const uint8_t handle[64], int64_t offset, void** dev_ptr) {
    if (!ctx || !handle || !dev_ptr || offset < 0) return KNN_ERR_ARG;
    KNN_TRY(set_device(ctx));
    const std::string key(reinterpret_cast<const char*>(handle), 64);
    for (auto& m : ctx->ipc_open)
        if (m.first == key) {
            *dev_ptr = static_cast<char*>(m.second) + offset;
            return KNN_OK;
        }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    void* base = nullptr;
    KNN_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    ctx->ipc_open.push_back({key, base});
    *dev_ptr = static_cast<char*>(base) + offset;
    return KNN_OK;
}

knn_status knn_ipc_close_all(knn_ctx_t ctx) {
    if (!ctx) return KNN_ERR_ARG;
    KNN_TRY(set_device(ctx));
    for (auto& m : ctx->ipc_open) cudaIpcCloseMemHandle(m.second);
    ctx->ipc_open.clear();
    return KNN_OK;
}

knn_status knn_merge(knn_ctx_t ctx, const float* part_dist, const int32_t* part_idx, int32_t G,
                     int64_t M, int32_t k, const int64_t* offsets_host, int32_t* out_idx,
                     float* out_dist, void* stream) {
    if (!ctx) return KNN_ERR_ARG;
    if (G < 1 || G > 64 || M < 0) return fail(ctx, KNN_ERR_ARG, "bad G=%d or M", G);
    if (M > INT32_MAX) return fail(ctx, KNN_ERR_ARG, "M must be < 2^31");
    if (k < 1) return fail(ctx, KNN_ERR_ARG, "k=%d < 1", k);
    if (k > KNN_MAX_K) return fail(ctx, KNN_ERR_UNSUPPORTED, "k=%d > %d", k, KNN_MAX_K);
    if (M > 0 && (!part_dist || !part_idx || !offsets_host || !out_idx || !out_dist))
        return fail(ctx, KNN_ERR_ARG, "null pointer");
    for (int g = 0; g < G; ++g)
        if (offsets_host[g] < 0 || offsets_host[g] > INT32_MAX)
            return fail(ctx, KNN_ERR_ARG, "offset %d out of range", g);
    if (M == 0) return KNN_OK;
    KNN_TRY(set_device(ctx));
    Timed t(ctx, KNN_KERNEL_MERGE, static_cast<cudaStream_t>(stream));
    KNN_CUDA(knn::launch_merge(part_dist, part_idx, G, M, k, offsets_host, out_idx, out_dist,
                               static_cast<cudaStream_t>(stream)));
    t.done();
    return KNN_OK;
}

}  // extern "C"
