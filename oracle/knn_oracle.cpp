// knn_oracle.cpp — CPU ORACLE for the brute-force k-NN / k-NNG of arXiv 1309.5478.
//
// THIS IS TEST INFRASTRUCTURE, NOT PART OF THE PRODUCT PATH.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// legs may load it.  It shares no code, header, table or helper with the CUDA path
// (paper_1309_5478_b200/csrc, include/knn.h), and it never imports or links it.
//
// What it computes is the plain definition the paper's method reaches exactly
// (§Introduction): "This process result in a distance matrix of size
// M x N ... The k-NNs ... is then found by sorting each row of the matrix and finding
// the k indices of the k smallest distances."  So this oracle
//   1. computes every distance directly in fp64 in the DIRECT form
//        d^2(q, c) = sum_t (q_t - c_t)^2        (t ascending, one double accumulator)
//      which is the quantity PAPER.md:80-82 writes as ||x||^2 + ||y||^2 - 2 x.y
//      (equal in exact arithmetic; the direct form is exactly symmetric and exactly 0
//      on the diagonal), and d_E = sqrt(d^2) for the Euclidean metric;
//   2. sorts each full row with std::sort by (distance, index) ascending — the index
//      tie-break is the reading R1 of DESIGN.md (smaller index first);
//   3. takes the first k.
// No blocking, fusion or reordering beyond that.  Build flags: -O2 -ffp-contract=off,
// no -ffast-math, so every sum is evaluated in the written order and is reproducible.
//
// Readings: R1 tie-break by smaller index; R2 output sorted;
// R3 graph mode excludes self by position; R5 squared distances >= 0
// (the direct form never goes negative); R6 -0 == +0; NaN ordered after +inf
// (knn_select rule); R14 cosine / Pearson keys are 1 - similarity, zero norm -> 3.0;
// R15 norms accumulated in fp64.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <thread>
#include <vector>

namespace {

// Run body(r) for r in [0, R) on `threads` std::threads, rows split in contiguous blocks.
template <class F>
void parallel_rows(int64_t R, int threads, F body) {
    if (threads <= 1 || R <= 1) {
        for (int64_t r = 0; r < R; ++r) body(r);
        return;
    }
    int T = (int)std::min<int64_t>(threads, R);
    std::vector<std::thread> pool;
    pool.reserve(T);
    for (int t = 0; t < T; ++t) {
        int64_t lo = R * t / T, hi = R * (t + 1) / T;
        pool.emplace_back([=, &body]() {
            for (int64_t r = lo; r < hi; ++r) body(r);
        });
    }
    for (auto& th : pool) th.join();
}

// Squared Euclidean distance, direct form, fp64, t ascending.
inline double sqdist64(const float* q, const float* c, int32_t d) {
    double s = 0.0;
    for (int32_t t = 0; t < d; ++t) {
        double diff = (double)q[t] - (double)c[t];
        s += diff * diff;
    }
    return s;
}

// Cosine key (d_C(x,y) = x.y / (||x|| ||y||), a similarity; reading R14,
// the selected key is 1 - d_C so that "k smallest" means nearest for every
// metric; a zero-norm vector gets the sentinel key 3.0).  fp64, t ascending.
inline double cosine64(const double* q, const double* c, int32_t d) {
    double dot = 0.0, nq = 0.0, nc = 0.0;
    for (int32_t t = 0; t < d; ++t) {
        dot += q[t] * c[t];
        nq += q[t] * q[t];
        nc += c[t] * c[t];
    }
    if (nq == 0.0 || nc == 0.0) return 3.0;
    return 1.0 - dot / (std::sqrt(nq) * std::sqrt(nc));
}

// x^ = x - mean(x) ("x^ = x - x_bar and x_bar is the mean of the entries
// in x"), in fp64.
inline void center64(const float* x, int32_t d, double* out) {
    double s = 0.0;
    for (int32_t t = 0; t < d; ++t) s += (double)x[t];
    const double mean = s / (double)d;
    for (int32_t t = 0; t < d; ++t) out[t] = (double)x[t] - mean;
}

// Metric 0 = squared Euclidean (the paper's d^2), 1 = Euclidean d_E = sqrt(d^2),
// 2 = cosine key 1 - d_C, 3 = Pearson key: the cosine key of the centred
// vectors ("the Pearson distance coefficient is essentially the Cosine
// distance of the centered data sets").
inline double metric64(const float* q, const float* c, int32_t d, int32_t metric) {
    if (metric == 2 || metric == 3) {
        std::vector<double> a(d), b(d);
        if (metric == 3) {
            center64(q, d, a.data());
            center64(c, d, b.data());
        } else {
            for (int32_t t = 0; t < d; ++t) {
                a[t] = q[t];
                b[t] = c[t];
            }
        }
        return cosine64(a.data(), b.data(), d);
    }
    double s = sqdist64(q, c, d);
    return metric == 1 ? std::sqrt(s) : s;
}

// Total order on fp32 keys used by knn_select (R6): -0 == +0, every NaN
// equal to every other NaN and greater than +inf.  Returns true iff a < b.
inline bool f32_less(float a, float b) {
    bool na = std::isnan(a), nb = std::isnan(b);
    if (na || nb) return !na && nb;
    return a < b;  // -0 < +0 is false in IEEE, so they compare equal
}
inline bool f32_equal(float a, float b) {
    bool na = std::isnan(a), nb = std::isnan(b);
    if (na || nb) return na && nb;
    return a == b;
}
// Canonical value written for a selected key: +0 for -0, +NaN for any NaN.
inline float f32_canon(float a) {
    if (std::isnan(a)) return std::numeric_limits<float>::quiet_NaN();
    if (a == 0.0f) return 0.0f;
    return a;
}

}  // namespace

extern "C" {

int oracle_version(void) { return 1; }

// ||x_j||^2 = sum_t x_j[t]^2 accumulated in fp64 ("transform iterator
// generates the square of individual elements ... reduction_by_key computes the square
// of the vector norms"; accumulator width R15).
int oracle_sqnorms(const float* X, int64_t N, int32_t d, double* out) {
    if (N < 0 || d < 1 || (!X && N) || (!out && N)) return 1;
    for (int64_t j = 0; j < N; ++j) {
        const float* x = X + j * (int64_t)d;
        double s = 0.0;
        for (int32_t t = 0; t < d; ++t) s += (double)x[t] * (double)x[t];
        out[j] = s;
    }
    return 0;
}

// Full distance rows for the queries Q[rows[r]], r < R, against all N corpus points:
// out[r*N + j] = d(Q[rows[r]], X[j]) in fp64 (metric 0: d^2, 1: d_E, 2: cosine key,
// 3: Pearson key).
int oracle_dist_rows(const float* Q, const int64_t* rows, int64_t R, const float* X, int64_t N,
                     int32_t d, int32_t metric, int32_t threads, double* out) {
    if (R < 0 || N < 1 || d < 1 || metric < 0 || metric > 3) return 1;
    parallel_rows(R, threads, [&](int64_t r) {
        const float* q = Q + rows[r] * (int64_t)d;
        double* o = out + r * N;
        for (int64_t j = 0; j < N; ++j) o[j] = metric64(q, X + j * (int64_t)d, d, metric);
    });
    return 0;
}

// The reference k-NN lists for sampled query rows (distance matrix, sort
// each row, take the k smallest).  For r < R the query is Q[rows[r]].
//   graph != 0: k-NNG mode, Q == X and the query's own position j == rows[r] is dropped
//               before sorting (reading R3); requires k <= N-1.
//   R64 (idx64/dist64, R×k): std::sort of j by (D64[j], j), first k — the end-to-end
//               reference.
//   R32 (idx32/dist32, R×k, optional): D32[j] = (float)D64[j] (round to nearest even),
//               std::sort of j by (D32[j], j), first k — what an exact select must
//               return on the fp32-rounded matrix.
int oracle_knn(const float* Q, int64_t M, const float* X, int64_t N, int32_t d, int32_t k,
               int32_t metric, int32_t graph, const int64_t* rows, int64_t R, int32_t threads,
               int32_t* idx64, double* dist64, int32_t* idx32, float* dist32) {
    if (M < 1 || N < 1 || d < 1 || k < 1 || metric < 0 || metric > 3) return 1;
    if (graph && (M != N || k > N - 1)) return 1;
    if (!graph && k > N) return 1;
    for (int64_t r = 0; r < R; ++r)
        if (rows[r] < 0 || rows[r] >= M) return 1;
    parallel_rows(R, threads, [&](int64_t r) {
        const int64_t i = rows[r];
        const float* q = Q + i * (int64_t)d;
        std::vector<double> D64(N);
        for (int64_t j = 0; j < N; ++j) D64[j] = metric64(q, X + j * (int64_t)d, d, metric);
        std::vector<int64_t> order;
        order.reserve(N);
        for (int64_t j = 0; j < N; ++j)
            if (!(graph && j == i)) order.push_back(j);
        std::vector<int64_t> o64 = order;
        std::sort(o64.begin(), o64.end(), [&](int64_t a, int64_t b) {
            if (D64[a] != D64[b]) return D64[a] < D64[b];
            return a < b;
        });
        for (int32_t s = 0; s < k; ++s) {
            idx64[r * k + s] = (int32_t)o64[s];
            dist64[r * k + s] = D64[o64[s]];
        }
        if (idx32) {
            std::vector<float> D32(N);
            for (int64_t j = 0; j < N; ++j) D32[j] = (float)D64[j];
            std::vector<int64_t> o32 = order;
            std::sort(o32.begin(), o32.end(), [&](int64_t a, int64_t b) {
                if (D32[a] != D32[b]) return D32[a] < D32[b];
                return a < b;
            });
            for (int32_t s = 0; s < k; ++s) {
                idx32[r * k + s] = (int32_t)o32[s];
                dist32[r * k + s] = D32[o32[s]];
            }
        }
    });
    return 0;
}

// Exact select on a given fp32 matrix (the parity reference for knn_select):
// for each row i < M of D (row stride ld), std::sort of j < N by (D[i,j], j) under the
// key order above, first k written as (idx, canonical value).  1 <= k <= N.
int oracle_select_f32(const float* D, int64_t M, int64_t N, int64_t ld, int32_t k,
                      int32_t threads, int32_t* idx, float* dist) {
    if (M < 0 || N < 1 || ld < N || k < 1 || k > N) return 1;
    parallel_rows(M, threads, [&](int64_t i) {
        const float* row = D + i * ld;
        std::vector<int64_t> o(N);
        std::iota(o.begin(), o.end(), 0);
        std::sort(o.begin(), o.end(), [&](int64_t a, int64_t b) {
            if (!f32_equal(row[a], row[b])) return f32_less(row[a], row[b]);
            return a < b;
        });
        for (int32_t s = 0; s < k; ++s) {
            idx[i * k + s] = (int32_t)o[s];
            dist[i * k + s] = f32_canon(row[o[s]]);
        }
    });
    return 0;
}

// Merge reference ("Batch execution will obviously require merging of
// results"): for each row, the union of G lists of k (value, local idx) pairs, where
// list g's indices are shifted by offsets[g], sorted by (value, global idx); first k.
// part_dist / part_idx are laid out [G][M][k].
int oracle_merge(const float* part_dist, const int32_t* part_idx, int32_t G, int64_t M, int32_t k,
                 const int64_t* offsets, int32_t* idx, float* dist) {
    if (G < 1 || M < 0 || k < 1) return 1;
    for (int64_t i = 0; i < M; ++i) {
        std::vector<std::pair<float, int64_t>> u;
        u.reserve((size_t)G * k);
        for (int32_t g = 0; g < G; ++g)
            for (int32_t s = 0; s < k; ++s) {
                int64_t off = ((int64_t)g * M + i) * k + s;
                u.emplace_back(part_dist[off], (int64_t)part_idx[off] + offsets[g]);
            }
        std::sort(u.begin(), u.end(), [](const std::pair<float, int64_t>& a,
                                         const std::pair<float, int64_t>& b) {
            if (!f32_equal(a.first, b.first)) return f32_less(a.first, b.first);
            return a.second < b.second;
        });
        for (int32_t s = 0; s < k; ++s) {
            idx[i * k + s] = (int32_t)u[s].second;
            dist[i * k + s] = f32_canon(u[s].first);
        }
    }
    return 0;
}

}  // extern "C"
