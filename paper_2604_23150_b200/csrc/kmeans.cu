// K7: request-clustering k-means on the device,
// bit-identical to the reference's host k-means.
//
// Restates kmeans / kmeanspp_init / assign_labels / repair_empty_clusters /
// objective_value (/root/reference/proj/core/src/clustering.cpp:39-230) and
// l2_normalize (:15-36). Every floating-point reduction keeps the reference's
// order and rounding (explicit __dadd_rn/__dmul_rn/__dsub_rn, no FMA
// contraction): per-row distances run one thread per row (rows staged in
// shared memory), sequential over the dimension; centroid sums run one lane
// per (cluster, dimension), sequential over rows in index order from
// shared-memory tiles streamed by loader warps; the k-means++ running totals
// and the objective are sequential sums in index order (one adding thread fed
// by loader warps). MPB_KMEANS_TRACE=1 prints per-iteration host timings. The RNG draws
// (std::mt19937_64 + libstdc++ uniform_int / uniform_real, data-independent)
// stay on the host, which drives the Lloyd loop with one small D2H read per
// step (cluster sizes, centroid movement). Empty clusters (rare) are repaired
// on the host exactly as the reference does.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <random>
#include <vector>

#include "internal.cuh"

namespace mpb {
namespace {

constexpr int kKMax = 16;  // register-resident distance accumulators per row

__device__ __forceinline__ double sqdist_dev(const double *a, const double *b, uint32_t dim) {
    double s = 0.0;
    for (uint32_t c = 0; c < dim; ++c) {
        const double d = __dsub_rn(a[c], b[c]);
        s = __dadd_rn(s, __dmul_rn(d, d));
    }
    return s;
}

__global__ void k_l2_normalize(const double *X, uint64_t n, uint32_t dim, double *out,
                               uint32_t *err) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double *a = X + i * dim;
    double ss = 0.0;
    for (uint32_t c = 0; c < dim; ++c) ss = __dadd_rn(ss, __dmul_rn(a[c], a[c]));
    if (ss == 0.0) {
        atomicOr(err, 1u);
        return;
    }
    const double inv = __ddiv_rn(1.0, __dsqrt_rn(ss));
    for (uint32_t c = 0; c < dim; ++c) out[i * dim + c] = __dmul_rn(a[c], inv);
}

// dmin[i] = sqdist(X_i, X_pick) (init) or min(dmin[i], sqdist(X_i, X_pick)).
__global__ void k_mindist(const double *X, uint64_t n, uint32_t dim, uint64_t pick, int init,
                          double *dmin) {
    extern __shared__ double s_c[];  // [dim]
    for (uint32_t c = threadIdx.x; c < dim; c += blockDim.x) s_c[c] = X[pick * dim + c];
    __syncthreads();
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double d = sqdist_dev(X + i * dim, s_c, dim);
    if (init) {
        dmin[i] = d;
    } else {
        const double m = dmin[i];
        dmin[i] = d < m ? d : m;  // std::min(m, d)
    }
}

// total = sum(v) in index order; then, when target >= 0, the first i with
// running sum >= target (n - 1 on rounding fall-through). One thread adds (the
// reference's sequential order); warps 1-7 stream the next tile into shared
// memory meanwhile, so the add chain never waits on global memory.
constexpr uint32_t kScanTile = 2048;
__global__ void __launch_bounds__(256) k_seq_scan(const double *v, uint64_t n, double target,
                                                  double *total_out, uint64_t *pick_out) {
    __shared__ double s_buf[2][kScanTile];
    __shared__ int s_done;
    const uint32_t warp = threadIdx.x >> 5;
    auto load = [&](uint64_t base, int b) {
        for (uint32_t j = threadIdx.x - 32; j < kScanTile; j += 224) {
            const uint64_t i = base + j;
            s_buf[b][j] = i < n ? v[i] : 0.0;
        }
    };
    if (warp != 0) load(0, 0);
    if (threadIdx.x == 0) s_done = 0;
    __syncthreads();
    double t = 0.0;
    uint64_t pick = n;
    int buf = 0;
    for (uint64_t base = 0; base < n; base += kScanTile, buf ^= 1) {
        if (warp != 0) {
            if (base + kScanTile < n) load(base + kScanTile, buf ^ 1);
        } else if (threadIdx.x == 0) {
            const uint32_t m = static_cast<uint32_t>(min(static_cast<uint64_t>(kScanTile), n - base));
            if (target < 0.0) {
                for (uint32_t j = 0; j < m; ++j) t = __dadd_rn(t, s_buf[buf][j]);
            } else {
                for (uint32_t j = 0; j < m; ++j) {
                    t = __dadd_rn(t, s_buf[buf][j]);
                    if (t >= target) {
                        pick = base + j;
                        s_done = 1;
                        break;
                    }
                }
            }
        }
        __syncthreads();
        if (s_done) break;
    }
    if (threadIdx.x == 0) {
        if (target < 0.0)
            *total_out = t;
        else
            *pick_out = pick == n ? n - 1 : pick;
    }
}

// labels[i] = argmin_k sqdist(X_i, C_k) (strict <: ties to the lowest k);
// sizes[k] += 1; dist[i] = the winning distance (objective / repair).
template <int KM>
__global__ void k_assign(const double *X, uint64_t n, uint32_t dim, const double *C, uint32_t K,
                         uint32_t *labels, uint32_t *sizes, double *dist) {
    extern __shared__ double s_C[];  // [K][dim], then this block's rows [blockDim][dim + 1]
    double *s_rows = s_C + size_t(K) * dim;
    for (uint32_t j = threadIdx.x; j < K * dim; j += blockDim.x) s_C[j] = C[j];
    // coalesced staging of the block's rows (padded stride: conflict-free reads)
    const uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x;
    const uint32_t nr = static_cast<uint32_t>(min(static_cast<uint64_t>(blockDim.x), n - r0));
    for (uint32_t j = threadIdx.x; j < nr * dim; j += blockDim.x) {
        const uint32_t r = j / dim, c = j - r * dim;
        s_rows[r * (dim + 1) + c] = X[r0 * dim + j];
    }
    __syncthreads();
    const uint64_t i = r0 + threadIdx.x;
    if (i >= n) return;
    const double *a = s_rows + threadIdx.x * (dim + 1);
    double best = INFINITY;
    uint32_t bk = 0;
    if (KM > 0 && K <= static_cast<uint32_t>(KM)) {
        // all K distance chains advance together over the dimension (each chain
        // still sums in dimension order)
        double s[KM > 0 ? KM : 1];
#pragma unroll
        for (int k = 0; k < (KM > 0 ? KM : 1); ++k) s[k] = 0.0;
        for (uint32_t c = 0; c < dim; ++c) {
            const double x = a[c];
#pragma unroll
            for (int k = 0; k < (KM > 0 ? KM : 1); ++k)
                if (static_cast<uint32_t>(k) < K) {
                    const double d = __dsub_rn(x, s_C[k * dim + c]);
                    s[k] = __dadd_rn(s[k], __dmul_rn(d, d));
                }
        }
#pragma unroll
        for (int k = 0; k < (KM > 0 ? KM : 1); ++k)
            if (static_cast<uint32_t>(k) < K && s[k] < best) {
                best = s[k];
                bk = k;
            }
    } else {
        for (uint32_t k = 0; k < K; ++k) {
            const double d = sqdist_dev(a, s_C + k * dim, dim);
            if (d < best) {
                best = d;
                bk = k;
            }
        }
    }
    labels[i] = bk;
    if (dist) dist[i] = best;
    if (sizes) atomicAdd(sizes + bk, 1u);
}

// dist[i] = sqdist(X_i, C[labels[i]]) (objective_value, clustering.cpp:159-166).
__global__ void k_label_dist(const double *X, uint64_t n, uint32_t dim, const double *C,
                             uint32_t K, const uint32_t *labels, double *dist) {
    extern __shared__ double s_C[];  // [K][dim]
    for (uint32_t j = threadIdx.x; j < K * dim; j += blockDim.x) s_C[j] = C[j];
    __syncthreads();
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    dist[i] = sqdist_dev(X + i * dim, s_C + static_cast<size_t>(labels[i]) * dim, dim);
}

// C[k][c] = (sum over rows i with labels[i] == k, in index order, of X[i][c]) / size_k.
// Block = a slice of cpb columns for ALL clusters (each row is read once):
// warp 0 lane (k, c) adds sequentially over rows from shared memory (the
// reference's order); warps 1-7 stage the next tile of labels + the slice's
// X values (double-buffered, 16-byte loads batched for memory-level
// parallelism), so the add chain never waits on global memory.
constexpr uint32_t kUpdRows = 256;
__global__ void __launch_bounds__(256) k_update(const double *X, uint64_t n, uint32_t dim,
                                                const uint32_t *labels, uint32_t K, uint32_t cpb,
                                                int vec, const uint32_t *sizes, double *C) {
    extern __shared__ double s_x[];  // [2][kUpdRows][cpb], then labels [2][kUpdRows]
    uint32_t *s_l = reinterpret_cast<uint32_t *>(s_x + 2 * kUpdRows * cpb);
    const uint32_t c0 = blockIdx.x * cpb;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t cols = min(cpb, dim - c0);
    auto load = [&](uint64_t base, int b) {
        double *dx = s_x + static_cast<size_t>(b) * kUpdRows * cpb;
        uint32_t *dl = s_l + b * kUpdRows;
        const uint32_t t = threadIdx.x - 32;  // 0..223
        if (vec) {  // 16-byte pieces: cpb/2 per row
            const uint32_t per = cpb / 2, total = kUpdRows * per;
#pragma unroll 4
            for (uint32_t j = t; j < total; j += 224) {
                const uint32_t r = j / per, q = j - r * per;
                const uint64_t i = base + r;
                double2 v = make_double2(0.0, 0.0);
                if (i < n) v = *reinterpret_cast<const double2 *>(X + i * dim + c0 + 2 * q);
                reinterpret_cast<double2 *>(dx)[j] = v;
            }
        } else {
            const uint32_t total = kUpdRows * cpb;
#pragma unroll 4
            for (uint32_t j = t; j < total; j += 224) {
                const uint32_t r = j / cpb, q = j - r * cpb;
                const uint64_t i = base + r;
                dx[j] = (i < n && q < cols) ? X[i * dim + c0 + q] : 0.0;
            }
        }
        for (uint32_t j = t; j < kUpdRows; j += 224) {
            const uint64_t i = base + j;
            dl[j] = i < n ? labels[i] : 0xFFFFFFFFu;
        }
    };
    if (warp != 0) load(0, 0);
    __syncthreads();
    const uint32_t k = lane / cpb, c = lane - k * cpb;
    const bool active = warp == 0 && k < K && c < cols;
    double s = 0.0;
    int buf = 0;
    for (uint64_t base = 0; base < n; base += kUpdRows, buf ^= 1) {
        if (warp != 0) {
            if (base + kUpdRows < n) load(base + kUpdRows, buf ^ 1);
        } else if (active) {
            const double *dx = s_x + static_cast<size_t>(buf) * kUpdRows * cpb + c;
            const uint32_t *dl = s_l + buf * kUpdRows;
            // branch-free: non-members add +0.0, which leaves s bit-identical
            // (s starts at +0.0 and round-to-nearest sums never produce -0.0)
#pragma unroll 8
            for (uint32_t r = 0; r < kUpdRows; ++r) {
                const double x = dx[r * cpb];
                s = __dadd_rn(s, dl[r] == k ? x : 0.0);
            }
        }
        __syncthreads();
    }
    if (active)
        C[static_cast<size_t>(k) * dim + c0 + c] = __ddiv_rn(s, static_cast<double>(sizes[k]));
}

// movement = max_k sqrt(sqdist(C_k, P_k)) (single thread, k order).
__global__ void k_movement(const double *C, const double *P, uint32_t K, uint32_t dim,
                           double *out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double m = 0.0;
    for (uint32_t k = 0; k < K; ++k) {
        const double v = __dsqrt_rn(sqdist_dev(C + size_t(k) * dim, P + size_t(k) * dim, dim));
        m = v > m ? v : m;  // std::max(m, v)
    }
    *out = m;
}

struct Scratch {
    double *dmin = nullptr, *dist = nullptr, *prev = nullptr;
    uint32_t *sizes = nullptr;
    double *d_small = nullptr;  // [0] total, [1] movement, [2] objective
    uint64_t *d_pick = nullptr;
    double *h_d = nullptr;      // pinned mirrors
    uint64_t *h_pick = nullptr;
    uint32_t *h_sizes = nullptr;
};

// Carves the k-means buffers out of the context's scratch / pinned areas.
mpb_status carve(mpb_context *ctx, uint64_t n, uint32_t dim, uint32_t K, Scratch &sc) {
    const size_t prev_b = (size_t(K) * dim * 8 + 255) / 256 * 256;
    const size_t need = 2 * ((n * 8 + 255) / 256 * 256) + prev_b + 256 + 256;
    MPB_CUDA(ctx->ensure_scratch(need));
    char *p = static_cast<char *>(ctx->scratch);
    sc.dmin = reinterpret_cast<double *>(p);
    p += (n * 8 + 255) / 256 * 256;
    sc.dist = reinterpret_cast<double *>(p);
    p += (n * 8 + 255) / 256 * 256;
    sc.prev = reinterpret_cast<double *>(p);
    p += prev_b;
    sc.d_small = reinterpret_cast<double *>(p);
    sc.d_pick = reinterpret_cast<uint64_t *>(p + 32);
    sc.sizes = reinterpret_cast<uint32_t *>(p + 256);
    const size_t hneed = 64 + size_t(K) * 4;
    if (ctx->pinned_bytes < hneed) {
        if (ctx->pinned) cudaFreeHost(ctx->pinned);
        ctx->pinned = nullptr;
        ctx->pinned_bytes = 0;
        MPB_CUDA(cudaMallocHost(&ctx->pinned, std::max<size_t>(hneed, 4096)));
        ctx->pinned_bytes = std::max<size_t>(hneed, 4096);
    }
    sc.h_d = static_cast<double *>(ctx->pinned);
    sc.h_pick = reinterpret_cast<uint64_t *>(static_cast<char *>(ctx->pinned) + 32);
    sc.h_sizes = reinterpret_cast<uint32_t *>(static_cast<char *>(ctx->pinned) + 64);
    return MPB_OK;
}

// Host-side repair of empty clusters (clustering.cpp:124-157): the farthest
// point of a cluster with more than one member moves into each empty cluster,
// in cluster order. Only labels, each row's distance to its own centroid
// (device-computed, unchanged by the repair for every row that can still be
// chosen) and the moved rows cross PCIe.
mpb_status host_repair(const double *dX, uint64_t n, uint32_t dim, double *dC, uint32_t K,
                       uint32_t *dlabels, const double *ddist, uint32_t *h_sizes, uint32_t *dsizes,
                       cudaStream_t st) {
    std::vector<uint32_t> labels(n);
    std::vector<double> dist(n);
    MPB_CUDA(cudaMemcpyAsync(labels.data(), dlabels, n * 4, cudaMemcpyDeviceToHost, st));
    MPB_CUDA(cudaMemcpyAsync(dist.data(), ddist, n * 8, cudaMemcpyDeviceToHost, st));
    MPB_CUDA(cudaStreamSynchronize(st));
    std::vector<size_t> size(K, 0);
    for (uint32_t l : labels) ++size[l];
    for (uint32_t k = 0; k < K; ++k) {
        if (size[k]) continue;
        double worst = -1.0;
        size_t victim = n;
        for (size_t i = 0; i < n; ++i) {
            if (size[labels[i]] <= 1) continue;
            if (dist[i] > worst) {
                worst = dist[i];
                victim = i;
            }
        }
        if (victim == n) return fail(MPB_INFEASIBLE_ERROR, "kmeans: cannot repair empty cluster");
        --size[labels[victim]];
        labels[victim] = k;
        size[k] = 1;
        MPB_CUDA(cudaMemcpyAsync(dlabels + victim, &labels[victim], 4, cudaMemcpyHostToDevice, st));
        MPB_CUDA(cudaMemcpyAsync(dC + size_t(k) * dim, dX + victim * dim, size_t(dim) * 8,
                                 cudaMemcpyDeviceToDevice, st));
        MPB_CUDA(cudaStreamSynchronize(st));  // &labels[victim] is pageable host memory
    }
    for (uint32_t k = 0; k < K; ++k) h_sizes[k] = static_cast<uint32_t>(size[k]);
    MPB_CUDA(cudaMemcpyAsync(dsizes, h_sizes, size_t(K) * 4, cudaMemcpyHostToDevice, st));
    MPB_CUDA(cudaStreamSynchronize(st));
    return MPB_OK;
}

}  // namespace
}  // namespace mpb

using namespace mpb;

extern "C" {

mpb_status mpb_l2_normalize_rows_device(mpb_context *ctx, const double *matrix, uint64_t rows,
                                        uint32_t cols, double *out) {
    if (!ctx || (rows && (!matrix || !out)))
        return fail(MPB_VALIDATION_ERROR, "mpb_l2_normalize_rows_device: NULL argument");
    if (rows == 0) return MPB_OK;
    k_l2_normalize<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, ctx->stream>>>(
        matrix, rows, cols, out, ctx->d_error);
    MPB_LAUNCHED(ctx);
    uint32_t flag = 0;
    MPB_CUDA(cudaMemcpyAsync(&flag, ctx->d_error, 4, cudaMemcpyDeviceToHost, ctx->stream));
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (flag) {
        MPB_CUDA(cudaMemsetAsync(ctx->d_error, 0, 4, ctx->stream));
        return fail(MPB_VALIDATION_ERROR, "l2_normalize: zero vector");
    }
    return MPB_OK;
}

mpb_status mpb_kmeans_device(mpb_context *ctx, const double *X, uint64_t n, uint32_t dim,
                             uint32_t K, uint64_t seed, uint32_t max_iterations, double tolerance,
                             uint32_t *labels, double *centroids, double *objective_out,
                             uint32_t *iterations_out, double *objective_history) {
    if (!ctx || !X || !labels || !centroids)
        return fail(MPB_VALIDATION_ERROR, "mpb_kmeans_device: NULL argument");
    if (K < 1) return fail(MPB_INFEASIBLE_ERROR, "kmeans: K must be >= 1");
    if (n < K)
        return fail(MPB_INFEASIBLE_ERROR,
                    "kmeans: " + std::to_string(n) + " rows < K=" + std::to_string(K));
    if (size_t(K) * dim * 8 > 160 * 1024)
        return fail(MPB_CONFIG_ERROR, "mpb_kmeans_device: K*dim centroids exceed shared memory");
    cudaStream_t st = ctx->stream;
    if (size_t(K) * 4 + 64 > (1u << 20)) return fail(MPB_CONFIG_ERROR, "kmeans: K too large");
    Scratch sc;
    if (mpb_status cs = carve(ctx, n, dim, K, sc); cs != MPB_OK) return cs;
    const unsigned rb = static_cast<unsigned>((n + 127) / 128);
    const size_t csmem = size_t(K) * dim * 8;
    const uint32_t ab = 64;  // assign: rows per block (staged in smem)
    const unsigned rba = static_cast<unsigned>((n + ab - 1) / ab);
    const size_t asmem = csmem + size_t(ab) * (dim + 1) * 8;
    if (asmem > 200 * 1024)
        return fail(MPB_CONFIG_ERROR, "mpb_kmeans_device: K*dim too large for the assign tile");
    if (K > 32) return fail(MPB_CONFIG_ERROR, "mpb_kmeans_device: K <= 32");
    // update: columns per block so that K * cpb <= 32 lanes (cpb a power of two)
    uint32_t cpb = 1;
    while (cpb * 2 * K <= 32 && cpb * 2 <= dim) cpb *= 2;
    const unsigned ucols = (dim + cpb - 1) / cpb;
    const int uvec = cpb >= 2 && dim % 2 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
    const size_t usmem = size_t(2) * kUpdRows * cpb * 8 + size_t(2) * kUpdRows * 4;
    MPB_CUDA(cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(usmem)));
    auto assign = K <= static_cast<uint32_t>(kKMax) ? k_assign<kKMax> : k_assign<0>;
    MPB_CUDA(cudaFuncSetAttribute(assign, cudaFuncAttributeMaxDynamicSharedMemorySize, int(asmem)));
    MPB_CUDA(cudaFuncSetAttribute(k_label_dist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(csmem)));

    // ---- k-means++ seeding (clustering.cpp:56-102); RNG on the host
    std::mt19937_64 rng(seed);
    std::vector<uint64_t> used;
    const uint64_t first = std::uniform_int_distribution<std::size_t>(0, n - 1)(rng);
    used.push_back(first);
    MPB_CUDA(cudaMemcpyAsync(centroids, X + first * dim, size_t(dim) * 8, cudaMemcpyDeviceToDevice, st));
    k_mindist<<<rb, 128, dim * 8, st>>>(X, n, dim, first, 1, sc.dmin);
    MPB_LAUNCHED(ctx);
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    for (uint32_t k = 1; k < K; ++k) {
        k_seq_scan<<<1, 256, 0, st>>>(sc.dmin, n, -1.0, sc.d_small, sc.d_pick);
        MPB_LAUNCHED(ctx);
        MPB_CUDA(cudaMemcpyAsync(sc.h_d, sc.d_small, 8, cudaMemcpyDeviceToHost, st));
        MPB_CUDA(cudaStreamSynchronize(st));
        const double total = sc.h_d[0];
        uint64_t pick = n;
        if (total > 0.0) {
            const double target = unit(rng) * total;
            k_seq_scan<<<1, 256, 0, st>>>(sc.dmin, n, target, sc.d_small, sc.d_pick);
            MPB_LAUNCHED(ctx);
            MPB_CUDA(cudaMemcpyAsync(sc.h_pick, sc.d_pick, 8, cudaMemcpyDeviceToHost, st));
            MPB_CUDA(cudaStreamSynchronize(st));
            pick = *sc.h_pick;
        } else {  // all points coincide with chosen centers: lowest unused row
            for (uint64_t i = 0; i < n && pick == n; ++i)
                if (std::find(used.begin(), used.end(), i) == used.end()) pick = i;
            if (pick == n) pick = 0;
        }
        used.push_back(pick);
        MPB_CUDA(cudaMemcpyAsync(centroids + size_t(k) * dim, X + pick * dim, size_t(dim) * 8,
                                 cudaMemcpyDeviceToDevice, st));
        k_mindist<<<rb, 128, dim * 8, st>>>(X, n, dim, pick, 0, sc.dmin);
        MPB_LAUNCHED(ctx);
    }

    // ---- Lloyd iterations (clustering.cpp:180-215)
    auto assign_repair = [&]() -> mpb_status {
        MPB_CUDA(cudaMemsetAsync(sc.sizes, 0, size_t(K) * 4, st));
        assign<<<rba, ab, asmem, st>>>(X, n, dim, centroids, K, labels, sc.sizes, sc.dist);
        MPB_LAUNCHED(ctx);
        MPB_CUDA(cudaMemcpyAsync(sc.h_sizes, sc.sizes, size_t(K) * 4, cudaMemcpyDeviceToHost, st));
        MPB_CUDA(cudaStreamSynchronize(st));
        bool empty = false;
        for (uint32_t k = 0; k < K; ++k) empty |= sc.h_sizes[k] == 0;
        if (!empty) return MPB_OK;
        // distances of every row to its own (pre-repair) centroid
        k_label_dist<<<rb, 128, csmem, st>>>(X, n, dim, centroids, K, labels, sc.dist);
        MPB_LAUNCHED(ctx);
        return host_repair(X, n, dim, centroids, K, labels, sc.dist, sc.h_sizes, sc.sizes, st);
    };
    static const bool trace = std::getenv("MPB_KMEANS_TRACE") != nullptr;
    uint32_t it = 0;
    for (; it < max_iterations; ++it) {
        auto t0 = std::chrono::steady_clock::now();
        mpb_status s = assign_repair();
        if (s != MPB_OK) return s;
        auto t1 = std::chrono::steady_clock::now();
        MPB_CUDA(cudaMemcpyAsync(sc.prev, centroids, size_t(K) * dim * 8, cudaMemcpyDeviceToDevice, st));
        k_update<<<ucols, 256, usmem, st>>>(X, n, dim, labels, K, cpb, uvec, sc.sizes, centroids);
        MPB_LAUNCHED(ctx);
        k_movement<<<1, 32, 0, st>>>(centroids, sc.prev, K, dim, sc.d_small + 1);
        MPB_LAUNCHED(ctx);
        if (objective_history) {  // objective_value after the update (clustering.cpp:207-208)
            k_label_dist<<<rb, 128, csmem, st>>>(X, n, dim, centroids, K, labels, sc.dist);
            MPB_LAUNCHED(ctx);
            k_seq_scan<<<1, 256, 0, st>>>(sc.dist, n, -1.0, sc.d_small + 2, sc.d_pick);
            MPB_LAUNCHED(ctx);
        }
        MPB_CUDA(cudaMemcpyAsync(sc.h_d + 1, sc.d_small + 1, objective_history ? 16 : 8,
                                 cudaMemcpyDeviceToHost, st));
        MPB_CUDA(cudaStreamSynchronize(st));
        if (objective_history) objective_history[it] = sc.h_d[2];
        if (trace) {
            auto t2 = std::chrono::steady_clock::now();
            std::fprintf(stderr, "[kmeans] it %u assign %.1f us update %.1f us move %.3g\n", it,
                         std::chrono::duration<double, std::micro>(t1 - t0).count(),
                         std::chrono::duration<double, std::micro>(t2 - t1).count(), sc.h_d[1]);
        }
        if (sc.h_d[1] < tolerance) {
            ++it;
            break;
        }
    }
    // final argmin assignment + repair + objective (clustering.cpp:220-224)
    mpb_status s = assign_repair();
    if (s != MPB_OK) return s;
    // each row's distance to its (possibly repaired) label's centroid, summed in order
    k_label_dist<<<rb, 128, csmem, st>>>(X, n, dim, centroids, K, labels, sc.dist);
    MPB_LAUNCHED(ctx);
    k_seq_scan<<<1, 256, 0, st>>>(sc.dist, n, -1.0, sc.d_small + 2, sc.d_pick);
    MPB_LAUNCHED(ctx);
    MPB_CUDA(cudaMemcpyAsync(sc.h_d + 2, sc.d_small + 2, 8, cudaMemcpyDeviceToHost, st));
    MPB_CUDA(cudaStreamSynchronize(st));
    if (objective_out) *objective_out = sc.h_d[2];
    if (iterations_out) *iterations_out = it;
    return MPB_OK;
}

}  // extern "C"
