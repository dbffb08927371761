// K6: bf16 expert-parallel dispatch / combine driven by the K3 permutation.
//
// Local halves (NCCL path): hidden-state gather into the send buffer and the
// weighted combine back into token order; the host runs the all-to-all-v in
// between. Fused NVLink path (P2P): every rank's recv buffer is mapped into
// every peer (symmetric memory over NVSwitch); k_put_counts writes this rank's
// per-destination counts into every peer's count matrix, k_dispatch_p2p
// gathers each sorted pair's row straight into the destination rank's recv
// buffer (remote 16-byte stores: gather and transfer are one pass), and
// k_combine_p2p reads each token's k returned rows straight out of the peers'
// buffers (remote loads) into the fp32 weighted sum — no send / back buffers,
// no second all-to-all. Rows of rank s for rank r land at
// sum_{s'<s} C[s'][r] + (position - first position for r) in r's buffer.
// One warp per row, 16-byte vectors; combine accumulates the k rows in a fixed
// order (bit-identical to the local combine).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace mpb {
namespace {

__global__ void __launch_bounds__(256) k_gather(const uint4 *X, const int32_t *sorted_pairs,
                                                uint64_t n, uint32_t k, uint32_t hv, uint4 *send) {
    const uint64_t row = static_cast<uint64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (row >= n) return;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t tok = static_cast<uint64_t>(sorted_pairs[row]) / k;
    const uint4 *src = X + tok * hv;
    uint4 *dst = send + row * hv;
    for (uint32_t i = lane; i < hv; i += 32) dst[i] = __ldg(src + i);
}

__global__ void __launch_bounds__(256) k_combine(const uint4 *recv, const int32_t *pair_pos,
                                                 const float *w, uint64_t T, uint32_t k,
                                                 uint32_t hv, uint4 *Y) {
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (t >= T) return;
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t i = lane; i < hv; i += 32) {
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (uint32_t j = 0; j < k; ++j) {
            const float wj = w[t * k + j];
            const uint4 v = __ldg(recv + static_cast<uint64_t>(pair_pos[t * k + j]) * hv + i);
            const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 f = __bfloat1622float2(h[q]);
                acc[2 * q] = fmaf(wj, f.x, acc[2 * q]);
                acc[2 * q + 1] = fmaf(wj, f.y, acc[2 * q + 1]);
            }
        }
        uint4 o;
        __nv_bfloat162 *oh = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
        for (int q = 0; q < 4; ++q) oh[q] = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
        Y[t * hv + i] = o;
    }
}

// C[me][r] = rows this rank sends to rank r (its contiguous slice of the
// sorted pairs), written into every peer's [world][world] count matrix.
__global__ void k_put_counts(const int64_t *ko, uint32_t span, uint32_t world, uint32_t me,
                             const uint64_t *peer_cnt) {
    const uint32_t q = threadIdx.x / world, r = threadIdx.x % world;
    if (q >= world) return;
    const int64_t c = ko[static_cast<size_t>(r + 1) * span] - ko[static_cast<size_t>(r) * span];
    reinterpret_cast<int64_t *>(peer_cnt[q])[me * world + r] = c;
}

struct P2PMap {
    int64_t first[9];  // first sorted position for rank r (r <= world)
    int64_t base[8];   // where this rank's rows start in rank r's recv buffer
};

__device__ __forceinline__ void p2p_map(const int64_t *C, const int64_t *ko, uint32_t span,
                                        uint32_t world, uint32_t me, P2PMap &m) {
    for (uint32_t r = 0; r <= world; ++r) m.first[r] = ko[static_cast<size_t>(r) * span];
    for (uint32_t r = 0; r < world; ++r) {
        int64_t b = 0;
        for (uint32_t s = 0; s < me; ++s) b += C[s * world + r];
        m.base[r] = b;
    }
}

__device__ __forceinline__ uint32_t rank_of_pos(const P2PMap &m, uint32_t world, int64_t pos) {
    uint32_t r = 0;
    while (r + 1 < world && pos >= m.first[r + 1]) ++r;
    return r;
}

__global__ void __launch_bounds__(256) k_dispatch_p2p(const uint4 *X, const int32_t *sorted_pairs,
                                                      uint64_t n, uint32_t k, uint32_t hv,
                                                      const int64_t *C, const int64_t *ko,
                                                      uint32_t span, uint32_t world, uint32_t me,
                                                      const uint64_t *peer_recv, uint64_t cap,
                                                      uint32_t *err) {
    __shared__ P2PMap m;
    if (threadIdx.x == 0) p2p_map(C, ko, span, world, me, m);
    __syncthreads();
    const uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (i0 >= n) return;
    // rotated start (see k_dispatch_p2p_tma)
    const uint64_t rot = static_cast<uint64_t>(m.first[(me + 1) % world]) % n;
    const uint64_t i = i0 + rot >= n ? i0 + rot - n : i0 + rot;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t r = rank_of_pos(m, world, static_cast<int64_t>(i));
    const uint64_t row = static_cast<uint64_t>(m.base[r] + static_cast<int64_t>(i) - m.first[r]);
    if (row >= cap) {
        if (lane == 0) atomicOr(err, kErrCapacity);
        return;
    }
    const uint64_t tok = static_cast<uint64_t>(sorted_pairs[i]) / k;
    const uint4 *src = X + tok * hv;
    uint4 *dst = reinterpret_cast<uint4 *>(peer_recv[r]) + row * hv;
    // batches of 8 independent 16-byte loads before their remote stores: more
    // bytes in flight per warp over NVLink
    uint32_t c = lane;
    for (; c + 7 * 32 < hv; c += 8 * 32) {
        uint4 v[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) v[b] = __ldg(src + c + b * 32);
#pragma unroll
        for (int b = 0; b < 8; ++b) dst[c + b * 32] = v[b];
    }
    for (; c < hv; c += 32) dst[c] = __ldg(src + c);
}

__global__ void __launch_bounds__(256) k_combine_p2p(const int32_t *pair_pos, const float *w,
                                                     uint64_t T, uint32_t k, uint32_t hv,
                                                     const int64_t *C, const int64_t *ko,
                                                     uint32_t span, uint32_t world, uint32_t me,
                                                     const uint64_t *peer_recv, uint4 *Y) {
    __shared__ P2PMap m;
    if (threadIdx.x == 0) p2p_map(C, ko, span, world, me, m);
    __syncthreads();
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (t >= T) return;
    const uint32_t lane = threadIdx.x & 31;
    if (k <= 8) {
        // the token's k rows located once; each lane then issues all k remote
        // loads of a column before accumulating them in j order (bit-identical
        // to the loop below, more bytes in flight per warp)
        const uint4 *rowp[8];
        float wj[8];
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
            rowp[j] = nullptr;
            wj[j] = 0.f;
            if (j < k) {
                const int64_t pos = pair_pos[t * k + j];
                const uint32_t r = rank_of_pos(m, world, pos);
                const uint64_t row = static_cast<uint64_t>(m.base[r] + pos - m.first[r]);
                rowp[j] = reinterpret_cast<const uint4 *>(peer_recv[r]) + row * hv;
                wj[j] = w[t * k + j];
            }
        }
        for (uint32_t c = lane; c < hv; c += 32) {
            uint4 v[8];
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j)
                if (j < k) v[j] = rowp[j][c];
            float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                if (j >= k) break;
                const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v[j]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 f = __bfloat1622float2(h[q]);
                    acc[2 * q] = fmaf(wj[j], f.x, acc[2 * q]);
                    acc[2 * q + 1] = fmaf(wj[j], f.y, acc[2 * q + 1]);
                }
            }
            uint4 o;
            __nv_bfloat162 *oh = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
            for (int q = 0; q < 4; ++q) oh[q] = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
            Y[t * hv + c] = o;
        }
        return;
    }
    for (uint32_t c = lane; c < hv; c += 32) {
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (uint32_t j = 0; j < k; ++j) {
            const float wj = w[t * k + j];
            const int64_t pos = pair_pos[t * k + j];
            const uint32_t r = rank_of_pos(m, world, pos);
            const uint64_t row = static_cast<uint64_t>(m.base[r] + pos - m.first[r]);
            const uint4 v = reinterpret_cast<const uint4 *>(peer_recv[r])[row * hv + c];
            const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 f = __bfloat1622float2(h[q]);
                acc[2 * q] = fmaf(wj, f.x, acc[2 * q]);
                acc[2 * q + 1] = fmaf(wj, f.y, acc[2 * q + 1]);
            }
        }
        uint4 o;
        __nv_bfloat162 *oh = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
        for (int q = 0; q < 4; ++q) oh[q] = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
        Y[t * hv + c] = o;
    }
}

// Pull variant of the dispatch: the DESTINATION copies its rows out of the
// sources' staged X (symmetric memory), in exactly the layout the push
// dispatch produces (source s's rows at sum_{s'<s} C[s'][me], in s's sorted
// order), so the combine and its output are unchanged. Remote reads run at the
// NVLink ingress rate of the pull combine (the pushed stores were measured at
// ~420 GB/s egress at 4 ranks). Warp per row, 8 independent 16-byte loads in
// flight per lane; the row's token id comes from the source's sorted pairs.
__global__ void __launch_bounds__(256) k_dispatch_pull(const int64_t *C, const uint64_t *peer_x,
                                                       const uint64_t *peer_sp, const uint64_t *peer_ko,
                                                       uint32_t k, uint32_t hv, uint32_t span,
                                                       uint32_t world, uint32_t me, uint4 *recv,
                                                       uint64_t cap, uint32_t *err) {
    __shared__ int64_t s_off[9], s_first[8];
    if (threadIdx.x < world)
        s_first[threadIdx.x] =
            reinterpret_cast<const int64_t *>(peer_ko[threadIdx.x])[static_cast<size_t>(me) * span];
    if (threadIdx.x == 0) {
        s_off[0] = 0;
        for (uint32_t s = 0; s < world; ++s) s_off[s + 1] = s_off[s] + C[s * world + me];
    }
    __syncthreads();
    const uint64_t total = static_cast<uint64_t>(s_off[world]);
    const uint32_t lane = threadIdx.x & 31;
    // rotated start: rows from source me+1 first, so the ranks do not all read
    // the same source at once (one hot NVLink port)
    const uint64_t rot = total ? static_cast<uint64_t>(s_off[(me + 1) % world]) % total : 0;
    for (uint64_t qq = static_cast<uint64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5); qq < total;
         qq += static_cast<uint64_t>(gridDim.x) * 8) {
        const uint64_t q = qq + rot >= total ? qq + rot - total : qq + rot;
        if (q >= cap) {
            if (lane == 0) atomicOr(err, kErrCapacity);
            continue;
        }
        uint32_t s = 0;
        while (s + 1 < world && static_cast<int64_t>(q) >= s_off[s + 1]) ++s;
        const int64_t j = static_cast<int64_t>(q) - s_off[s];
        int32_t pair = 0;
        if (lane == 0) pair = reinterpret_cast<const int32_t *>(peer_sp[s])[s_first[s] + j];
        pair = __shfl_sync(0xffffffffu, pair, 0);
        const uint4 *src = reinterpret_cast<const uint4 *>(peer_x[s]) +
                           (static_cast<uint64_t>(pair) / k) * hv;
        uint4 *dst = recv + q * hv;
        uint32_t c = lane;
        for (; c + 7 * 32 < hv; c += 8 * 32) {
            uint4 v[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) v[b] = __ldcg(src + c + b * 32);
#pragma unroll
            for (int b = 0; b < 8; ++b) dst[c + b * 32] = v[b];
        }
        for (; c < hv; c += 32) dst[c] = __ldcg(src + c);
    }
}

// TMA variant of the dispatch: one issuing thread per CTA streams rows
// through a ring of kRing shared-memory row buffers — bulk load of the token's
// row from local HBM, then bulk store straight into the destination rank's
// receive buffer (large NVLink transactions, no per-lane stores). Rows are
// dealt round-robin over the CTAs; loads run kRing-1 rows ahead.
constexpr int kRing = 8;
__global__ void __launch_bounds__(32) k_dispatch_p2p_tma(const uint8_t *X, const int32_t *sorted_pairs,
                                                         uint64_t n, uint32_t k, uint32_t row_bytes,
                                                         const int64_t *C, const int64_t *ko,
                                                         uint32_t span, uint32_t world, uint32_t me,
                                                         const uint64_t *peer_recv, uint64_t cap,
                                                         uint32_t *err) {
    extern __shared__ __align__(128) uint8_t s_buf[];  // [kRing][row_bytes]
    __shared__ P2PMap m;
    __shared__ __align__(8) uint64_t bars[kRing];
    if (threadIdx.x != 0) return;
    p2p_map(C, ko, span, world, me, m);
    for (int i = 0; i < kRing; ++i) ptx::mbar_init(&bars[i], 1);
    ptx::fence_barrier_init();
    const uint64_t first = blockIdx.x, step = gridDim.x;
    const uint64_t cnt = first < n ? (n - first + step - 1) / step : 0;
    // rotated start: this rank's rows for rank me+1 first, so the ranks do not
    // all push into the same destination at once (one hot NVLink port)
    const uint64_t rot = static_cast<uint64_t>(m.first[(me + 1) % world]) % n;
    auto row_of = [&](uint64_t j) {
        const uint64_t i = first + j * step + rot;
        return i >= n ? i - n : i;
    };
    auto load = [&](uint64_t j) {
        const int slot = static_cast<int>(j % kRing);
        const uint64_t tok = static_cast<uint64_t>(sorted_pairs[row_of(j)]) / k;
        ptx::mbar_arrive_expect_tx(&bars[slot], row_bytes);
        ptx::bulk_load(s_buf + static_cast<size_t>(slot) * row_bytes, X + tok * row_bytes, row_bytes,
                       &bars[slot]);
    };
    for (uint64_t j = 0; j < cnt && j < kRing; ++j) load(j);
    for (uint64_t j = 0; j < cnt; ++j) {
        const int slot = static_cast<int>(j % kRing);
        ptx::mbar_wait(&bars[slot], static_cast<uint32_t>((j / kRing) & 1));
        const uint64_t i = row_of(j);
        const uint32_t r = rank_of_pos(m, world, static_cast<int64_t>(i));
        const uint64_t row = static_cast<uint64_t>(m.base[r] + static_cast<int64_t>(i) - m.first[r]);
        if (row < cap) {
            ptx::bulk_store(reinterpret_cast<uint8_t *>(peer_recv[r]) + row * row_bytes,
                            s_buf + static_cast<size_t>(slot) * row_bytes, row_bytes);
        } else {
            atomicOr(err, kErrCapacity);
        }
        ptx::bulk_commit();
        if (j >= 1 && j - 1 + kRing < cnt) {
            ptx::bulk_wait_read<1>();  // row j-1's store has left its buffer
            load(j - 1 + kRing);
        }
    }
    ptx::bulk_wait<0>();  // every store complete before the CTA exits
}

// Return leg, pushed: every row this rank received goes back to its source
// rank s, into s's symmetric `back` buffer at the row's position in s's
// sorted order (s's slice for this rank starts at sum_{r'<me} C[s][r']).
// Remote stores only; the source then combines from local memory.
__global__ void __launch_bounds__(256) k_return_p2p(const uint4 *recv, uint64_t rows,
                                                    uint32_t hv, const int64_t *C,
                                                    uint32_t world, uint32_t me,
                                                    const uint64_t *peer_back) {
    __shared__ int64_t s_base[9];   // first recv row from source s (s <= world)
    __shared__ int64_t s_first[8];  // where this rank's slice starts in s's order
    if (threadIdx.x == 0) {
        int64_t b = 0;
        for (uint32_t q = 0; q < world; ++q) {
            s_base[q] = b;
            b += C[q * world + me];
            int64_t f = 0;
            for (uint32_t r = 0; r < me; ++r) f += C[q * world + r];
            s_first[q] = f;
        }
        s_base[world] = b;
    }
    __syncthreads();
    const uint64_t row0 = static_cast<uint64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    const uint64_t total = static_cast<uint64_t>(s_base[world]);
    if (row0 >= rows || row0 >= total) return;
    // rotated start: rows of source me+1 first (no single hot destination)
    const uint64_t rot = static_cast<uint64_t>(s_base[(me + 1) % world]) % total;
    const uint64_t row = row0 + rot >= total ? row0 + rot - total : row0 + rot;
    if (row >= rows) return;  // capacity overflow (dispatch flagged kErrCapacity)
    const uint32_t lane = threadIdx.x & 31;
    uint32_t q = 0;
    while (q + 1 < world && static_cast<int64_t>(row) >= s_base[q + 1]) ++q;
    const uint64_t pos = static_cast<uint64_t>(s_first[q] + static_cast<int64_t>(row) - s_base[q]);
    const uint4 *src = recv + row * hv;
    uint4 *dst = reinterpret_cast<uint4 *>(peer_back[q]) + pos * hv;
    for (uint32_t c = lane; c < hv; c += 32) dst[c] = src[c];
}

}  // namespace
}  // namespace mpb

using namespace mpb;

extern "C" {

mpb_status mpb_dispatch_gather(mpb_context *ctx, const void *X, const int32_t *sorted_pairs,
                               uint64_t n_pairs, uint32_t k, uint32_t H, void *send) {
    if (!ctx || (n_pairs && (!X || !sorted_pairs || !send)))
        return fail(MPB_VALIDATION_ERROR, "mpb_dispatch_gather: NULL argument");
    if (H % 8 != 0 || k == 0) return fail(MPB_CONFIG_ERROR, "mpb_dispatch_gather: need H % 8 == 0, k >= 1");
    if (n_pairs == 0) return MPB_OK;
    k_gather<<<static_cast<unsigned>((n_pairs + 7) / 8), 256, 0, ctx->stream>>>(
        static_cast<const uint4 *>(X), sorted_pairs, n_pairs, k, H / 8, static_cast<uint4 *>(send));
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

mpb_status mpb_combine_scatter(mpb_context *ctx, const void *recv, const int32_t *pair_pos,
                               const float *weights, uint64_t T, uint32_t k, uint32_t H, void *Y) {
    if (!ctx || (T && (!recv || !pair_pos || !weights || !Y)))
        return fail(MPB_VALIDATION_ERROR, "mpb_combine_scatter: NULL argument");
    if (H % 8 != 0 || k == 0) return fail(MPB_CONFIG_ERROR, "mpb_combine_scatter: need H % 8 == 0, k >= 1");
    if (T == 0) return MPB_OK;
    k_combine<<<static_cast<unsigned>((T + 7) / 8), 256, 0, ctx->stream>>>(
        static_cast<const uint4 *>(recv), pair_pos, weights, T, k, H / 8, static_cast<uint4 *>(Y));
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

mpb_status mpb_a2a_put_counts(mpb_context *ctx, const int64_t *key_offsets, uint32_t span,
                              uint32_t world, uint32_t rank, const uint64_t *peer_counts) {
    if (!ctx || !key_offsets || !peer_counts)
        return fail(MPB_VALIDATION_ERROR, "mpb_a2a_put_counts: NULL argument");
    if (world < 1 || world > 8 || rank >= world)
        return fail(MPB_CONFIG_ERROR, "mpb_a2a_put_counts: need 1 <= world <= 8, rank < world");
    k_put_counts<<<1, 64, 0, ctx->stream>>>(key_offsets, span, world, rank, peer_counts);
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

mpb_status mpb_dispatch_p2p(mpb_context *ctx, const void *X, const int32_t *sorted_pairs,
                            uint64_t n_pairs, uint32_t k, uint32_t H, const int64_t *counts,
                            const int64_t *key_offsets, uint32_t span, uint32_t world,
                            uint32_t rank, const uint64_t *peer_recv, uint64_t capacity_rows) {
    if (!ctx || !counts || !key_offsets || !peer_recv || (n_pairs && (!X || !sorted_pairs)))
        return fail(MPB_VALIDATION_ERROR, "mpb_dispatch_p2p: NULL argument");
    if (H % 8 != 0 || k == 0) return fail(MPB_CONFIG_ERROR, "mpb_dispatch_p2p: need H % 8 == 0, k >= 1");
    if (world < 1 || world > 8 || rank >= world)
        return fail(MPB_CONFIG_ERROR, "mpb_dispatch_p2p: need 1 <= world <= 8, rank < world");
    if (n_pairs == 0) return MPB_OK;
    static const bool tma = [] {
        const char *v = std::getenv("MPB_P2P_TMA");
        return !(v && v[0] == '0');
    }();
    const size_t row_bytes = size_t(H) * 2;
    if (tma && (reinterpret_cast<uintptr_t>(X) & 15) == 0 && kRing * row_bytes <= 200 * 1024) {
        const size_t smem = kRing * row_bytes;
        MPB_CUDA(cudaFuncSetAttribute(k_dispatch_p2p_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(smem)));
        const unsigned ctas = static_cast<unsigned>(std::min<uint64_t>(n_pairs, ctx->num_sms * 2ull));
        k_dispatch_p2p_tma<<<ctas, 32, smem, ctx->stream>>>(
            static_cast<const uint8_t *>(X), sorted_pairs, n_pairs, k, static_cast<uint32_t>(row_bytes),
            counts, key_offsets, span, world, rank, peer_recv, capacity_rows, ctx->d_error);
        MPB_LAUNCHED(ctx);
        return MPB_OK;
    }
    k_dispatch_p2p<<<static_cast<unsigned>((n_pairs + 7) / 8), 256, 0, ctx->stream>>>(
        static_cast<const uint4 *>(X), sorted_pairs, n_pairs, k, H / 8, counts, key_offsets, span,
        world, rank, peer_recv, capacity_rows, ctx->d_error);
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

mpb_status mpb_dispatch_pull(mpb_context *ctx, const int64_t *counts, const uint64_t *peer_x,
                             const uint64_t *peer_sorted_pairs, const uint64_t *peer_key_offsets,
                             uint32_t k, uint32_t H, uint32_t span, uint32_t world, uint32_t rank,
                             void *recv, uint64_t capacity_rows) {
    if (!ctx || !counts || !peer_x || !peer_sorted_pairs || !peer_key_offsets || !recv)
        return fail(MPB_VALIDATION_ERROR, "mpb_dispatch_pull: NULL argument");
    if (H % 8 != 0 || k == 0) return fail(MPB_CONFIG_ERROR, "mpb_dispatch_pull: need H % 8 == 0, k >= 1");
    if (world < 1 || world > 8 || rank >= world)
        return fail(MPB_CONFIG_ERROR, "mpb_dispatch_pull: need 1 <= world <= 8, rank < world");
    k_dispatch_pull<<<static_cast<unsigned>(ctx->num_sms) * 4, 256, 0, ctx->stream>>>(
        counts, peer_x, peer_sorted_pairs, peer_key_offsets, k, H / 8, span, world, rank,
        static_cast<uint4 *>(recv), capacity_rows, ctx->d_error);
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

mpb_status mpb_combine_p2p(mpb_context *ctx, const int32_t *pair_pos, const float *weights,
                           uint64_t T, uint32_t k, uint32_t H, const int64_t *counts,
                           const int64_t *key_offsets, uint32_t span, uint32_t world,
                           uint32_t rank, const uint64_t *peer_recv, void *Y) {
    if (!ctx || !counts || !key_offsets || !peer_recv || (T && (!pair_pos || !weights || !Y)))
        return fail(MPB_VALIDATION_ERROR, "mpb_combine_p2p: NULL argument");
    if (H % 8 != 0 || k == 0) return fail(MPB_CONFIG_ERROR, "mpb_combine_p2p: need H % 8 == 0, k >= 1");
    if (world < 1 || world > 8 || rank >= world)
        return fail(MPB_CONFIG_ERROR, "mpb_combine_p2p: need 1 <= world <= 8, rank < world");
    if (T == 0) return MPB_OK;
    k_combine_p2p<<<static_cast<unsigned>((T + 7) / 8), 256, 0, ctx->stream>>>(
        pair_pos, weights, T, k, H / 8, counts, key_offsets, span, world, rank, peer_recv,
        static_cast<uint4 *>(Y));
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

mpb_status mpb_return_p2p(mpb_context *ctx, const void *recv, uint64_t recv_rows, uint32_t H,
                          const int64_t *counts, uint32_t world, uint32_t rank,
                          const uint64_t *peer_back) {
    if (!ctx || !recv || !counts || !peer_back)
        return fail(MPB_VALIDATION_ERROR, "mpb_return_p2p: NULL argument");
    if (H % 8 != 0) return fail(MPB_CONFIG_ERROR, "mpb_return_p2p: need H % 8 == 0");
    if (world < 1 || world > 8 || rank >= world)
        return fail(MPB_CONFIG_ERROR, "mpb_return_p2p: need 1 <= world <= 8, rank < world");
    if (recv_rows == 0) return MPB_OK;
    k_return_p2p<<<static_cast<unsigned>((recv_rows + 7) / 8), 256, 0, ctx->stream>>>(
        static_cast<const uint4 *>(recv), recv_rows, H / 8, counts, world, rank, peer_back);
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

}  // extern "C"
