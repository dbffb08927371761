// K6 (local halves): bf16 hidden-state gather into the dispatch send buffer
// and weighted combine back into token order, both driven by the K3
// permutation. Between them the host runs the all-to-all (NCCL) with the
// per-destination counts from key_offsets. One warp per row, 16-byte vector
// loads/stores; combine accumulates the k rows of a token in fp32 in a fixed
// order (deterministic, no atomics).
#include <cuda_bf16.h>

#include "internal.cuh"

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

}  // extern "C"
