// Top-k over materialised fp32 logits (one warp per token).
//
// Selection order: larger logit first, equal logits -> lower expert id, NaN
// below everything — the reference's "lowest index wins" rule (strict
// compares + std::stable_sort, /root/reference/proj/core/src/placement.cpp:
// 143-152, clustering.cpp:113-120). Each lane holds E/32 logits in registers;
// k rounds of a warp-wide (value, id) arg-max pick the winners. Softmax is
// over all E logits (max-subtracted, fp32), sigmoid is per pick.
#include <cfloat>

#include "internal.cuh"

namespace mpb {

__device__ __forceinline__ bool topk_beats(float a, uint32_t ia, float b, uint32_t ib) {
    const bool na = isnan(a), nb = isnan(b);
    if (na || nb) return (na && nb) ? ia < ib : nb;
    if (a != b) return a > b;
    return ia < ib;
}

namespace {

template <int VPL>
__global__ void __launch_bounds__(256) k_topk_logits(const float *logits, uint64_t T, uint32_t E,
                                                     uint32_t k, int score_fn, int renorm,
                                                     int32_t *idx_out, float *w_out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (t >= T) return;
    const float *x = logits + t * E;
    float v[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
        const uint32_t e = lane + 32u * i;
        v[i] = e < E ? __ldg(x + e) : -INFINITY;
    }
    uint32_t taken = 0;
#pragma unroll
    for (int i = 0; i < VPL; ++i)
        if (lane + 32u * i >= E) taken |= 1u << i;
    float wsel[16];
    int32_t isel[16];
    for (uint32_t r = 0; r < k; ++r) {
        float bv = NAN;
        uint32_t bi = 0xFFFFFFFFu;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
            if (taken & (1u << i)) continue;
            const uint32_t e = lane + 32u * i;
            if (bi == 0xFFFFFFFFu || topk_beats(v[i], e, bv, bi)) {
                bv = v[i];
                bi = e;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oi != 0xFFFFFFFFu && (bi == 0xFFFFFFFFu || topk_beats(ov, oi, bv, bi))) {
                bv = ov;
                bi = oi;
            }
        }
        if (bi != 0xFFFFFFFFu && (bi & 31u) == lane) taken |= 1u << (bi >> 5);
        wsel[r] = bv;
        isel[r] = static_cast<int32_t>(bi);
    }
    float w[16];
    if (score_fn == MPB_SCORE_SOFTMAX) {
        float m = -INFINITY;
#pragma unroll
        for (int i = 0; i < VPL; ++i)
            if (!isnan(v[i])) m = fmaxf(m, v[i]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < VPL; ++i)
            if (!isnan(v[i]) && lane + 32u * i < E) s += expf(v[i] - m);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        for (uint32_t r = 0; r < k; ++r) w[r] = isnan(wsel[r]) ? 0.f : expf(wsel[r] - m) / s;
    } else {
        for (uint32_t r = 0; r < k; ++r)
            w[r] = isnan(wsel[r]) ? 0.f : 1.f / (1.f + expf(-wsel[r]));
    }
    if (renorm) {
        float s = 0.f;
        for (uint32_t r = 0; r < k; ++r) s += w[r];
        for (uint32_t r = 0; r < k; ++r) w[r] = s > 0.f ? w[r] / s : 0.f;
    }
    for (uint32_t r = lane; r < k; r += 32) {
        // register arrays indexed by a lane-dependent r: pick via shuffle-free select
        float wr = 0.f;
        int32_t ir = 0;
        for (uint32_t q = 0; q < k; ++q)
            if (q == r) {
                wr = w[q];
                ir = isel[q];
            }
        idx_out[t * k + r] = ir;
        w_out[t * k + r] = wr;
    }
}

}  // namespace
}  // namespace mpb

using namespace mpb;

extern "C" mpb_status mpb_topk_logits(mpb_context *ctx, const float *logits, uint64_t T,
                                      uint32_t E, uint32_t k, int score_fn, int renorm,
                                      int32_t *idx, float *weights) {
    if (!ctx || (T && (!logits || !idx || !weights)))
        return fail(MPB_VALIDATION_ERROR, "mpb_topk_logits: NULL argument");
    if (E == 0 || E > 1024) return fail(MPB_CONFIG_ERROR, "mpb_topk_logits: need 1 <= E <= 1024");
    if (k == 0 || k > 16 || k > E)
        return fail(MPB_CONFIG_ERROR, "mpb_topk_logits: need 1 <= k <= min(16, E)");
    if (score_fn != MPB_SCORE_SOFTMAX && score_fn != MPB_SCORE_SIGMOID)
        return fail(MPB_CONFIG_ERROR, "mpb_topk_logits: unknown score_fn");
    if (T == 0) return MPB_OK;
    const unsigned blocks = static_cast<unsigned>((T + 7) / 8);
    const uint32_t vpl = (E + 31) / 32;
#define MPB_TOPK_CASE(V)                                                                         \
    k_topk_logits<V><<<blocks, 256, 0, ctx->stream>>>(logits, T, E, k, score_fn, renorm, idx,  \
                                                      weights)
    if (vpl <= 1) MPB_TOPK_CASE(1);
    else if (vpl <= 2) MPB_TOPK_CASE(2);
    else if (vpl <= 4) MPB_TOPK_CASE(4);
    else if (vpl <= 8) MPB_TOPK_CASE(8);
    else if (vpl <= 16) MPB_TOPK_CASE(16);
    else MPB_TOPK_CASE(32);
#undef MPB_TOPK_CASE
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}
