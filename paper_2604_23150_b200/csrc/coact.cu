// K4: expert x expert co-activation via warp-ballot expert masks + popc.
//
// C[i][j] = #tokens whose top-k holds both i and j. For every group of 32
// tokens the CTA needs one 32-bit mask per expert (bit u set when token u
// picked that expert) — a ballot over the token group. It is built without
// atomics: warp w takes token group w (lane = token), each lane sets its k
// picks in E/32 register words, and a 5-step shuffle butterfly transposes each
// 32x32 bit block so lane b ends up holding the ballot mask of expert
// 32*word + b (one coalesced smem store per word). Then C[i][j] +=
// popc(m_i & m_j): each thread owns one 8x8 tile of the upper triangle in 64
// registers and streams the masks of all its CTA's token groups. Tiles are
// split evenly over grid.x, tokens over grid.y; per-chunk tiles are stored as
// plain u32 partials (no global atomics) and k_coact_reduce folds them into
// the symmetric uint64 matrix.
// Work: E^2/2 AND+POPC+ADD per 32 tokens (POPC-bound); HBM: T*k*4 bytes.
// (No reference implementation: the closest analogue is aggregate_usage,
// /root/reference/proj/core/src/placement.cpp:96-125.)
#include "internal.cuh"

namespace mpb {
namespace {

constexpr int kGroups = 8;     // 32-token groups per shared-memory round (256 tokens)
constexpr int kMaxWords = 32;  // E8 <= 1024

__device__ __forceinline__ void tile_of(uint32_t t, uint32_t NB, uint32_t &ib, uint32_t &jb) {
    // row-major enumeration of ib <= jb
    uint32_t i = 0, rem = t;
    while (rem >= NB - i) {
        rem -= NB - i;
        ++i;
    }
    ib = i;
    jb = i + rem;
}

// Lane r holds row r of a 32x32 bit matrix (bit c = element (r, c)); after
// the butterfly lane c holds column c (bit r = element (r, c)).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, uint32_t lane) {
    const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const uint32_t s = 16u >> i, M = masks[i];
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
        x = (lane & s) ? ((x & ~M) | ((y & ~M) >> s)) : ((x & M) | ((y & M) << s));
    }
    return x;
}

template <int WORDS, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) k_coact_partial(const int32_t *idx, uint64_t T, uint32_t k, uint32_t NT,
                                uint32_t tiles_per_cta, uint64_t tpc, uint32_t *partials) {
    constexpr uint32_t E8 = WORDS * 32;
    extern __shared__ uint32_t s_mask_all[];  // [2][kGroups][E8] double-buffered
    const uint32_t NB = E8 / 8;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tile = blockIdx.x * tiles_per_cta + threadIdx.x;
    const bool has_tile = threadIdx.x < tiles_per_cta && tile < NT;
    uint32_t ib = 0, jb = 0;
    if (has_tile) tile_of(tile, NB, ib, jb);
    uint32_t acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0;

    const uint64_t t0 = static_cast<uint64_t>(blockIdx.y) * tpc;
    const uint64_t t1 = min(T, t0 + tpc);
    uint32_t buf = 0;
    for (uint64_t tb = t0; tb < t1; tb += kGroups * 32, buf ^= 1) {
        uint32_t *s_mask = s_mask_all + buf * kGroups * E8;
        // ---- masks: warp g builds token group g (lane = token); the other
        // buffer may still be read by slower tile owners of the previous round
        // (one barrier per round suffices)
        for (uint32_t g = warp; g < kGroups; g += blockDim.x / 32) {
            const uint64_t t = tb + g * 32 + lane;
            uint32_t words[WORDS];
#pragma unroll
            for (int w = 0; w < WORDS; ++w) words[w] = 0;
            if (t < t1) {
                // issue all of the token's loads before using any (k <= 16 here;
                // larger k falls through to the tail loop)
                const int32_t *x = idx + t * k;
                int32_t ev[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) ev[j] = j < static_cast<int>(k) ? __ldg(x + j) : -1;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int32_t e = ev[j];
                    if (e < 0 || static_cast<uint32_t>(e) >= E8) continue;
#pragma unroll
                    for (int w = 0; w < WORDS; ++w)
                        words[w] |= (static_cast<uint32_t>(e) >> 5) == static_cast<uint32_t>(w)
                                        ? (1u << (e & 31))
                                        : 0u;
                }
                for (uint32_t j = 16; j < k; ++j) {
                    const int32_t e = __ldg(x + j);
                    if (e < 0 || static_cast<uint32_t>(e) >= E8) continue;
#pragma unroll
                    for (int w = 0; w < WORDS; ++w)
                        words[w] |= (static_cast<uint32_t>(e) >> 5) == static_cast<uint32_t>(w)
                                        ? (1u << (e & 31))
                                        : 0u;
                }
            }
#pragma unroll
            for (int w = 0; w < WORDS; ++w)
                s_mask[g * E8 + w * 32 + lane] = transpose32(words[w], lane);
        }
        __syncthreads();
        if (has_tile) {
#pragma unroll 2
            for (int g = 0; g < kGroups; ++g) {
                const uint4 *mi = reinterpret_cast<const uint4 *>(s_mask + g * E8 + ib * 8);
                const uint4 *mj = reinterpret_cast<const uint4 *>(s_mask + g * E8 + jb * 8);
                const uint4 a0 = mi[0], a1 = mi[1], b0 = mj[0], b1 = mj[1];
                const uint32_t A[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const uint32_t Bm[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int b = 0; b < 8; ++b) acc[a][b] += __popc(A[a] & Bm[b]);
            }
        }
    }
    if (has_tile) {
        uint4 *out = reinterpret_cast<uint4 *>(
            partials + (static_cast<size_t>(blockIdx.y) * NT + tile) * 64);
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            out[a * 2] = make_uint4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
            out[a * 2 + 1] = make_uint4(acc[a][4], acc[a][5], acc[a][6], acc[a][7]);
        }
    }
}

__global__ void k_coact_reduce(const uint32_t *partials, uint32_t chunks, uint32_t NT, uint32_t E,
                               uint32_t E8, uint64_t *coact) {
    const uint64_t cell = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (cell >= static_cast<uint64_t>(NT) * 64) return;
    unsigned long long s = 0;
    const uint32_t *p = partials + cell;
    const size_t stride = static_cast<size_t>(NT) * 64;
    uint32_t c = 0;
    for (; c + 8 <= chunks; c += 8) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(p + (c + u) * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; c < chunks; ++c) s += __ldg(p + c * stride);
    const uint32_t tile = static_cast<uint32_t>(cell / 64), ab = static_cast<uint32_t>(cell % 64);
    uint32_t ib, jb;
    tile_of(tile, E8 / 8, ib, jb);
    const uint32_t i = ib * 8 + ab / 8, j = jb * 8 + ab % 8;
    if (i >= E || j >= E) return;
    coact[static_cast<size_t>(i) * E + j] += s;
    if (ib != jb) coact[static_cast<size_t>(j) * E + i] += s;
}

template <int WORDS>
mpb_status launch_partial(mpb_context *ctx, dim3 grid, uint32_t threads, size_t smem,
                          const int32_t *idx, uint64_t T, uint32_t k, uint32_t NT, uint32_t tpcta,
                          uint64_t tpc, uint32_t *partials) {
    // E <= 256: <= 288 threads; larger E: up to 512 threads (one CTA per SM:
    // 64 register accumulators per thread)
    constexpr int MAXT = WORDS <= 8 ? 288 : 512;
    constexpr int MINB = 1;
    auto kern = k_coact_partial<WORDS, MAXT, MINB>;
    MPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<grid, threads, smem, ctx->stream>>>(idx, T, k, NT, tpcta, tpc, partials);
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

}  // namespace
}  // namespace mpb

using namespace mpb;

extern "C" mpb_status mpb_coactivation(mpb_context *ctx, const int32_t *idx, uint64_t T,
                                       uint32_t k, uint32_t E, uint64_t *coact) {
    if (!ctx || !coact || (T && !idx))
        return fail(MPB_VALIDATION_ERROR, "mpb_coactivation: NULL argument");
    if (E == 0 || E > 32 * kMaxWords)
        return fail(MPB_CONFIG_ERROR, "mpb_coactivation: need 1 <= E <= 1024");
    if (T == 0 || k == 0) return MPB_OK;
    const uint32_t words = (E + 31) / 32;
    const uint32_t W = words <= 2 ? 2 : words <= 4 ? 4 : words <= 8 ? 8 : words <= 16 ? 16 : 32;
    const uint32_t E8 = W * 32;
    const uint32_t NB = E8 / 8;
    const uint32_t NT = NB * (NB + 1) / 2;
    // tiles split evenly over G CTAs of <= 512 threads (multiple of 32, >= 8 warps
    // so every token group has its mask-building warp)
    const uint32_t cap = W <= 8 ? 288u : 512u;
    const uint32_t G = (NT + cap - 1) / cap;
    const uint32_t tpcta = (NT + G - 1) / G;
    const uint32_t threads = std::max(256u, (tpcta + 31) / 32 * 32);
    uint64_t chunks = std::max<uint64_t>(1, static_cast<uint64_t>(ctx->num_sms) / G);
    uint64_t tpc = (T + chunks - 1) / chunks;
    tpc = (tpc + 31) / 32 * 32;  // token groups never straddle chunks
    chunks = (T + tpc - 1) / tpc;
    MPB_CUDA(ctx->ensure_scratch(size_t(chunks) * NT * 64 * 4));
    auto *partials = static_cast<uint32_t *>(ctx->scratch);
    const size_t smem = size_t(2) * kGroups * E8 * 4;
    dim3 grid(G, static_cast<uint32_t>(chunks));
    mpb_status st;
    switch (W) {
    case 2: st = launch_partial<2>(ctx, grid, threads, smem, idx, T, k, NT, tpcta, tpc, partials); break;
    case 4: st = launch_partial<4>(ctx, grid, threads, smem, idx, T, k, NT, tpcta, tpc, partials); break;
    case 8: st = launch_partial<8>(ctx, grid, threads, smem, idx, T, k, NT, tpcta, tpc, partials); break;
    case 16: st = launch_partial<16>(ctx, grid, threads, smem, idx, T, k, NT, tpcta, tpc, partials); break;
    default: st = launch_partial<32>(ctx, grid, threads, smem, idx, T, k, NT, tpcta, tpc, partials); break;
    }
    if (st != MPB_OK) return st;
    const uint64_t cells = uint64_t(NT) * 64;
    k_coact_reduce<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, ctx->stream>>>(
        partials, static_cast<uint32_t>(chunks), NT, E, E8, coact);
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}
