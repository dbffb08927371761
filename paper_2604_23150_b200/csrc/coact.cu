// K4: expert x expert co-activation via warp-ballot expert masks + popc.
//
// C[i][j] = #tokens whose top-k holds both i and j. For every group of 32
// tokens the CTA builds one 32-bit mask per expert in shared memory (bit u set
// when token u picked that expert — a ballot over the token group), so
// C[i][j] += popc(m_i & m_j). Each thread owns one 8x8 tile of the upper
// triangle in registers (64 accumulators) and streams the masks of all its
// CTA's token groups; tiles are spread over grid.x, tokens over grid.y.
// Per-chunk tiles are written as plain u32 partials (no global atomics) and
// k_coact_reduce folds them into the symmetric uint64 matrix.
// Work: E^2/2 AND+POPC+ADD per 32 tokens; HBM: T*k*4 bytes of idx.
// (No reference implementation: the closest analogue is aggregate_usage,
// /root/reference/proj/core/src/placement.cpp:96-125.)
#include "internal.cuh"

namespace mpb {
namespace {

constexpr int kCoThreads = 128;
constexpr int kGroups = 8;  // 32-token groups per shared-memory round (256 tokens)

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

__global__ void __launch_bounds__(kCoThreads) k_coact_partial(const int32_t *idx, uint64_t T,
                                                              uint32_t k, uint32_t E8,
                                                              uint32_t NT, uint64_t tpc,
                                                              uint32_t *partials) {
    extern __shared__ uint32_t s_mask[];  // [kGroups][E8]
    const uint32_t NB = E8 / 8;
    const uint32_t tile = blockIdx.x * kCoThreads + threadIdx.x;
    const bool has_tile = tile < NT;
    uint32_t ib = 0, jb = 0;
    if (has_tile) tile_of(tile, NB, ib, jb);
    uint32_t acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0;

    const uint64_t t0 = static_cast<uint64_t>(blockIdx.y) * tpc;
    const uint64_t t1 = min(T, t0 + tpc);
    for (uint64_t tb = t0; tb < t1; tb += kGroups * 32) {
        for (uint32_t i = threadIdx.x; i < kGroups * E8; i += kCoThreads) s_mask[i] = 0;
        __syncthreads();
        // ballot: token u of this round sets bit (u % 32) of mask[u / 32][e]
        for (uint32_t u = threadIdx.x; u < kGroups * 32; u += kCoThreads) {
            const uint64_t t = tb + u;
            if (t >= t1) break;
            const int32_t *x = idx + t * k;
            for (uint32_t j = 0; j < k; ++j) {
                const int32_t e = __ldg(x + j);
                if (e >= 0 && static_cast<uint32_t>(e) < E8)
                    atomicOr(s_mask + (u >> 5) * E8 + e, 1u << (u & 31));
            }
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
        __syncthreads();
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
    for (uint32_t c = 0; c < chunks; ++c) s += partials[static_cast<size_t>(c) * NT * 64 + cell];
    const uint32_t tile = static_cast<uint32_t>(cell / 64), ab = static_cast<uint32_t>(cell % 64);
    uint32_t ib, jb;
    tile_of(tile, E8 / 8, ib, jb);
    const uint32_t i = ib * 8 + ab / 8, j = jb * 8 + ab % 8;
    if (i >= E || j >= E) return;
    coact[static_cast<size_t>(i) * E + j] += s;
    if (ib != jb) coact[static_cast<size_t>(j) * E + i] += s;
}

}  // namespace
}  // namespace mpb

using namespace mpb;

extern "C" mpb_status mpb_coactivation(mpb_context *ctx, const int32_t *idx, uint64_t T,
                                       uint32_t k, uint32_t E, uint64_t *coact) {
    if (!ctx || !coact || (T && !idx))
        return fail(MPB_VALIDATION_ERROR, "mpb_coactivation: NULL argument");
    if (E == 0 || E > 1024) return fail(MPB_CONFIG_ERROR, "mpb_coactivation: need 1 <= E <= 1024");
    if (T == 0 || k == 0) return MPB_OK;
    const uint32_t E8 = (E + 7) / 8 * 8;
    const uint32_t NB = E8 / 8;
    const uint32_t NT = NB * (NB + 1) / 2;
    const uint32_t tile_groups = (NT + kCoThreads - 1) / kCoThreads;
    const uint64_t target = 2ull * ctx->num_sms;
    uint64_t chunks = std::max<uint64_t>(1, (target + tile_groups - 1) / tile_groups);
    uint64_t tpc = (T + chunks - 1) / chunks;
    tpc = std::max<uint64_t>(kGroups * 32, (tpc + kGroups * 32 - 1) / (kGroups * 32) * (kGroups * 32));
    chunks = (T + tpc - 1) / tpc;
    if (chunks > 65535) {
        chunks = 65535;
        tpc = (T + chunks - 1) / chunks;
        tpc = (tpc + kGroups * 32 - 1) / (kGroups * 32) * (kGroups * 32);
        chunks = (T + tpc - 1) / tpc;
    }
    MPB_CUDA(ctx->ensure_scratch(size_t(chunks) * NT * 64 * 4));
    auto *partials = static_cast<uint32_t *>(ctx->scratch);
    const size_t smem = size_t(kGroups) * E8 * 4;
    MPB_CUDA(cudaFuncSetAttribute(k_coact_partial, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    dim3 grid(tile_groups, static_cast<uint32_t>(chunks));
    k_coact_partial<<<grid, kCoThreads, smem, ctx->stream>>>(idx, T, k, E8, NT, tpc, partials);
    MPB_LAUNCHED(ctx);
    const uint64_t cells = uint64_t(NT) * 64;
    k_coact_reduce<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, ctx->stream>>>(
        partials, static_cast<uint32_t>(chunks), NT, E, E8, coact);
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}
