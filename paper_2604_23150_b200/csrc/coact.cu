// K4: expert x expert co-activation.
//
// E <= 256 and k <= 16 (every shape the pipeline runs): tcgen05 kind::i8
// tensor-core kernel k_coact_mma below (C = X^T X over the 0/1 routing
// matrix, exact s32 accumulation). Otherwise the popc kernel described here.
// Top-k ids are distinct per token; ids outside [0, E) are ignored.
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
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"
#include "tc_ptx.cuh"

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

// ---------------------------------------------------------------------------
// Tensor-core path (E <= 256, k <= 16): C = X^T X with X the [T x E] 0/1
// routing matrix, on tcgen05 kind::i8 (u8 x u8 -> s32: exact integer counts).
// Per 128-token chunk the producers build X in shared memory in its natural
// token-major order, as an MN-major SW128 u8 operand: token t's row of
// experts is 128-byte MN blocks (expert e in block e/128), rows grouped by 8
// tokens into 1024-byte swizzle atoms. Each producer thread owns one token:
// it zeroes the token's row (16-byte stores, swizzled so a warp's stores hit
// distinct banks) and sets its k expert bytes — no transposes. One thread
// issues the MMAs (both operands MN-major views of the same tile): the upper
// triangle as tile 0 (experts 0..127 x all) and, when E > 128, tile 1
// (experts 128.. x 128..); both accumulate in TMEM over the CTA's token
// range. The epilogue writes the CTA's u16 partial (upper triangle only;
// <= 65535 tokens per CTA) and k_coact_mma_reduce folds the partials into C.
// Work per 128 tokens: 128*128*(N0+N1) MACs on the tensor pipe; E/16 + k
// shared stores per token; HBM: T*k*4 bytes of ids (+ the partials,
// L2-resident).
constexpr int kMmaStages = 4;
constexpr int kMmaMaxK = 16;
constexpr int kMmaThreads = 320;  // warp 0: TMEM + MMA; warps 1-8: producers + epilogue; 9: ids

template <int WORDS>
__global__ void __launch_bounds__(kMmaThreads, 1)
    k_coact_mma(const int32_t *idx, uint64_t T, uint32_t k, uint32_t E, uint32_t N0, uint32_t N1,
                uint32_t chunks_per_cta, uint32_t *partials, uint64_t *direct) {
    constexpr bool kTwo = WORDS == 8;
    constexpr uint32_t kRows = WORDS * 32;   // experts (padded) = partial row length
    constexpr uint32_t kBlock = 128 * 128;   // one 128-expert MN block of 128 token rows
    constexpr uint32_t kTile = kRows * 128;  // bytes per stage
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    uint8_t *tiles = smem;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kMmaStages * kTile);
    uint64_t *full = bars, *empty = bars + kMmaStages, *idfull = bars + 2 * kMmaStages,
             *idempty = bars + 3 * kMmaStages, *tfull = bars + 4 * kMmaStages;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(tfull + 1);
    int32_t *ring = reinterpret_cast<int32_t *>(bars + 4 * kMmaStages + 2);  // [S][128][k]
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kMmaStages; ++s) {
            ptx::mbar_init(&full[s], 128);
            ptx::mbar_init(&empty[s], 1);
            ptx::mbar_init(&idfull[s], 1);
            ptx::mbar_init(&idempty[s], 128);
        }
        ptx::mbar_init(tfull, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<kTwo ? 512 : 256>(s_tmem);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *s_tmem;
    pdl_trigger();
    pdl_wait();  // ids (previous kernels) and the partials buffer (WAR) from here on

    const uint64_t tok0 = static_cast<uint64_t>(blockIdx.x) * chunks_per_cta * 128;
    const uint64_t tok1 = min(T, tok0 + static_cast<uint64_t>(chunks_per_cta) * 128);
    const uint32_t nch = tok0 < tok1 ? static_cast<uint32_t>((tok1 - tok0 + 127) / 128) : 0;

    if (warp == 0) {
        if (lane == 0 && nch) {
            const uint32_t id0 = ptx::idesc_u8_s32_mn(128, N0);
            const uint32_t id1 = ptx::idesc_u8_s32_mn(128, N1);
            for (uint32_t n = 0; n < nch; ++n) {
                const uint32_t s = n % kMmaStages;
                ptx::mbar_wait(&full[s], (n / kMmaStages) & 1);
                ptx::tc_fence_after();
                const uint32_t base = ptx::smem_u32(tiles + s * kTile);
#pragma unroll
                for (uint32_t kk = 0; kk < 4; ++kk) {  // K = 32 tokens per MMA
                    const uint32_t acc = (n | kk) != 0;
                    // K = 32 tokens = 4 swizzle atoms of 8 token rows
                    const uint64_t d0 = ptx::sw128_mnmajor_desc(base + kk * 4096, kBlock);
                    ptx::mma_u8(tmem, d0, d0, id0, acc);
                    if (kTwo) {
                        const uint64_t d1 = ptx::sw128_mnmajor_desc(base + kBlock + kk * 4096, kBlock);
                        ptx::mma_u8(tmem + 256, d1, d1, id1, acc);
                    }
                }
                ptx::mma_commit(&empty[s]);
            }
            ptx::mma_commit(tfull);
        }
        __syncwarp();
    } else if (warp == 9) {
        // ids loader: chunk n's [ntok x k] int32 block -> ring slot n % S with
        // one bulk copy (async proxy; the sub-16-byte tail by plain copies)
        if (lane == 0) {
            const bool aligned = (reinterpret_cast<uintptr_t>(idx) & 15) == 0;
            for (uint32_t n = 0; n < nch; ++n) {
                const uint32_t s = n % kMmaStages;
                if (n >= kMmaStages) ptx::mbar_wait(&idempty[s], ((n / kMmaStages) - 1) & 1);
                // the producers' generic reads of this slot (ordered by the idempty
                // barrier) must also be ordered before the async-proxy bulk write
                // that overwrites it: without this proxy fence a bulk copy can land
                // under a producer still reading the previous chunk's ids
                ptx::fence_proxy_async_smem();
                const uint64_t t = tok0 + static_cast<uint64_t>(n) * 128;
                const uint32_t ntok = static_cast<uint32_t>(min(static_cast<uint64_t>(128), tok1 - t));
                const uint32_t bytes = ntok * k * 4;
                const uint32_t bulk = aligned ? bytes & ~15u : 0;
                const int32_t *src = idx + t * k;
                int32_t *dst = ring + s * 128 * k;
                for (uint32_t i = bulk / 4; i < bytes / 4; ++i) dst[i] = __ldg(src + i);
                ptx::mbar_arrive_expect_tx(&idfull[s], bulk);
                if (bulk) ptx::bulk_load(dst, src, bulk, &idfull[s]);
            }
        }
        __syncwarp();
    } else {
        const uint32_t pw = warp - 1, set = pw >> 2, g = pw & 3;
        const uint32_t u = g * 32 + lane;  // token within the chunk
        for (uint32_t n = set; n < nch; n += 2) {
            const uint32_t s = n % kMmaStages;
            const uint32_t tile = ptx::smem_u32(tiles + s * kTile);
            ptx::mbar_wait(&idfull[s], (n / kMmaStages) & 1);  // this chunk's ids landed
            int32_t ids[kMmaMaxK];
            const bool ok = tok0 + static_cast<uint64_t>(n) * 128 + u < tok1;
            {
                const uint32_t ids_s = ptx::smem_u32(ring + (s * 128 + u) * k);
#pragma unroll
                for (int j = 0; j < kMmaMaxK; ++j) {
                    ids[j] = -1;
                    if (ok && j < static_cast<int>(k))
                        asm volatile("ld.shared.s32 %0, [%1];" : "=r"(ids[j]) : "r"(ids_s + 4 * j) : "memory");
                }
            }
            ptx::mbar_arrive(&idempty[s]);
            if (n >= kMmaStages) ptx::mbar_wait(&empty[s], ((n / kMmaStages) - 1) & 1);
            // token u's row: (u/8)*1024 + (u%8)*128 in each MN block; 16-byte
            // chunk c of the row lives at physical chunk c ^ (u%8)
            const uint32_t row = tile + (u >> 3) * 1024 + (u & 7) * 128;
            {
#pragma unroll
                for (int b = 0; b < (kTwo ? 2 : 1); ++b)
#pragma unroll
                    for (uint32_t c = 0; c < 8; ++c)
                        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(
                                         row + b * kBlock + ((c ^ (u & 7)) << 4)),
                                     "r"(0u)
                                     : "memory");
#pragma unroll
                for (int j = 0; j < kMmaMaxK; ++j) {
                    const uint32_t e = static_cast<uint32_t>(ids[j]);
                    if (e < E)
                        asm volatile("st.shared.u8 [%0], %1;" ::"r"(
                                         row + (e >> 7) * kBlock + ((((e >> 4) & 7) ^ (u & 7)) << 4) +
                                         (e & 15)),
                                     "r"(1u)
                                     : "memory");
                }
            }
            ptx::fence_proxy_async_smem();
            ptx::mbar_arrive(&full[s]);
        }
        // ---- epilogue: TMEM lane quarter (warp % 4) holds tile rows 32*(warp%4) + lane;
        // the two warp sets take alternate 32-column slices
        if (nch) {
            ptx::mbar_wait(tfull, 0);
            ptx::tc_fence_after();
            const uint32_t q = warp & 3, r = q * 32 + lane;
            uint16_t *out = reinterpret_cast<uint16_t *>(partials) +
                            static_cast<size_t>(blockIdx.x) * kRows * kRows;
            auto dump = [&](uint32_t tcol, uint32_t orow, uint32_t ocol) {
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(tmem + ((q * 32) << 16) + tcol, v);
                ptx::tmem_ld_wait();
                if (direct) {  // few CTAs (decode batches): straight into C, no reduce launch
                    if (orow >= E) return;
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const uint32_t col = ocol + i;
                        if (!v[i] || col < orow || col >= E) continue;
                        atomicAdd(reinterpret_cast<unsigned long long *>(direct) + size_t(orow) * E + col,
                                  static_cast<unsigned long long>(v[i]));
                        if (col != orow)
                            atomicAdd(reinterpret_cast<unsigned long long *>(direct) + size_t(col) * E + orow,
                                      static_cast<unsigned long long>(v[i]));
                    }
                    return;
                }
                uint4 *o = reinterpret_cast<uint4 *>(out + static_cast<size_t>(orow) * kRows + ocol);
#pragma unroll
                for (int w = 0; w < 4; ++w)
                    o[w] = make_uint4(v[8 * w] | (v[8 * w + 1] << 16),
                                          v[8 * w + 2] | (v[8 * w + 3] << 16),
                                          v[8 * w + 4] | (v[8 * w + 5] << 16),
                                          v[8 * w + 6] | (v[8 * w + 7] << 16));
            };
            // tile 0: row r, cols >= the quarter's first row
            for (uint32_t c = q * 32 + set * 32; c < N0; c += 64) dump(c, r, c);
            if (kTwo)  // tile 1: row 128 + r, col 128 + c
                for (uint32_t c = q * 32 + set * 32; c < N1; c += 64) dump(256 + c, 128 + r, 128 + c);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<kTwo ? 512 : 256>(tmem);
}

constexpr uint64_t kDirectMaxCtas = 32;  // direct-to-C epilogue up to this many CTAs (4,096 tokens: 1 chunk each)

// Row i of C (one CTA of 8 warps per row): warp w sums partials w, w+8, ...
// with lane L owning columns 8L..8L+7 (coalesced 16-byte loads, 8 in flight);
// the warps' sums meet in shared memory; C[i][j] and C[j][i] += sum, j >= i.
__global__ void __launch_bounds__(256) k_coact_mma_reduce(const uint32_t *partials, uint32_t ctas,
                                                          uint32_t E, uint32_t kRows,
                                                          uint64_t *coact) {
    __shared__ uint32_t s_red[8][256];
    pdl_trigger();
    pdl_wait();
    const uint32_t i = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t pstride = static_cast<size_t>(kRows) * kRows / 8;  // uint4 per partial
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (8 * lane < kRows && 8 * lane + 7 >= i) {
        const uint4 *p = reinterpret_cast<const uint4 *>(partials) +
                         (static_cast<size_t>(i) * kRows) / 8 + lane;
        for (uint32_t c0 = w; c0 < ctas; c0 += 64) {
            uint4 v[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const uint32_t c = c0 + 8 * b;
                v[b] = c < ctas ? __ldg(p + c * pstride) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                acc[0] += v[b].x & 0xFFFFu;
                acc[1] += v[b].x >> 16;
                acc[2] += v[b].y & 0xFFFFu;
                acc[3] += v[b].y >> 16;
                acc[4] += v[b].z & 0xFFFFu;
                acc[5] += v[b].z >> 16;
                acc[6] += v[b].w & 0xFFFFu;
                acc[7] += v[b].w >> 16;
            }
        }
    }
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) s_red[w][(8 * lane + jj) & 255] = acc[jj];
    __syncthreads();
    const uint32_t j = threadIdx.x;
    if (j >= i && j < E) {
        uint32_t sum = 0;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) sum += s_red[ww][j];
        coact[static_cast<size_t>(i) * E + j] += sum;
        if (i != j) coact[static_cast<size_t>(j) * E + i] += sum;
    }
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
    static const bool force_popc = std::getenv("MPB_COACT_POPC") != nullptr;
    if (E <= 256 && k <= static_cast<uint32_t>(kMmaMaxK) && !force_popc) {
        const bool two = E > 128;
        const uint32_t E16 = (E + 15) / 16 * 16;
        const uint32_t N0 = E16, N1 = two ? E16 - 128 : 0;
        const uint32_t E8 = two ? 256 : 128;
        const size_t smem = 1024 + size_t(kMmaStages) * E8 * 128 + (4 * kMmaStages + 2) * 8 +
                            size_t(kMmaStages) * 128 * k * 4;
        auto kern = two ? k_coact_mma<8> : k_coact_mma<4>;
        MPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        // one CTA per SM at most, >= 2 chunks of 128 tokens each;
        // u16 partials need <= 511 chunks per CTA: longer inputs take several
        // launches, each accumulating into C
        // (decode-size batches that fit the direct epilogue: one chunk per CTA)
        static const char *env = std::getenv("MPB_COACT_CHUNKS_PER_CTA");
        const uint64_t want = env ? std::max(1, std::atoi(env)) : ((T + 127) / 128 <= kDirectMaxCtas ? 1 : 2);
        const uint64_t max_tokens = uint64_t(ctx->num_sms) * 511 * 128;
        for (uint64_t t0 = 0; t0 < T; t0 += max_tokens) {
            const uint64_t Tn = std::min<uint64_t>(max_tokens, T - t0);
            const uint64_t chunks = (Tn + 127) / 128;
            uint64_t ctas = std::min<uint64_t>(ctx->num_sms, std::max<uint64_t>(1, chunks / want));
            const uint64_t cpc = (chunks + ctas - 1) / ctas;
            ctas = (chunks + cpc - 1) / cpc;
            // a few CTAs (decode-size batches): each adds its upper triangle
            // straight into C with 64-bit atomics (integer sums: the same C),
            // no partials and no reduce launch (MPB_COACT_DIRECT=0: off)
            const char *denv = std::getenv("MPB_COACT_DIRECT");
            const bool direct = ctas <= kDirectMaxCtas && !(denv && denv[0] == '0');
            uint32_t *partials = nullptr;
            if (!direct) {
                MPB_CUDA(ctx->ensure_scratch(size_t(ctas) * E8 * E8 * 2));
                partials = static_cast<uint32_t *>(ctx->scratch);
            }
            MPB_CUDA(launch_pdl(kern, dim3(static_cast<unsigned>(ctas)), dim3(kMmaThreads), smem,
                                ctx->stream, idx + t0 * k, Tn, k, E, N0, N1,
                                static_cast<uint32_t>(cpc), partials, direct ? coact : nullptr));
            MPB_LAUNCHED(ctx);
            if (direct) continue;
            MPB_CUDA(launch_pdl(k_coact_mma_reduce, dim3(E), dim3(256), 0, ctx->stream, partials,
                                static_cast<uint32_t>(ctas), E, E8, coact));
            MPB_LAUNCHED(ctx);
        }
        return MPB_OK;
    }
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
