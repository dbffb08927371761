// K5: batched placement-cost evaluator (sm_100a).
//
// simulate_layer (/root/reference/proj/core/src/simulator.cpp:43-99) only
// depends on a batch through its demand per (source node, expert): the
// destination of a pair is fixed by (node(src), expert) under a placement
// (simulator.cpp:74-80), bytes are count * hidden * bpe (:57-58, :81), and
// inter/intra is node(dest) != node(src) (:82-85). So P candidates x B batches
// reduce to P*B lookups over a [nodes x E] demand table:
//   k_batch_demand : CSR matrix rows sampled into B batches -> node_demand
//                    (the BatchAssignment assembly of compare_strategies,
//                    simulator.cpp:154-181), smem-privatised counters.
//   k_score        : one CTA per candidate (its LUT in smem), one warp per
//                    batch; integer pair counts per destination rank.
//   k_finalize     : LayerSim doubles with the reference's exact expression
//                    order (:27-41, :90-98), correctly rounded dadd/dmul/ddiv
//                    intrinsics so the result is bit-identical to the host.
// Algorithmic bytes per (candidate, batch): nodes*E*8 (demand) + nodes*E
// (LUT, reused across batches from smem) + (2 + D)*8 out.
#include <cstdlib>

#include "internal.cuh"

namespace mpb {
namespace {

__global__ void __launch_bounds__(256) k_batch_demand(const uint32_t *row_ptr, const uint32_t *cols,
                                                      const uint32_t *vals, uint32_t R,
                                                      const uint32_t *rows, const uint8_t *src,
                                                      uint32_t S, const uint8_t *g2n, uint32_t D,
                                                      uint32_t nodes, uint32_t E, int use_smem,
                                                      uint64_t *node_demand, uint32_t *err) {
    // u64 counters: a batch's summed demand for one cell may pass 2^32
    extern __shared__ unsigned long long s_nd[];  // [nodes*E]
    const uint32_t b = blockIdx.x;
    uint64_t *out = node_demand + static_cast<size_t>(b) * nodes * E;
    if (use_smem) {
        for (uint32_t i = threadIdx.x; i < nodes * E; i += blockDim.x) s_nd[i] = 0;
    } else {
        for (uint32_t i = threadIdx.x; i < nodes * E; i += blockDim.x) out[i] = 0;
    }
    __syncthreads();
    // one warp per sampled slot, lanes over the row's non-zeros
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t i = warp; i < S; i += blockDim.x / 32) {
        const uint32_t r = rows[static_cast<size_t>(b) * S + i];
        const uint32_t s = src[static_cast<size_t>(b) * S + i];
        if (r >= R || s >= D) {
            if (lane == 0) atomicOr(err, kErrSourceRange);
            continue;
        }
        const uint32_t n = g2n[s];
        for (uint32_t z = row_ptr[r] + lane; z < row_ptr[r + 1]; z += 32) {
            const uint32_t e = cols[z];
            if (e >= E) {
                atomicOr(err, kErrExpertRange);
                continue;
            }
            if (use_smem)
                atomicAdd(s_nd + n * E + e, static_cast<unsigned long long>(vals[z]));
            else
                atomicAdd(reinterpret_cast<unsigned long long *>(out) + n * E + e,
                          static_cast<unsigned long long>(vals[z]));
        }
    }
    __syncthreads();
    if (use_smem)
        for (uint32_t i = threadIdx.x; i < nodes * E; i += blockDim.x) out[i] = s_nd[i];
}

struct CostParams {
    double hidden, bpe, inter_bw, intra_bw, etpt, overhead;
};

// One LayerSim from a cell's integer pair counts — simulate_layer's doubles in
// the reference's order of operations (shared by k_finalize and the fused
// scorer, so both produce the same bits).
__device__ __forceinline__ void finalize_cell(uint64_t i, uint64_t inter, uint64_t intra,
                                              const uint64_t *rank, uint32_t D, const CostParams &c,
                                              uint32_t tp_exp, int spans, double *out, double *payload) {
    // bytes_per_token = double(hidden) * double(bpe) (simulator.cpp:57-58)
    const double bpt = __dmul_rn(c.hidden, c.bpe);
    double mx = 0.0, straggler = 0.0;
    for (uint32_t d = 0; d < D; ++d) {
        const double pairs = static_cast<double>(rank[d]);
        const double bytes = __dmul_rn(pairs, bpt);
        if (payload) payload[i * D + d] = bytes;
        if (d == 0 || bytes > mx) mx = bytes;
        if (d == 0 || pairs > straggler) straggler = pairs;
    }
    const double bw = spans ? c.inter_bw : c.intra_bw;
    // max_payload / tp_exp / bandwidth (simulator.cpp:40)
    const double dispatch = __ddiv_rn(__ddiv_rn(mx, static_cast<double>(tp_exp)), bw);
    const double compute = __dmul_rn(c.etpt, straggler);
    // dispatch + compute + combine + overhead, left to right (simulator.cpp:96-97)
    const double layer = __dadd_rn(__dadd_rn(__dadd_rn(dispatch, compute), dispatch), c.overhead);
    double *o = out + i * 6;
    o[0] = __dmul_rn(static_cast<double>(inter), bpt);
    o[1] = __dmul_rn(static_cast<double>(intra), bpt);
    o[2] = dispatch;
    o[3] = compute;
    o[4] = dispatch;
    o[5] = layer;
}

// optional fused finalize of the scorer (out == nullptr: off)
struct FinalizeArgs {
    CostParams c;
    uint32_t tp_exp;
    int spans;
    double *out;
    double *payload;
};

constexpr int kScoreWarps = 8;
constexpr uint32_t kScoreMaxD = 32;  // lane-private rank accumulators in smem

// Batch-major scorer: one CTA per (batch, candidate range). The batch's demand
// is folded by source node into shared memory once; each warp then prices
// one candidate at a time by streaming its [nodes x E] destination table from
// L2 (coalesced bytes), accumulating pair counts per destination rank in
// lane-private shared-memory columns (no atomics), and reducing at the end.
template <bool kPrivate>
__global__ void __launch_bounds__(kScoreWarps * 32) k_score(const uint64_t *demand, uint32_t B,
                                                            uint32_t rows,
                                                            const uint8_t *row_node_g,
                                                            const uint8_t *luts, uint32_t P,
                                                            const uint8_t *g2n_g, uint32_t D,
                                                            uint32_t nodes, uint32_t E,
                                                            uint64_t *inter_out,
                                                            uint64_t *intra_out,
                                                            uint64_t *rank_out, uint32_t *err,
                                                            FinalizeArgs fin, uint32_t b0) {
    extern __shared__ unsigned long long s_raw[];
    const uint32_t NE = nodes * E;
    unsigned long long *s_nd = s_raw;                        // [nodes*E]
    unsigned long long *s_acc = s_nd + NE;  // [warps][D][32] lane-private, or [warps][D]
    const uint32_t cols = kPrivate ? 32u : 1u;
    uint8_t *s_g2n = reinterpret_cast<uint8_t *>(s_acc + kScoreWarps * D * cols);
    const uint32_t b = b0 + blockIdx.x;  // batches [b0, b0 + gridDim.x) of B
    pdl_trigger();
    for (uint32_t i = threadIdx.x; i < D; i += blockDim.x) s_g2n[i] = g2n_g[i];
    for (uint32_t i = threadIdx.x; i < NE; i += blockDim.x) s_nd[i] = 0;
    pdl_wait();  // the demand / outputs belong to the previous kernels
    __syncthreads();
    const uint64_t *a = demand + static_cast<size_t>(b) * rows * E;
    for (uint32_t i = threadIdx.x; i < rows * E; i += blockDim.x) {
        const unsigned long long v = a[i];
        if (v) atomicAdd(&s_nd[static_cast<uint32_t>(row_node_g[i / E]) * E + i % E], v);
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long *acc = s_acc + warp * D * cols;
    for (uint32_t p = blockIdx.y * kScoreWarps + warp; p < P; p += gridDim.y * kScoreWarps) {
        if (kPrivate)
            for (uint32_t d = 0; d < D; ++d) acc[d * 32 + lane] = 0;
        else
            for (uint32_t d = lane; d < D; d += 32) acc[d] = 0;
        __syncwarp();
        const uint8_t *lut = luts + static_cast<size_t>(p) * NE;
        unsigned long long inter = 0, intra = 0;
        // four LUT bytes per lane in flight before any is used (the L2 latency
        // of the candidate's table is paid once per 128 cells, not per cell)
        for (uint32_t i0 = lane; i0 < NE; i0 += 128) {
            uint32_t dd[4];
            unsigned long long vv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t i = i0 + 32u * u;
                dd[u] = i < NE ? __ldg(lut + i) : 255u;
                vv[u] = i < NE ? s_nd[i] : 0ull;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t i = i0 + 32u * u, d = dd[u];
                const unsigned long long v = vv[u];
                if (!v) continue;
                if (d >= D) {  // 255 = uncovered; any other out-of-range group too
                    atomicOr(err, kErrUncovered);
                    continue;
                }
                if (kPrivate)
                    acc[d * 32 + lane] += v;
                else
                    atomicAdd(acc + d, v);
                if (s_g2n[d] == i / E)
                    intra += v;
                else
                    inter += v;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            inter += __shfl_xor_sync(0xffffffffu, inter, o);
            intra += __shfl_xor_sync(0xffffffffu, intra, o);
        }
        __syncwarp();
        const size_t cell = static_cast<size_t>(p) * B + b;
        if (lane == 0) {
            inter_out[cell] = inter;
            intra_out[cell] = intra;
        }
        for (uint32_t d = lane; d < D; d += 32) {
            unsigned long long t = 0;
            if (kPrivate)
                for (uint32_t l = 0; l < 32; ++l) t += acc[d * 32 + ((l + lane) & 31)];
            else
                t = acc[d];
            rank_out[cell * D + d] = t;
        }
        __syncwarp();  // the warp's rank totals are visible to lane 0
        if (fin.out && lane == 0)
            finalize_cell(cell, inter, intra, rank_out + cell * D, D, fin.c, fin.tp_exp, fin.spans,
                          fin.out, fin.payload);
    }
}

constexpr uint32_t kFastMaxD = 16;  // static smem: lane-private rank columns for D <= 16

// Fast path of the scorer for nodes*E <= 512 with E % 16 == 0 (every BASELINE
// shape): lane l owns the 16 consecutive (node, expert) cells 16l..16l+15 of
// the batch's folded demand in REGISTERS, and reads a candidate's destination
// table as one 16-byte load — one L2 round trip per candidate, prefetched one
// candidate ahead. Rank totals pass to the finalizing lane through shared
// memory (no global read-back). Same integer sums and the same finalize_cell:
// bit-identical to k_score.
struct Job16 {
    const uint64_t *demand;
    uint32_t B, rows;
    const uint8_t *row_node_g;
    const uint8_t *luts;
    uint32_t P;
    const uint8_t *g2n_g;
    uint32_t D, nodes, E;
    uint64_t *inter_out, *intra_out, *rank_out;
    FinalizeArgs fin;
};

__device__ __forceinline__ void score16_body(const Job16 &J, uint32_t *err, uint32_t b0) {
    const uint64_t *demand = J.demand;
    const uint32_t B = J.B, rows = J.rows, P = J.P, D = J.D, nodes = J.nodes, E = J.E;
    const uint8_t *row_node_g = J.row_node_g, *luts = J.luts, *g2n_g = J.g2n_g;
    uint64_t *inter_out = J.inter_out, *intra_out = J.intra_out, *rank_out = J.rank_out;
    const FinalizeArgs &fin = J.fin;
    __shared__ unsigned long long s_nd[512];
    __shared__ unsigned long long s_acc[kScoreWarps][kFastMaxD][32];
    __shared__ unsigned long long s_rank[kScoreWarps][kFastMaxD];
    __shared__ uint8_t s_g2n[256];
    const uint32_t NE = nodes * E;
    const uint32_t b = b0 + blockIdx.x;  // batches [b0, b0 + gridDim.x) of B
    pdl_trigger();
    for (uint32_t i = threadIdx.x; i < D; i += blockDim.x) s_g2n[i] = g2n_g[i];
    for (uint32_t i = threadIdx.x; i < NE; i += blockDim.x) s_nd[i] = 0;
    pdl_wait();  // the demand / outputs belong to the previous kernels
    __syncthreads();
    const uint64_t *a = demand + static_cast<size_t>(b) * rows * E;
    for (uint32_t i = threadIdx.x; i < rows * E; i += blockDim.x) {
        const unsigned long long v = a[i];
        if (v) atomicAdd(&s_nd[static_cast<uint32_t>(row_node_g[i / E]) * E + i % E], v);
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool active = lane * 16 < NE;
    unsigned long long v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = active ? s_nd[lane * 16 + j] : 0ull;
    const uint32_t my_node = active ? lane * 16 / E : 0u;  // 16 cells never straddle a node
    unsigned long long(*acc)[32] = s_acc[warp];
    const uint32_t stride = gridDim.y * kScoreWarps;
    uint32_t p = blockIdx.y * kScoreWarps + warp;
    uint4 nxt = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    if (p < P && active) nxt = __ldg(reinterpret_cast<const uint4 *>(luts + static_cast<size_t>(p) * NE) + lane);
    for (; p < P; p += stride) {
        const uint4 cur = nxt;
        if (p + stride < P && active)  // next candidate's table in flight during this one
            nxt = __ldg(reinterpret_cast<const uint4 *>(luts + static_cast<size_t>(p + stride) * NE) + lane);
        for (uint32_t d = 0; d < D; ++d) acc[d][lane] = 0;
        __syncwarp();
        unsigned long long inter = 0, intra = 0;
        const uint32_t w4[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t d = (w4[j >> 2] >> (8 * (j & 3))) & 0xFFu;
            if (!v[j]) continue;
            if (d >= D) {
                atomicOr(err, kErrUncovered);
                continue;
            }
            acc[d][lane] += v[j];
            if (s_g2n[d] == my_node)
                intra += v[j];
            else
                inter += v[j];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            inter += __shfl_xor_sync(0xffffffffu, inter, o);
            intra += __shfl_xor_sync(0xffffffffu, intra, o);
        }
        __syncwarp();
        const size_t cell = static_cast<size_t>(p) * B + b;
        if (lane == 0) {
            inter_out[cell] = inter;
            intra_out[cell] = intra;
        }
        for (uint32_t d = lane; d < D; d += 32) {
            unsigned long long t = 0;
            for (uint32_t l = 0; l < 32; ++l) t += acc[d][(l + lane) & 31];
            rank_out[cell * D + d] = t;
            s_rank[warp][d] = t;
        }
        __syncwarp();  // the warp's rank totals are visible to lane 0
        if (fin.out && lane == 0)
            finalize_cell(cell, inter, intra, reinterpret_cast<const uint64_t *>(s_rank[warp]), D, fin.c,
                          fin.tp_exp, fin.spans, fin.out,
                          fin.payload);
        __syncwarp();
    }
}

__global__ void __launch_bounds__(kScoreWarps * 32) k_score16(Job16 job, uint32_t *err, uint32_t b0) {
    score16_body(job, err, b0);
}

// Two scoring jobs of the same batch range in ONE launch (blockIdx.z = job):
// the step's candidate and baseline tables, no second stream, no fork / join.
__global__ void __launch_bounds__(kScoreWarps * 32) k_score16x2(Job16 j0, Job16 j1, uint32_t *err,
                                                                uint32_t b0) {
    if (blockIdx.z == 0)
        score16_body(j0, err, b0);
    else
        score16_body(j1, err, b0);
}

__global__ void k_finalize(const uint64_t *inter, const uint64_t *intra, const uint64_t *rank,
                           uint64_t N, uint32_t D, CostParams c, uint32_t tp_exp, int spans,
                           double *out, double *payload) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= N) return;
    finalize_cell(i, inter[i], intra[i], rank + i * D, D, c, tp_exp, spans, out, payload);
}

}  // namespace
}  // namespace mpb

using namespace mpb;

extern "C" {

mpb_status mpb_batch_demand(mpb_context *ctx, const uint32_t *row_ptr, const uint32_t *cols,
                            const uint32_t *vals, uint32_t R, const uint32_t *rows,
                            const uint8_t *src, uint32_t B, uint32_t S, const uint8_t *group_to_node,
                            uint32_t D, uint32_t nodes, uint32_t E, uint64_t *node_demand) {
    if (!ctx || !row_ptr || !rows || !src || !group_to_node || !node_demand)
        return fail(MPB_VALIDATION_ERROR, "mpb_batch_demand: NULL argument");
    if (B == 0) return MPB_OK;
    const size_t smem = size_t(nodes) * E * 8;
    const int use_smem = smem <= 160 * 1024;
    if (use_smem)
        MPB_CUDA(cudaFuncSetAttribute(k_batch_demand, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(smem)));
    k_batch_demand<<<B, 256, use_smem ? smem : 0, ctx->stream>>>(
        row_ptr, cols, vals, R, rows, src, S, group_to_node, D, nodes, E, use_smem, node_demand,
        ctx->d_error);
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

}  // extern "C"

namespace {
mpb_status check_cost(const double *cost, uint32_t tp_exp) {
    // CostModelParams::validate (simulator.cpp:14-25)
    if (cost[0] < 1 || cost[1] < 1)
        return fail(MPB_CONFIG_ERROR, "cost model: hidden_dim and bytes_per_element must be >= 1");
    if (cost[2] <= 0.0 || cost[3] <= 0.0)
        return fail(MPB_CONFIG_ERROR, "cost model: bandwidths must be positive");
    if (cost[3] < cost[2])
        return fail(MPB_CONFIG_ERROR, "cost model: intra_node_bandwidth must be >= inter_node_bandwidth");
    if (cost[4] <= 0.0)
        return fail(MPB_CONFIG_ERROR, "cost model: expert_time_per_token must be positive");
    if (cost[5] < 0.0)
        return fail(MPB_CONFIG_ERROR, "cost model: fixed_layer_overhead must be >= 0");
    if (tp_exp == 0) return fail(MPB_CONFIG_ERROR, "topology: tp_exp must be >= 1");
    return MPB_OK;
}

mpb_status launch_score(mpb_context *ctx, const char *fn, const uint64_t *demand, uint32_t B,
                        uint32_t rows, const uint8_t *row_node, const uint8_t *luts, uint32_t P,
                        const uint8_t *group_to_node, uint32_t D, uint32_t nodes, uint32_t E,
                        uint64_t *inter, uint64_t *intra, uint64_t *rank_pairs, FinalizeArgs fin,
                        uint32_t b0, uint32_t nb) {
    if (!ctx || !demand || !row_node || !luts || !group_to_node || !inter || !intra || !rank_pairs)
        return fail(MPB_VALIDATION_ERROR, std::string(fn) + ": NULL argument");
    if (rows == 0 || rows > 255) return fail(MPB_CONFIG_ERROR, std::string(fn) + ": need 1 <= rows <= 255");
    if (D == 0 || D > 255 || nodes == 0)
        return fail(MPB_CONFIG_ERROR, std::string(fn) + ": need 1 <= D <= 255, nodes >= 1");
    if (P == 0 || B == 0) return MPB_OK;
    const bool priv = D <= kScoreMaxD;
    const size_t smem =
        size_t(nodes) * E * 8 + size_t(kScoreWarps) * D * (priv ? 32 : 1) * 8 + D + 8;
    if (smem > 200 * 1024) return fail(MPB_CONFIG_ERROR, std::string(fn) + ": nodes*E too large");
    // register-resident fast path: 16 cells per lane, one 16-byte LUT load per candidate
    const bool fast = size_t(nodes) * E <= 512 && E % 16 == 0 && D <= kFastMaxD &&
                      (reinterpret_cast<uintptr_t>(luts) & 15) == 0 && !std::getenv("MPB_SCORE_SLOW");
    auto kern = priv ? k_score<true> : k_score<false>;
    if (!fast)
        MPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    // one CTA per batch; split candidates over grid.y until the machine is full
    const uint32_t want = 4u * static_cast<uint32_t>(ctx->num_sms);
    if (b0 + nb > B) return fail(MPB_CONFIG_ERROR, std::string(fn) + ": batch range past B");
    if (nb == 0) return MPB_OK;
    uint32_t gy = std::max(1u, want / std::max(1u, nb));
    gy = std::min(gy, (P + kScoreWarps - 1) / kScoreWarps);
    gy = std::min(gy, 65535u);
    dim3 grid(nb, gy);
    // programmatic launch: the prologue (smem zeroing, g2n staging) overlaps
    // the previous kernel's drain; the demand is read after griddepcontrol.wait
    if (fast) {
        const Job16 job{demand, B, rows, row_node, luts, P, group_to_node, D, nodes, E, inter, intra,
                        rank_pairs, fin};
        MPB_CUDA(launch_pdl(k_score16, grid, dim3(kScoreWarps * 32), 0, ctx->stream, job, ctx->d_error, b0));
    } else {
        MPB_CUDA(launch_pdl(kern, grid, dim3(kScoreWarps * 32), smem, ctx->stream, demand, B, rows,
                            row_node, luts, P, group_to_node, D, nodes, E, inter, intra, rank_pairs,
                            ctx->d_error, fin, b0));
    }
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}
}  // namespace

extern "C" {

mpb_status mpb_score_placements(mpb_context *ctx, const uint64_t *demand, uint32_t B,
                                uint32_t rows, const uint8_t *row_node, const uint8_t *luts,
                                uint32_t P, const uint8_t *group_to_node, uint32_t D,
                                uint32_t nodes, uint32_t E, uint64_t *inter, uint64_t *intra,
                                uint64_t *rank_pairs) {
    return launch_score(ctx, "mpb_score_placements", demand, B, rows, row_node, luts, P,
                        group_to_node, D, nodes, E, inter, intra, rank_pairs,
                        FinalizeArgs{CostParams{}, 1, 0, nullptr, nullptr}, 0, B);
}

mpb_status mpb_score_placements_finalize(mpb_context *ctx, const uint64_t *demand, uint32_t B,
                                         uint32_t rows, const uint8_t *row_node, const uint8_t *luts,
                                         uint32_t P, const uint8_t *group_to_node, uint32_t D,
                                         uint32_t nodes, uint32_t E, uint64_t *inter, uint64_t *intra,
                                         uint64_t *rank_pairs, const double *cost, uint32_t tp_exp,
                                         int spans_nodes, double *out, double *payload) {
    if (!ctx || !cost || !out)
        return fail(MPB_VALIDATION_ERROR, "mpb_score_placements_finalize: NULL argument");
    if (mpb_status st = check_cost(cost, tp_exp)) return st;
    return launch_score(ctx, "mpb_score_placements_finalize", demand, B, rows, row_node, luts, P,
                        group_to_node, D, nodes, E, inter, intra, rank_pairs,
                        FinalizeArgs{CostParams{cost[0], cost[1], cost[2], cost[3], cost[4], cost[5]},
                                     tp_exp, spans_nodes, out, payload},
                        0, B);
}

mpb_status mpb_finalize_layer_sims(mpb_context *ctx, const uint64_t *inter, const uint64_t *intra,
                                   const uint64_t *rank_pairs, uint64_t N, uint32_t D,
                                   const double *cost, uint32_t tp_exp, int spans_nodes,
                                   double *out, double *payload) {
    if (!ctx || !inter || !intra || !rank_pairs || !cost || !out)
        return fail(MPB_VALIDATION_ERROR, "mpb_finalize_layer_sims: NULL argument");
    if (mpb_status st = check_cost(cost, tp_exp)) return st;
    if (N == 0) return MPB_OK;
    CostParams c{cost[0], cost[1], cost[2], cost[3], cost[4], cost[5]};
    const unsigned blocks = static_cast<unsigned>((N + 255) / 256);
    k_finalize<<<blocks, 256, 0, ctx->stream>>>(inter, intra, rank_pairs, N, D, c, tp_exp,
                                                spans_nodes, out, payload);
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

}  // extern "C"

namespace mpb {
// Two finalized scoring jobs over the same batch range in one launch when both
// take the register-resident path (else one launch each, in job order).
mpb_status score_finalize_pair(mpb_context *ctx, const mpb_score_job &a, const mpb_score_job &b,
                               uint32_t b0, uint32_t nb) {
    auto eligible = [](const mpb_score_job &j) {
        return size_t(j.nodes) * j.E <= 512 && j.E % 16 == 0 && j.D <= kFastMaxD && j.D >= 1 &&
               j.rows >= 1 && j.rows <= 255 && (reinterpret_cast<uintptr_t>(j.luts) & 15) == 0 && j.out &&
               j.demand && j.row_node && j.luts && j.group_to_node && j.inter && j.intra && j.rank_pairs;
    };
    if (!ctx || !eligible(a) || !eligible(b) || a.B != b.B || std::getenv("MPB_SCORE_SLOW") ||
        b0 + nb > a.B) {
        if (mpb_status st = score_finalize_range(ctx, a, b0, nb)) return st;
        return score_finalize_range(ctx, b, b0, nb);
    }
    if (mpb_status st = check_cost(a.cost, a.tp_exp)) return st;
    if (mpb_status st = check_cost(b.cost, b.tp_exp)) return st;
    if (nb == 0 || (a.P == 0 && b.P == 0)) return MPB_OK;
    auto job = [](const mpb_score_job &j) {
        return Job16{j.demand, j.B, j.rows, j.row_node, j.luts, j.P, j.group_to_node, j.D, j.nodes, j.E,
                     j.inter, j.intra, j.rank_pairs,
                     FinalizeArgs{CostParams{j.cost[0], j.cost[1], j.cost[2], j.cost[3], j.cost[4], j.cost[5]},
                                  j.tp_exp, j.spans_nodes, j.out, j.payload}};
    };
    const uint32_t want = 4u * static_cast<uint32_t>(ctx->num_sms);
    const uint32_t P = std::max(a.P, b.P);
    uint32_t gy = std::max(1u, want / std::max(1u, nb));
    gy = std::min(gy, (P + kScoreWarps - 1) / kScoreWarps);
    gy = std::min(gy, 65535u);
    MPB_CUDA(launch_pdl(k_score16x2, dim3(nb, gy, 2), dim3(kScoreWarps * 32), 0, ctx->stream, job(a), job(b),
                        ctx->d_error, b0));
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

// Batches [b0, b0 + nb) of an mpb_score_placements_finalize job (the step plan
// prices each chunk of layers as soon as its statistics are in).
mpb_status score_finalize_range(mpb_context *ctx, const mpb_score_job &j, uint32_t b0, uint32_t nb) {
    if (!ctx || !j.out) return fail(MPB_VALIDATION_ERROR, "score_finalize_range: NULL argument");
    if (mpb_status st = check_cost(j.cost, j.tp_exp)) return st;
    return launch_score(ctx, "mpb_step score", j.demand, j.B, j.rows, j.row_node, j.luts, j.P,
                        j.group_to_node, j.D, j.nodes, j.E, j.inter, j.intra, j.rank_pairs,
                        FinalizeArgs{CostParams{j.cost[0], j.cost[1], j.cost[2], j.cost[3], j.cost[4],
                                                j.cost[5]},
                                     j.tp_exp, j.spans_nodes, j.out, j.payload},
                        b0, nb);
}
}  // namespace mpb
