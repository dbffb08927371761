// K1: router GEMM + fused top-k on tcgen05 tensor cores (sm_100a).
//
// logits[T, E] = X[T, H] . W[E, H]^T with bf16 inputs and fp32 accumulation,
// followed in the same kernel by softmax/sigmoid top-k selection. The whole
// expert dimension (E = N <= 256) is one UMMA tile, so one 128-token tile's
// logits live in TMEM (128 lanes x N fp32 columns) and the epilogue owns one
// token per thread: no logits ever reach HBM (unless requested for parity
// tests). No reference implementation exists (the reference samples routes
// synthetically, /root/reference/proj/core/src/trace.cpp:240-259); selection
// follows its lowest-index-wins tie rule (placement.cpp:143-152).
//
// Persistent, warp-specialised CTA (one per SM, 384 threads); for E = 256 the
// default is a 2-CTA cluster per 256-token tile with cta_group::2 UMMA (see
// k_router's PAIR mode):
//   warp 0     TMA producer: X tile [128 x 64] (evict-first) + W tile [N x 64]
//              (evict-last, L2-resident across CTAs) per k-block into a
//              STAGES-deep 128B-swizzled smem ring (mbarrier full/empty)
//   warp 1     MMA issuer: 4 x tcgen05.mma (M=128, N, K=16) per k-block into a
//              double-buffered TMEM accumulator; tcgen05.commit frees smem
//              slots and hands finished accumulators to the epilogue
//   warp 2     TMEM allocator (2*N columns)
//   warps 4-7  epilogue: tcgen05.ld 32 columns at a time, running top-k in
//              registers (static-index insertion network), max / sum-exp,
//              then release the accumulator so the next tile's MMAs overlap
// Roofline: FLOP/token = 2*H*E; bytes/token = 2*H (X) + 8*k out.
#include <cudaTypedefs.h>

#include <cfloat>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace mpb {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 bytes: one 128B swizzle atom per row
#ifndef MPB_ROUTER_KBLOCKS
#define MPB_ROUTER_KBLOCKS 1  // 64-column K blocks per pipeline stage (build-time knob)
#endif
constexpr int kKB = MPB_ROUTER_KBLOCKS;
constexpr int kStageK = kBK * kKB;  // K columns per stage
constexpr int kThreadsR = 384;  // 4 non-epilogue + 8 epilogue warps

#ifndef MPB_ROUTER_PREFETCH
#define MPB_ROUTER_PREFETCH 0  // X k-steps prefetched into L2 ahead of the TMA loads
#endif
constexpr uint32_t kPrefetch = MPB_ROUTER_PREFETCH;

#ifndef MPB_ROUTER_STAGES_CAP
#define MPB_ROUTER_STAGES_CAP 8  // build-time knob for stage-count experiments
#endif

template <int N, int KMAX, bool PAIR>
struct RCfg {
    static constexpr int A_BLOCK = kBM * kBK * 2;                       // one 64-col box
    static constexpr int B_BLOCK = (PAIR ? N / 2 : N) * kBK * 2;       // pair: half of W
    static constexpr int A_BYTES = A_BLOCK * kKB;
    static constexpr int B_BYTES = B_BLOCK * kKB;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr uint32_t TMEM_COLS = 2 * N < 32 ? 32 : 2 * N;
    static constexpr int ROWS_PER_TILE = PAIR ? 2 * kBM : kBM;
    // per epilogue thread: 16 parked logits, later its half's top-k (values,
    // ids) + max + sum for the merge; odd stride keeps banks conflict-free
    static constexpr int PARK_ROW = (2 * KMAX + 2 > 16 ? 2 * KMAX + 2 : 16) | 1;
    static constexpr int PARK = 256 * PARK_ROW * 4;
    static constexpr int BUDGET = 232448 - 1024 - PARK - 256;
    static constexpr int STAGES = BUDGET / STAGE > MPB_ROUTER_STAGES_CAP ? MPB_ROUTER_STAGES_CAP
                                                                         : BUDGET / STAGE;
    static constexpr int SMEM = 1024 + STAGES * STAGE + PARK + (2 * STAGES + 6) * 8 + 16;
};

#ifdef MPB_ROUTER_TRACE
// Experiment builds only: per-CTA %globaltimer stamps of the kernel's phases
// (tools/router_trace.py). slot: 0 entry, 1 after griddepcontrol.wait,
// 2 producer's first TMA issued, 3 MMA warp's last commit, 4 epilogue: last
// accumulator ready, 5 epilogue: last fix-up done, 6 epilogue: last item
// done, 7 exit; 8 = role of the last item, 9 = items.
__device__ unsigned long long g_router_trace[2 * 148 * 16];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");
    return t;
}
#define RTRACE(slot, val) g_router_trace[blockIdx.x * 16 + (slot)] = (val)
#else
#define RTRACE(slot, val) ((void)0)
#endif

struct RouterParams {
    uint64_t T;
    uint32_t H;
    uint32_t k;
    int score_fn;
    int renorm;
    uint32_t num_tiles;
    int32_t *idx;
    float *w;
    float *logits;
    // split-K tail (wave quantisation): the last partial wave's tiles are split in
    // S K parts run by S units; parts 1..S-1 dump their fp32 partials, part 0 adds
    // them (in part order) and finishes the tile. S = 1: no split
    uint32_t splits;
    float *partial;      // [slot][part-1][rank][N/16 chunks][128 rows][16]
    uint32_t *flags;     // [slot][rank]: partials ready, reset to 0 by the finisher
    uint32_t E;          // real experts (<= N): columns >= E are padding, never selected
    // grouped launch over several layers: tile t belongs to layer t / tiles_per_layer;
    // maps = [layer][X, W] descriptors in global memory (nullptr: the kernel
    // parameters tmX / tmW, one layer); idx / w are [layers][T][k]
    const CUtensorMap *maps;
    uint32_t tiles_per_layer;
    uint32_t layers;
    // split-K tail through distributed shared memory (single-CTA tiles): the S
    // K-part units of a tail tile form one cluster (cluster_tail != 0)
    uint32_t cluster_tail;
    // fused dispatch demand (mpb_router_topk_demand, one layer): every selected
    // (token, expert) adds 1 to demand[src[token]][expert] (and demand2 under
    // src2) as it is written; nullptr: off
    const uint8_t *src, *src2;
    unsigned long long *demand, *demand2;
    uint32_t D;
    uint32_t *err;
};

// The fused demand count of one selected (token, expert) pair (the layout's
// K2 demand histogram, simulator.cpp:64-80 semantics: source group >= D is
// flagged, not counted).
__device__ __forceinline__ void count_demand(const RouterParams &p, uint64_t token, uint32_t e) {
    const uint32_t s = p.src[token];
    if (s < p.D)
        atomicAdd(p.demand + static_cast<size_t>(s) * p.E + e, 1ull);
    else
        atomicOr(p.err, kErrSourceRange);
    if (p.demand2) {
        const uint32_t s2 = p.src2[token];
        if (s2 < p.D)
            atomicAdd(p.demand2 + static_cast<size_t>(s2) * p.E + e, 1ull);
        else
            atomicOr(p.err, kErrSourceRange);
    }
}

// Work item n of a scheduling unit: full waves of whole tiles, then (split
// tail) unit u takes K part (u % S) of tail tile u / S. role 0 = whole tile,
// 1 = K part 0 + fix-up with the other parts' partials, 2 = K part > 0, dump only.
struct WorkItem {
    uint32_t tile, k0, k1, role, slot, part;
};

__device__ __forceinline__ bool next_item(uint32_t n, uint32_t unit, uint32_t units,
                                          uint32_t num_tiles, uint32_t nk, uint32_t S,
                                          WorkItem &w) {
    if (S <= 1) {
        const uint32_t t = unit + n * units;
        if (t >= num_tiles) return false;
        w = {t, 0, nk, 0, 0, 0};
        return true;
    }
    const uint32_t waves = num_tiles / units;
    if (n < waves) {
        w = {unit + n * units, 0, nk, 0, 0, 0};
        return true;
    }
    const uint32_t rem = num_tiles - waves * units;
    if (n == waves && unit < S * rem) {
        const uint32_t slot = unit / S, h = unit - slot * S;
        w = {waves * units + slot, h * nk / S, (h + 1) * nk / S, h ? 2u : 1u, slot, h};
        return true;
    }
    return false;
}

// r[i] for a per-lane dynamic i in [0, 16): a 4-level select tree on the
// index bits keeps the chunk in registers (an indexed register array would be
// demoted to local memory; a shared-memory park costs a store of the chunk and
// a dependent load per insertion).
__device__ __forceinline__ float pick16(const uint32_t (&r)[16], int i) {
    uint32_t a[8], b[4], c[2];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = (i & 1) ? r[2 * j + 1] : r[2 * j];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = (i & 2) ? a[2 * j + 1] : a[2 * j];
#pragma unroll
    for (int j = 0; j < 2; ++j) c[j] = (i & 4) ? b[2 * j + 1] : b[2 * j];
    return __uint_as_float((i & 8) ? c[1] : c[0]);
}

// (v, id) ranks before (w, jd): larger logit, equal logits -> lower expert id.
__device__ __forceinline__ bool ranks_before(float v, int id, float w, int jd) {
    return v > w || (v == w && id < jd);
}

// Order-preserving u32 key of a logit for the top-k: larger key ranks first.
// Real values (+-inf included) descend, -0 == +0 (a tie), NaN (key 1) ranks
// after every real value; 0 is reserved for padding / taken columns. Equal keys
// are broken by the lower expert id: exactly the oracle's beats()
// (oracle/moeplace_oracle.c, the reference's lowest-index tie rule,
// placement.cpp:143-152).
__device__ __forceinline__ uint32_t rank_key(float v) {
    if (v != v) return 1u;
    uint32_t b = __float_as_uint(v);
    if (b == 0x80000000u) b = 0u;
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // -inf -> 0x007FFFFF
}
__device__ __forceinline__ float key_value(uint32_t key) {
    return key == 1u ? __uint_as_float(0x7FC00000u)
                     : __uint_as_float((key & 0x80000000u) ? (key & 0x7FFFFFFFu) : ~key);
}

// Compare-exchange of (key, slot) pairs into descending key order (equal keys:
// the lower slot first, i.e. the lower expert id of the lane's columns).
__device__ __forceinline__ void cx_desc(uint32_t &ka, uint32_t &sa, uint32_t &kb, uint32_t &sb) {
    const bool sw = kb > ka || (kb == ka && sb < sa);
    const uint32_t k0 = sw ? kb : ka, k1 = sw ? ka : kb, s0 = sw ? sb : sa, s1 = sw ? sa : sb;
    ka = k0;
    kb = k1;
    sa = s0;
    sb = s1;
}

// Sum and top-k of a cluster-tail row share (RPS = 8R rows) from shared memory.
// Warp ew (of the 8 epilogue warps) owns rows ew, ew+8, ...; lane l holds
// columns l, l+32, ... of each (conflict-free LDS; the K parts summed in part
// order 0..S-1: the global tail's fp32 order, bit-identical logits). Each lane
// sorts its V rank keys once (a 1- or 5-exchange network); the row's top-k is
// then k rounds of: redux.sync max over the 32 lane heads, a ballot of the
// lanes holding it (several only on an exact tie: the lowest column id wins,
// warp-uniform slow path), the winning lane pops its head. The R rows are
// interleaved so one row's reductions hide the others' latency; no branches
// outside the tie path, no dynamic register indexing. Lane j ends with slot j.
// Weights: softmax shifts by the row max (the first round's winner); with
// renormalisation the softmax denominator cancels and is never formed.
// Micro-benchmark (tools/micro/sel_bench.cu, 32 rows x 128 logits, top-8):
// 5.2K SM cycles against 8.6K for the per-thread insertion + shuffle merge.
template <int N, int KMAX, int R>
__device__ __forceinline__ void tail_select(const RouterParams &p, const float *rx, const float *tile,
                                            uint32_t h, uint32_t ew, uint32_t lane,
                                            uint64_t row_tile0, uint64_t out_row_tile0) {
    constexpr uint32_t RS = N + 4, V = N / 32;
    static_assert(V == 2 || V == 4, "cluster tail: N = 64 or 128");
    constexpr uint32_t RPS = 8u * R, SP = 128u / RPS;  // SP = S: 4 K parts (R = 4) or 2 (R = 8)
    constexpr float kL2E = 1.4426950408889634f;
    uint32_t key[R][V], perm[R];
    // every row's sums first (all loads in flight: no global store between
    // them that the compiler would have to order them against), then the
    // optional logits, then the rank keys
    const float *share[SP];
#pragma unroll
    for (uint32_t part = 0; part < SP; ++part)
        share[part] = part == h ? tile : rx + static_cast<size_t>(part < h ? part : part - 1) * RPS * RS;
    float xs[R][V];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int i = 0; i < static_cast<int>(V); ++i) {
            const uint32_t off = (ew + 8u * r) * RS + lane + 32u * i;
            float tot = share[0][off];
#pragma unroll
            for (uint32_t part = 1; part < SP; ++part) tot += share[part][off];
            xs[r][i] = tot;
        }
    if (p.logits)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t rr = ew + 8u * r;
            if (row_tile0 + h * RPS + rr >= p.T) continue;
            float *out = p.logits + (out_row_tile0 + h * RPS + rr) * p.E;
#pragma unroll
            for (int i = 0; i < static_cast<int>(V); ++i)
                if (lane + 32u * i < p.E) out[lane + 32u * i] = xs[r][i];
        }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const float *x = xs[r];
        uint32_t sl[V];
#pragma unroll
        for (int i = 0; i < static_cast<int>(V); ++i) {
            key[r][i] = lane + 32u * i < p.E ? rank_key(x[i]) : 0u;  // padding: 0, never selected
            sl[i] = i;
        }
        cx_desc(key[r][0], sl[0], key[r][1], sl[1]);
        if constexpr (V == 4) {
            cx_desc(key[r][2], sl[2], key[r][3], sl[3]);
            cx_desc(key[r][0], sl[0], key[r][2], sl[2]);
            cx_desc(key[r][1], sl[1], key[r][3], sl[3]);
            cx_desc(key[r][1], sl[1], key[r][2], sl[2]);
        }
        perm[r] = 0;
#pragma unroll
        for (int i = 0; i < static_cast<int>(V); ++i) perm[r] |= sl[i] << (2 * i);
    }
#ifdef MPB_ROUTER_TRACE
    if (ew == 0 && lane == 0) RTRACE(5, gtime());
#endif
    const uint32_t k = p.k;
    const bool softmax = p.score_fn == MPB_SCORE_SOFTMAX;
    uint32_t skey[R], sid[R], mkey[R];
    float spart[R];  // the lane's share of the softmax denominator (formed only without renormalisation)
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        if (static_cast<uint32_t>(j) >= k) break;
        uint32_t km[R], b[R];
#pragma unroll
        for (int r = 0; r < R; ++r) km[r] = __reduce_max_sync(0xffffffffu, key[r][0]);
        if (j == 0) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                mkey[r] = km[r];
                spart[r] = 0.f;
                if (softmax && !p.renorm) {  // every column still at its place: sum them now
                    const float mlog = (km[r] <= 1u ? -INFINITY : key_value(km[r])) * kL2E;
#pragma unroll
                    for (int i = 0; i < static_cast<int>(V); ++i)
                        spart[r] += key[r][i] > 1u ? exp2f(fmaf(key_value(key[r][i]), kL2E, -mlog)) : 0.f;
                }
            }
        }
        bool tie = false;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            b[r] = __ballot_sync(0xffffffffu, key[r][0] == km[r]);
            tie |= __popc(b[r]) != 1;
        }
        if (tie) {  // equal keys at several lane heads: the lowest column id (slot, then lane)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const bool at = key[r][0] == km[r];
                const uint32_t ms = __reduce_min_sync(0xffffffffu, at ? (perm[r] & 3u) : 0xffu);
                b[r] = __ballot_sync(0xffffffffu, at && (perm[r] & 3u) == ms);
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t wl = __ffs(b[r]) - 1;
            const uint32_t id = __shfl_sync(0xffffffffu, lane + 32u * (perm[r] & 3u), wl);
            skey[r] = lane == static_cast<uint32_t>(j) ? km[r] : skey[r];
            sid[r] = lane == static_cast<uint32_t>(j) ? id : sid[r];
            const bool pop = lane == wl;
#pragma unroll
            for (int i = 0; i + 1 < static_cast<int>(V); ++i) key[r][i] = pop ? key[r][i + 1] : key[r][i];
            key[r][V - 1] = pop ? 0u : key[r][V - 1];
            perm[r] = pop ? perm[r] >> 2 : perm[r];
        }
    }
    float e[R], tsum[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const float mlog = (mkey[r] <= 1u ? -INFINITY : key_value(mkey[r])) * kL2E;
        const float v = key_value(skey[r]);
        e[r] = lane < k && !isnan(v) ? (softmax ? exp2f(fmaf(v, kL2E, -mlog)) : 1.f / (1.f + expf(-v))) : 0.f;
        tsum[r] = e[r];
    }
#pragma unroll
    for (uint32_t o = 16; o >= 1; o >>= 1)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            tsum[r] += __shfl_xor_sync(0xffffffffu, tsum[r], o);
            spart[r] += __shfl_xor_sync(0xffffffffu, spart[r], o);
        }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t rr = ew + 8u * r;
        if (lane < k && row_tile0 + h * RPS + rr < p.T) {
            const uint64_t o = (out_row_tile0 + h * RPS + rr) * p.k + lane;
            p.idx[o] = static_cast<int32_t>(sid[r]);
            p.w[o] = p.renorm ? (tsum[r] > 0.f ? e[r] / tsum[r] : 0.f) : softmax ? e[r] / spart[r] : e[r];
            if (p.demand) count_demand(p, row_tile0 + h * RPS + rr, sid[r]);
        }
    }
}

// Split-K tail through distributed shared memory (single-CTA tiles, PAIR off).
// The S = p.splits K-part units of a tail tile are one cluster; CTA h (K part
// h, cluster rank h) ends with rows [h*RPS, (h+1)*RPS) of the tile (RPS =
// 128/S), i.e. a reduce-scatter of the fp32 partial accumulators:
//   1. once its own MMAs are done (its pipeline smem is free) every CTA tells
//      its peers so (remote mbarrier arrive);
//   2. the epilogue warps stage the TMEM rows the CTA does not own in local
//      shared memory (its own share straight into the sum tile); once every
//      peer's pipeline smem is free one thread bulk-copies each share into its
//      owner's smem (cp.async.bulk shared::cluster, completion counted in bytes
//      on the owner's mbarrier) — no global memory, no flags;
//   3.+4. one warp per owned row sums it in K-part order 0..S-1 (the fp32
//      order of the global-memory tail) in registers and selects its top-k by
//      k warp arg-max rounds (tail_select).
// The whole 128-row epilogue of a decode batch's tiles is thus spread over the S
// CTAs and over 8 warps per row group instead of 2.
template <int N, int KMAX>
__device__ __forceinline__ void cluster_tail(const RouterParams &p, const WorkItem &it,
                                             uint32_t taddr_q, uint8_t *stage_base,
                                             uint64_t *peer_free, uint64_t *rx_full, uint32_t warp,
                                             uint32_t lane, uint64_t row_tile0, uint64_t out_row_tile0) {
    if constexpr (N > 128) {  // the host runs the cluster tail only for N <= 128
        return;
    } else {
    const uint32_t S = p.splits, h = it.part;
    const uint32_t RPS = 128u / S;
    constexpr uint32_t RS = N + 4;  // padded row stride (floats): conflict-free 16-byte stores
    constexpr int NH = N / 2;
    float *rx = reinterpret_cast<float *>(stage_base);                  // [S-1][RPS][RS]
    float *tile = rx + static_cast<size_t>(S - 1) * RPS * RS;            // [RPS][RS]
    float *snd = tile + static_cast<size_t>(RPS) * RS;                   // [S-1][RPS][RS]
    const uint32_t t = threadIdx.x - 128u;                               // epilogue thread 0..255
    const uint32_t q = warp & 3, half = (warp - 4) >> 2;
    const uint32_t share_bytes = RPS * RS * 4u;  // one row share, padded rows, contiguous
    // cluster_tail == 2 (MPB_ROUTER_ST_ASYNC=1, experiment): every thread
    // pushes its half rows of the other owners' shares straight from registers
    // into the owners' smem with st.async instead of staging + bulk copies
    const bool push = p.cluster_tail == 2;
    if (t == 0) {
        ptx::mbar_arrive_expect_tx(rx_full, (S - 1) * (push ? RPS * N * 4u : share_bytes));
        for (uint32_t c = 0; c < S; ++c)
            if (c != h) ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(peer_free), c));
    }
    const uint32_t owner = q * S / 4u;
    const uint32_t rloc = q * 32u + lane - owner * RPS;  // row within the owner's share
    {  // stage this CTA's partial of every row: other owners' shares for the bulk
       // copies, its own share into the tile (local, conflict-free 16-byte stores)
        const uint32_t i = owner < h ? owner : owner - 1;
        float *dst = owner == h ? tile + static_cast<size_t>(rloc) * RS
                                : snd + (static_cast<size_t>(i) * RPS + rloc) * RS;
        uint32_t r[NH];  // the thread's half row: every TMEM load in flight before one wait
#pragma unroll
        for (int c = 0; c < NH; c += 16) ptx::tmem_ld_32x32b_x16(taddr_q + half * NH + c, *reinterpret_cast<uint32_t(*)[16]>(r + c));
        ptx::tmem_ld_wait();
        if (push && owner != h) {
            const uint32_t j = h < owner ? h : h - 1;  // my slot at the owner
            const uint32_t dst_c = ptx::mapa(
                ptx::smem_u32(rx + (static_cast<size_t>(j) * RPS + rloc) * RS + half * NH), owner);
            const uint32_t bar_c = ptx::mapa(ptx::smem_u32(rx_full), owner);
            ptx::mbar_wait_cluster(peer_free, 0);  // every peer's pipeline smem is free
#pragma unroll
            for (int c = 0; c < NH; c += 4) ptx::st_async_v4(dst_c + 4u * c, r[c], r[c + 1], r[c + 2], r[c + 3], bar_c);
        } else {
#pragma unroll
            for (int c = 0; c < NH; c += 4)
                *reinterpret_cast<float4 *>(dst + half * NH + c) =
                    make_float4(__uint_as_float(r[c]), __uint_as_float(r[c + 1]), __uint_as_float(r[c + 2]),
                                __uint_as_float(r[c + 3]));
            if (owner != h) ptx::fence_proxy_async_smem();  // generic writes -> visible to the bulk-copy engine
        }
    }
    asm volatile("bar.sync 5, 256;" ::: "memory");  // every share staged
    if (t == 0 && !push) {
        ptx::mbar_wait_cluster(peer_free, 0);  // every peer's pipeline smem is free
#ifdef MPB_ROUTER_TRACE
        RTRACE(14, gtime());
#endif
        for (uint32_t o = 0; o < S; ++o) {
            if (o == h) continue;
            const uint32_t i = o < h ? o : o - 1;  // my share slot for owner o / my slot at o
            const uint32_t j = h < o ? h : h - 1;
            ptx::bulk_s2s(ptx::mapa(ptx::smem_u32(rx + static_cast<size_t>(j) * RPS * RS), o),
                          ptx::smem_u32(snd + static_cast<size_t>(i) * RPS * RS), share_bytes,
                          ptx::mapa(ptx::smem_u32(rx_full), o));
        }
    }
    ptx::mbar_wait_cluster(rx_full, 0);  // the peers' partials of my rows have landed
#ifdef MPB_ROUTER_TRACE
    if (t == 0) RTRACE(15, gtime());
#endif
    // sum + top-k of the RPS owned rows (tail_select): one warp per row
    if (S == 4)
        tail_select<N, KMAX, 4>(p, rx, tile, h, warp - 4u, lane, row_tile0, out_row_tile0);
    else
        tail_select<N, KMAX, 8>(p, rx, tile, h, warp - 4u, lane, row_tile0, out_row_tile0);
#ifdef MPB_ROUTER_TRACE
    if (t == 0) RTRACE(6, gtime());
#endif
    }
}

// Hands an accumulator's TMEM back to the MMA issuer after this thread's
// tcgen05.ld reads: single CTA — every epilogue thread arrives; pair — one lane
// per warp arrives on the LEADER's barrier (locally or through DSMEM).
template <bool PAIR>
__device__ __forceinline__ void release_tmem(uint64_t *bar, uint32_t rank, uint32_t lane) {
    ptx::tc_fence_before();
    if constexpr (PAIR) {
        __syncwarp();
        if (lane == 0) {
            if (rank == 0)
                ptx::mbar_arrive(bar);
            else
                ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(bar), 0));
        }
    } else {
        ptx::mbar_arrive(bar);
    }
}

// PAIR = false: one CTA per 128-token tile, UMMA M=128 x N (cta_group::1).
// PAIR = true : a 2-CTA cluster per 256-token tile, UMMA M=256 x N issued by the
//   leader with cta_group::2 — each CTA stages its own 128 X rows and HALF of
//   W's rows; the tensor cores read the peer's operands across the SM pair, so
//   W's L2->SM traffic per FLOP halves. Each CTA's TMEM holds full 256-expert
//   rows for its 128 tokens, so the top-k epilogue stays CTA-local.
template <int N, int KMAX, bool PAIR>
__global__ void __launch_bounds__(kThreadsR, 1)
    k_router(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
             RouterParams p) {
    using Cfg = RCfg<N, KMAX, PAIR>;
    constexpr int S = Cfg::STAGES;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned (SW128 operands); offset arithmetic on smem_raw keeps the
    // pointers in the shared window, so the epilogue's park / merge rows compile
    // to LDS / STS rather than generic loads and stores
    uint8_t *base = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *sA = base;
    uint8_t *sB = base + S * Cfg::A_BYTES;
    float *s_park = reinterpret_cast<float *>(base + S * Cfg::STAGE);
    uint64_t *full = reinterpret_cast<uint64_t *>(base + S * Cfg::STAGE + Cfg::PARK);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + 2;
    uint64_t *peer_free = tempty + 2;  // cluster tail: peers' pipeline smem is free (S-1 arrivals)
    uint64_t *rx_full = peer_free + 1;  // cluster tail: peers' partials of my rows (tx bytes)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rx_full + 1);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = PAIR ? ptx::cluster_ctarank() : 0u;
    const uint32_t unit = PAIR ? blockIdx.x >> 1 : blockIdx.x;     // tile-scheduling unit
    const uint32_t units = PAIR ? gridDim.x >> 1 : gridDim.x;
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(p.maps ? p.maps : &tmX);
        ptx::tma_prefetch_desc(p.maps ? p.maps + 1 : &tmW);
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            // single: every epilogue thread arrives; pair: one lane per epilogue
            // warp of both CTAs arrives on the leader's barrier
            ptx::mbar_init(&tempty[a], PAIR ? 16 : 256);
        }
        if (!PAIR && p.cluster_tail) {
            ptx::mbar_init(peer_free, p.splits - 1);
            ptx::mbar_init(rx_full, 1);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) {
        if constexpr (PAIR)
            ptx::tmem_alloc_2sm<Cfg::TMEM_COLS>(tmem_slot);
        else
            ptx::tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
    }
    ptx::tc_fence_before();
    if (PAIR || p.cluster_tail)
        ptx::cluster_sync();  // barrier inits visible to the peers before any remote arrive
    else
        __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t nk = p.H / kStageK;
    // PDL: setup above overlapped the previous kernel; X, W, idx/w and the
    // split-tail workspace are touched only after it completed
    if (threadIdx.x == 0) RTRACE(0, gtime());
    pdl_trigger();
    pdl_wait();
    if (threadIdx.x == 0) RTRACE(1, gtime());

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer ----------------
        const uint64_t pol_x = ptx::policy_evict_first();
        const uint64_t pol_w = ptx::policy_evict_last();
        int stage = 0;
        uint32_t phase = 0;
        WorkItem it;
        // X L2 prefetch cursor, kPrefetch k-steps ahead of the loads in the same
        // (tile, k-block) order: HBM latency is covered by L2 prefetches that hold
        // no shared memory, so the smem ring only has to cover the L2 latency
        uint32_t pn = 0, pkb = 0;
        WorkItem pit;
        bool pvalid = kPrefetch > 0 && next_item(0, unit, units, p.num_tiles, nk, p.splits, pit);
        if (pvalid) pkb = pit.k0;
        auto prefetch_one = [&]() {
            if (!pvalid) return;
            const uint32_t pl = pit.tile / p.tiles_per_layer;
            ptx::tma_prefetch_2d(p.maps ? p.maps + 2 * pl : &tmX, static_cast<int32_t>(pkb * kStageK),
                                 static_cast<int32_t>((pit.tile - pl * p.tiles_per_layer) * Cfg::ROWS_PER_TILE +
                                                      rank * kBM));
            if (++pkb >= pit.k1) {
                pvalid = next_item(++pn, unit, units, p.num_tiles, nk, p.splits, pit);
                if (pvalid) pkb = pit.k0;
            }
        };
        if constexpr (kPrefetch > 0)
            for (uint32_t i = 0; i < kPrefetch; ++i) prefetch_one();
        for (uint32_t n = 0; next_item(n, unit, units, p.num_tiles, nk, p.splits, it); ++n) {
            const uint32_t layer = it.tile / p.tiles_per_layer;
            const int32_t m0 = static_cast<int32_t>((it.tile - layer * p.tiles_per_layer) * Cfg::ROWS_PER_TILE +
                                                    rank * kBM);
            const CUtensorMap *mX = p.maps ? p.maps + 2 * layer : &tmX;
            const CUtensorMap *mW = p.maps ? p.maps + 2 * layer + 1 : &tmW;
            for (uint32_t kb = it.k0; kb < it.k1; ++kb) {
                prefetch_one();
#ifdef MPB_ROUTER_TRACE
                if (n == 0 && kb == it.k0) RTRACE(2, gtime());
#endif
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                if constexpr (PAIR) {
#if (defined(MPB_EXP) && MPB_EXP == 1) || defined(MPB_EXP_FEEDNOW)  // experiment: W for the first tile only
                    const bool wl = n == 0;
#else
                    constexpr bool wl = true;
#endif
#if defined(MPB_EXP) && MPB_EXP == 2  // experiment: X rows from an L2-resident window
                    const int32_t mx0 = m0 & 2047;
#else
                    const int32_t mx0 = m0;
#endif
                    // both CTAs' loads complete on the leader's full barrier
                    if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], wl ? 2 * Cfg::STAGE : 2 * Cfg::A_BYTES);
                    const uint32_t bar = ptx::mapa(ptx::smem_u32(&full[stage]), 0);
#pragma unroll
                    for (int j = 0; j < kKB; ++j) {
                        const int32_t kc = static_cast<int32_t>(kb * kStageK + j * kBK);
#if defined(MPB_EXP_CONTIG)  // experiment: the same bytes as one contiguous stream per tile
                        ptx::tma_load_2d_2sm(mX, bar, sA + stage * Cfg::A_BYTES + j * Cfg::A_BLOCK,
                                             0, static_cast<int32_t>(((mx0 / kBM) * nk + kb) * kBM), pol_x);
#else
                        ptx::tma_load_2d_2sm(mX, bar, sA + stage * Cfg::A_BYTES + j * Cfg::A_BLOCK,
                                             kc, mx0, pol_x);
#endif
                        if (wl)
                            ptx::tma_load_2d_2sm(mW, bar, sB + stage * Cfg::B_BYTES + j * Cfg::B_BLOCK,
                                                 kc, static_cast<int32_t>(rank) * (N / 2), pol_w);
                    }
                } else {
                    ptx::mbar_arrive_expect_tx(&full[stage], Cfg::STAGE);
#pragma unroll
                    for (int j = 0; j < kKB; ++j) {
                        const int32_t kc = static_cast<int32_t>(kb * kStageK + j * kBK);
                        ptx::tma_load_2d(mX, &full[stage], sA + stage * Cfg::A_BYTES + j * Cfg::A_BLOCK,
                                         kc, m0, pol_x);
                        ptx::tma_load_2d(mW, &full[stage], sB + stage * Cfg::B_BYTES + j * Cfg::B_BLOCK,
                                         kc, 0, pol_w);
                    }
                }
                if (++stage == S) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1 && lane == 0 && rank == 0) {
        // ---------------- MMA issuer (pair: leader CTA only) ----------------
        constexpr uint32_t idesc = ptx::idesc_bf16_f32<PAIR ? 2 * kBM : kBM, N>();
        int stage = 0;
        uint32_t phase = 0, acc = 0, aphase = 0;
        WorkItem it;
        for (uint32_t n = 0; next_item(n, unit, units, p.num_tiles, nk, p.splits, it); ++n) {
            ptx::mbar_wait(&tempty[acc], aphase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tmem_base + acc * N;
            for (uint32_t kb = it.k0; kb < it.k1; ++kb) {
                ptx::mbar_wait(&full[stage], phase);
                ptx::tc_fence_after();
#pragma unroll
                for (int j = 0; j < kKB; ++j) {
                    const uint64_t ad = ptx::sw128_kmajor_desc(
                        ptx::smem_u32(sA + stage * Cfg::A_BYTES + j * Cfg::A_BLOCK));
                    const uint64_t bd = ptx::sw128_kmajor_desc(
                        ptx::smem_u32(sB + stage * Cfg::B_BYTES + j * Cfg::B_BLOCK));
#if defined(MPB_EXP) && MPB_EXP == 3  // experiment: loads only (no MMAs) — the feed's own rate
                    if (kb != it.k0 + 1) continue;
#endif
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {  // +32 bytes along K per UMMA_K = 16
                        const uint32_t accum = (kb != it.k0) | (j != 0) | (kk != 0);
                        if constexpr (PAIR)
                            ptx::mma_bf16_2sm(d, ad + 2 * kk, bd + 2 * kk, idesc, accum);
                        else
                            ptx::mma_bf16(d, ad + 2 * kk, bd + 2 * kk, idesc, accum);
                    }
                }
                if constexpr (PAIR)
                    ptx::mma_commit_2sm_mc(&empty[stage], 0x3);  // frees the stage in both CTAs
                else
                    ptx::mma_commit(&empty[stage]);
                if (++stage == S) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if constexpr (PAIR)
                ptx::mma_commit_2sm_mc(&tfull[acc], 0x3);
            else
                ptx::mma_commit(&tfull[acc]);
            RTRACE(3, gtime());
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: one token row per thread pair ----------------
        // Warp w reads TMEM lanes [32q, 32q+32), q = w % 4; warps 4-7 take
        // expert columns [0, N/2) and warps 8-11 [N/2, N) of the same rows, so
        // two warps per SM sub-partition hide each other's latency.
        // Columns are scanned in ascending expert id: a new value displaces a
        // kept entry only if strictly larger (equal logits keep the lower id),
        // so the per-column test is one compare against the current k-th
        // value, and an insertion is a branch-free shift of a sorted register
        // list (values parked in smem so one copy of the network serves all
        // columns). The column-half lists merge through smem (half 1's ids are
        // all larger). NaN / -inf logits only fill slots the others leave empty.
        const uint32_t q = warp & 3, half = (warp - 4) >> 2;
        const uint32_t row_in_tile = q * 32 + lane;
        float *park = s_park + ((half * 128) + row_in_tile) * Cfg::PARK_ROW;
        float *peer = s_park + (128 + row_in_tile) * Cfg::PARK_ROW;
        constexpr int NH = N / 2;
        const int off = KMAX - static_cast<int>(p.k);
        uint32_t acc = 0, aphase = 0;
        WorkItem it;
        for (uint32_t n = 0; next_item(n, unit, units, p.num_tiles, nk, p.splits, it); ++n) {
            ptx::mbar_wait(&tfull[acc], aphase);
            ptx::tc_fence_after();
#ifdef MPB_ROUTER_TRACE
            if (warp == 4 && lane == 0) {
                RTRACE(4, gtime());
                RTRACE(8, it.role);
                RTRACE(9, n + 1);
            }
#endif
            const uint32_t layer = it.tile / p.tiles_per_layer;
            if (!PAIR && it.role != 0 && p.cluster_tail) {
                const uint64_t r0 = static_cast<uint64_t>(it.tile - layer * p.tiles_per_layer) * Cfg::ROWS_PER_TILE;
                cluster_tail<N, KMAX>(p, it, tmem_base + acc * N + ((q * 32) << 16), base, peer_free,
                                      rx_full, warp, lane, r0, static_cast<uint64_t>(layer) * p.T + r0);
                release_tmem<PAIR>(&tempty[acc], rank, lane);
                acc ^= 1;
                if (acc == 0) aphase ^= 1;
                continue;
            }
            const uint64_t row = static_cast<uint64_t>(it.tile - layer * p.tiles_per_layer) * Cfg::ROWS_PER_TILE +
                                 rank * kBM + row_in_tile;  // token within the layer
            const uint64_t out_row = static_cast<uint64_t>(layer) * p.T + row;
            const uint32_t taddr = tmem_base + acc * N + ((q * 32) << 16);
            if (it.role != 0) {
                // split-K tail: partial [slot][part-1][rank][chunk][quarter][row] float4 — a
                // warp's 16-byte accesses to one (chunk, quarter) cover 512 contiguous bytes
                constexpr size_t kPartFloats = static_cast<size_t>(N) * kBM;
                const size_t part_stride = (PAIR ? 2 : 1) * kPartFloats;  // between K parts
                float *part0 = p.partial + static_cast<size_t>(it.slot) * (p.splits - 1) * part_stride +
                               rank * kPartFloats;
                uint32_t *flag = p.flags + it.slot * (PAIR ? 2 : 1) + rank;
                if (it.role == 2) {
                    float *part = part0 + (it.part - 1) * part_stride;
#pragma unroll 1
                    for (int c = half * NH; c < (half + 1) * NH; c += 16) {
                        uint32_t r[16];
                        ptx::tmem_ld_32x32b_x16(taddr + c, r);
                        ptx::tmem_ld_wait();
                        float4 *dst = reinterpret_cast<float4 *>(part) + (c / 16) * 4 * kBM + row_in_tile;
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            dst[i * kBM] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                                 __uint_as_float(r[4 * i + 2]),
                                                 __uint_as_float(r[4 * i + 3]));
                    }
                    __threadfence();
                    asm volatile("bar.sync 5, 256;" ::: "memory");  // every epilogue thread dumped
                    if (warp == 4 && lane == 0)
                        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(flag) : "memory");
                    release_tmem<PAIR>(&tempty[acc], rank, lane);
                    acc ^= 1;
                    if (acc == 0) aphase ^= 1;
                    continue;
                }
                // role 1: wait for the other K parts, add them into TMEM (in part
                // order: a fixed fp32 summation order), then finish. One thread
                // polls (an acquire load invalidates L1); the named barrier hands
                // its view to the other epilogue threads, whose partial loads go
                // to L2 (ld.cg)
                if (warp == 4 && lane == 0) {
                    uint32_t seen;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(flag) : "memory");
                    } while (seen != p.splits - 1);
                }
                asm volatile("bar.sync 5, 256;" ::: "memory");
#pragma unroll 1
                for (int c = half * NH; c < (half + 1) * NH; c += 16) {
                    uint32_t r[16];
                    ptx::tmem_ld_32x32b_x16(taddr + c, r);
                    const float4 *src =
                        reinterpret_cast<const float4 *>(part0) + (c / 16) * 4 * kBM + row_in_tile;
                    constexpr uint32_t kMaxParts = 4;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        float4 v[kMaxParts - 1];  // every part's float4 in flight at once
#pragma unroll
                        for (uint32_t h = 1; h < kMaxParts; ++h)
                            if (h < p.splits) v[h - 1] = __ldcg(src + (h - 1) * (part_stride / 4) + i * kBM);
                        if (i == 0) ptx::tmem_ld_wait();
#pragma unroll
                        for (uint32_t h = 1; h < kMaxParts; ++h)
                            if (h < p.splits) {
                                r[4 * i] = __float_as_uint(__uint_as_float(r[4 * i]) + v[h - 1].x);
                                r[4 * i + 1] = __float_as_uint(__uint_as_float(r[4 * i + 1]) + v[h - 1].y);
                                r[4 * i + 2] = __float_as_uint(__uint_as_float(r[4 * i + 2]) + v[h - 1].z);
                                r[4 * i + 3] = __float_as_uint(__uint_as_float(r[4 * i + 3]) + v[h - 1].w);
                            }
                    }
                    ptx::tmem_st_32x32b_x16(taddr + c, r);
                }
                ptx::tmem_st_wait();
                // every epilogue thread has read the partial: re-arm the flag for the
                // next launch (self-resetting, so CUDA-graph replays stay correct)
                asm volatile("bar.sync 5, 256;" ::: "memory");
                if (warp == 4 && lane == 0)
                    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(0u) : "memory");
            }
#ifdef MPB_ROUTER_TRACE
            if (warp == 4 && lane == 0) RTRACE(5, gtime());
#endif
            float tv[KMAX];
            int ti[KMAX];
#pragma unroll
            for (int j = 0; j < KMAX; ++j) {
                tv[j] = j < off ? INFINITY : -INFINITY;  // sentinels above, empty slots below
                ti[j] = j < off ? -1 : 0x7FFFFFFF;
            }
            // pass 1 (TMEM reads are cheap): the half-row's max m and a lower bound
            // t0 on its k-th largest logit — the minimum over >= KMAX column groups
            // of each group's maximum (each group holds a logit >= t0, so at least
            // KMAX >= k logits are >= t0). Pass 2 inserts only candidates >= t0: a
            // handful per row instead of nearly every column of the first chunks.
            // NaN never raises a group maximum (an all-NaN or all -inf group gives
            // -inf: no filtering), so the NaN / -inf fill below is unaffected.
            constexpr int GS = NH / KMAX >= 16 ? 16 : NH / KMAX;  // group size, divides 16
            float m = -INFINITY, t0 = INFINITY;
#pragma unroll 1
            for (int c = half * NH; c < (half + 1) * NH; c += 16) {
                uint32_t r[16];
                ptx::tmem_ld_32x32b_x16(taddr + c, r);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int g = 0; g < 16; g += GS) {
                    float gm = -INFINITY;
#pragma unroll
                    for (int i = g; i < g + GS; ++i)
                        if (static_cast<uint32_t>(c + i) < p.E) gm = fmaxf(gm, __uint_as_float(r[i]));
                    t0 = fminf(t0, gm);
                    m = fmaxf(m, gm);
                }
            }
            if (KMAX == 1) t0 = m;
            float *lrow = (p.logits && row < p.T) ? p.logits + out_row * p.E : nullptr;
#ifdef MPB_ROUTER_TRACE
            long long cy_ld = 0, cy_ins = 0, n_ins = 0;
#endif
#pragma unroll 1
            for (int c = half * NH; c < (half + 1) * NH; c += 16) {
                uint32_t r[16];
#ifdef MPB_ROUTER_TRACE
                const long long c0 = clock64();
#endif
                ptx::tmem_ld_32x32b_x16(taddr + c, r);
                ptx::tmem_ld_wait();
#ifdef MPB_ROUTER_TRACE
                const long long c1 = clock64();
                cy_ld += c1 - c0;
#endif
                const bool padded = static_cast<uint32_t>(c + 16) > p.E;
                if (padded)  // padding columns (E < N): -inf, never selected
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (static_cast<uint32_t>(c + i) >= p.E) r[i] = __float_as_uint(-INFINITY);
                if (lrow) {
                    if (!padded && (p.E & 3) == 0) {
                        float4 *dst = reinterpret_cast<float4 *>(lrow + c);
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            dst[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                                 __uint_as_float(r[4 * i + 2]),
                                                 __uint_as_float(r[4 * i + 3]));
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (static_cast<uint32_t>(c + i) < p.E) lrow[c + i] = __uint_as_float(r[i]);
                    }
                }
                const float thr = fmaxf(tv[KMAX - 1], t0);  // v > thr, or v == t0 > tv[KMAX-1]
                uint32_t hit = 0;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float v = __uint_as_float(r[i]);
                    hit |= static_cast<uint32_t>(v > thr || (v == t0 && v > tv[KMAX - 1])) << i;
                }
#ifdef MPB_ROUTER_TRACE
                const long long c2 = clock64();
                n_ins += __popc(hit);
#endif
                if (hit) {
                    while (hit) {
                        const int i = __ffs(hit) - 1;
                        hit &= hit - 1;
                        const float v = pick16(r, i);  // register select tree, no smem round trip
                        const int e = c + i;
                        // sorted-list insertion: slot j takes slot j-1 if v goes above it
#pragma unroll
                        for (int j = KMAX - 1; j >= 0; --j) {
                            const bool here = v > tv[j];
                            const bool above = j > 0 && v > tv[j > 0 ? j - 1 : 0];
                            tv[j] = above ? tv[j > 0 ? j - 1 : 0] : (here ? v : tv[j]);
                            ti[j] = above ? ti[j > 0 ? j - 1 : 0] : (here ? e : ti[j]);
                        }
                    }
                }
#ifdef MPB_ROUTER_TRACE
                cy_ins += clock64() - c2;
#endif
            }
#ifdef MPB_ROUTER_TRACE
            if (warp == 4 && lane == 0) {
                RTRACE(10, gtime());
                RTRACE(13, cy_ld);
                RTRACE(14, cy_ins);
                RTRACE(15, n_ins);
            }
#endif
            float ssum = 0.f;
            if (p.score_fn == MPB_SCORE_SOFTMAX) {
                const float mlog = m * 1.4426950408889634f;
#pragma unroll 1
                for (int c = half * NH; c < (half + 1) * NH; c += 16) {
                    uint32_t r[16];
                    ptx::tmem_ld_32x32b_x16(taddr + c, r);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float v = __uint_as_float(r[i]);
                        const bool real = static_cast<uint32_t>(c + i) < p.E;
                        ssum += (real && v == v) ? exp2f(fmaf(v, 1.4426950408889634f, -mlog)) : 0.f;
                    }
                }
            }
#ifdef MPB_ROUTER_TRACE
            if (warp == 4 && lane == 0) RTRACE(11, gtime());
#endif
            // ---- merge the two column halves (named barrier per lane quadrant)
            if (half == 1) {
#pragma unroll
                for (int j = 0; j < KMAX; ++j) {
                    park[j] = tv[j];
                    park[KMAX + j] = __int_as_float(ti[j]);
                }
                park[2 * KMAX] = m;
                park[2 * KMAX + 1] = ssum;
            }
            asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
            if (half == 1) {
                release_tmem<PAIR>(&tempty[acc], rank, lane);
            } else {
#pragma unroll 1
                for (int jj = off; jj < KMAX; ++jj) {
                    const float v = peer[jj];
                    const int e = __float_as_int(peer[KMAX + jj]);
                    if (!(v > tv[KMAX - 1])) break;  // peer list is sorted
#pragma unroll
                    for (int j = KMAX - 1; j >= 0; --j) {
                        const bool here = v > tv[j];
                        const bool above = j > 0 && v > tv[j > 0 ? j - 1 : 0];
                        tv[j] = above ? tv[j > 0 ? j - 1 : 0] : (here ? v : tv[j]);
                        ti[j] = above ? ti[j > 0 ? j - 1 : 0] : (here ? e : ti[j]);
                    }
                }
                const float m1 = peer[2 * KMAX], s1 = peer[2 * KMAX + 1];
                const float mm = fmaxf(m, m1);
                if (p.score_fn == MPB_SCORE_SOFTMAX) {
                    const float a0 = m == -INFINITY ? 0.f : exp2f((m - mm) * 1.4426950408889634f);
                    const float a1 = m1 == -INFINITY ? 0.f : exp2f((m1 - mm) * 1.4426950408889634f);
                    ssum = ssum * a0 + s1 * a1;
                }
                m = mm;
                const bool short_row = ti[KMAX - 1] == 0x7FFFFFFF;
                if (__any_sync(0xffffffffu, short_row)) {
                    // rare: fewer than k logits above -inf — fill with -inf ids, then
                    // NaN ids, ascending (NaN ranks lowest). tcgen05.ld is warp-collective:
                    // the whole warp loads, only the short rows place
#pragma unroll 1
                    for (int pass = 0; pass < 2; ++pass)
#pragma unroll 1
                        for (int c = 0; c < N; c += 16) {
                            uint32_t r[16];
                            ptx::tmem_ld_32x32b_x16(taddr + c, r);
                            ptx::tmem_ld_wait();
#pragma unroll
                            for (int i = 0; i < 16; ++i) {
                                const float v = __uint_as_float(r[i]);
                                const bool want = pass == 0 ? v == -INFINITY : v != v;
                                if (!short_row || !want || static_cast<uint32_t>(c + i) >= p.E) continue;
                                bool placed = false;
#pragma unroll
                                for (int j = 0; j < KMAX; ++j)
                                    if (!placed && ti[j] == 0x7FFFFFFF) {
                                        ti[j] = c + i;
                                        tv[j] = v;
                                        placed = true;
                                    }
                            }
                        }
                }
                release_tmem<PAIR>(&tempty[acc], rank, lane);
#ifdef MPB_ROUTER_TRACE
                if (warp == 4 && lane == 0) RTRACE(12, gtime());
#endif
                if (row < p.T) {
                    const float mlog = m * 1.4426950408889634f;
                    float w[KMAX];
                    float wsum = 0.f;
#pragma unroll
                    for (int j = 0; j < KMAX; ++j) {
                        const float v = tv[j];
                        float x;
                        if (j < off || isnan(v))
                            x = 0.f;
                        else if (p.score_fn == MPB_SCORE_SOFTMAX)
                            x = exp2f(fmaf(v, 1.4426950408889634f, -mlog)) / ssum;
                        else
                            x = 1.f / (1.f + expf(-v));
                        w[j] = x;
                        wsum += x;
                    }
#pragma unroll
                    for (int j = 0; j < KMAX; ++j) {
                        if (j < off) continue;
                        const float x = p.renorm ? (wsum > 0.f ? w[j] / wsum : 0.f) : w[j];
                        p.idx[out_row * p.k + (j - off)] = ti[j];
                        p.w[out_row * p.k + (j - off)] = x;
                        if (p.demand) count_demand(p, row, static_cast<uint32_t>(ti[j]));
                    }
                }
            }
            // half 1 must not overwrite its park row before half 0 read it
            asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
#ifdef MPB_ROUTER_TRACE
            if (warp == 4 && lane == 0) RTRACE(6, gtime());
#endif
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
    }
    ptx::tc_fence_before();
    if (PAIR || p.cluster_tail)
        ptx::cluster_sync();
    else
        __syncthreads();
    if (threadIdx.x == 0) RTRACE(7, gtime());
    if (warp == 2) {
        ptx::tc_fence_after();
        if constexpr (PAIR)
            ptx::tmem_dealloc_2sm<Cfg::TMEM_COLS>(tmem_base);
        else
            ptx::tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

bool make_map(CUtensorMap *map, const void *ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
#ifdef MPB_EXP_PROMO
                    static_cast<CUtensorMapL2promotion>(MPB_EXP_PROMO),
#else
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
#endif
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// How many clusters of S CTAs of this kernel can be resident at once (the
// split tail's CTAs wait on each other, so its units must all be resident);
// cached per (kernel, S).
template <typename K>
uint32_t max_active_clusters(K kern, int smem, uint32_t S) {
    static std::mutex mu;
    static std::map<std::pair<const void *, uint32_t>, uint32_t> cache;
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_pair(reinterpret_cast<const void *>(kern), S);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    cfg.gridDim = dim3(S * 64);
    cfg.blockDim = dim3(kThreadsR);
    cfg.dynamicSmemBytes = smem;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
    cudaGetLastError();
    cache[key] = static_cast<uint32_t>(n);
    return static_cast<uint32_t>(n);
}

template <int N, int KMAX, bool PAIR>
mpb_status launch_router_n(mpb_context *ctx, const CUtensorMap &mx, const CUtensorMap &mw,
                           RouterParams p) {
    using Cfg = RCfg<N, KMAX, PAIR>;
    constexpr int smem = Cfg::SMEM;
    auto kern = k_router<N, KMAX, PAIR>;
    MPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[2];
    cfg.blockDim = dim3(kThreadsR);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    uint32_t units;
    p.tiles_per_layer = static_cast<uint32_t>((p.T + Cfg::ROWS_PER_TILE - 1) / Cfg::ROWS_PER_TILE);
    p.num_tiles = p.tiles_per_layer * p.layers;
    if constexpr (PAIR)
        units = std::min<uint32_t>(p.num_tiles, static_cast<uint32_t>(ctx->num_sms) / 2);
    else
        units = std::min<uint32_t>(p.num_tiles, static_cast<uint32_t>(ctx->num_sms));
    // split-K tail: when the last wave would leave at least half the units idle,
    // its tiles are split in S K parts over S times as many units (S <= 4, at
    // least kMinPartK k-steps per part); S = 2 for every multi-wave shape so far
    // (DSv3, Maverick), up to 4 for small decode batches (a few tiles only)
    const uint32_t full_units = PAIR ? static_cast<uint32_t>(ctx->num_sms) / 2
                                     : static_cast<uint32_t>(ctx->num_sms);
    const uint32_t nk = p.H / kStageK;
    const uint32_t waves = p.num_tiles / full_units;
    const uint32_t rem = p.num_tiles - waves * full_units;
    constexpr uint32_t kMaxSplits = 4, kMinPartK = 4;  // 8 measured slower at T=1024 (fix-up); <= the epilogue's kMaxParts
    uint32_t S = 1;
    if (rem > 0 && !std::getenv("MPB_ROUTER_NO_SPLIT")) {
        S = std::min(full_units / rem, kMaxSplits);
        if (const char *e = std::getenv("MPB_ROUTER_MAX_SPLITS")) S = std::min<uint32_t>(S, std::atoi(e));
        S = std::min(S, std::max<uint32_t>(nk / kMinPartK, nk >= 2 ? 2u : 1u));
        if (S < 2 || nk < 2) S = 1;
    }
    // single-CTA tiles: the split tail runs through distributed shared memory,
    // the S K parts of a tile in one cluster (S a power of two dividing the units)
    // When some SMs cannot host a whole cluster (GPC granularity) the split runs
    // on the resident clusters if every tile is in the tail (decode batches);
    // otherwise (whole waves before the tail) only if all units fit.
    bool ct = false;
    if (!PAIR && N <= 128 && S > 1 && !std::getenv("MPB_ROUTER_GLOBAL_TAIL")) {
        if (S == 3) S = 2;
        const uint32_t cap = std::min(full_units, max_active_clusters(kern, smem, S) * S) / S * S;
        if (waves == 0 && S * rem <= cap) {
            ct = true;
            units = cap;
        } else if (cap == full_units && full_units % S == 0) {
            ct = true;
            units = full_units;
        }
    }
    p.splits = S;
    const char *sa = std::getenv("MPB_ROUTER_ST_ASYNC");
    p.cluster_tail = ct ? ((sa && sa[0] == '1') ? 2u : 1u) : 0u;
    if (S > 1 && ct) {
        // units set above
    } else if (S > 1) {
        units = full_units;
        const size_t ranks = PAIR ? 2 : 1;
        const size_t flag_bytes = 4096;
        const size_t need = flag_bytes + size_t(rem) * (S - 1) * ranks * N * kBM * sizeof(float);
        MPB_CUDA(ctx->grow(&ctx->router_ws, &ctx->router_ws_bytes, need, 0, flag_bytes));
        // flags: count of K parts > 0 whose partial is ready (reset by the finisher)
        p.flags = static_cast<uint32_t *>(ctx->router_ws);
        p.partial = reinterpret_cast<float *>(static_cast<char *>(ctx->router_ws) + flag_bytes);
    }
    if constexpr (PAIR) {
        cfg.gridDim = dim3(2 * units);
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    } else if (ct) {
        cfg.gridDim = dim3(units);
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = S;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    } else {
        cfg.gridDim = dim3(units);
        cfg.attrs = attr;
        cfg.numAttrs = 0;
    }
    // PDL only when this context owns the whole GPU: an early-launched CTA may
    // land on (and spin on) an SM outside the context's budget, starving the
    // kernels that another context runs there
    if (pdl_enabled() && (ctx->num_sms == ctx->device_sms || ctx->confined)) {
        attr[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
        ++cfg.numAttrs;
    }
    MPB_CUDA(cudaLaunchKernelEx(&cfg, kern, mx, mw, p));
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

template <int N, bool PAIR>
mpb_status launch_router_k(mpb_context *ctx, const CUtensorMap &mx, const CUtensorMap &mw,
                           const RouterParams &p) {
    if (p.k <= 1) return launch_router_n<N, 1, PAIR>(ctx, mx, mw, p);
    if (p.k <= 2) return launch_router_n<N, 2, PAIR>(ctx, mx, mw, p);
    if (p.k <= 4) return launch_router_n<N, 4, PAIR>(ctx, mx, mw, p);
    if (p.k <= 8) return launch_router_n<N, 8, PAIR>(ctx, mx, mw, p);
    return launch_router_n<N, 16, PAIR>(ctx, mx, mw, p);
}

}  // namespace
}  // namespace mpb

using namespace mpb;

namespace {
// shared validation + tile-width choice of the single and grouped entry points
mpb_status router_check(const char *fn, uint64_t T, uint32_t H, uint32_t E, uint32_t k, int score_fn) {
    if (E == 0 || E > 256) return fail(MPB_CONFIG_ERROR, std::string(fn) + ": need 1 <= E <= 256");
    if (H == 0 || H % kStageK != 0)
        return fail(MPB_CONFIG_ERROR, std::string(fn) + ": H must be a multiple of " + std::to_string(kStageK));
    if (k == 0 || k > 16 || k > E) return fail(MPB_CONFIG_ERROR, std::string(fn) + ": need 1 <= k <= 16");
    if (score_fn != MPB_SCORE_SOFTMAX && score_fn != MPB_SCORE_SIGMOID)
        return fail(MPB_CONFIG_ERROR, std::string(fn) + ": unknown score_fn");
    if (T > 0x7fffffffull) return fail(MPB_CONFIG_ERROR, std::string(fn) + ": T too large");
    return MPB_OK;
}

// E = 256 (tensor-bound): 2-SM CTA pairs (UMMA M=256) by default;
// MPB_ROUTER_SINGLE=1 forces the single-CTA kernel. E <= 128 is HBM-bound:
// single-CTA tiles already stream X at the HBM roofline. The tile width N is
// the next of 64 / 128 / 256: W rows past E come in as TMA out-of-bounds zeros
// and their columns are masked in the epilogue.
uint32_t router_tile_n(uint32_t E, bool *pair) {
    const char *v = std::getenv("MPB_ROUTER_SINGLE");
    const bool single = v && v[0] == '1';
    const uint32_t N = E <= 64 ? 64 : E <= 128 ? 128 : 256;
    *pair = N == 256 && !single;
    return N;
}

mpb_status router_dispatch(mpb_context *ctx, uint32_t N, bool pair, const CUtensorMap &mx,
                           const CUtensorMap &mw, const RouterParams &p) {
    if (pair) return launch_router_k<256, true>(ctx, mx, mw, p);
    if (N == 64) return launch_router_k<64, false>(ctx, mx, mw, p);
    if (N == 128) return launch_router_k<128, false>(ctx, mx, mw, p);
    return launch_router_k<256, false>(ctx, mx, mw, p);
}
}  // namespace

extern "C" mpb_status mpb_router_topk(mpb_context *ctx, const void *X, const void *W, uint64_t T,
                                      uint32_t H, uint32_t E, uint32_t k, int score_fn, int renorm,
                                      int32_t *idx, float *weights, float *logits_out) {
    if (!ctx || (T && (!X || !W || !idx || !weights)))
        return fail(MPB_VALIDATION_ERROR, "mpb_router_topk: NULL argument");
    if (mpb_status st = router_check("mpb_router_topk", T, H, E, k, score_fn)) return st;
    if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(W)) & 15)
        return fail(MPB_CONFIG_ERROR, "mpb_router_topk: X and W must be 16-byte aligned");
    if (T == 0) return MPB_OK;
    RouterParams p{T, H, k, score_fn, renorm, 0, idx, weights, logits_out, 1, nullptr, nullptr, E,
                   nullptr, 0, 1, 0, nullptr, nullptr, nullptr, nullptr, 0, nullptr};
    bool pair;
    const uint32_t N = router_tile_n(E, &pair);
    CUtensorMap mx, mw;
    if (!make_map(&mx, X, T, H, kBM) || !make_map(&mw, W, E, H, pair ? N / 2 : N))
        return fail(MPB_CUDA_ERROR, "mpb_router_topk: cuTensorMapEncodeTiled failed");
    return router_dispatch(ctx, N, pair, mx, mw, p);
}

extern "C" mpb_status mpb_router_topk_demand(mpb_context *ctx, const void *X, const void *W, uint64_t T,
                                             uint32_t H, uint32_t E, uint32_t k, int score_fn, int renorm,
                                             int32_t *idx, float *weights, float *logits_out,
                                             const uint8_t *src_group, const uint8_t *src_group2,
                                             uint32_t D, uint64_t *demand, uint64_t *demand2) {
    if (!ctx || (T && (!X || !W || !idx || !weights || !src_group || !demand)) || (src_group2 && !demand2))
        return fail(MPB_VALIDATION_ERROR, "mpb_router_topk_demand: NULL argument");
    if (mpb_status st = router_check("mpb_router_topk_demand", T, H, E, k, score_fn)) return st;
    if (D == 0 || D > 255) return fail(MPB_CONFIG_ERROR, "mpb_router_topk_demand: need 1 <= D <= 255");
    if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(W)) & 15)
        return fail(MPB_CONFIG_ERROR, "mpb_router_topk_demand: X and W must be 16-byte aligned");
    if (T == 0) return MPB_OK;
    RouterParams p{T, H, k, score_fn, renorm, 0, idx, weights, logits_out, 1, nullptr, nullptr, E,
                   nullptr, 0, 1, 0, src_group, src_group2,
                   reinterpret_cast<unsigned long long *>(demand),
                   src_group2 ? reinterpret_cast<unsigned long long *>(demand2) : nullptr, D, ctx->d_error};
    bool pair;
    const uint32_t N = router_tile_n(E, &pair);
    CUtensorMap mx, mw;
    if (!make_map(&mx, X, T, H, kBM) || !make_map(&mw, W, E, H, pair ? N / 2 : N))
        return fail(MPB_CUDA_ERROR, "mpb_router_topk_demand: cuTensorMapEncodeTiled failed");
    return router_dispatch(ctx, N, pair, mx, mw, p);
}

extern "C" mpb_status mpb_router_topk_layers(mpb_context *ctx, uint32_t layers, const void *const *X,
                                             const void *const *W, uint64_t T, uint32_t H, uint32_t E,
                                             uint32_t k, int score_fn, int renorm, int32_t *idx,
                                             float *weights, float *logits_out) {
    if (!ctx || (layers && T && (!X || !W || !idx || !weights)))
        return fail(MPB_VALIDATION_ERROR, "mpb_router_topk_layers: NULL argument");
    if (mpb_status st = router_check("mpb_router_topk_layers", T, H, E, k, score_fn)) return st;
    if (layers == 0 || T == 0) return MPB_OK;
    if (static_cast<uint64_t>(layers) * ((T + kBM - 1) / kBM) > 0xffffffffull)
        return fail(MPB_CONFIG_ERROR, "mpb_router_topk_layers: too many tiles");
    for (uint32_t l = 0; l < layers; ++l) {
        if (!X[l] || !W[l]) return fail(MPB_VALIDATION_ERROR, "mpb_router_topk_layers: NULL X / W");
        if ((reinterpret_cast<uintptr_t>(X[l]) | reinterpret_cast<uintptr_t>(W[l])) & 15)
            return fail(MPB_CONFIG_ERROR, "mpb_router_topk_layers: X and W must be 16-byte aligned");
    }
    bool pair;
    const uint32_t N = router_tile_n(E, &pair);
    // descriptor table: encoded and uploaded once per (shape, pointers); the
    // kernel reads the descriptors from global memory
    std::vector<uint64_t> key{T, H, E, N, pair ? 1u : 0u};
    for (uint32_t l = 0; l < layers; ++l) {
        key.push_back(reinterpret_cast<uint64_t>(X[l]));
        key.push_back(reinterpret_cast<uint64_t>(W[l]));
    }
    auto it = ctx->router_maps.find(key);
    if (it == ctx->router_maps.end()) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        MPB_CUDA(cudaStreamIsCapturing(ctx->stream, &cs));
        if (cs != cudaStreamCaptureStatusNone)
            return fail(MPB_CONFIG_ERROR,
                        "mpb_router_topk_layers: first call for these buffers inside a stream capture "
                        "(call once before capturing)");
        if (ctx->router_maps.size() >= 256) {  // bounded lookup; captured graphs may still read the
            for (auto &kv : ctx->router_maps) ctx->retired.push_back(kv.second);  // old tables
            ctx->router_maps.clear();
        }
        std::vector<CUtensorMap> maps(2 * static_cast<size_t>(layers));
        for (uint32_t l = 0; l < layers; ++l)
#if defined(MPB_EXP_CONTIG)
            if (!make_map(&maps[2 * l], X[l], T * H / kBK, kBK, kBM) ||
#else
            if (!make_map(&maps[2 * l], X[l], T, H, kBM) ||
#endif
                !make_map(&maps[2 * l + 1], W[l], E, H, pair ? N / 2 : N))
                return fail(MPB_CUDA_ERROR, "mpb_router_topk_layers: cuTensorMapEncodeTiled failed");
        void *d = nullptr;
        MPB_CUDA(cudaMalloc(&d, maps.size() * sizeof(CUtensorMap)));
        const cudaError_t e = cudaMemcpy(d, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(d);
            return cuda_fail(e, "mpb_router_topk_layers");
        }
        it = ctx->router_maps.emplace(std::move(key), d).first;
    }
    RouterParams p{T, H, k, score_fn, renorm, 0, idx, weights, logits_out, 1, nullptr, nullptr, E,
                   static_cast<const CUtensorMap *>(it->second), 0, layers, 0, nullptr, nullptr, nullptr,
                   nullptr, 0, nullptr};
    CUtensorMap unused{};
    return router_dispatch(ctx, N, pair, unused, unused, p);
}

#ifdef MPB_ROUTER_TRACE
extern "C" __attribute__((visibility("default"))) int mpb_debug_router_trace(unsigned long long *out,
                                                                             size_t n) {
    if (!out) {  // reset
        static unsigned long long zeros[2 * 148 * 16] = {};
        return cudaMemcpyToSymbol(g_router_trace, zeros, sizeof(zeros)) == cudaSuccess ? 0 : 9;
    }
    return cudaMemcpyFromSymbol(out, g_router_trace, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : 9;
}
#endif
