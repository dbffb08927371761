// K2 dispatch histograms + K3 stable token permutation (sm_100a).
//
// Replaces the per-(request, expert) accounting loop of simulate_layer
// (/root/reference/proj/core/src/simulator.cpp:64-88) at token granularity
// and adds the permutation the reference never materialises.
//
// HBM layout: idx[T*k] int32 (pair p = t*k + j), src_group[T] / tag[T] uint8.
// Three launches, all streaming idx with coalesced 128-bit loads:
//   1. count   : per block (2048 pairs) shared-memory-privatised histograms
//                (demand[src][e], demand2[src2][e] for a second routing of the
//                same tokens, tag_pop[tag][e]); the block's slot counts are
//                derived from its demand cells (one add per non-zero cell, not
//                per pair); bins flushed with one global atomic each, slot
//                counts written block-major as bhist[block][slot].
//   2. scan    : one CTA per 32 slots scans their bhist columns down the block
//                axis (exclusive, in place) and writes the slot totals.
//   3. scatter : every block scans the NS slot totals in smem (slot bases; block
//                0 emits key_offsets), re-reads its chunk (L2-resident), ranks
//                pairs stably inside each warp (per-warp slot counters; the
//                rank among lower lanes from per-bit ballots of the slot id,
//                no MATCH.ANY) and writes sorted_pairs / pair_pos.
// Algorithmic bytes per pair: 4 (idx) + 8 (perm out) [+ 1/k src + 1/k tag].
#include <algorithm>
#include <cstdlib>

#include "internal.cuh"

namespace mpb {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kChunkQuantum = kWarps * 128;  // block chunks: multiples of 1024 pairs
constexpr uint32_t kNone = 0xFFFFFFFFu;

struct LayoutParams {
    const int32_t *idx;
    uint64_t P;  // T * k
    uint64_t T;
    uint32_t k;
    const uint8_t *src_group;
    uint32_t src_base, src_span;
    const uint16_t *tag;
    uint32_t n_tags;
    const uint8_t *src2;
    const uint8_t *g2n;
    const uint16_t *slot_lut;
    const uint16_t *cell_slot;  // [D][E]: slot of a pair from source group s to expert e
    uint32_t D, E, NS;
    uint64_t *demand;
    uint64_t *demand2;
    uint64_t *tag_pop;
    uint32_t *bhist;   // [nblocks][NS] block-major
    uint32_t *totals;  // [NS]
    uint32_t nb;
    uint32_t chunk;     // pairs per block (multiple of kChunkQuantum)
    uint32_t key_bits;  // bits of a slot id with kNone mapped to all-ones (NS < 2^key_bits - 1)
    uint32_t *err;
    int demand_smem;
    int cell_smem;
    int demand2_smem;
    int tag_smem;
};

__device__ __forceinline__ uint32_t source_of(const LayoutParams &p, uint64_t t) {
    return p.src_group ? static_cast<uint32_t>(p.src_group[t])
                       : p.src_base + static_cast<uint32_t>((t * p.src_span) / p.T);
}

__device__ __forceinline__ bool vec_ok(const int32_t *base, uint64_t q, uint64_t P) {
    return q + 3 < P && ((reinterpret_cast<uintptr_t>(base + q) & 15) == 0);
}

// Loads pairs q..q+3 (128-bit when aligned and in range).
__device__ __forceinline__ void load4(const int32_t *idx, uint64_t q, uint64_t P, int32_t v[4]) {
    if (vec_ok(idx, q, P)) {
        int4 x = __ldg(reinterpret_cast<const int4 *>(idx + q));
        v[0] = x.x;
        v[1] = x.y;
        v[2] = x.z;
        v[3] = x.w;
    } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = q + c < P ? __ldg(idx + q + c) : -1;
    }
}

// Resolves pair (t, e): slot id (kNone if invalid), flags errors.
__device__ __forceinline__ uint32_t resolve(const LayoutParams &p, uint64_t pair, int32_t e,
                                            uint32_t &src_out, uint64_t &t_out) {
    if (pair >= p.P) return kNone;
    const uint64_t t = pair / p.k;
    const uint32_t src = source_of(p, t);
    t_out = t;
    src_out = src;
    if (e < 0 || static_cast<uint32_t>(e) >= p.E) {
        atomicOr(p.err, kErrExpertRange);
        return kNone;
    }
    if (src >= p.D) {
        atomicOr(p.err, kErrSourceRange);
        return kNone;
    }
    const uint32_t n = p.g2n[src];
    const uint16_t slot = __ldg(p.slot_lut + static_cast<size_t>(n) * p.E + e);
    if (slot == 0xFFFF) {
        atomicOr(p.err, kErrUncovered);
        return kNone;
    }
    return slot;
}

// Per-token fields of the pairs q..q+3 (pair ids < 2^31, so 32-bit math):
// one division per 4 pairs, token loads only when the token changes.
struct TokenCursor {
    uint32_t t, r, src, s2, tg;
};

__device__ __forceinline__ void load_token(const LayoutParams &p, TokenCursor &c) {
    if (c.t >= p.T) return;
    c.src = p.src_group ? static_cast<uint32_t>(__ldg(p.src_group + c.t))
                        : p.src_base + static_cast<uint32_t>((uint64_t(c.t) * p.src_span) / p.T);
    c.s2 = p.src2 ? static_cast<uint32_t>(__ldg(p.src2 + c.t)) : 0u;
    c.tg = p.tag ? static_cast<uint32_t>(__ldg(p.tag + c.t)) : kNone;
}

__device__ __forceinline__ void cursor_start(const LayoutParams &p, uint32_t q, TokenCursor &c) {
    c.t = q / p.k;
    c.r = q - c.t * p.k;
    load_token(p, c);
}

__device__ __forceinline__ void cursor_next(const LayoutParams &p, TokenCursor &c) {
    if (++c.r == p.k) {
        c.r = 0;
        ++c.t;
        load_token(p, c);
    }
}

template <bool kPerm>
__device__ __forceinline__ void count_body(const LayoutParams &p, uint32_t *sm) {
    const uint32_t DE = p.D * p.E;
    uint32_t *s_demand = sm;
    uint32_t *s_demand2 = s_demand + (p.demand_smem ? DE : 0);
    uint32_t *s_tag = s_demand2 + (p.demand2_smem ? DE : 0);
    uint32_t *s_slot = s_tag + (p.tag_smem ? p.n_tags * p.E : 0);
    const uint32_t nsm = (p.demand_smem ? DE : 0) + (p.demand2_smem ? DE : 0) +
                         (p.tag_smem ? p.n_tags * p.E : 0) + (kPerm ? p.NS : 0);
    // the (source, expert) -> slot table, staged for the flush
    uint16_t *s_cell = reinterpret_cast<uint16_t *>(sm + nsm);
    pdl_trigger();
    if (kPerm && p.cell_smem)  // placement data: not produced by earlier kernels
        for (uint32_t i = threadIdx.x; i < DE; i += kThreads) s_cell[i] = __ldg(p.cell_slot + i);
    for (uint32_t i = threadIdx.x; i < nsm; i += kThreads) sm[i] = 0;
    pdl_wait();
    __syncthreads();

    const uint32_t base = blockIdx.x * p.chunk;
    const uint32_t P = static_cast<uint32_t>(p.P);
    const uint32_t rounds = p.chunk / (kThreads * 4);
    if (p.demand_smem && (!p.src2 || p.demand2_smem) && (!p.tag || p.tag_smem)) {
        // fast path: every histogram is block-private; coverage is checked per
        // non-zero cell at flush time instead of per pair
#pragma unroll 2
        for (uint32_t h = 0; h < rounds; ++h) {
            const uint32_t q = base + h * kThreads * 4 + threadIdx.x * 4;
            if (q >= P) break;
            int32_t v[4];
            load4(p.idx, q, p.P, v);
            TokenCursor tc;
            cursor_start(p, q, tc);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (c) cursor_next(p, tc);
                if (q + c >= P) break;
                const uint32_t e = static_cast<uint32_t>(v[c]);
                if (e >= p.E) {
                    atomicOr(p.err, kErrExpertRange);
                    continue;
                }
                if (tc.src >= p.D) {
                    atomicOr(p.err, kErrSourceRange);
                    continue;
                }
                atomicAdd(s_demand + tc.src * p.E + e, 1u);
                if (p.src2) {
                    if (tc.s2 < p.D)
                        atomicAdd(s_demand2 + tc.s2 * p.E + e, 1u);
                    else
                        atomicOr(p.err, kErrSourceRange);
                }
                if (tc.tg < p.n_tags) atomicAdd(s_tag + tc.tg * p.E + e, 1u);
            }
        }
    } else {
    for (uint32_t h = 0; h < rounds; ++h) {
        const uint64_t q = base + static_cast<uint64_t>(h) * kThreads * 4 + threadIdx.x * 4;
        int32_t v[4];
        load4(p.idx, q, p.P, v);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t src = 0;
            uint64_t t = 0;
            const uint32_t slot = resolve(p, q + c, v[c], src, t);
            if (slot == kNone) continue;
            const uint32_t e = static_cast<uint32_t>(v[c]);
            if (p.demand_smem) {
                atomicAdd(s_demand + src * p.E + e, 1u);
            } else {
                atomicAdd(reinterpret_cast<unsigned long long *>(p.demand) + src * p.E + e, 1ull);
                if (kPerm) atomicAdd(s_slot + slot, 1u);
            }
            if (p.src2) {
                const uint32_t s2 = p.src2[t];
                if (s2 >= p.D) {
                    atomicOr(p.err, kErrSourceRange);
                } else if (p.demand2_smem) {
                    atomicAdd(s_demand2 + s2 * p.E + e, 1u);
                } else {
                    atomicAdd(reinterpret_cast<unsigned long long *>(p.demand2) + s2 * p.E + e,
                              1ull);
                }
            }
            if (p.tag) {
                const uint32_t tg = p.tag[t];
                if (tg < p.n_tags) {
                    if (p.tag_smem)
                        atomicAdd(s_tag + tg * p.E + e, 1u);
                    else
                        atomicAdd(reinterpret_cast<unsigned long long *>(p.tag_pop) + tg * p.E + e,
                                  1ull);
                }
            }
        }
    }
    }
    __syncthreads();
    if (p.demand_smem) {
#pragma unroll 4
        for (uint32_t i = threadIdx.x; i < DE; i += kThreads) {
            const uint32_t c = s_demand[i];
            // the block's slot counts (and coverage) from its (src, expert) cells
            const uint16_t slot = (kPerm && p.cell_smem) ? s_cell[i] : __ldg(p.cell_slot + i);
            if (!c) continue;
            if (slot == 0xFFFF) {
                atomicOr(p.err, kErrUncovered);
                continue;
            }
            atomicAdd(reinterpret_cast<unsigned long long *>(p.demand) + i,
                      static_cast<unsigned long long>(c));
            if (kPerm) atomicAdd(s_slot + slot, c);
        }
    }
    if (p.demand2_smem)
#pragma unroll 4
        for (uint32_t i = threadIdx.x; i < DE; i += kThreads)
            if (s_demand2[i])
                atomicAdd(reinterpret_cast<unsigned long long *>(p.demand2) + i,
                          static_cast<unsigned long long>(s_demand2[i]));
    if (p.tag && p.tag_smem)
#pragma unroll 4
        for (uint32_t i = threadIdx.x; i < p.n_tags * p.E; i += kThreads)
            if (s_tag[i])
                atomicAdd(reinterpret_cast<unsigned long long *>(p.tag_pop) + i,
                          static_cast<unsigned long long>(s_tag[i]));
    if (kPerm) {
        __syncthreads();
        for (uint32_t sl = threadIdx.x; sl < p.NS; sl += kThreads)
            p.bhist[static_cast<size_t>(blockIdx.x) * p.NS + sl] = s_slot[sl];
    }
}

template <bool kPerm>
__global__ void __launch_bounds__(kThreads) k_layout_count(LayoutParams p) {
    extern __shared__ uint32_t sm[];
    count_body<kPerm>(p, sm);
}

// Block-wide exclusive scan of one value per thread (kThreads threads).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *s_warp, uint32_t &total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kWarps ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < kWarps) s_warp[lane] = w;
    }
    __syncthreads();
    total = s_warp[kWarps - 1];
    const uint32_t r = (warp ? s_warp[warp - 1] : 0) + incl - v;
    __syncthreads();
    return r;
}

// One CTA per 32 slots: exclusive scan down the block axis of bhist[.][slot]
// in place + slot totals. Lane = slot (coalesced 128-byte rows); warp w owns a
// contiguous range of blocks: per-warp sums, prefix over warps, then rewrite.
__device__ __forceinline__ void scan_columns(uint32_t *bhist, uint32_t nb, uint32_t NS,
                                             uint32_t *totals, uint32_t group) {
    __shared__ uint32_t s_part[kWarps][32];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t slot = group * 32 + lane;
    const bool ok = slot < NS;
    const uint32_t per = (nb + kWarps - 1) / kWarps;
    const uint32_t b0 = min(nb, warp * per), b1 = min(nb, b0 + per);
    uint32_t *col = bhist + slot;
    uint32_t sum = 0;
    if (ok) {
        uint32_t b = b0;
        for (; b + 8 <= b1; b += 8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = col[static_cast<size_t>(b + u) * NS];
#pragma unroll
            for (int u = 0; u < 8; ++u) sum += v[u];
        }
        for (; b < b1; ++b) sum += col[static_cast<size_t>(b) * NS];
    }
    s_part[warp][lane] = sum;
    __syncthreads();
    uint32_t run = 0;
    for (uint32_t w = 0; w < warp; ++w) run += s_part[w][lane];
    if (warp == kWarps - 1 && ok) totals[slot] = run + sum;
    if (ok) {
        uint32_t b = b0;
        for (; b + 8 <= b1; b += 8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = col[static_cast<size_t>(b + u) * NS];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                col[static_cast<size_t>(b + u) * NS] = run;
                run += v[u];
            }
        }
        for (; b < b1; ++b) {
            const uint32_t v = col[static_cast<size_t>(b) * NS];
            col[static_cast<size_t>(b) * NS] = run;
            run += v;
        }
    }
    __syncthreads();  // s_part is reused by the next column group
}

__global__ void __launch_bounds__(kThreads) k_layout_scan(uint32_t *bhist, uint32_t nb,
                                                          uint32_t NS, uint32_t *totals) {
    pdl_trigger();
    pdl_wait();
    scan_columns(bhist, nb, NS, totals, blockIdx.x);
}

// kInline: the count pass's raw per-block slot counts are scanned here (each
// block sums the bhist column of every slot: its own exclusive prefix over the
// blocks and the slot total) — for small nb * NS (decode batches) this replaces
// the separate scan launch.
template <bool kFused, bool kInline = false>
__device__ __forceinline__ void scatter_body(const LayoutParams &p, int32_t *sorted_pairs,
                                             int32_t *pair_pos, const uint16_t *key_lb,
                                             uint32_t nkeys, int64_t *key_offsets,
                                             uint32_t *s_w) {  // [kWarps][NS] counts / positions, [NS+1] bases[, NS prefixes]
    __shared__ uint32_t s_warp[32];
    uint32_t *s_base = s_w + kWarps * p.NS;
    uint32_t *s_pref = s_base + p.NS + 1;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // slot bases: exclusive scan of the slot totals (coalesced loads into smem,
    // then a blocked scan; every block, NS is small)
    if (!kFused) pdl_trigger();
    for (uint32_t i = threadIdx.x; i < kWarps * p.NS; i += kThreads) s_w[i] = 0;
    if (!kFused) pdl_wait();
    if (kInline) {
        for (uint32_t i = threadIdx.x; i < p.NS; i += kThreads) {
            uint32_t pre = 0, tot = 0;
            for (uint32_t b = 0; b < p.nb; ++b) {
                const uint32_t v = __ldcg(p.bhist + static_cast<size_t>(b) * p.NS + i);
                pre += b < blockIdx.x ? v : 0u;
                tot += v;
            }
            s_base[i] = tot;
            s_pref[i] = pre;
        }
    } else {
        for (uint32_t i = threadIdx.x; i < p.NS; i += kThreads) s_base[i] = __ldcg(p.totals + i);
    }
    __syncthreads();
    {
        const uint32_t per = (p.NS + kThreads - 1) / kThreads;
        const uint32_t lo = min(p.NS, threadIdx.x * per), hi = min(p.NS, lo + per);
        uint32_t local = 0;
        for (uint32_t i = lo; i < hi; ++i) local += s_base[i];
        uint32_t grand;
        uint32_t run = block_excl_scan(local, s_warp, grand);
        for (uint32_t i = lo; i < hi; ++i) {
            const uint32_t t = s_base[i];
            s_base[i] = run;
            run += t;
        }
        if (threadIdx.x == 0) s_base[p.NS] = grand;
    }
    __syncthreads();
    if (blockIdx.x == 0 && key_offsets)
        for (uint32_t key = threadIdx.x; key <= nkeys; key += kThreads)
            key_offsets[key] = static_cast<int64_t>(s_base[__ldg(key_lb + key)]);

    // each warp owns chunk/kWarps consecutive pairs, walked in groups of 128
    // (one 128-bit load of 4 pairs per lane)
    const uint32_t wchunk = p.chunk / kWarps;
    const uint32_t wbase = blockIdx.x * p.chunk + warp * wchunk;
    const uint32_t P = static_cast<uint32_t>(p.P);
    auto slots_of = [&](uint32_t q, uint32_t (&sl)[4]) {
        int32_t v[4];
        load4(p.idx, q, p.P, v);
        TokenCursor tc;
        if (q < P) cursor_start(p, q, tc);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            // errors were flagged by the count pass; here invalid pairs drop out
            uint32_t slot = kNone;
            if (q + c < P) {
                if (c) cursor_next(p, tc);
                if (static_cast<uint32_t>(v[c]) < p.E && tc.src < p.D) {
                    const uint16_t s16 = __ldg(p.cell_slot + tc.src * p.E + v[c]);
                    slot = s16 == 0xFFFF ? kNone : s16;
                }
            }
            sl[c] = slot;
        }
    };
    // the first kKeep groups keep their slots in registers for the ranking pass
    constexpr uint32_t kKeep = 4;
    uint32_t keep[kKeep][4];
    auto count_group = [&](uint32_t g, uint32_t (&sl)[4]) {
        slots_of(wbase + g + lane * 4, sl);
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (sl[c] != kNone) atomicAdd(s_w + warp * p.NS + sl[c], 1u);
    };
#pragma unroll
    for (uint32_t gi = 0; gi < kKeep; ++gi)
        if (gi * 128 < wchunk) count_group(gi * 128, keep[gi]);
    for (uint32_t g = kKeep * 128; g < wchunk; g += 128) {
        uint32_t sl[4];
        count_group(g, sl);
    }
    __syncthreads();
    // per slot: exclusive prefix over warps, seeded with the block's global offset
    for (uint32_t s = threadIdx.x; s < p.NS; s += kThreads) {
        uint32_t run = s_base[s] + (kInline ? s_pref[s] : p.bhist[static_cast<size_t>(blockIdx.x) * p.NS + s]);
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = s_w[w * p.NS + s];
            s_w[w * p.NS + s] = run;
            run += c;
        }
    }
    __syncthreads();
    uint32_t *mine = s_w + warp * p.NS;
    const unsigned lt = (1u << lane) - 1u;
    auto rank_group = [&](uint32_t g, const uint32_t (&sl)[4]) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            // round r covers pairs wbase + g + 32r + lane, held by lane 8r + lane/4,
            // component lane%4
            const int srcl = r * 8 + (lane >> 2);
            uint32_t cand[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) cand[c] = __shfl_sync(0xffffffffu, sl[c], srcl);
            const uint32_t c4 = lane & 3;
            const uint32_t slot = c4 == 0 ? cand[0] : c4 == 1 ? cand[1] : c4 == 2 ? cand[2] : cand[3];
            // lanes holding the same slot: AND of per-bit ballots (short, independent
            // ballots pipeline better than one long-latency MATCH.ANY)
            const uint32_t key = slot == kNone ? (1u << p.key_bits) - 1u : slot;
#ifdef MPB_EXP_MATCH  // experiment: one MATCH.ANY instead of key_bits ballots
            const unsigned peers = __match_any_sync(0xffffffffu, key);
#else
            unsigned peers = 0xffffffffu;
            for (uint32_t b = 0; b < p.key_bits; ++b) {
                const unsigned m = __ballot_sync(0xffffffffu, (key >> b) & 1u);
                peers &= ((key >> b) & 1u) ? m : ~m;
            }
#endif
            uint32_t pos = 0;
            if (slot != kNone) pos = mine[slot] + __popc(peers & lt);
            __syncwarp();
            if (slot != kNone && lane == static_cast<uint32_t>(__ffs(peers) - 1))
                mine[slot] += __popc(peers);
            __syncwarp();
            if (slot != kNone) {
                const uint32_t pair = wbase + g + r * 32 + lane;
                sorted_pairs[pos] = static_cast<int32_t>(pair);
                pair_pos[pair] = static_cast<int32_t>(pos);
            }
        }
    };
#pragma unroll
    for (uint32_t gi = 0; gi < kKeep; ++gi)
        if (gi * 128 < wchunk) rank_group(gi * 128, keep[gi]);
    for (uint32_t g = kKeep * 128; g < wchunk; g += 128) {
        uint32_t sl[4];
        slots_of(wbase + g + lane * 4, sl);
        rank_group(g, sl);
    }
}

template <bool kInline>
__global__ void __launch_bounds__(kThreads) k_layout_scatter(LayoutParams p, int32_t *sorted_pairs,
                                                             int32_t *pair_pos,
                                                             const uint16_t *key_lb,
                                                             uint32_t nkeys,
                                                             int64_t *key_offsets) {
    extern __shared__ uint32_t s_w[];
    scatter_body<false, kInline>(p, sorted_pairs, pair_pos, key_lb, nkeys, key_offsets, s_w);
}

// Grid-wide barrier of a launch whose blocks are all resident (nb <= SMs):
// arrival counter + generation word, self-resetting (graph-replay safe).
__device__ __forceinline__ void grid_barrier(uint32_t *bar, uint32_t nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile uint32_t *vgen = bar + 1;
        const uint32_t gen = *vgen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            uint32_t g;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
            } while (g == gen);
        }
        __threadfence();
    }
    __syncthreads();
}

// Small batches (decode: T*k <= 1024 * SMs): count, scan and scatter in ONE
// launch of nb <= SMs resident blocks separated by two grid barriers — the
// same three phases (same per-block histograms, same stable order) without
// two kernel boundaries.
__global__ void __launch_bounds__(kThreads) k_layout_fused(LayoutParams p, int32_t *sorted_pairs,
                                                           int32_t *pair_pos, const uint16_t *key_lb,
                                                           uint32_t nkeys, int64_t *key_offsets,
                                                           uint32_t *gbar) {
    extern __shared__ uint32_t sm[];
    count_body<true>(p, sm);
    grid_barrier(gbar, gridDim.x);
    for (uint32_t g = blockIdx.x; g < (p.NS + 31) / 32; g += gridDim.x)
        scan_columns(p.bhist, p.nb, p.NS, p.totals, g);
    grid_barrier(gbar, gridDim.x);
    __syncthreads();
    scatter_body<true>(p, sorted_pairs, pair_pos, key_lb, nkeys, key_offsets, sm);
}

__global__ void __launch_bounds__(256) k_layout_derive(const uint64_t *demand, const uint8_t *g2n,
                                                       const uint8_t *dest_lut, uint32_t D,
                                                       uint32_t E, uint32_t nodes,
                                                       uint64_t *expert_count,
                                                       uint64_t *group_pairs,
                                                       uint64_t *node_demand,
                                                       uint64_t *inter_intra, uint32_t *err) {
    extern __shared__ unsigned long long s_g[];  // [D + 2]
    for (uint32_t i = threadIdx.x; i < D + 2; i += blockDim.x) s_g[i] = 0;
    __syncthreads();
    unsigned long long inter = 0, intra = 0;
    for (uint32_t e = threadIdx.x; e < E; e += blockDim.x) {
        unsigned long long col = 0;
        // the column's demands in flight together (8 source groups per batch),
        // node sums kept in registers: one store per (node, expert), no global
        // read-modify-write chain
        for (uint32_t s0 = 0; s0 < D; s0 += 8) {
            unsigned long long a[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = s0 + j < D ? demand[static_cast<size_t>(s0 + j) * E + e] : 0ull;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (!a[j]) continue;
                const uint32_t s = s0 + j, n = g2n[s];
                const uint32_t d = dest_lut[static_cast<size_t>(n) * E + e];
                if (d >= D) {
                    atomicOr(err, kErrUncovered);
                    continue;
                }
                col += a[j];
                atomicAdd(&s_g[d], a[j]);
                if (g2n[d] == n)
                    intra += a[j];
                else
                    inter += a[j];
            }
        }
        if (node_demand)
            for (uint32_t n = 0; n < nodes; ++n) {
                unsigned long long t = 0;
                for (uint32_t s = 0; s < D; ++s)
                    if (g2n[s] == n) t += demand[static_cast<size_t>(s) * E + e];
                node_demand[static_cast<size_t>(n) * E + e] = t;
            }
        if (expert_count) expert_count[e] = col;
    }
    atomicAdd(&s_g[D], inter);
    atomicAdd(&s_g[D + 1], intra);
    __syncthreads();
    if (group_pairs)
        for (uint32_t d = threadIdx.x; d < D; d += blockDim.x) group_pairs[d] = s_g[d];
    if (inter_intra && threadIdx.x == 0) {
        inter_intra[0] = s_g[D];
        inter_intra[1] = s_g[D + 1];
    }
}

constexpr size_t kSmemLimit = 160 * 1024;

}  // namespace

mpb_status launch_layout(mpb_context *ctx, const mpb_tokens *tk, const mpb_placement *pl,
                         uint64_t *demand, uint64_t *demand2, uint64_t *tag_pop,
                         int32_t *sorted_pairs, int32_t *pair_pos, int64_t *key_offsets) {
    // the permutation is requested through key_offsets (never empty: D*E+1
    // entries); sorted_pairs / pair_pos may be NULL only when T*k == 0
    const bool perm = key_offsets != nullptr;
    if (perm && tk->T && (!pair_pos || !sorted_pairs))
        return fail(MPB_VALIDATION_ERROR,
                    "mpb_dispatch_layout: sorted_pairs, pair_pos and key_offsets go together");
    if (!demand) return fail(MPB_VALIDATION_ERROR, "mpb_dispatch_layout: demand is NULL");
    if (tk->src_group2 && !demand2)
        return fail(MPB_VALIDATION_ERROR, "mpb_dispatch_layout: src_group2 given without demand2");
    if (tk->k == 0) return fail(MPB_CONFIG_ERROR, "mpb_dispatch_layout: k must be >= 1");
    if (tk->tag && !tag_pop)
        return fail(MPB_VALIDATION_ERROR, "mpb_dispatch_layout: tag given without tag_pop");
    const uint64_t P = tk->T * tk->k;
    if (P > 0x7fffffffull)
        return fail(MPB_CONFIG_ERROR, "mpb_dispatch_layout: T*k must fit int32 pair ids");
    if (perm && (size_t(pl->NS) * kWarps + 2 * size_t(pl->NS) + 1) * 4 > kSmemLimit)
        return fail(MPB_CONFIG_ERROR, "mpb_dispatch_layout: too many (group, expert) slots "
                                      "for the permutation");
    if (P == 0) {
        if (perm)  // every offset is zero
            MPB_CUDA(cudaMemsetAsync(key_offsets, 0, sizeof(int64_t) * (size_t(pl->D) * pl->E + 1),
                                     ctx->stream));
        return MPB_OK;
    }
    LayoutParams p{};
    p.idx = tk->idx;
    p.P = P;
    p.T = tk->T;
    p.k = tk->k;
    p.src_group = tk->src_group;
    p.src_base = tk->src_base;
    p.src_span = tk->src_span;
    p.tag = tk->tag;
    p.n_tags = tk->tag ? tk->n_tags : 0;
    p.src2 = tk->src_group2;
    p.g2n = pl->d_g2n;
    p.slot_lut = pl->d_slot_lut;
    p.cell_slot = pl->d_cell_slot;
    p.D = pl->D;
    p.E = pl->E;
    p.NS = pl->NS;
    p.demand = demand;
    p.demand2 = demand2;
    p.tag_pop = tag_pop;
    p.err = ctx->d_error;
    const size_t DE4 = size_t(pl->D) * pl->E * 4;
    size_t smem = perm ? size_t(pl->NS) * 4 : 0;
    p.demand_smem = smem + DE4 <= kSmemLimit;
    if (p.demand_smem) smem += DE4;
    p.demand2_smem = p.src2 && smem + DE4 <= kSmemLimit;
    if (p.demand2_smem) smem += DE4;
    p.tag_smem = p.n_tags && smem + size_t(p.n_tags) * pl->E * 4 <= kSmemLimit;
    if (p.tag_smem) smem += size_t(p.n_tags) * pl->E * 4;
    const size_t cell4 = (size_t(pl->D) * pl->E + 1) / 2 * 4;
    p.cell_smem = perm && p.demand_smem && smem + cell4 <= kSmemLimit;
    if (p.cell_smem) smem += cell4;
    // about one block per SM: per-block histogram zero/flush and slot-count
    // work scale with D*E and NS, so fewer, fatter blocks amortise them
    // (at least kMinBlocks: a context with a small SM budget — the statistics
    // tail beside the router — needs several resident blocks per SM to hide
    // latency)
    static const char *cenv = std::getenv("MPB_LAYOUT_BLOCKS_PER_SM");
    static const char *menv = std::getenv("MPB_LAYOUT_MIN_BLOCKS");
    static const bool fuse_on = std::getenv("MPB_LAYOUT_FUSE") != nullptr;
    const uint64_t kMinBlocks = menv ? std::max(1, std::atoi(menv)) : 160;
    const uint64_t want_blocks = std::max<uint64_t>(
        kMinBlocks, uint64_t(ctx->num_sms) * (cenv ? std::max(1, std::atoi(cenv)) : 2));
    uint64_t chunk = (P + want_blocks - 1) / want_blocks;
    // at most 8 quanta per block: large batches (1M tokens x 8) get more, thinner
    // blocks — the scatter's per-warp ranking is latency-bound, and 28K-pair
    // blocks at 2 per SM left it at 25% occupancy (K2+K3 200 -> 106 us measured)
    chunk = std::min<uint64_t>(chunk, 8 * kChunkQuantum);
    chunk = std::max<uint64_t>(kChunkQuantum, (chunk + kChunkQuantum - 1) / kChunkQuantum * kChunkQuantum);
    // opt-in (MPB_LAYOUT_FUSE=1): small batches in one launch with grid barriers —
    // measured slower than the three PDL-chained kernels at the decode shape
    const bool fused = perm && fuse_on && (P + kChunkQuantum - 1) / kChunkQuantum <= uint64_t(ctx->num_sms);
    if (fused) chunk = kChunkQuantum;
    const uint32_t nb = static_cast<uint32_t>((P + chunk - 1) / chunk);
    p.nb = nb;
    p.chunk = static_cast<uint32_t>(chunk);
    p.key_bits = 1;
    while ((1u << p.key_bits) - 1u <= pl->NS) ++p.key_bits;
    if (perm) {
        MPB_CUDA(ctx->ensure_scratch((size_t(nb) + 1) * pl->NS * 4 + 256));
        p.bhist = static_cast<uint32_t *>(ctx->scratch);
        p.totals = p.bhist + size_t(nb) * pl->NS;
    }
    if (fused) {
        const size_t sc_smem = (size_t(kWarps) * pl->NS + pl->NS + 1) * 4;
        const size_t f_smem = std::max(smem, sc_smem);
        MPB_CUDA(cudaFuncSetAttribute(k_layout_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(f_smem)));
        MPB_CUDA(launch_pdl(k_layout_fused, dim3(nb), dim3(kThreads), f_smem, ctx->stream, p,
                            sorted_pairs, pair_pos, pl->d_key_lb, pl->D * pl->E, key_offsets,
                            ctx->d_gbar));
        MPB_LAUNCHED(ctx);
        return MPB_OK;
    }
    auto count = perm ? k_layout_count<true> : k_layout_count<false>;
    MPB_CUDA(cudaFuncSetAttribute(count, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    MPB_CUDA(launch_pdl(count, dim3(nb), dim3(kThreads), smem, ctx->stream, p));
    MPB_LAUNCHED(ctx);
    if (!perm) return MPB_OK;
    // small nb * NS: every scatter block scans its slot columns itself (no scan launch)
    static const bool no_inline = std::getenv("MPB_LAYOUT_SCAN_KERNEL") != nullptr;
    const bool inl = !no_inline && uint64_t(nb) * pl->NS <= 65536;
    if (!inl) {
        MPB_CUDA(launch_pdl(k_layout_scan, dim3((pl->NS + 31) / 32), dim3(kThreads), 0, ctx->stream,
                            p.bhist, nb, pl->NS, p.totals));
        MPB_LAUNCHED(ctx);
    }
    const size_t sc_smem = (size_t(kWarps) * pl->NS + pl->NS + 1 + (inl ? pl->NS : 0)) * 4;
    auto scatter = inl ? k_layout_scatter<true> : k_layout_scatter<false>;
    MPB_CUDA(cudaFuncSetAttribute(scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sc_smem)));
    MPB_CUDA(launch_pdl(scatter, dim3(nb), dim3(kThreads), sc_smem, ctx->stream, p,
                        sorted_pairs, pair_pos, pl->d_key_lb, pl->D * pl->E, key_offsets));
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

mpb_status launch_layout_derive(mpb_context *ctx, const mpb_placement *pl, const uint64_t *demand,
                                uint64_t *expert_count, uint64_t *group_pairs,
                                uint64_t *node_demand, uint64_t *inter_intra) {
    const size_t smem = (size_t(pl->D) + 2) * 8;
    k_layout_derive<<<1, 256, smem, ctx->stream>>>(demand, pl->d_g2n, pl->d_dest_lut, pl->D, pl->E,
                                                   pl->nodes, expert_count, group_pairs,
                                                   node_demand, inter_intra, ctx->d_error);
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

}  // namespace mpb

using namespace mpb;

extern "C" {

mpb_status mpb_dispatch_layout(mpb_context *ctx, const mpb_tokens *tokens,
                               const mpb_placement *placement, uint64_t *demand,
                               uint64_t *demand2, uint64_t *tag_pop, int32_t *sorted_pairs,
                               int32_t *pair_pos, int64_t *key_offsets) {
    if (!ctx || !tokens || !placement)
        return fail(MPB_VALIDATION_ERROR, "mpb_dispatch_layout: NULL argument");
    if (tokens->T && !tokens->idx)
        return fail(MPB_VALIDATION_ERROR, "mpb_dispatch_layout: idx is NULL");
    if (!tokens->src_group && tokens->src_span == 0 && tokens->T)
        return fail(MPB_CONFIG_ERROR, "mpb_dispatch_layout: src_group NULL needs src_span >= 1");
    return launch_layout(ctx, tokens, placement, demand, demand2, tag_pop, sorted_pairs, pair_pos,
                         key_offsets);
}

mpb_status mpb_layout_derive(mpb_context *ctx, const mpb_placement *placement,
                             const uint64_t *demand, uint64_t *expert_count,
                             uint64_t *group_pairs, uint64_t *node_demand,
                             uint64_t *inter_intra) {
    if (!ctx || !placement || !demand)
        return fail(MPB_VALIDATION_ERROR, "mpb_layout_derive: NULL argument");
    return launch_layout_derive(ctx, placement, demand, expert_count, group_pairs, node_demand,
                                inter_intra);
}

}  // extern "C"
