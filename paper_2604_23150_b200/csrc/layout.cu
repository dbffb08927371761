// K2 dispatch histograms + K3 stable token permutation (sm_100a).
//
// Replaces the per-(request, expert) accounting loop of simulate_layer
// (/root/reference/proj/core/src/simulator.cpp:64-88) at token granularity
// and adds the permutation the reference never materialises.
//
// HBM layout: idx[T*k] int32 (pair p = t*k + j), src_group[T] / tag[T] uint8.
// Decode-size batches (T*k <= 128K pairs): ONE launch of one thread-block
// cluster (k_layout_cluster below). Larger batches: three launches, all
// streaming idx with coalesced 128-bit loads:
//   1. count   : per block (up to 8K pairs) shared-memory-privatised histograms
//                (demand[src][e], demand2[src2][e] for a second routing of the
//                same tokens, tag_pop[tag][e]); the block's slot counts are
//                derived from its demand cells (one add per non-zero cell, not
//                per pair); bins flushed with one global atomic each, slot
//                counts written slot-major as bhist[slot][block].
//   2. scan    : one CTA per slot scans its bhist row (exclusive, in place,
//                coalesced) and writes the slot total.
//   3. scatter : one pass over the block's chunk (L2-resident): slots, the
//                stable rank of every pair inside its warp (per-warp slot
//                counters; the rank among lower lanes from per-bit ballots of
//                the slot id, no MATCH.ANY) into a shared-memory stash; then the
//                slot bases (block 0 emits key_offsets) and the stash written
//                out as sorted_pairs / pair_pos.
// Algorithmic bytes per pair: 4 (idx) + 8 (perm out) [+ 1/k src + 1/k tag].
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>

#include "internal.cuh"
#include "tc_ptx.cuh"

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
    // several layers in one launch (blockIdx.y = layer): idx [L][P], demand /
    // demand2 [L][D][E], each layer's block counts + totals bh_stride words apart
    uint32_t layers;
    uint32_t bh_stride;
};

// The view of layer blockIdx.y of a multi-layer launch (tag_pop: shared sums).
__device__ __forceinline__ LayoutParams layer_view(LayoutParams p) {
    if (p.layers > 1) {
        const size_t l = blockIdx.y, DE = size_t(p.D) * p.E;
        p.idx += l * p.P;
        p.demand += l * DE;
        if (p.demand2) p.demand2 += l * DE;
        if (p.bhist) {
            p.bhist += l * p.bh_stride;
            p.totals += l * p.bh_stride;
        }
    }
    return p;
}

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

// Histogram increments of the pairs q..q+3 (all < P) into the block's shared
// tables, and the demand cell of each pair (kNone when it is dropped):
// e >= E -> kErrExpertRange, source >= D -> kErrSourceRange (the pair counts
// nowhere); second source >= D -> kErrSourceRange (demand2 skipped); tags >=
// n_tags are not counted. kK4 (k % 4 == 0): the four pairs are one token — one
// metadata lookup, no cursor, predicated atomics instead of nested branches.
template <bool kK4>
__device__ __forceinline__ void hist4(const LayoutParams &p, uint32_t q, uint32_t P,
                                      const int32_t (&v)[4], uint32_t *s_demand,
                                      uint32_t *s_demand2, uint32_t *s_tag, uint32_t (&cells)[4]) {
    if constexpr (kK4) {
        const uint32_t t = q / p.k;
        const uint32_t src = p.src_group ? static_cast<uint32_t>(__ldg(p.src_group + t))
                                         : p.src_base + static_cast<uint32_t>((uint64_t(t) * p.src_span) / p.T);
        const uint32_t s2 = p.src2 ? static_cast<uint32_t>(__ldg(p.src2 + t)) : 0u;
        const uint32_t tg = p.tag ? static_cast<uint32_t>(__ldg(p.tag + t)) : kNone;
        const bool src_ok = src < p.D, s2_ok = s2 < p.D, tg_ok = tg < p.n_tags;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t e = static_cast<uint32_t>(v[c]);
            const bool e_ok = e < p.E;
            const bool ok = e_ok && src_ok;
            if (!ok) atomicOr(p.err, e_ok ? kErrSourceRange : kErrExpertRange);
            const uint32_t cell = src * p.E + e;
            if (ok) atomicAdd(s_demand + cell, 1u);
            if (p.src2) {
                if (ok && s2_ok) atomicAdd(s_demand2 + s2 * p.E + e, 1u);
                if (ok && !s2_ok) atomicOr(p.err, kErrSourceRange);
            }
            if (ok && tg_ok) atomicAdd(s_tag + tg * p.E + e, 1u);
            cells[c] = ok ? cell : kNone;
        }
    } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) cells[c] = kNone;
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
            cells[c] = tc.src * p.E + e;
            atomicAdd(s_demand + cells[c], 1u);
            if (p.src2) {
                if (tc.s2 < p.D)
                    atomicAdd(s_demand2 + tc.s2 * p.E + e, 1u);
                else
                    atomicOr(p.err, kErrSourceRange);
            }
            if (tc.tg < p.n_tags) atomicAdd(s_tag + tc.tg * p.E + e, 1u);
        }
    }
}

// The (source, expert) cells of the pairs q..q+3 without counting (kNone:
// dropped; the count pass flagged the errors).
template <bool kK4>
__device__ __forceinline__ void cells4(const LayoutParams &p, uint32_t q, uint32_t P,
                                       const int32_t (&v)[4], uint32_t (&cells)[4]) {
    if constexpr (kK4) {
        const uint32_t t = q / p.k;
        const uint32_t src = p.src_group ? static_cast<uint32_t>(__ldg(p.src_group + t))
                                         : p.src_base + static_cast<uint32_t>((uint64_t(t) * p.src_span) / p.T);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t e = static_cast<uint32_t>(v[c]);
            cells[c] = (e < p.E && src < p.D) ? src * p.E + e : kNone;
        }
    } else {
        TokenCursor tc;
        cursor_start(p, q, tc);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (c) cursor_next(p, tc);
            const uint32_t e = static_cast<uint32_t>(v[c]);
            cells[c] = (q + c < P && e < p.E && tc.src < p.D) ? tc.src * p.E + e : kNone;
        }
    }
}

// Lanes of the warp holding the same key: AND of per-bit ballots of the key
// (short, independent ballots pipeline better than one long-latency
// MATCH.ANY). KB > 0: the bit count at compile time (unrolled); 0: p.key_bits.
template <int KB>
__device__ __forceinline__ unsigned same_key_lanes(uint32_t key, uint32_t key_bits) {
    unsigned peers = 0xffffffffu;
    if constexpr (KB > 0) {
#pragma unroll
        for (int b = 0; b < KB; ++b) {
            const bool bit = (key >> b) & 1u;
            const unsigned m = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? m : ~m;
        }
    } else {
        for (uint32_t b = 0; b < key_bits; ++b) {
            const bool bit = (key >> b) & 1u;
            const unsigned m = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? m : ~m;
        }
    }
    return peers;
}

constexpr uint32_t kCountCluster = 8;  // count CTAs whose histogram tables are summed over DSMEM

// kClu (fast path only: every table in smem): the kernel runs in clusters of
// kCountCluster CTAs, which sum their tables over distributed shared memory
// before the flush — each cell is flushed with one global atomic per cluster
// instead of one per CTA.
template <bool kPerm, bool kClu>
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
        const bool k4 = p.k % 4 == 0;  // (block and lane offsets are multiples of 4)
#pragma unroll 2
        for (uint32_t h = 0; h < rounds; ++h) {
            const uint32_t q = base + h * kThreads * 4 + threadIdx.x * 4;
            if (q >= P) break;
            int32_t v[4];
            load4(p.idx, q, p.P, v);
            uint32_t cells[4];
            if (k4)
                hist4<true>(p, q, P, v, s_demand, s_demand2, s_tag, cells);
            else
                hist4<false>(p, q, P, v, s_demand, s_demand2, s_tag, cells);
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
    if constexpr (kClu) {
        // the block's slot counts from its own cells (coverage is flagged on
        // the cluster sums below)
        if (kPerm) {
            for (uint32_t i = threadIdx.x; i < DE; i += kThreads) {
                const uint32_t c = s_demand[i];
                const uint16_t slot = p.cell_smem ? s_cell[i] : __ldg(p.cell_slot + i);
                if (c && slot != 0xFFFF) atomicAdd(s_slot + slot, c);
            }
            __syncthreads();
            for (uint32_t sl = threadIdx.x; sl < p.NS; sl += kThreads)
                p.bhist[static_cast<size_t>(sl) * p.nb + blockIdx.x] = s_slot[sl];
        }
        ptx::cluster_sync();  // every CTA's tables are final
        const uint32_t crank = ptx::cluster_ctarank();
        auto reduce = [&](const uint32_t *tab, uint32_t n, uint64_t *dst, bool check) {
            const uint32_t lo = crank * n / kCountCluster, hi = (crank + 1) * n / kCountCluster;
            for (uint32_t i = lo + threadIdx.x; i < hi; i += kThreads) {
                const uint32_t a = ptx::smem_u32(tab + i);
                uint32_t v[kCountCluster];
#pragma unroll
                for (uint32_t r = 0; r < kCountCluster; ++r) v[r] = ptx::ld_dsmem_u32(ptx::mapa(a, r));
                uint32_t c = 0;
#pragma unroll
                for (uint32_t r = 0; r < kCountCluster; ++r) c += v[r];
                if (!c) continue;
                if (check && (p.cell_smem ? s_cell[i] : __ldg(p.cell_slot + i)) == 0xFFFF) {
                    atomicOr(p.err, kErrUncovered);
                    continue;
                }
                atomicAdd(reinterpret_cast<unsigned long long *>(dst) + i, static_cast<unsigned long long>(c));
            }
        };
        reduce(s_demand, DE, p.demand, true);
        if (p.src2) reduce(s_demand2, DE, p.demand2, false);
        if (p.tag) reduce(s_tag, p.n_tags * p.E, p.tag_pop, false);
        ptx::cluster_sync();  // peers may still be reading this CTA's tables
        return;
    }
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
            p.bhist[static_cast<size_t>(sl) * p.nb + blockIdx.x] = s_slot[sl];
    }
}

template <bool kPerm, bool kClu>
__global__ void __launch_bounds__(kThreads) k_layout_count(LayoutParams p) {
    extern __shared__ uint32_t sm[];
    count_body<kPerm, kClu>(layer_view(p), sm);
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

// One CTA per slot: exclusive scan of the slot's row of block counts
// bhist[slot][0..nb) in place (slot-major: coalesced) and the slot total.
// Thread t owns the contiguous blocks [t*per, (t+1)*per): thread sums, a block
// scan of the sums, then the rewrite (one batch of loads each way for
// nb <= 8 * kThreads).
__global__ void __launch_bounds__(kThreads) k_layout_scan(uint32_t *bhist, uint32_t nb,
                                                          uint32_t NS, uint32_t *totals,
                                                          uint32_t layer_stride) {
    __shared__ uint32_t s_warp[32];
    bhist += static_cast<size_t>(blockIdx.y) * layer_stride;  // multi-layer launch: layer blockIdx.y
    totals += static_cast<size_t>(blockIdx.y) * layer_stride;
    pdl_trigger();
    pdl_wait();
    const uint32_t slot = blockIdx.x;
    uint32_t *row = bhist + static_cast<size_t>(slot) * nb;
    const uint32_t per = (nb + kThreads - 1) / kThreads;
    const uint32_t b0 = min(nb, threadIdx.x * per), b1 = min(nb, b0 + per);
    uint32_t sum = 0;
    for (uint32_t b = b0; b < b1; b += 8) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = b + u < b1 ? row[b + u] : 0u;
#pragma unroll
        for (int u = 0; u < 8; ++u) sum += v[u];
    }
    uint32_t total;
    uint32_t run = block_excl_scan(sum, s_warp, total);
    if (threadIdx.x == 0) totals[slot] = total;
    for (uint32_t b = b0; b < b1; b += 8) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = b + u < b1 ? row[b + u] : 0u;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (b + u < b1) {
                row[b + u] = run;
                run += v[u];
            }
    }
}

// One read of the block's chunk:
//   pass 1a: each warp resolves the slots of its consecutive pairs (one 128-bit
//            load of 4 pairs per lane per group, several groups in flight) into
//            a shared-memory stash;
//   pass 1b: 32 pairs per round in pair order, the stable rank of every pair
//            among the warp's earlier pairs of the same slot (per-bit ballots of
//            the slot id; the warp's running per-slot counters in smem), packed
//            (slot, rank) in place;
//   bases  : slot bases from the slot totals (block scan; block 0 emits
//            key_offsets), this block's prefix per slot from the scan kernel,
//            then the per-warp prefixes;
//   pass 2 : the stash is read back in pair order (coalesced pair_pos stores)
//            and every pair written at base + rank.
template <int KB>
__global__ void __launch_bounds__(kThreads) k_layout_scatter(LayoutParams p, int32_t *sorted_pairs,
                                                             int32_t *pair_pos,
                                                             const uint16_t *key_lb,
                                                             uint32_t nkeys,
                                                             int64_t *key_offsets) {
    extern __shared__ uint32_t s_w[];  // [kWarps][NS] counters -> bases, [NS+1] bases, [NS] prefixes, stash
    if (p.layers > 1) {  // layer blockIdx.y of a multi-layer launch
        sorted_pairs += static_cast<size_t>(blockIdx.y) * p.P;
        pair_pos += static_cast<size_t>(blockIdx.y) * p.P;
        key_offsets += static_cast<size_t>(blockIdx.y) * (nkeys + 1);
        p = layer_view(p);
    }
    __shared__ uint32_t s_warp[32];
    const uint32_t NS = p.NS;
    uint32_t *s_base = s_w + kWarps * NS;
    uint32_t *s_pref = s_base + NS + 1;
    uint32_t *stash = s_w + ((kWarps + 2) * NS + 1 + 3) / 4 * 4;  // 16-byte aligned
    uint16_t *s_cell = reinterpret_cast<uint16_t *>(stash + p.chunk);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t DE = p.D * p.E;
    pdl_trigger();
    for (uint32_t i = threadIdx.x; i < kWarps * NS; i += kThreads) s_w[i] = 0;
    if (p.cell_smem)
        for (uint32_t i = threadIdx.x; i < DE; i += kThreads) s_cell[i] = __ldg(p.cell_slot + i);
    const uint16_t *cell = p.cell_smem ? s_cell : p.cell_slot;
    // (idx may come from the kernel before the count pass: everything global
    // is read after the wait)
    pdl_wait();
    __syncthreads();

    // ---- pass 1a: slots of the warp's pairs into the stash (lane-major, 4 pairs
    // per lane per group; loads of several groups in flight)
    const uint32_t wchunk = p.chunk / kWarps;
    const uint32_t cbase = blockIdx.x * p.chunk;
    const uint32_t wbase = cbase + warp * wchunk;
    const uint32_t P = static_cast<uint32_t>(p.P);
    uint32_t *mine = s_w + warp * NS;
    uint32_t *wstash = stash + warp * wchunk;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t wn = P > wbase ? min(wchunk, P - wbase) : 0u;  // the warp's pairs
    const bool k4 = p.k % 4 == 0;
#pragma unroll 4
    for (uint32_t g = 0; g < wn; g += 128) {
        const uint32_t q = wbase + g + lane * 4;
        uint4 sl = make_uint4(kNone, kNone, kNone, kNone);
        if (q < P) {
            int32_t v[4];
            load4(p.idx, q, p.P, v);
            uint32_t o[4];
            if (k4)
                cells4<true>(p, q, P, v, o);
            else
                cells4<false>(p, q, P, v, o);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                // errors were flagged by the count pass; here invalid pairs drop out
                const uint16_t s16 = o[c] == kNone ? uint16_t(0xFFFF) : cell[o[c]];
                o[c] = s16 == 0xFFFF ? kNone : s16;
            }
            sl = make_uint4(o[0], o[1], o[2], o[3]);
        }
        *reinterpret_cast<uint4 *>(wstash + g + lane * 4) = sl;
    }
    __syncwarp();
    // ---- pass 1b: stable ranks in pair order, 32 pairs per round (packed in place)
    for (uint32_t g = 0; g < wn; g += 32) {
        const uint32_t slot = wstash[g + lane];
        const uint32_t key = slot == kNone ? (1u << p.key_bits) - 1u : slot;
        const unsigned peers = same_key_lanes<KB>(key, p.key_bits);
        uint32_t x = kNone;
        if (slot != kNone) x = (slot << 16) | (mine[slot] + __popc(peers & lt));
        __syncwarp();
        if (slot != kNone && lane == static_cast<uint32_t>(__ffs(peers) - 1)) mine[slot] += __popc(peers);
        wstash[g + lane] = x;
        __syncwarp();
    }

    // ---- bases
    for (uint32_t i = threadIdx.x; i < NS; i += kThreads) {
        s_base[i] = __ldcg(p.totals + i);
        s_pref[i] = __ldcg(p.bhist + static_cast<size_t>(i) * p.nb + blockIdx.x);
    }
    __syncthreads();
    {
        const uint32_t per = (NS + kThreads - 1) / kThreads;
        const uint32_t lo = min(NS, threadIdx.x * per), hi = min(NS, lo + per);
        uint32_t local = 0;
        for (uint32_t i = lo; i < hi; ++i) local += s_base[i];
        uint32_t grand;
        uint32_t run = block_excl_scan(local, s_warp, grand);
        for (uint32_t i = lo; i < hi; ++i) {
            const uint32_t t = s_base[i];
            s_base[i] = run;
            run += t;
        }
        if (threadIdx.x == 0) s_base[NS] = grand;
    }
    __syncthreads();
    if (blockIdx.x == 0 && key_offsets)
        for (uint32_t key = threadIdx.x; key <= nkeys; key += kThreads)
            key_offsets[key] = static_cast<int64_t>(s_base[__ldg(key_lb + key)]);
    // per slot: exclusive prefix over warps, seeded with the block's global offset
    for (uint32_t sl = threadIdx.x; sl < NS; sl += kThreads) {
        uint32_t run = s_base[sl] + s_pref[sl];
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = s_w[w * NS + sl];
            s_w[w * NS + sl] = run;
            run += c;
        }
    }
    __syncthreads();

    // ---- pass 2: stash in pair order
    const uint32_t n = P > cbase ? min(p.chunk, P - cbase) : 0u;
    for (uint32_t w = 0; w < kWarps; ++w) {
        const uint32_t *bases = s_w + w * NS;
        const uint32_t i1 = min(n, (w + 1) * wchunk);
        for (uint32_t i = w * wchunk + threadIdx.x; i < i1; i += kThreads) {
            const uint32_t x = stash[i];
            if (x == kNone) continue;
            const uint32_t pos = bases[x >> 16] + (x & 0xFFFFu);
            sorted_pairs[pos] = static_cast<int32_t>(cbase + i);
            pair_pos[cbase + i] = static_cast<int32_t>(pos);
        }
    }
}

// Decode-size batches (T*k <= 16 CTAs x 8K pairs): the whole layout in ONE
// launch of ONE thread-block cluster — no bhist round trip through global
// memory, no scan launch, no second pass over idx.
//   phase 1: each warp walks its G groups of 128 pairs once: histogram atomics
//            into the CTA's shared tables (count_body's fast-path semantics),
//            slot lookup, and the pair's stable rank among the warp's earlier
//            pairs of the same slot (per-bit ballots, as k_layout_scatter); the
//            (slot, rank) of every pair stays in registers;
//   phase 2: per-warp slot prefixes and the CTA's slot totals, which every CTA
//            pushes into every peer's shared memory (st.shared::cluster);
//            the CTA's histogram cells go to global memory (one atomic per
//            non-zero cell, as the count kernel's flush); ONE cluster barrier;
//            every CTA then holds all totals locally: its prefix over earlier
//            CTAs, the slot bases (block scan), key_offsets from CTA 0;
//   phase 3: each pair is written at base[slot] + cta_prefix + warp_prefix +
//            rank (the same stable order as count/scan/scatter).
constexpr int kCThreads = 512;
constexpr int kCWarps = kCThreads / 32;
constexpr uint32_t kCGroupPairs = kCWarps * 128;  // pairs per CTA per group
constexpr uint32_t kCMax = 16;                     // CTAs per cluster (non-portable size)

using ptx::cluster_ctarank;
using ptx::cluster_sync;
using ptx::mapa;
using ptx::smem_u32;
using ptx::st_dsmem_u32;

#ifdef MPB_LAYOUT_TRACE
// Experiment builds only: per-CTA %globaltimer stamps of the last launch's
// phases (0 entry, 1 cluster barrier, 2 griddepcontrol.wait, 3 warp 0 done
// with phase 1, 4 all warps, 5 flush issued, 6 second barrier, 7 exit).
__device__ unsigned long long g_lc_trace[kCMax * 8];
__device__ __forceinline__ unsigned long long lc_time() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");
    return t;
}
#define LCTRACE(slot) \
    if (threadIdx.x == 0) g_lc_trace[cluster_ctarank() * 8 + (slot)] = lc_time()
#else
#define LCTRACE(slot) ((void)0)
#endif

template <int G, int KB>
__global__ void __launch_bounds__(kCThreads) k_layout_cluster(LayoutParams p, int32_t *sorted_pairs,
                                                              int32_t *pair_pos,
                                                              const uint16_t *key_lb,
                                                              uint32_t nkeys, int64_t *key_offsets) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t s_warp[32];
    const uint32_t DE = p.D * p.E;
    const uint32_t NS = p.NS;
    const uint32_t n_dem2 = p.src2 ? DE : 0u, n_tag = p.tag ? p.n_tags * p.E : 0u;
    const uint32_t crank = cluster_ctarank(), csize = gridDim.x;
    uint32_t *s_demand = sm;
    uint32_t *s_demand2 = s_demand + DE;
    uint32_t *s_tag = s_demand2 + n_dem2;
    uint32_t *s_cnt = s_tag + n_tag;         // [kCWarps][NS]: counts, then write bases
    uint32_t *s_all = s_cnt + kCWarps * NS;  // [csize][NS]: every CTA's slot totals
    uint32_t *s_base = s_all + csize * NS;   // [NS + 1] slot bases (+ this CTA's prefix)
    uint16_t *s_cell = reinterpret_cast<uint16_t *>(s_base + NS + 1);
    const uint32_t nzero = DE + n_dem2 + n_tag + kCWarps * NS;
    LCTRACE(0);
    pdl_trigger();
    for (uint32_t i = threadIdx.x; i < DE; i += kCThreads) s_cell[i] = __ldg(p.cell_slot + i);
    for (uint32_t i = threadIdx.x; i < nzero; i += kCThreads) sm[i] = 0;
    // every CTA must be running before any peer stores into its shared memory
    cluster_sync();
    LCTRACE(1);
    pdl_wait();
    LCTRACE(2);

    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t P = static_cast<uint32_t>(p.P);
    const uint32_t wbase = crank * (G * kCGroupPairs) + warp * (G * 128);
    uint32_t *mine = s_cnt + warp * NS;
    const unsigned lt = (1u << lane) - 1u;
    uint32_t res[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const uint32_t q = wbase + g * 128 + lane * 4;
        uint32_t sl[4] = {kNone, kNone, kNone, kNone};
        if (q < P) {
            int32_t v[4];
            load4(p.idx, q, p.P, v);
            uint32_t cells[4];
            if (p.k % 4 == 0)
                hist4<true>(p, q, P, v, s_demand, s_demand2, s_tag, cells);
            else
                hist4<false>(p, q, P, v, s_demand, s_demand2, s_tag, cells);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint16_t s16 = cells[c] == kNone ? uint16_t(0xFFFF) : s_cell[cells[c]];
                sl[c] = s16 == 0xFFFF ? kNone : s16;
            }
        }
        // stable rank inside the warp: round r covers pairs wbase + 128g + 32r + lane
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int srcl = r * 8 + (lane >> 2);
            uint32_t cand[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) cand[c] = __shfl_sync(0xffffffffu, sl[c], srcl);
            const uint32_t c4 = lane & 3;
            const uint32_t slot = c4 == 0 ? cand[0] : c4 == 1 ? cand[1] : c4 == 2 ? cand[2] : cand[3];
            const uint32_t key = slot == kNone ? (1u << p.key_bits) - 1u : slot;
            const unsigned peers = same_key_lanes<KB>(key, p.key_bits);
            uint32_t x = kNone;
            if (slot != kNone) x = (slot << 16) | (mine[slot] + __popc(peers & lt));
            __syncwarp();
            if (slot != kNone && lane == static_cast<uint32_t>(__ffs(peers) - 1))
                mine[slot] += __popc(peers);
            __syncwarp();
            res[g][r] = x;
        }
    }
    LCTRACE(3);
    __syncthreads();
    LCTRACE(4);
    // per slot: exclusive prefix over this CTA's warps (in place); the CTA total
    // goes into row `crank` of every CTA's s_all
    for (uint32_t s = threadIdx.x; s < NS; s += kCThreads) {
        uint32_t run = 0;
#pragma unroll 4
        for (int w = 0; w < kCWarps; ++w) {
            const uint32_t c = s_cnt[w * NS + s];
            s_cnt[w * NS + s] = run;
            run += c;
        }
        const uint32_t a = smem_u32(s_all + crank * NS + s);
        for (uint32_t c = 0; c < csize; ++c) st_dsmem_u32(mapa(a, c), run);
    }
    // this CTA's histogram cells (coverage checked per non-zero demand cell)
    for (uint32_t i = threadIdx.x; i < DE; i += kCThreads) {
        const uint32_t c = s_demand[i];
        if (!c) continue;
        if (s_cell[i] == 0xFFFF) {
            atomicOr(p.err, kErrUncovered);
            continue;
        }
        atomicAdd(reinterpret_cast<unsigned long long *>(p.demand) + i, static_cast<unsigned long long>(c));
    }
    for (uint32_t i = threadIdx.x; i < n_dem2; i += kCThreads)
        if (s_demand2[i])
            atomicAdd(reinterpret_cast<unsigned long long *>(p.demand2) + i,
                      static_cast<unsigned long long>(s_demand2[i]));
    for (uint32_t i = threadIdx.x; i < n_tag; i += kCThreads)
        if (s_tag[i])
            atomicAdd(reinterpret_cast<unsigned long long *>(p.tag_pop) + i,
                      static_cast<unsigned long long>(s_tag[i]));
    LCTRACE(5);
    cluster_sync();  // every CTA's totals are in every CTA's s_all
    LCTRACE(6);
    uint32_t *s_pre = s_demand;  // the histogram tables are flushed: reuse
    for (uint32_t s = threadIdx.x; s < NS; s += kCThreads) {
        uint32_t pre = 0, tot = 0;
        for (uint32_t c = 0; c < csize; ++c) {
            const uint32_t v = s_all[c * NS + s];
            pre += c < crank ? v : 0u;
            tot += v;
        }
        s_pre[s] = pre;
        s_base[s] = tot;
    }
    __syncthreads();
    {  // slot bases: block-wide exclusive scan of the cluster totals
        const uint32_t per = (NS + kCThreads - 1) / kCThreads;
        const uint32_t lo = min(NS, threadIdx.x * per), hi = min(NS, lo + per);
        uint32_t local = 0;
        for (uint32_t i = lo; i < hi; ++i) local += s_base[i];
        uint32_t incl = local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = lane < kCWarps ? s_warp[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            if (lane < kCWarps) s_warp[lane] = w;
        }
        __syncthreads();
        uint32_t run = (warp ? s_warp[warp - 1] : 0) + incl - local;
        for (uint32_t i = lo; i < hi; ++i) {
            const uint32_t t = s_base[i];
            s_base[i] = run;
            run += t;
        }
        if (threadIdx.x == kCThreads - 1) s_base[NS] = run;
    }
    __syncthreads();
    if (crank == 0 && key_offsets)
        for (uint32_t key = threadIdx.x; key <= nkeys; key += kCThreads)
            key_offsets[key] = static_cast<int64_t>(s_base[__ldg(key_lb + key)]);
    for (uint32_t i = threadIdx.x; i < kCWarps * NS; i += kCThreads) {
        const uint32_t s = i % NS;
        s_cnt[i] += s_base[s] + s_pre[s];
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t x = res[g][r];
            if (x == kNone) continue;
            const uint32_t pos = mine[x >> 16] + (x & 0xFFFFu);
            const uint32_t pair = wbase + g * 128 + r * 32 + lane;
            sorted_pairs[pos] = static_cast<int32_t>(pair);
            pair_pos[pair] = static_cast<int32_t>(pos);
        }
    LCTRACE(7);
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
// The single-cluster layout when the batch fits one cluster: false when not
// taken (MPB_LAYOUT_CLUSTER=0 disables it), else `st` is the launch status.
bool launch_layout_cluster(mpb_context *ctx, LayoutParams p, const mpb_placement *pl,
                           int32_t *sorted_pairs, int32_t *pair_pos, int64_t *key_offsets,
                           mpb_status &st) {
    static const char *env = std::getenv("MPB_LAYOUT_CLUSTER");
    if (env && env[0] == '0') return false;
    const uint32_t DE = p.D * p.E, NS = p.NS;
    // (the slot prefixes reuse the demand table: DE >= NS)
    const size_t smem = (size_t(DE) + (p.src2 ? DE : 0) + (p.tag ? size_t(p.n_tags) * p.E : 0) +
                         size_t(kCWarps) * NS + size_t(kCMax) * NS + NS + 1) * 4 +
                        (size_t(DE) + 1) / 2 * 4;
    if (NS > DE) return false;
    if (smem > kSmemLimit) return false;
    // smallest group count whose cluster (<= 16 CTAs, one per SM) holds the batch
    static const char *cenv = std::getenv("MPB_LAYOUT_CLUSTER_MAX");
    const uint64_t cmax = cenv ? std::min<uint64_t>(kCMax, std::max(1, std::atoi(cenv))) : kCMax;
    const uint64_t P = p.P;
    int G = 0;
    uint32_t C = 0;
    for (int g : {1, 2, 4}) {
        const uint64_t c = (P + uint64_t(g) * kCGroupPairs - 1) / (uint64_t(g) * kCGroupPairs);
        if (c <= cmax) {
            G = g;
            C = static_cast<uint32_t>(c);
            break;
        }
    }
    if (!G || C > uint32_t(ctx->num_sms)) return false;
    p.key_bits = 1;
    while ((1u << p.key_bits) - 1u <= NS) ++p.key_bits;
    auto pick = [&](auto g) {
        constexpr int GG = decltype(g)::value;
        return p.key_bits <= 8 ? k_layout_cluster<GG, 8>
                               : p.key_bits == 9 ? k_layout_cluster<GG, 9> : k_layout_cluster<GG, 0>;
    };
    auto kern = G == 1 ? pick(std::integral_constant<int, 1>{})
                       : G == 2 ? pick(std::integral_constant<int, 2>{}) : pick(std::integral_constant<int, 4>{});
    st = MPB_OK;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e == cudaSuccess && C > 8)
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) {
        st = cuda_fail(e, "k_layout_cluster attributes");
        return true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kCThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    {  // a cluster this size must fit the device (checked once per shape)
        static std::mutex mu;
        static std::map<std::pair<uint32_t, size_t>, int> fits;
        std::lock_guard<std::mutex> lock(mu);
        auto key = std::make_pair(C * 8 + uint32_t(G), smem);
        auto it = fits.find(key);
        if (it == fits.end()) {
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
            cudaGetLastError();
            it = fits.emplace(key, n).first;
        }
        if (it->second < 1) return false;
    }
    e = cudaLaunchKernelEx(&cfg, kern, p, sorted_pairs, pair_pos,
                           static_cast<const uint16_t *>(pl->d_key_lb), DE, key_offsets);
    ctx->launches++;
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) st = cuda_fail(e, "k_layout_cluster launch");
    return true;
}

}  // namespace

mpb_status launch_layout(mpb_context *ctx, const mpb_tokens *tk, const mpb_placement *pl,
                         uint64_t *demand, uint64_t *demand2, uint64_t *tag_pop,
                         int32_t *sorted_pairs, int32_t *pair_pos, int64_t *key_offsets,
                         uint32_t layers) {
    if (layers == 0) return MPB_OK;
    if (layers > 65535) return fail(MPB_CONFIG_ERROR, "mpb_dispatch_layout_layers: too many layers");
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
    if (perm && (size_t(pl->NS) * kWarps + 2 * size_t(pl->NS) + 1 + 8 * kChunkQuantum) * 4 > kSmemLimit)
        return fail(MPB_CONFIG_ERROR, "mpb_dispatch_layout: too many (group, expert) slots "
                                      "for the permutation");
    if (P == 0) {
        if (perm)  // every offset is zero
            MPB_CUDA(cudaMemsetAsync(key_offsets, 0,
                                     sizeof(int64_t) * (size_t(pl->D) * pl->E + 1) * layers, ctx->stream));
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
    p.layers = layers;
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
    const uint64_t kMinBlocks = menv ? std::max(1, std::atoi(menv)) : 160;
    const uint64_t want_blocks = std::max<uint64_t>(
        kMinBlocks, uint64_t(ctx->num_sms) * (cenv ? std::max(1, std::atoi(cenv)) : 2));
    uint64_t chunk = (P + want_blocks - 1) / want_blocks;
    // at most 8 quanta per block: large batches (1M tokens x 8) get more, thinner
    // blocks — the scatter's per-warp ranking is latency-bound, and 28K-pair
    // blocks at 2 per SM left it at 25% occupancy (K2+K3 200 -> 106 us measured)
    static const char *qenv = std::getenv("MPB_LAYOUT_MAX_QUANTA");
    chunk = std::min<uint64_t>(chunk, uint64_t(qenv ? std::max(1, std::atoi(qenv)) : 8) * kChunkQuantum);
    chunk = std::max<uint64_t>(kChunkQuantum, (chunk + kChunkQuantum - 1) / kChunkQuantum * kChunkQuantum);
    uint32_t nb = static_cast<uint32_t>((P + chunk - 1) / chunk);
    p.nb = nb;
    p.chunk = static_cast<uint32_t>(chunk);
    p.key_bits = 1;
    while ((1u << p.key_bits) - 1u <= pl->NS) ++p.key_bits;
    // per layer: block counts [nb][NS] then totals [NS], 256-byte aligned regions
    auto bh_words = [&](uint32_t n) { return ((size_t(n) + 1) * pl->NS + 63) / 64 * 64; };
    if (perm) {
        p.bh_stride = static_cast<uint32_t>(bh_words(nb));
        MPB_CUDA(ctx->ensure_scratch(size_t(p.bh_stride) * layers * 4 + 256));
        p.bhist = static_cast<uint32_t *>(ctx->scratch);
        p.totals = p.bhist + size_t(nb) * pl->NS;
    }
    if (layers == 1 && perm && p.demand_smem && (!p.src2 || p.demand2_smem) && (!p.tag || p.tag_smem)) {
        mpb_status st = MPB_OK;
        if (launch_layout_cluster(ctx, p, pl, sorted_pairs, pair_pos, key_offsets, st)) return st;
    }
    // fast path (every table in smem) and enough blocks: clusters of
    // kCountCluster CTAs sum their tables before the flush
    static const char *ccenv = std::getenv("MPB_LAYOUT_COUNT_CLUSTER");
    const bool clu = !(ccenv && ccenv[0] == '0') && p.demand_smem && (!p.src2 || p.demand2_smem) &&
                     (!p.tag || p.tag_smem) && nb >= 8 * kCountCluster;
    if (clu) {  // empty trailing blocks round the grid up to whole clusters
        p.nb = nb = (nb + kCountCluster - 1) / kCountCluster * kCountCluster;
        if (perm) {
            p.bh_stride = static_cast<uint32_t>(bh_words(nb));
            MPB_CUDA(ctx->ensure_scratch(size_t(p.bh_stride) * layers * 4 + 256));
            p.bhist = static_cast<uint32_t *>(ctx->scratch);
            p.totals = p.bhist + size_t(nb) * pl->NS;
        }
        auto count = perm ? k_layout_count<true, true> : k_layout_count<false, true>;
        MPB_CUDA(cudaFuncSetAttribute(count, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(nb, layers);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kCountCluster;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl_enabled() ? 2 : 1;
        MPB_CUDA(cudaLaunchKernelEx(&cfg, count, p));
    } else {
        auto count = perm ? k_layout_count<true, false> : k_layout_count<false, false>;
        MPB_CUDA(cudaFuncSetAttribute(count, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        MPB_CUDA(launch_pdl(count, dim3(nb, layers), dim3(kThreads), smem, ctx->stream, p));
    }
    MPB_LAUNCHED(ctx);
    if (!perm) return MPB_OK;
    MPB_CUDA(launch_pdl(k_layout_scan, dim3(pl->NS, layers), dim3(kThreads), 0, ctx->stream, p.bhist, nb,
                        pl->NS, p.totals, p.bh_stride));
    MPB_LAUNCHED(ctx);
    // counters / bases, slot bases, block prefixes, the chunk's stash, the cell table
    size_t sc_smem = ((size_t(kWarps) + 2) * pl->NS + 1 + 3) / 4 * 16 + size_t(p.chunk) * 4;
    p.cell_smem = sc_smem + (size_t(pl->D) * pl->E + 1) / 2 * 4 <= kSmemLimit;
    if (p.cell_smem) sc_smem += (size_t(pl->D) * pl->E + 1) / 2 * 4;
    auto scatter = p.key_bits <= 8 ? k_layout_scatter<8> : p.key_bits == 9 ? k_layout_scatter<9>
                                                                            : k_layout_scatter<0>;
    MPB_CUDA(cudaFuncSetAttribute(scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sc_smem)));
    MPB_CUDA(launch_pdl(scatter, dim3(nb, layers), dim3(kThreads), sc_smem, ctx->stream, p,
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

mpb_status mpb_dispatch_layout_layers(mpb_context *ctx, uint32_t layers, const mpb_tokens *tokens,
                                      const mpb_placement *placement, uint64_t *demand,
                                      uint64_t *demand2, uint64_t *tag_pop, int32_t *sorted_pairs,
                                      int32_t *pair_pos, int64_t *key_offsets) {
    if (!ctx || !tokens || !placement)
        return fail(MPB_VALIDATION_ERROR, "mpb_dispatch_layout_layers: NULL argument");
    if (layers && tokens->T && !tokens->idx)
        return fail(MPB_VALIDATION_ERROR, "mpb_dispatch_layout_layers: idx is NULL");
    if (!tokens->src_group && tokens->src_span == 0 && tokens->T)
        return fail(MPB_CONFIG_ERROR, "mpb_dispatch_layout_layers: src_group NULL needs src_span >= 1");
    return launch_layout(ctx, tokens, placement, demand, demand2, tag_pop, sorted_pairs, pair_pos,
                         key_offsets, layers);
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

#ifdef MPB_LAYOUT_TRACE
extern "C" __attribute__((visibility("default"))) int mpb_debug_layout_trace(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, mpb::g_lc_trace, sizeof(mpb::g_lc_trace)) == cudaSuccess ? 0 : 9;
}
#endif
