// The routed step's host schedule (mpb_step_*): C++ inside the library.
//
// The reference's planner loop (/root/reference/proj/core/src/pipeline.cpp:
// 316-443) routes, accounts and prices on the host, layer after layer. Here one
// step over L layers is a fixed launch schedule on two streams owned by the
// plan, built once and replayed (eagerly or from CUDA graphs):
//
//   LAYERS  main stream (high priority, SM budget device - side_sms):
//             memset(stats) ; for each chunk c of layers [l0, l1):
//               ev_r0[c] ; mpb_router_topk_layers(l0..l1) ; ev_r1[c] ; ev_done[c]
//           side stream (low priority, side_sms): for each chunk c:
//               wait ev_done[c] ; for l in [l0, l1): mpb_dispatch_layout(l) ;
//               mpb_coactivation(layers l0..l1 as one token list)
//                                          -- beside router chunk c+1
//           main waits for the side stream's last tail.
//           One layer (nothing to overlap): router on every SM, then the layout
//           on main with the co-activation beside it on the side stream.
//   SCORE   score_jobs[0] on main, the others on side, joined.
//
// Chunks taper at the end (..., 4, 2, 1 layers) so the tails left after the
// last router are short. Every layer owns its idx / weights slice, so routers
// never wait on tails. Both phases order after the work already on the
// caller's stream and before anything enqueued after them.
#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only: the functions are resolved at run time

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include "internal.cuh"

namespace {
// NCCL, resolved at run time: the libnccl.so.2 already loaded in the process
// (torch's), else the system one. No link-time dependency.
struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    bool ok = false;
};
const NcclApi &nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
        if (!h) return a;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.init_rank = reinterpret_cast<decltype(a.init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(h, "ncclCommDestroy"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
        a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
        a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.get_unique_id && a.init_rank && a.destroy && a.all_reduce && a.all_gather &&
               a.group_start && a.group_end && a.error_string;
        return a;
    }();
    return api;
}
}  // namespace

#define MPB_NCCL(call)                                                                      \
    do {                                                                                    \
        ncclResult_t r_ = (call);                                                           \
        if (r_ != ncclSuccess)                                                              \
            return ::mpb::fail(MPB_CUDA_ERROR, std::string("NCCL error in " #call ": ") +     \
                                                   nccl().error_string(r_));                \
    } while (0)

struct mpb_step {
    mpb_context *ctx = nullptr;  // the caller's (ordering) context
    mpb_context *main = nullptr, *side = nullptr;
    cudaStream_t s_main = nullptr, s_side = nullptr;
    mpb_step_desc d{};
    std::vector<const void *> X, W;
    std::vector<mpb_score_job> jobs;
    std::vector<std::pair<uint32_t, uint32_t>> chunks;
    bool overlapped = false;
    // one layer, one GPU: the router counts the demand tables itself
    // (mpb_router_topk_demand) and the layout writes its copy into scratch, so
    // the layout + permutation, the pricing and the co-activation all follow
    // the router at once (MPB_ROUTER_DEMAND=0: off)
    bool fused_ok = false;
    // MPB_TAIL_BOOST = n: the last n router chunks run on a smaller grid budget
    // and the side stream's grids double from the tails that run beside them,
    // so the statistics backlog left after the last router drains sooner
    uint32_t tail_boost = 0, side_sms = 0, dev_sms = 0;
    // overlapped step: a chunk's layouts in ONE launch set
    // (mpb_dispatch_layout_layers); the permutations of all but the step's
    // last layer land in this scratch ([max chunk][T*k] x 2 + key offsets),
    // the last layer's in the caller's buffers, as with per-layer launches
    // MPB_LAYOUT_BATCH = layers per batched launch set (default 4; 0 or 1: one
    // mpb_dispatch_layout per layer). Whole 8-layer chunks halve the time after
    // the last router but their (blocks x layers) grids spill onto the routers'
    // SMs between router launches (router 0.220 -> 0.240 ms/layer); interleaved
    // A/B at DSv3 (16 rounds): 4 layers -1.7 / -2.1%, 8 layers +1.9% vs per layer.
    uint32_t layout_batch = 0;  // layers per batched launch set (0: off)
    void *perm_scratch = nullptr;
    // one GPU: the last main_tail_chunks chunks' tails run on the main stream
    // right after the last routers, beside the side stream's backlog (no join
    // first); the side stream's permutations then go to side_perm (one layer)
    // so the caller's buffers still end with the step's last layer
    // (MPB_MAIN_TAIL_CHUNKS, default 1 = the last chunk after a join)
    uint32_t main_tail_chunks = 1;
    void *side_perm = nullptr;
    uint32_t max_chunk = 0;
    uint64_t *scratch_demand = nullptr;  // [2][D][E]
    // fused single layer: a third stream for the pricing (the layout follows
    // the router on main, the co-activation runs on side)
    cudaStream_t s_lay = nullptr;
    mpb_context *lay = nullptr;
    cudaEvent_t ev_join2 = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_fork = nullptr, ev_join = nullptr,
                ev_zero = nullptr;
    std::vector<cudaEvent_t> ev_done;
    // router timing: kRing sets of (start, end) events per chunk; run r of the
    // LAYERS phase records into set r % kRing, so the per-layer router time can
    // be averaged over every run of a timed region (graphs: the event-record
    // nodes are re-pointed at the run's set before each launch)
    static constexpr uint32_t kRing = 64;
    std::vector<cudaEvent_t> ev_r0, ev_r1;  // [kRing][chunk]
    uint64_t runs = 0, timing_from = 0;
    // graphs: the LAYERS phase, the SCORE phase (a caller that all-reduces the
    // statistics itself runs them separately) and both in one graph
    using RecNodes = std::vector<std::pair<cudaGraphNode_t, uint32_t>>;  // (node, chunk*2 + end)
    cudaGraph_t graph_layers = nullptr, graph_all = nullptr;
    RecNodes rec_layers, rec_all;
    cudaGraphExec_t g_layers = nullptr, g_score = nullptr, g_all = nullptr;
    uint64_t launches[4] = {0, 0, 0, 0};  // per phase mask (1, 2, 3)
    bool capturing = false;
    // stream the phases order against: the caller's stream, or during capture
    // a plan-owned origin stream (the legacy default stream cannot capture)
    cudaStream_t origin = nullptr, s_cap = nullptr;
    // multi-GPU (mpb_step_attach_comm)
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0;
    std::vector<mpb_gather_spec> gather;
    // MPB_STEP_PROBE=1 (experiments, eager runs only): timing events at the
    // step's start, after each chunk's router (main) and after each chunk's
    // statistics tails + pricing (their stream), and at the end
    bool probe = false;
    cudaEvent_t ev_p0 = nullptr, ev_p1 = nullptr;
    std::vector<cudaEvent_t> ev_pr, ev_pt;
};

namespace {

using namespace mpb;

std::vector<std::pair<uint32_t, uint32_t>> taper_chunks(uint32_t L, uint32_t G) {
    std::vector<uint32_t> tail;
    uint32_t sum = 0;
    for (uint32_t c = 1; c < G && sum + c <= L; c *= 2) {
        tail.insert(tail.begin(), c);
        sum += c;
    }
    const uint32_t rest = L - sum;
    std::vector<uint32_t> sizes;
    if (rest % G) sizes.push_back(rest % G);
    for (uint32_t i = 0; i < rest / G; ++i) sizes.push_back(G);
    sizes.insert(sizes.end(), tail.begin(), tail.end());
    std::vector<std::pair<uint32_t, uint32_t>> out;
    uint32_t l0 = 0;
    for (uint32_t n : sizes) {
        out.emplace_back(l0, l0 + n);
        l0 += n;
    }
    return out;
}

bool fused_single(const mpb_step *s) { return s->fused_ok && !s->comm; }

mpb_status record(mpb_step *s, cudaEvent_t ev, cudaStream_t st, bool timing) {
#ifdef MPB_EXP_NO_TIMING  // experiment: the step without its router timing events
    if (timing) return MPB_OK;
#endif
    // timing events inside a capture must be external nodes to stay readable
    MPB_CUDA(cudaEventRecordWithFlags(ev, st, (timing && s->capturing) ? cudaEventRecordExternal : 0));
    return MPB_OK;
}

mpb_status tail(mpb_step *s, mpb_context *c, uint32_t l, bool scratch_demand = false,
                bool scratch_perm = false) {
    const mpb_step_desc &d = s->d;
    const uint32_t D = d.deployed->D, E = d.E;
    const size_t pairs = static_cast<size_t>(d.T) * d.k;
    mpb_tokens tk{d.idx + l * pairs, d.T, d.k, d.src_group, 0, 0, d.tag, d.n_tags, d.src_group2};
    uint64_t *dem = d.demand + static_cast<size_t>(l) * D * E;
    uint64_t *dem2 = d.demand2 ? d.demand2 + static_cast<size_t>(l) * D * E : nullptr;
    if (scratch_demand) {  // the router counted the demand; the layout's copy is discarded
        dem = s->scratch_demand;
        dem2 = d.demand2 ? s->scratch_demand + static_cast<size_t>(D) * E : nullptr;
    }
    int32_t *sp = d.sorted_pairs, *pp = d.pair_pos;
    int64_t *ko = d.key_offsets;
    if (scratch_perm && ko) {  // a permutation the step's later layers overwrite anyway
        sp = static_cast<int32_t *>(s->side_perm);
        pp = sp + pairs;
        ko = reinterpret_cast<int64_t *>(pp + pairs);
    }
    if (mpb_status st = mpb_dispatch_layout(c, &tk, d.deployed, dem, dem2, d.tag_pop, sp, pp, ko))
        return st;
    return MPB_OK;
}

// Layers [l0, l1) of the statistics tail in one launch set; their permutations
// go to the plan's scratch (the caller's buffers keep the step's last layer).
mpb_status tail_batch(mpb_step *s, mpb_context *c, uint32_t l0, uint32_t l1) {
    const mpb_step_desc &d = s->d;
    const uint32_t D = d.deployed->D, E = d.E;
    const size_t pairs = static_cast<size_t>(d.T) * d.k;
    const size_t DE = static_cast<size_t>(D) * E;
    mpb_tokens tk{d.idx + l0 * pairs, d.T, d.k, d.src_group, 0, 0, d.tag, d.n_tags, d.src_group2};
    int32_t *sp = static_cast<int32_t *>(s->perm_scratch);
    int32_t *pp = sp + size_t(s->max_chunk) * pairs;
    int64_t *ko = reinterpret_cast<int64_t *>(pp + size_t(s->max_chunk) * pairs);
    return mpb_dispatch_layout_layers(c, l1 - l0, &tk, d.deployed, d.demand + l0 * DE,
                                      d.demand2 ? d.demand2 + l0 * DE : nullptr, d.tag_pop, sp, pp, ko);
}

// In-place all-reduce (sum, uint64) of layers [l0, l1) of the per-layer demand
// tables, plus the whole-step tag / co-activation tables when `whole`.
mpb_status reduce_stats(mpb_step *s, uint32_t l0, uint32_t l1, bool whole, cudaStream_t st) {
    if (!s->comm) return MPB_OK;
    const mpb_step_desc &d = s->d;
    const size_t DE = static_cast<size_t>(d.deployed->D) * d.E;
    const NcclApi &n = nccl();
    MPB_NCCL(n.group_start());
    MPB_NCCL(n.all_reduce(d.demand + l0 * DE, d.demand + l0 * DE, (l1 - l0) * DE, ncclUint64, ncclSum,
                          s->comm, st));
    if (d.demand2)
        MPB_NCCL(n.all_reduce(d.demand2 + l0 * DE, d.demand2 + l0 * DE, (l1 - l0) * DE, ncclUint64,
                              ncclSum, s->comm, st));
    if (whole && d.tag_pop && d.n_tags)
        MPB_NCCL(n.all_reduce(d.tag_pop, d.tag_pop, size_t(d.n_tags) * d.E, ncclUint64, ncclSum, s->comm, st));
    if (whole && d.coact)
        MPB_NCCL(n.all_reduce(d.coact, d.coact, size_t(d.E) * d.E, ncclUint64, ncclSum, s->comm, st));
    MPB_NCCL(n.group_end());
    return MPB_OK;
}

// In-place all-gather of the sharded score outputs (rank r's slice at r * bytes).
mpb_status gather_scores(mpb_step *s, cudaStream_t st) {
    if (!s->comm || s->gather.empty()) return MPB_OK;
    const NcclApi &n = nccl();
    MPB_NCCL(n.group_start());
    for (const mpb_gather_spec &g : s->gather) {
        char *base = static_cast<char *>(g.buf);
        MPB_NCCL(n.all_gather(base + size_t(s->rank) * g.bytes_per_rank, base, g.bytes_per_rank, ncclUint8,
                              s->comm, st));
    }
    MPB_NCCL(n.group_end());
    return MPB_OK;
}

mpb_status launch_router(mpb_step *s, size_t c) {
    const mpb_step_desc &d = s->d;
    const size_t pairs = static_cast<size_t>(d.T) * d.k;
    const auto [l0, l1] = s->chunks[c];
    const size_t set = (s->runs % mpb_step::kRing) * s->chunks.size();
    // one layer: both stamps go on the side stream (run_layers takes the start
    // stamp there), so no event-record node sits on the main stream's router ->
    // layout chain (each costs ~3 us in a graph)
    // consecutive routers share a stamp: the end of chunk c-1 is the start of c
    if (s->overlapped && c == 0)
        if (mpb_status st = record(s, s->ev_r0[set + c], s->s_main, true)) return st;
    mpb_status st;
    if (fused_single(s))
        st = mpb_router_topk_demand(s->main, s->X[l0], s->W[l0], d.T, d.H, d.E, d.k, d.score_fn, d.renorm,
                                    d.idx + l0 * pairs, d.weights + l0 * pairs, nullptr, d.src_group,
                                    d.src_group2, d.deployed->D, d.demand, d.demand2);
    else if (l1 - l0 == 1)
        st = mpb_router_topk(s->main, s->X[l0], s->W[l0], d.T, d.H, d.E, d.k, d.score_fn, d.renorm,
                             d.idx + l0 * pairs, d.weights + l0 * pairs, nullptr);
    else
        st = mpb_router_topk_layers(s->main, l1 - l0, s->X.data() + l0, s->W.data() + l0, d.T, d.H, d.E,
                                    d.k, d.score_fn, d.renorm, d.idx + l0 * pairs,
                                    d.weights + l0 * pairs, nullptr);
    if (st) return st;
    if (s->overlapped) {
        if ((st = record(s, s->ev_r1[set + c], s->s_main, true))) return st;
        MPB_CUDA(cudaEventRecord(s->ev_done[c], s->s_main));
        if (s->probe && !s->capturing) MPB_CUDA(cudaEventRecord(s->ev_pr[c], s->s_main));
    } else {
        // one layer: the end stamp is taken on the (idle) side stream, so no
        // event-record node sits between the router and the layout on the main
        // stream (which would cut their programmatic-launch overlap)
        MPB_CUDA(cudaEventRecord(s->ev_done[c], s->s_main));
        MPB_CUDA(cudaStreamWaitEvent(s->s_side, s->ev_done[c], 0));
        if ((st = record(s, s->ev_r1[set + c], s->s_side, true))) return st;
    }
    return MPB_OK;
}

mpb_status run_layers(mpb_step *s) {
    const mpb_step_desc &d = s->d;
    const size_t pairs = static_cast<size_t>(d.T) * d.k;
    MPB_CUDA(cudaEventRecord(s->ev_in, s->origin));
    MPB_CUDA(cudaStreamWaitEvent(s->s_main, s->ev_in, 0));
    MPB_CUDA(cudaStreamWaitEvent(s->s_side, s->ev_in, 0));
    // the statistics buffer is zeroed on the side stream, beside the first
    // router (nothing reads or writes it before that router's tails); the main
    // stream's own tails (single layer / last chunk) wait for it
    if (!s->overlapped) {  // the router's start stamp: the side passes the point the router waits on
        const size_t set = (s->runs % mpb_step::kRing) * s->chunks.size();
        if (mpb_status st = record(s, s->ev_r0[set], s->s_side, true)) return st;
    }
    // fused single layer: the router itself counts into the buffer, so the
    // zeroing is on its own stream (a memset node ahead of it, no cross-stream
    // event on the critical chain)
    const bool zero_on_main = fused_single(s) && d.zero_base && d.zero_bytes;
    if (zero_on_main) {
        MPB_CUDA(cudaMemsetAsync(d.zero_base, 0, d.zero_bytes, s->s_main));
    } else if (d.zero_base && d.zero_bytes) {
        MPB_CUDA(cudaMemsetAsync(d.zero_base, 0, d.zero_bytes, s->s_side));
        MPB_CUDA(cudaEventRecord(s->ev_zero, s->s_side));
    }
    const bool probe = s->probe && !s->capturing;
    if (probe) MPB_CUDA(cudaEventRecord(s->ev_p0, s->s_main));
    bool main_zeroed = !(d.zero_base && d.zero_bytes) || zero_on_main;
    auto main_waits_zero = [&]() -> mpb_status {
        if (!main_zeroed) {
            MPB_CUDA(cudaStreamWaitEvent(s->s_main, s->ev_zero, 0));
            main_zeroed = true;
        }
        return MPB_OK;
    };
    mpb_status st;
    if (s->overlapped) {
        // router c+1 is enqueued before the tails of chunk c, so the main stream
        // never idles while the host enqueues the side stream's launches
        const size_t nc = s->chunks.size();
        const uint32_t boost = std::min<uint32_t>(s->tail_boost, static_cast<uint32_t>(nc) - 1);
        auto budgets = [&](bool boosted) {
            const uint32_t side = boosted ? 2 * s->side_sms : s->side_sms;
            mpb_context_set_sm_budget(s->side, side);
            mpb_context_set_sm_budget(s->main, s->dev_sms - side);
        };
        if (boost) budgets(false);
        if ((st = launch_router(s, 0))) return st;
        for (size_t c = 0; c < nc; ++c) {
            if (boost && c + 1 == nc - boost) budgets(true);  // routers nc-boost.. and the tails beside them
            if (c + 1 < nc && (st = launch_router(s, c + 1))) return st;
            mpb_context *tc = s->side;
            const uint32_t on_main = s->comm ? 1u : s->main_tail_chunks;
            if (d.score_per_chunk && on_main > 1 && c + on_main >= nc) {
                // one GPU: the last chunks' tails on the main stream's grids right
                // after the last routers, beside the side stream's backlog
                if ((st = main_waits_zero())) return st;
                tc = s->main;
            } else if (d.score_per_chunk && c + 1 == nc) {
                // nothing runs beside the last chunk's tails: they take the main
                // stream's grids, after the side stream's earlier tails
                MPB_CUDA(cudaEventRecord(s->ev_join, s->s_side));
                MPB_CUDA(cudaStreamWaitEvent(s->s_main, s->ev_join, 0));
                main_zeroed = true;
                tc = s->main;
            } else {
                MPB_CUDA(cudaStreamWaitEvent(s->s_side, s->ev_done[c], 0));
            }
            const auto [l0, l1] = s->chunks[c];
            if (s->layout_batch && d.key_offsets) {
                // layers [l0, lb) batched into the scratch permutations; the
                // step's last layer (if in this chunk) into the caller's
                const uint32_t lb = l1 == d.layers ? l1 - 1 : l1;
                for (uint32_t b0 = l0; b0 < lb; b0 += s->layout_batch)
                    if ((st = tail_batch(s, tc, b0, std::min(lb, b0 + s->layout_batch)))) return st;
                for (uint32_t l = lb; l < l1; ++l)
                    if ((st = tail(s, tc, l))) return st;
            } else {
                const bool sp_side = tc == s->side && s->side_perm;
                for (uint32_t l = l0; l < l1; ++l)
                    if ((st = tail(s, tc, l, false, sp_side))) return st;
            }
            // the co-activation sums over tokens and layers alike: the chunk's
            // contiguous [l1 - l0][T][k] routing is ONE token list (one launch pair
            // per chunk instead of per layer; integer sums, the same matrix)
            if (d.coact && (st = mpb_coactivation(tc, d.idx + l0 * pairs, uint64_t(l1 - l0) * d.T, d.k,
                                                  d.E, d.coact)))
                return st;
            // multi-GPU: this chunk's demand becomes global before it is priced
            if ((st = reduce_stats(s, l0, l1, c + 1 == nc, tc->stream))) return st;
            if (d.score_per_chunk) {
                if (s->jobs.size() == 2 && s->jobs[0].B == d.layers && s->jobs[1].B == d.layers) {
                    if ((st = score_finalize_pair(tc, s->jobs[0], s->jobs[1], l0, l1 - l0))) return st;
                } else {
                    for (const mpb_score_job &j : s->jobs)
                        if (j.B == d.layers && (st = score_finalize_range(tc, j, l0, l1 - l0))) return st;
                }
                if (c + 1 == nc && (st = gather_scores(s, tc->stream))) return st;
            }
            if (probe) MPB_CUDA(cudaEventRecord(s->ev_pt[c], tc->stream));
        }
    } else if (fused_single(s)) {
        // router (with the demand count), then three branches at once: the
        // layout + permutation, the pricing and the co-activation
        if ((st = main_waits_zero())) return st;
        if ((st = launch_router(s, 0))) return st;
        MPB_CUDA(cudaEventRecord(s->ev_fork, s->s_main));
        MPB_CUDA(cudaStreamWaitEvent(s->s_side, s->ev_fork, 0));
        MPB_CUDA(cudaStreamWaitEvent(s->s_lay, s->ev_fork, 0));
        if (d.coact && (st = mpb_coactivation(s->side, d.idx, d.T, d.k, d.E, d.coact))) return st;
        // the longer of the two (the layout) follows the router on its own
        // stream (programmatic launch overlaps its prologue with the router's
        // drain); the pricing goes to the third stream
        const char *lm = std::getenv("MPB_DECODE_LAYOUT_MAIN");
        const bool layout_main = !(lm && lm[0] == '0');
        mpb_context *c_lay = layout_main ? s->main : s->lay, *c_score = layout_main ? s->lay : s->main;
        if ((st = tail(s, c_lay, 0, true))) return st;
        if (s->jobs.size() == 2 && s->jobs[0].B == d.layers && s->jobs[1].B == d.layers) {
            if ((st = score_finalize_pair(c_score, s->jobs[0], s->jobs[1], 0, 1))) return st;
        } else {
            for (const mpb_score_job &j : s->jobs)
                if (j.B == d.layers && (st = score_finalize_range(c_score, j, 0, 1))) return st;
        }
        MPB_CUDA(cudaEventRecord(s->ev_join2, s->s_lay));
        MPB_CUDA(cudaStreamWaitEvent(s->s_main, s->ev_join2, 0));
    } else {
        for (size_t c = 0; c < s->chunks.size(); ++c) {
            if ((st = launch_router(s, c))) return st;
            if ((st = main_waits_zero())) return st;
            for (uint32_t l = s->chunks[c].first; l < s->chunks[c].second; ++l) {
                if (d.coact) {  // co-activation beside the layout (both only read idx)
                    MPB_CUDA(cudaEventRecord(s->ev_fork, s->s_main));
                    MPB_CUDA(cudaStreamWaitEvent(s->s_side, s->ev_fork, 0));
                    if ((st = mpb_coactivation(s->side, d.idx + l * pairs, d.T, d.k, d.E, d.coact))) return st;
                }
                if ((st = tail(s, s->main, l))) return st;
                if (d.coact) {
                    MPB_CUDA(cudaEventRecord(s->ev_join, s->s_side));
                    MPB_CUDA(cudaStreamWaitEvent(s->s_main, s->ev_join, 0));
                }
            }
        }
    }
    MPB_CUDA(cudaEventRecord(s->ev_join, s->s_side));
    MPB_CUDA(cudaStreamWaitEvent(s->s_main, s->ev_join, 0));
    if (!s->overlapped && (st = reduce_stats(s, 0, d.layers, true, s->s_main))) return st;
    if (probe) MPB_CUDA(cudaEventRecord(s->ev_p1, s->s_main));
    MPB_CUDA(cudaEventRecord(s->ev_out, s->s_main));
    MPB_CUDA(cudaStreamWaitEvent(s->origin, s->ev_out, 0));
    return MPB_OK;
}

bool score_in_layers(const mpb_step *s, const mpb_score_job &j) {
    return (s->overlapped || fused_single(s)) && s->d.score_per_chunk && j.B == s->d.layers;
}

mpb_status run_score(mpb_step *s) {
    bool any = false;
    for (const mpb_score_job &j : s->jobs) any = any || !score_in_layers(s, j);
    if (!any) return MPB_OK;
    MPB_CUDA(cudaEventRecord(s->ev_in, s->origin));
    MPB_CUDA(cudaStreamWaitEvent(s->s_main, s->ev_in, 0));
    if (s->jobs.size() == 2 && s->jobs[0].B == s->jobs[1].B && !score_in_layers(s, s->jobs[0]) &&
        !score_in_layers(s, s->jobs[1])) {
        // both tables in one launch on the main stream (no side stream, no join)
        if (mpb_status st = score_finalize_pair(s->main, s->jobs[0], s->jobs[1], 0, s->jobs[0].B)) return st;
        if (mpb_status st = gather_scores(s, s->s_main)) return st;
        MPB_CUDA(cudaEventRecord(s->ev_out, s->s_main));
        MPB_CUDA(cudaStreamWaitEvent(s->origin, s->ev_out, 0));
        return MPB_OK;
    }
    MPB_CUDA(cudaStreamWaitEvent(s->s_side, s->ev_in, 0));
    for (size_t j = 0; j < s->jobs.size(); ++j) {
        const mpb_score_job &b = s->jobs[j];
        if (score_in_layers(s, b)) continue;
        mpb_context *c = j == 0 ? s->main : s->side;
        if (mpb_status st = mpb_score_placements_finalize(
                c, b.demand, b.B, b.rows, b.row_node, b.luts, b.P, b.group_to_node, b.D, b.nodes, b.E,
                b.inter, b.intra, b.rank_pairs, b.cost, b.tp_exp, b.spans_nodes, b.out, b.payload))
            return st;
    }
    MPB_CUDA(cudaEventRecord(s->ev_join, s->s_side));
    MPB_CUDA(cudaStreamWaitEvent(s->s_main, s->ev_join, 0));
    if (mpb_status st = gather_scores(s, s->s_main)) return st;
    MPB_CUDA(cudaEventRecord(s->ev_out, s->s_main));
    MPB_CUDA(cudaStreamWaitEvent(s->origin, s->ev_out, 0));
    return MPB_OK;
}

mpb_status run_phases(mpb_step *s, uint32_t phases) {
    if (!s->capturing) s->origin = s->ctx->stream;
    if (phases & MPB_STEP_LAYERS)
        if (mpb_status st = run_layers(s)) return st;
    if (phases & MPB_STEP_SCORE)
        if (mpb_status st = run_score(s)) return st;
    return MPB_OK;
}

uint64_t launch_total(const mpb_step *s) {
    return s->main->launches + s->side->launches + (s->lay ? s->lay->launches : 0);
}

}  // namespace

extern "C" {

mpb_status mpb_step_create(mpb_context *ctx, const mpb_step_desc *desc, mpb_step **out) {
    if (!ctx || !desc || !out) return fail(MPB_VALIDATION_ERROR, "mpb_step_create: NULL argument");
    *out = nullptr;
    const mpb_step_desc &d = *desc;
    if (!d.layers || !d.T || !d.X || !d.W || !d.idx || !d.weights || !d.deployed || !d.demand)
        return fail(MPB_VALIDATION_ERROR, "mpb_step_create: missing layers / X / W / idx / weights / "
                                          "deployed placement / demand");
    if (d.deployed->E != d.E) return fail(MPB_CONFIG_ERROR, "mpb_step_create: placement E != E");
    if (d.n_score_jobs && !d.score_jobs) return fail(MPB_VALIDATION_ERROR, "mpb_step_create: NULL score_jobs");
    if ((d.sorted_pairs || d.pair_pos || d.key_offsets) && !(d.sorted_pairs && d.pair_pos && d.key_offsets))
        return fail(MPB_VALIDATION_ERROR, "mpb_step_create: permutation outputs: all three or none");
    auto *s = new mpb_step();
    s->ctx = ctx;
    s->d = d;
    s->X.assign(d.X, d.X + d.layers);
    s->W.assign(d.W, d.W + d.layers);
    s->d.X = s->d.W = nullptr;
    if (d.n_score_jobs) s->jobs.assign(d.score_jobs, d.score_jobs + d.n_score_jobs);
    s->d.score_jobs = nullptr;
    s->overlapped = d.layers > 1;
    const uint32_t side_sms = d.side_sms ? d.side_sms : 20;
    const uint32_t G = d.router_group ? d.router_group : 8;
    if (s->overlapped)
        s->chunks = taper_chunks(d.layers, G);
    else
        s->chunks.emplace_back(0, 1);
    auto cleanup = [&](mpb_status st) {
        mpb_step_destroy(s);
        return st;
    };
    int lo = 0, hi = 0;
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
    // the router chain gets the high-priority stream: when SMs free up, the
    // block scheduler serves its CTAs before the tails'
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&s->s_main, cudaStreamNonBlocking, hi);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&s->s_side, cudaStreamNonBlocking, lo);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->s_cap, cudaStreamNonBlocking);
    for (cudaEvent_t *ev : {&s->ev_in, &s->ev_out, &s->ev_fork, &s->ev_join, &s->ev_zero})
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    const size_t nc = s->chunks.size();
    s->ev_done.assign(nc, nullptr);
    s->ev_r0.assign(nc * mpb_step::kRing, nullptr);
    s->ev_r1.assign(nc * mpb_step::kRing, nullptr);
    for (size_t c = 0; c < nc && e == cudaSuccess; ++c) {
        e = cudaEventCreateWithFlags(&s->ev_done[c], cudaEventDisableTiming);
    }
    for (size_t i = 0; i < s->ev_r0.size() && e == cudaSuccess; ++i) {
        e = cudaEventCreate(&s->ev_r0[i]);
        if (e == cudaSuccess) e = cudaEventCreate(&s->ev_r1[i]);
    }
    if (const char *pe = std::getenv("MPB_STEP_PROBE"); pe && pe[0] == '1' && e == cudaSuccess) {
        s->probe = true;
        s->ev_pr.assign(nc, nullptr);
        s->ev_pt.assign(nc, nullptr);
        e = cudaEventCreate(&s->ev_p0);
        if (e == cudaSuccess) e = cudaEventCreate(&s->ev_p1);
        for (size_t c = 0; c < nc && e == cudaSuccess; ++c) {
            e = cudaEventCreate(&s->ev_pr[c]);
            if (e == cudaSuccess) e = cudaEventCreate(&s->ev_pt[c]);
        }
    }
    {
        const char *fe = std::getenv("MPB_ROUTER_DEMAND");
        s->fused_ok = !s->overlapped && d.layers == 1 && d.score_per_chunk && d.src_group && d.demand &&
                      d.deployed && d.deployed->D <= 255 && d.E <= 256 && !(fe && fe[0] == '0');
        if (s->fused_ok && e == cudaSuccess)
            e = cudaMalloc(&s->scratch_demand, 2 * sizeof(uint64_t) * d.deployed->D * d.E);
    }
    if (s->overlapped && e == cudaSuccess) {
        if (const char *mt = std::getenv("MPB_MAIN_TAIL_CHUNKS"))
            s->main_tail_chunks = static_cast<uint32_t>(std::max(1, std::atoi(mt)));
        if (s->main_tail_chunks > 1 && d.key_offsets && d.deployed) {
            const size_t pairs = static_cast<size_t>(d.T) * d.k;
            const size_t DE1 = static_cast<size_t>(d.deployed->D) * d.E + 1;
            e = cudaMalloc(&s->side_perm, 2 * pairs * 4 + DE1 * 8 + 16);
        }
    }
    if (s->overlapped && e == cudaSuccess) {
        const char *lb = std::getenv("MPB_LAYOUT_BATCH");
        s->layout_batch = (d.key_offsets && d.deployed) ? (lb ? static_cast<uint32_t>(std::max(0, std::atoi(lb))) : 4u)
                                                        : 0u;
        if (s->layout_batch == 1) s->layout_batch = 0;  // one layer: the plain per-layer call
        for (const auto &ch : s->chunks) s->max_chunk = std::max(s->max_chunk, ch.second - ch.first);
        if (s->layout_batch) {
            const size_t pairs = static_cast<size_t>(d.T) * d.k;
            const size_t DE1 = static_cast<size_t>(d.deployed->D) * d.E + 1;
            const size_t bytes = size_t(s->max_chunk) * (2 * pairs * 4 + DE1 * 8) + 16;
            e = cudaMalloc(&s->perm_scratch, bytes);
        }
    }
    if (e != cudaSuccess) return cleanup(cuda_fail(e, "mpb_step_create"));
    if (mpb_status st = mpb_context_create(ctx->device, s->s_main, &s->main)) return cleanup(st);
    if (mpb_status st = mpb_context_create(ctx->device, s->s_side, &s->side)) return cleanup(st);
    if (s->fused_ok) {
        cudaError_t e3 = cudaStreamCreateWithPriority(&s->s_lay, cudaStreamNonBlocking, lo);
        if (e3 == cudaSuccess) e3 = cudaEventCreateWithFlags(&s->ev_join2, cudaEventDisableTiming);
        if (e3 != cudaSuccess) return cleanup(cuda_fail(e3, "mpb_step_create"));
        if (mpb_status st = mpb_context_create(ctx->device, s->s_lay, &s->lay)) return cleanup(st);
    }
    if (s->overlapped) {
        const uint32_t dev_sms = static_cast<uint32_t>(ctx->device_sms);
        if (side_sms >= dev_sms) return cleanup(fail(MPB_CONFIG_ERROR, "mpb_step_create: side_sms >= SMs"));
        mpb_context_set_sm_budget(s->side, side_sms);
        mpb_context_set_sm_budget(s->main, dev_sms - side_sms);
        s->side_sms = side_sms;
        s->dev_sms = dev_sms;
        if (const char *tb = std::getenv("MPB_TAIL_BOOST"))
            s->tail_boost = 2 * side_sms < dev_sms ? static_cast<uint32_t>(std::max(0, std::atoi(tb))) : 0;
    }
    *out = s;
    return MPB_OK;
}

mpb_status mpb_step_destroy(mpb_step *s) {
    if (!s) return MPB_OK;
    if (s->s_main) cudaStreamSynchronize(s->s_main);
    if (s->s_side) cudaStreamSynchronize(s->s_side);
    if (s->s_lay) cudaStreamSynchronize(s->s_lay);
    if (s->g_layers) cudaGraphExecDestroy(s->g_layers);
    if (s->graph_layers) cudaGraphDestroy(s->graph_layers);
    if (s->g_all) cudaGraphExecDestroy(s->g_all);
    if (s->graph_all) cudaGraphDestroy(s->graph_all);
    if (s->g_score) cudaGraphExecDestroy(s->g_score);
    if (s->comm) nccl().destroy(s->comm);
    mpb_context_destroy(s->main);
    mpb_context_destroy(s->side);
    if (s->lay) mpb_context_destroy(s->lay);
    if (s->ev_join2) cudaEventDestroy(s->ev_join2);
    if (s->s_lay) cudaStreamDestroy(s->s_lay);
    for (cudaEvent_t ev : {s->ev_in, s->ev_out, s->ev_fork, s->ev_join, s->ev_zero, s->ev_p0, s->ev_p1})
        if (ev) cudaEventDestroy(ev);
    for (auto *v : {&s->ev_done, &s->ev_r0, &s->ev_r1, &s->ev_pr, &s->ev_pt})
        for (cudaEvent_t ev : *v)
            if (ev) cudaEventDestroy(ev);
    if (s->scratch_demand) cudaFree(s->scratch_demand);
    if (s->perm_scratch) cudaFree(s->perm_scratch);
    if (s->side_perm) cudaFree(s->side_perm);
    if (s->s_main) cudaStreamDestroy(s->s_main);
    if (s->s_side) cudaStreamDestroy(s->s_side);
    if (s->s_cap) cudaStreamDestroy(s->s_cap);
    delete s;
    return MPB_OK;
}

}  // extern "C"

namespace {

// Points the graph's router timing nodes at ring set `runs % kRing`.
mpb_status retarget_timing(mpb_step *s, cudaGraphExec_t g, const mpb_step::RecNodes &rec) {
    const size_t set = (s->runs % mpb_step::kRing) * s->chunks.size();
    for (const auto &[node, which] : rec)
        MPB_CUDA(cudaGraphExecEventRecordNodeSetEvent(
            g, node, (which & 1) ? s->ev_r1[set + which / 2] : s->ev_r0[set + which / 2]));
    return MPB_OK;
}

// Captures `phases` into an executable graph (on the plan's origin stream); for
// graphs with the LAYERS phase, finds the router timing nodes.
mpb_status capture_graph(mpb_step *s, uint32_t phases, cudaGraphExec_t *exec, cudaGraph_t *keep,
                         mpb_step::RecNodes *rec) {
    MPB_CUDA(cudaStreamBeginCapture(s->s_cap, cudaStreamCaptureModeRelaxed));
    s->capturing = true;
    s->origin = s->s_cap;
    mpb_status st = run_phases(s, phases);
    s->capturing = false;
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(s->s_cap, &g);
    if (st) {
        if (g) cudaGraphDestroy(g);
        return st;
    }
    if (e != cudaSuccess) return cuda_fail(e, "mpb_step_capture: cudaStreamEndCapture");
    // per-node priorities (captured from the streams): the routers keep their
    // high priority over the statistics tails inside the graph too
    const cudaError_t e2 = cudaGraphInstantiate(exec, g, cudaGraphInstantiateFlagUseNodePriority);
    if (e2 != cudaSuccess) {
        cudaGraphDestroy(g);
        return cuda_fail(e2, "mpb_step_capture: cudaGraphInstantiate");
    }
    if (!(phases & MPB_STEP_LAYERS)) {
        cudaGraphDestroy(g);
        return MPB_OK;
    }
    *keep = g;  // node handles stay valid while the graph lives
    size_t n = 0;
    MPB_CUDA(cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    MPB_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
    const size_t set = (s->runs % mpb_step::kRing) * s->chunks.size();
    for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType t;
        MPB_CUDA(cudaGraphNodeGetType(nd, &t));
        if (t != cudaGraphNodeTypeEventRecord) continue;
        cudaEvent_t ev;
        MPB_CUDA(cudaGraphEventRecordNodeGetEvent(nd, &ev));
        for (size_t c = 0; c < s->chunks.size(); ++c) {
            if (ev == s->ev_r0[set + c]) rec->emplace_back(nd, static_cast<uint32_t>(2 * c));
            if (ev == s->ev_r1[set + c]) rec->emplace_back(nd, static_cast<uint32_t>(2 * c + 1));
        }
    }
#ifdef MPB_EXP_NO_TIMING
    return MPB_OK;
#endif
    if (rec->size() != (s->overlapped ? s->chunks.size() + 1 : 2 * s->chunks.size()))
        return fail(MPB_CUDA_ERROR, "mpb_step_capture: router timing nodes not found in the graph");
    return MPB_OK;
}

}  // namespace

extern "C" {

mpb_status mpb_step_run(mpb_step *s, uint32_t phases) {
    if (!s) return fail(MPB_VALIDATION_ERROR, "mpb_step_run: NULL step");
    if (s->g_all && (phases & 3) == 3) {  // single GPU: the whole step, one graph
        if (mpb_status st = retarget_timing(s, s->g_all, s->rec_all)) return st;
        MPB_CUDA(cudaGraphLaunch(s->g_all, s->ctx->stream));
        ++s->runs;
        return MPB_OK;
    }
    if (s->g_layers || s->g_score) {
        if ((phases & MPB_STEP_LAYERS) && s->g_layers) {
            if (mpb_status st = retarget_timing(s, s->g_layers, s->rec_layers)) return st;
            MPB_CUDA(cudaGraphLaunch(s->g_layers, s->ctx->stream));
            ++s->runs;
        }
        if ((phases & MPB_STEP_SCORE) && s->g_score) MPB_CUDA(cudaGraphLaunch(s->g_score, s->ctx->stream));
        return MPB_OK;
    }
    const uint64_t n0 = launch_total(s);
    if (mpb_status st = run_phases(s, phases)) return st;
    s->launches[phases & 3] = launch_total(s) - n0;
    if (phases & MPB_STEP_LAYERS) ++s->runs;
    return MPB_OK;
}

mpb_status mpb_step_capture(mpb_step *s) {
    if (!s) return fail(MPB_VALIDATION_ERROR, "mpb_step_capture: NULL step");
    if (s->g_layers || s->g_score || s->g_all) return MPB_OK;
    // one eager run sizes every workspace and uploads the router descriptor tables
    for (uint32_t ph : {MPB_STEP_LAYERS, MPB_STEP_SCORE}) {
        const uint64_t n0 = launch_total(s);
        if (mpb_status st = run_phases(s, ph)) return st;
        s->launches[ph] = launch_total(s) - n0;
        if (ph == MPB_STEP_LAYERS) ++s->runs;
    }
    if (mpb_status st = mpb_step_sync(s)) return st;
    mpb_status st = capture_graph(s, MPB_STEP_LAYERS, &s->g_layers, &s->graph_layers, &s->rec_layers);
    bool any = false;
    for (const mpb_score_job &j : s->jobs) any = any || !score_in_layers(s, j);
    if (!st && any) {
        cudaGraph_t unused = nullptr;
        mpb_step::RecNodes none;
        st = capture_graph(s, MPB_STEP_SCORE, &s->g_score, &unused, &none);
    }
    if (!st) st = capture_graph(s, MPB_STEP_LAYERS | MPB_STEP_SCORE, &s->g_all, &s->graph_all, &s->rec_all);
    if (st) {  // all or nothing: a failed capture leaves the plan eager
        for (cudaGraphExec_t *g : {&s->g_layers, &s->g_score, &s->g_all})
            if (*g) cudaGraphExecDestroy(*g), *g = nullptr;
        for (cudaGraph_t *g : {&s->graph_layers, &s->graph_all})
            if (*g) cudaGraphDestroy(*g), *g = nullptr;
        s->rec_layers.clear();
        s->rec_all.clear();
        cudaGetLastError();
    }
    return st;
}

mpb_status mpb_step_sync(mpb_step *s) {
    if (!s) return fail(MPB_VALIDATION_ERROR, "mpb_step_sync: NULL step");
    MPB_CUDA(cudaStreamSynchronize(s->ctx->stream));
    mpb_status a = mpb_context_sync(s->main);
    mpb_status b = mpb_context_sync(s->side);
    mpb_status c = s->lay ? mpb_context_sync(s->lay) : MPB_OK;
    return a ? a : b ? b : c;
}

mpb_status mpb_step_timing_reset(mpb_step *s) {
    if (!s) return fail(MPB_VALIDATION_ERROR, "mpb_step_timing_reset: NULL step");
    s->timing_from = s->runs;
    return MPB_OK;
}

mpb_status mpb_step_router_ms(const mpb_step *s, float *ms, uint32_t *n_runs) {
    if (!s || !ms) return fail(MPB_VALIDATION_ERROR, "mpb_step_router_ms: NULL argument");
    uint64_t from = std::max(s->timing_from, s->runs > mpb_step::kRing ? s->runs - mpb_step::kRing : 0);
    if (from >= s->runs) from = s->runs ? s->runs - 1 : 0;  // nothing since the reset: the last run
    const size_t nc = s->chunks.size();
    for (uint32_t l = 0; l < s->d.layers; ++l) ms[l] = 0.f;
    for (uint64_t r = from; r < s->runs; ++r) {
        const size_t set = (r % mpb_step::kRing) * nc;
        for (size_t c = 0; c < nc; ++c) {
            float t = 0.f;
            const cudaEvent_t start = (s->overlapped && c > 0) ? s->ev_r1[set + c - 1] : s->ev_r0[set + c];
            MPB_CUDA(cudaEventElapsedTime(&t, start, s->ev_r1[set + c]));
            const auto [l0, l1] = s->chunks[c];
            for (uint32_t l = l0; l < l1; ++l) ms[l] += t / static_cast<float>(l1 - l0);
        }
    }
    const uint64_t n = s->runs - from;
    for (uint32_t l = 0; l < s->d.layers && n; ++l) ms[l] /= static_cast<float>(n);
    if (n_runs) *n_runs = static_cast<uint32_t>(n);
    return MPB_OK;
}

mpb_status mpb_step_info(const mpb_step *s, uint32_t phases, uint64_t *launches, uint32_t *chunks,
                         uint32_t *n_chunks) {
    if (!s) return fail(MPB_VALIDATION_ERROR, "mpb_step_info: NULL step");
    if (launches) {
        uint64_t n = s->launches[phases & 3];
        if (!n && phases == (MPB_STEP_LAYERS | MPB_STEP_SCORE))
            n = s->launches[MPB_STEP_LAYERS] + s->launches[MPB_STEP_SCORE];
        *launches = n;
    }
    if (n_chunks) *n_chunks = static_cast<uint32_t>(s->chunks.size());
    if (chunks)
        for (size_t c = 0; c < s->chunks.size(); ++c) chunks[c] = s->chunks[c].second - s->chunks[c].first;
    return MPB_OK;
}

mpb_status mpb_nccl_get_unique_id(uint8_t id[128]) {
    if (!id) return fail(MPB_VALIDATION_ERROR, "mpb_nccl_get_unique_id: NULL id");
    if (!nccl().ok) return fail(MPB_CONFIG_ERROR, "mpb_nccl_get_unique_id: libnccl.so.2 not found");
    ncclUniqueId u;
    MPB_NCCL(nccl().get_unique_id(&u));
    std::memcpy(id, u.internal, sizeof(u.internal));
    return MPB_OK;
}

mpb_status mpb_step_attach_comm(mpb_step *s, const uint8_t id[128], int world, int rank,
                                const mpb_gather_spec *gather, uint32_t n_gather) {
    if (!s || !id) return fail(MPB_VALIDATION_ERROR, "mpb_step_attach_comm: NULL argument");
    if (world < 1 || rank < 0 || rank >= world) return fail(MPB_CONFIG_ERROR, "mpb_step_attach_comm: bad rank");
    if (s->g_layers || s->g_score || s->g_all)
        return fail(MPB_CONFIG_ERROR, "mpb_step_attach_comm: attach before mpb_step_capture");
    if (n_gather && !gather) return fail(MPB_VALIDATION_ERROR, "mpb_step_attach_comm: NULL gather");
    if (!nccl().ok) return fail(MPB_CONFIG_ERROR, "mpb_step_attach_comm: libnccl.so.2 not found");
    if (s->comm) {
        nccl().destroy(s->comm);
        s->comm = nullptr;
    }
    s->world = world;
    s->rank = rank;
    s->gather.assign(gather, gather + n_gather);
    if (world == 1) return MPB_OK;
    ncclUniqueId u;
    std::memcpy(u.internal, id, sizeof(u.internal));
    MPB_CUDA(cudaSetDevice(s->ctx->device));
    MPB_NCCL(nccl().init_rank(&s->comm, world, u, rank));
    return MPB_OK;
}

}  // extern "C"

// Experiments (MPB_STEP_PROBE=1, eager runs): the last run's timeline in ms from
// its start — out[c] = router chunk c done, out[nc + c] = chunk c's statistics
// tails + pricing done, out[2 nc] = step end. Returns the number written.
extern "C" MPB_API int mpb_debug_step_probe(const mpb_step *s, float *out,
                                                                          size_t n) {
    if (!s || !s->probe || !out) return -1;
    const size_t nc = s->chunks.size();
    if (n < 2 * nc + 1) return -1;
    if (cudaEventSynchronize(s->ev_p1) != cudaSuccess) return -1;
    for (size_t c = 0; c < nc; ++c) {
        if (cudaEventElapsedTime(&out[c], s->ev_p0, s->ev_pr[c]) != cudaSuccess) return -1;
        if (cudaEventElapsedTime(&out[nc + c], s->ev_p0, s->ev_pt[c]) != cudaSuccess) return -1;
    }
    if (cudaEventElapsedTime(&out[2 * nc], s->ev_p0, s->ev_p1) != cudaSuccess) return -1;
    return static_cast<int>(2 * nc + 1);
}

// Tests: 1 when this plan's single-layer step counts the demand in the router
// (mpb_router_topk_demand) and prices it beside the layout.
extern "C" MPB_API int mpb_debug_step_fused(const mpb_step *s) {
    return s && fused_single(s) ? 1 : 0;
}
