/*
 * moeplace_b200 — C ABI of the B200-native MoE routing-and-placement hot path.
 *
 * Drop-in boundary for the reference's cost evaluator, metrics and routing
 * (arxiv/paper_2604_23150, /root/reference/proj/core). Plain pointers and
 * sizes only (no C++ or torch types); every device function is asynchronous on
 * the context's CUDA stream; status codes map 1:1 onto the reference's
 * exception classes (proj/core/include/moeplace/errors.hpp:11-66).
 *
 * Which reference interface each entry point replaces:
 *   mpb_placement_create   Placement + Topology holder resolution
 *                          (placement.hpp:35-65, simulator.cpp:52-55,74-80)
 *   mpb_router_topk        (new) router GEMM + top-k; feeds what route_tokens
 *                          produces (trace.cpp:240-259)
 *   mpb_router_topk_layers (new) the same for several layers in one launch
 *   mpb_router_topk_demand (new) mpb_router_topk + simulate_layer's demand
 *                          count (simulator.cpp:64-80) in its epilogue
 *   mpb_topk_logits        (new) top-k over given logits, tie rule of
 *                          placement.cpp:143-152
 *   mpb_dispatch_layout    simulate_layer's per-destination accounting
 *                          (simulator.cpp:61-88) + the token permutation
 *   mpb_dispatch_layout_layers  the same for several layers in one launch set
 *   mpb_layout_derive      per_rank_payload / tokens_per_group / inter-intra
 *                          split (simulator.cpp:81-88); column sums
 *                          (pipeline.cpp:76-82, simulator.cpp:253-258)
 *   mpb_coactivation       (new) expert x expert co-activation
 *   mpb_sample_batches / mpb_route_sources / mpb_batch_demand
 *                          compare_strategies batch sampling + assembly
 *                          (simulator.cpp:154-181)
 *   mpb_score_placements   simulate_layer over P candidates x B batches
 *                          (simulator.cpp:43-99)
 *   mpb_finalize_layer_sims padded_all_to_all_time + LayerSim times
 *   mpb_score_placements_finalize  the two above in one launch
 *                          (simulator.cpp:27-41, 90-98), bit-exact doubles
 *   mpb_dispatch_gather / mpb_combine_scatter  (new) physical bf16 dispatch /
 *                          combine around the all-to-all
 *   mpb_step_*             the host schedule of one routed step over all
 *                          layers (pipeline.cpp:316-443's route -> account ->
 *                          price loop), in C++ inside the library
 */
#ifndef MOEPLACE_B200_H
#define MOEPLACE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPB_ABI_VERSION 1
#define MPB_API __attribute__((visibility("default")))

/* Status codes: 1:1 with moeplace::Error subclasses (errors.hpp:11-66). */
typedef enum {
    MPB_OK = 0,
    MPB_ERROR = 1,                       /* moeplace::Error (generic)          */
    MPB_PARSE_ERROR = 2,                 /* moeplace::ParseError               */
    MPB_VALIDATION_ERROR = 3,            /* moeplace::ValidationError          */
    MPB_CONFIG_ERROR = 4,                /* moeplace::ConfigError              */
    MPB_EMPTY_SELECTION_ERROR = 5,       /* moeplace::EmptySelectionError      */
    MPB_UNDEFINED_CORRELATION_ERROR = 6, /* moeplace::UndefinedCorrelationError */
    MPB_INFEASIBLE_ERROR = 7,            /* moeplace::InfeasibleError          */
    MPB_LOOKUP_ERROR = 8,                /* moeplace::LookupError              */
    MPB_CUDA_ERROR = 9                   /* CUDA runtime failure (no reference analogue) */
} mpb_status;

typedef struct mpb_context mpb_context;
typedef struct mpb_placement mpb_placement;

/* ---- context ---------------------------------------------------------- */
MPB_API int mpb_abi_version(void);
/* Thread-local message of the last non-OK status. */
MPB_API const char *mpb_last_error_message(void);
/* Binds `device`; stream may be NULL (legacy default stream) or a cudaStream_t. */
MPB_API mpb_status mpb_context_create(int device, void *stream, mpb_context **out);
MPB_API mpb_status mpb_context_destroy(mpb_context *ctx);
MPB_API mpb_status mpb_context_set_stream(mpb_context *ctx, void *stream);
/* Caps the SMs this context's grids are sized for (persistent router units,
 * layout blocks, co-activation CTAs); 0 restores the device count. Two
 * contexts with disjoint budgets run their kernels concurrently (e.g. the
 * router of layer l+1 beside the statistics of layer l). */
MPB_API mpb_status mpb_context_set_sm_budget(mpb_context *ctx, uint32_t sms);
/* Like mpb_context_set_sm_budget, for a context whose stream belongs to an SM
 * partition (mpb_sm_partition_create): the hardware confines its kernels to
 * `sms` SMs, so early-launched (programmatic) CTAs cannot land elsewhere. */
MPB_API mpb_status mpb_context_set_sm_partition(mpb_context *ctx, uint32_t sms);
/* Splits the device's SMs into two green-context partitions, side >= side_sms
 * SMs (the hardware rounds up to its granularity, 8 on B200) and main = the
 * rest, and returns one stream (cudaStream_t) on each; kernels launched into a
 * stream run only on its partition's SMs. Reports the actual SM counts. */
MPB_API mpb_status mpb_sm_partition_create(int device, uint32_t side_sms, int main_priority,
                                           int side_priority, void **main_stream,
                                           void **side_stream, uint32_t *main_sms,
                                           uint32_t *side_sms_out);
MPB_API mpb_status mpb_sm_partition_destroy(void *main_stream);
/* Synchronises the stream and reports input errors the kernels flagged
 * (uncovered expert, id >= E, source group >= D -> MPB_VALIDATION_ERROR,
 * exactly where simulate_layer throws, simulator.cpp:66-71). Clears the flag. */
MPB_API mpb_status mpb_context_sync(mpb_context *ctx);
/* Number of kernels this context launched since creation (instrumentation). */
MPB_API uint64_t mpb_context_launch_count(const mpb_context *ctx);

/* ---- placement ---------------------------------------------------------
 * groups_flat concatenates D groups (group_sizes[d] experts each, host).
 * group_to_node[D] (host). Builds the device lookup tables: destination
 * group per (source node, expert) — same-node copy first, else the lowest
 * group id (simulator.cpp:74-80) — and the permutation's slot tables.
 * Like simulate_layer, coverage is checked lazily: an uncovered expert is an
 * error only when a token routes to it. D <= 255, E <= 65535, nodes <= D. */
MPB_API mpb_status mpb_placement_create(mpb_context *ctx, const uint32_t *groups_flat,
                                        const uint32_t *group_sizes, uint32_t D, uint32_t E,
                                        const uint32_t *group_to_node, mpb_placement **out);
MPB_API mpb_status mpb_placement_destroy(mpb_placement *p);
/* Device pointer to the [nodes x E] uint8 destination table (255 = uncovered),
 * the form mpb_score_placements consumes; nodes = max(group_to_node)+1. */
MPB_API const uint8_t *mpb_placement_dest_lut(const mpb_placement *p, uint32_t *nodes);
/* Same table computed on the host into dest_lut[nodes*E] (no device needed). */
MPB_API mpb_status mpb_build_dest_lut(const uint32_t *groups_flat, const uint32_t *group_sizes,
                                      uint32_t D, uint32_t E, const uint32_t *group_to_node,
                                      uint8_t *dest_lut);

/* ---- routing (gate) ----------------------------------------------------
 * score_fn: MPB_SCORE_SOFTMAX (softmax over all E) or MPB_SCORE_SIGMOID.
 * Selection is on the fp32 logits, descending, equal logits -> lower expert
 * id (the reference's lowest-index-wins rule), NaN ranks lowest. renorm != 0
 * divides the k weights by their sum. k <= 16. */
#define MPB_SCORE_SOFTMAX 0
#define MPB_SCORE_SIGMOID 1

/* Fused router: logits = X[T,H] . W[E,H]^T (bf16 in, fp32 accumulate on
 * tcgen05 tensor cores) -> top-k. X, W row-major bf16 (device); H % 64 == 0,
 * E in {64, 128, 256}. logits_out [T,E] fp32 is optional (NULL = not
 * materialised; used by parity tests). */
MPB_API mpb_status mpb_router_topk(mpb_context *ctx, const void *X, const void *W, uint64_t T,
                                   uint32_t H, uint32_t E, uint32_t k, int score_fn, int renorm,
                                   int32_t *idx, float *weights, float *logits_out);
/* mpb_router_topk for `layers` independent layers of the same shape in ONE
 * persistent launch: X[l] [T,H] and W[l] [E,H] (host arrays of device
 * pointers); idx / weights are [layers][T][k] (device); logits_out
 * [layers][T][E] fp32 is optional (NULL in the step; parity tests check the
 * grouped launch's top-k against the oracle on these logits). Results equal
 * mpb_router_topk per layer up to the fp32 order of the split-K tail (the last
 * wave of the whole launch). Only one exposed last-tile epilogue per launch
 * instead of one per layer. The TMA descriptors are encoded and uploaded on
 * the first call for a given (shape, X, W) set and cached in the context (the
 * first call must not be inside a stream capture). */
MPB_API mpb_status mpb_router_topk_layers(mpb_context *ctx, uint32_t layers, const void *const *X,
                                          const void *const *W, uint64_t T, uint32_t H, uint32_t E,
                                          uint32_t k, int score_fn, int renorm, int32_t *idx,
                                          float *weights, float *logits_out);
/* mpb_router_topk that also counts the dispatch demand as it writes each
 * selected (token, expert): demand[src_group[t]][e] += 1 (uint64 [D][E],
 * device, accumulated — the caller zeroes it), and demand2 under src_group2
 * when given (the same counts mpb_dispatch_layout produces: integer sums,
 * bit-identical). A source group >= D is flagged (MPB_VALIDATION_ERROR at
 * mpb_context_sync), not counted. Lets a single-layer step price the demand
 * right after the router while the permutation is built beside it. */
MPB_API mpb_status mpb_router_topk_demand(mpb_context *ctx, const void *X, const void *W, uint64_t T,
                                          uint32_t H, uint32_t E, uint32_t k, int score_fn, int renorm,
                                          int32_t *idx, float *weights, float *logits_out,
                                          const uint8_t *src_group, const uint8_t *src_group2, uint32_t D,
                                          uint64_t *demand, uint64_t *demand2);
/* Top-k over given fp32 logits [T,E] (device), E <= 1024. */
MPB_API mpb_status mpb_topk_logits(mpb_context *ctx, const float *logits, uint64_t T, uint32_t E,
                                   uint32_t k, int score_fn, int renorm, int32_t *idx,
                                   float *weights);

/* ---- dispatch layout (histograms + permutation) -------------------------
 * Tokens t < T carry k expert ids idx[t*k + j]; pair p = t*k + j. Source EP
 * group: src_group[t] (device uint8), or when src_group == NULL,
 * src_base + (t * src_span) / T (contiguous token blocks).
 * src_group2 (optional) is a second routing of the same tokens (e.g. the
 * round-robin baseline next to the cluster routing) accounted in the same
 * pass into demand2.
 * Outputs (device, ACCUMULATED with += so shards/layers can be fused; the
 * caller zeroes them):
 *   demand[D*E]       pairs per (source group, expert)        (uint64)
 *   demand2[D*E]      same under src_group2 (when given)
 *   tag_pop[n_tags*E] pairs per (tag[t], expert) if tag != NULL (uint64; tag[t]
 *                     uint16, tags >= n_tags are ignored):
 *                     per-domain popularity / per-stage vectors
 * Permutation (optional, all three or none; device):
 *   sorted_pairs[T*k] pairs ordered by (dest group, expert id, p) — stable
 *   pair_pos[T*k]     inverse: position of pair p
 *   key_offsets[D*E+1] start of key (d, e) = d*E + e in sorted order */
typedef struct {
    const int32_t *idx;
    uint64_t T;
    uint32_t k;
    const uint8_t *src_group;
    uint32_t src_base;
    uint32_t src_span;
    const uint16_t *tag;
    uint32_t n_tags;
    const uint8_t *src_group2;
} mpb_tokens;

MPB_API mpb_status mpb_dispatch_layout(mpb_context *ctx, const mpb_tokens *tokens,
                                       const mpb_placement *placement, uint64_t *demand,
                                       uint64_t *demand2, uint64_t *tag_pop,
                                       int32_t *sorted_pairs, int32_t *pair_pos,
                                       int64_t *key_offsets);
/* mpb_dispatch_layout for `layers` layers of the same T, k and placement in
 * ONE set of launches (grids over (block, layer)): tokens->idx is [layers][T][k];
 * demand / demand2 [layers][D][E], sorted_pairs / pair_pos [layers][T*k],
 * key_offsets [layers][D*E+1]; tag_pop sums over the layers. Per-token arrays
 * (src_group, src_group2, tag) are shared by every layer. Results equal
 * `layers` single-layer calls (integer counts, stable permutations). */
MPB_API mpb_status mpb_dispatch_layout_layers(mpb_context *ctx, uint32_t layers, const mpb_tokens *tokens,
                                              const mpb_placement *placement, uint64_t *demand,
                                              uint64_t *demand2, uint64_t *tag_pop,
                                              int32_t *sorted_pairs, int32_t *pair_pos,
                                              int64_t *key_offsets);

/* From demand[D*E] (device): expert_count[E] (column sums), group_pairs[D]
 * (tokens_per_group / per_rank payload in pairs), node_demand[nodes*E],
 * inter_intra[2] = {inter-node pairs, intra-node pairs}. Overwritten (not
 * accumulated). Any output may be NULL. */
MPB_API mpb_status mpb_layout_derive(mpb_context *ctx, const mpb_placement *placement,
                                     const uint64_t *demand, uint64_t *expert_count,
                                     uint64_t *group_pairs, uint64_t *node_demand,
                                     uint64_t *inter_intra);

/* ---- co-activation --------------------------------------------------------
 * coact[E*E] (device uint64, accumulated): number of tokens whose k picks
 * contain both i and j (symmetric; diagonal = tokens that picked i). Picks
 * within a token must be distinct (top-k guarantees it). Warp-ballot expert
 * masks + popc into register/shared tiles. */
MPB_API mpb_status mpb_coactivation(mpb_context *ctx, const int32_t *idx, uint64_t T, uint32_t k,
                                    uint32_t E, uint64_t *coact);

/* ---- batched placement scoring ------------------------------------------
 * Batch demand for compare_strategies: B batches x S sampled matrix rows.
 * matrix CSR (device): row_ptr[R+1], cols[nnz] (expert), vals[nnz] (integer
 * token counts); rows[B*S] sampled row ids; src[B*S] source group per slot.
 * node_demand[B][nodes][E] (device uint64) is overwritten. */
MPB_API mpb_status mpb_batch_demand(mpb_context *ctx, const uint32_t *row_ptr,
                                    const uint32_t *cols, const uint32_t *vals, uint32_t R,
                                    const uint32_t *rows, const uint8_t *src, uint32_t B,
                                    uint32_t S, const uint8_t *group_to_node, uint32_t D,
                                    uint32_t nodes, uint32_t E, uint64_t *node_demand);

/* On-device compare_strategies sampler (simulator.cpp:115-118, 155-177):
 * for batch b < B, rows[b*S+i] = uniform_int[0, R-1] draws of
 * std::mt19937_64(std::seed_seq{seed, b, 1}) and picks[b*S+i] = index into
 * row rows[b*S+i]'s routing group set drawn from mt19937_64(seed_seq{seed, b,
 * 2}) only when set_size[row] > 1 (else 0) — libstdc++ Lemire downscaling,
 * bit-identical to the host. set_size[R] device uint32 (NULL = all 1). */
MPB_API mpb_status mpb_sample_batches(mpb_context *ctx, uint64_t seed, uint32_t B, uint32_t R,
                                      uint32_t S, const uint32_t *set_size, uint32_t *rows,
                                      uint32_t *picks);
/* Source group per sampled slot: cluster_routed ? groups[set_off[row] + pick]
 * : i % D (the baselines' batch-position rule, simulator.cpp:171-180).
 * set_off[R+1], groups[] device uint32 (ignored when !cluster_routed). */
MPB_API mpb_status mpb_route_sources(mpb_context *ctx, const uint32_t *rows, const uint32_t *picks,
                                     uint32_t B, uint32_t S, const uint32_t *set_off,
                                     const uint32_t *groups, uint32_t D, int cluster_routed,
                                     uint8_t *src);

/* demand[B][rows][E] (uint64) x luts[P][nodes][E] (uint8, 255 = uncovered)
 * -> inter[P*B], intra[P*B], rank_pairs[P*B*D] pair counts (device). Row r
 * of a demand table originates on node row_node[r] (device uint8 [rows]):
 * rows = nodes with row_node = identity for node-level demand, or rows = D
 * with row_node = group_to_node for the per-source-group demand of
 * mpb_dispatch_layout. group_to_node[D] device uint8; D <= 255. */
MPB_API mpb_status mpb_score_placements(mpb_context *ctx, const uint64_t *demand, uint32_t B,
                                        uint32_t rows, const uint8_t *row_node,
                                        const uint8_t *luts, uint32_t P,
                                        const uint8_t *group_to_node, uint32_t D, uint32_t nodes,
                                        uint32_t E, uint64_t *inter, uint64_t *intra,
                                        uint64_t *rank_pairs);

/* LayerSim doubles for N scored (candidate, batch) cells, bit-identical to
 * simulate_layer: cost = {hidden_dim, bytes_per_element, inter_bw, intra_bw,
 * expert_time_per_token, fixed_layer_overhead} (host array), tp_exp and
 * spans_nodes (any group on another node than group 0) as in
 * simulator.cpp:27-41. out[N][6] = {inter, intra, dispatch, compute, combine,
 * layer}; payload[N][D] bytes (nullable). */
MPB_API mpb_status mpb_finalize_layer_sims(mpb_context *ctx, const uint64_t *inter,
                                           const uint64_t *intra, const uint64_t *rank_pairs,
                                           uint64_t N, uint32_t D, const double *cost,
                                           uint32_t tp_exp, int spans_nodes, double *out,
                                           double *payload);
/* mpb_score_placements with mpb_finalize_layer_sims fused into its epilogue
 * (one launch; each cell's LayerSim computed by the warp that priced it, the
 * same operations in the same order: bit-identical to the two calls). */
MPB_API mpb_status mpb_score_placements_finalize(
    mpb_context *ctx, const uint64_t *demand, uint32_t B, uint32_t rows, const uint8_t *row_node,
    const uint8_t *luts, uint32_t P, const uint8_t *group_to_node, uint32_t D, uint32_t nodes,
    uint32_t E, uint64_t *inter, uint64_t *intra, uint64_t *rank_pairs, const double *cost,
    uint32_t tp_exp, int spans_nodes, double *out, double *payload);

/* ---- physical dispatch / combine (bf16 hidden states) --------------------
 * gather:  send[pos][:] = X[sorted_pairs[pos] / k][:] for pos < n_pairs
 * combine: Y[t][:] = sum_j w[t*k+j] * recv[pair_pos[t*k+j]][:] (fp32 accumulate)
 * X, send, recv, Y bf16 row-major with H columns; H % 8 == 0. */
MPB_API mpb_status mpb_dispatch_gather(mpb_context *ctx, const void *X, const int32_t *sorted_pairs,
                                       uint64_t n_pairs, uint32_t k, uint32_t H, void *send);
MPB_API mpb_status mpb_combine_scatter(mpb_context *ctx, const void *recv, const int32_t *pair_pos,
                                       const float *weights, uint64_t T, uint32_t k, uint32_t H,
                                       void *Y);

/* Fused NVLink dispatch / combine (K6-P2P): `peer_recv` [world] holds the
 * device addresses of every rank's receive buffer mapped into this process
 * (symmetric memory over NVSwitch), `peer_counts` [world] every rank's
 * [world][world] int64 count matrix. mpb_a2a_put_counts writes this rank's
 * per-destination counts (from key_offsets; span = keys per rank = groups per
 * rank * E) into every peer; after a cross-rank barrier mpb_dispatch_p2p
 * writes each sorted pair's hidden-state row straight into the destination
 * rank's buffer, and (after the experts and another barrier)
 * mpb_combine_p2p reads each token's k rows out of the peers' buffers into
 * the weighted sum — the same result as gather + all-to-all-v + combine,
 * bit for bit, with no staging buffers. Rows past `capacity_rows` raise
 * MPB_VALIDATION_ERROR at the next mpb_context_sync. */
MPB_API mpb_status mpb_a2a_put_counts(mpb_context *ctx, const int64_t *key_offsets,
                                      uint32_t span, uint32_t world, uint32_t rank,
                                      const uint64_t *peer_counts);
MPB_API mpb_status mpb_dispatch_p2p(mpb_context *ctx, const void *X, const int32_t *sorted_pairs,
                                    uint64_t n_pairs, uint32_t k, uint32_t H,
                                    const int64_t *counts, const int64_t *key_offsets,
                                    uint32_t span, uint32_t world, uint32_t rank,
                                    const uint64_t *peer_recv, uint64_t capacity_rows);
/* Pull variant of mpb_dispatch_p2p: each rank copies the rows destined to it
 * out of every source's staged hidden states into its own receive buffer.
 * peer_x / peer_sorted_pairs / peer_key_offsets: device arrays of every
 * rank's (symmetric-memory) X [T,H] bf16, sorted pairs and key offsets;
 * counts: this rank's [world][world] count matrix (mpb_a2a_put_counts). The
 * receive buffer ends up identical to the push dispatch's. */
MPB_API mpb_status mpb_dispatch_pull(mpb_context *ctx, const int64_t *counts, const uint64_t *peer_x,
                                     const uint64_t *peer_sorted_pairs,
                                     const uint64_t *peer_key_offsets, uint32_t k, uint32_t H,
                                     uint32_t span, uint32_t world, uint32_t rank, void *recv,
                                     uint64_t capacity_rows);
/* Return leg pushed instead of pulled: every received row (the first
 * `recv_rows` rows of this rank's buffer, grouped by source rank) is written
 * into its source rank's `back` buffer at its position in that rank's sorted
 * order; after a barrier the source runs mpb_combine_scatter on `back`. */
MPB_API mpb_status mpb_return_p2p(mpb_context *ctx, const void *recv, uint64_t recv_rows,
                                  uint32_t H, const int64_t *counts, uint32_t world,
                                  uint32_t rank, const uint64_t *peer_back);
MPB_API mpb_status mpb_combine_p2p(mpb_context *ctx, const int32_t *pair_pos,
                                   const float *weights, uint64_t T, uint32_t k, uint32_t H,
                                   const int64_t *counts, const int64_t *key_offsets,
                                   uint32_t span, uint32_t world, uint32_t rank,
                                   const uint64_t *peer_recv, void *Y);

/* ---- the routed step (C++ host schedule) ----------------------------------
 * One routed pass of every MoE layer over one batch, scheduled by the library
 * on two streams of its own — the host side of the reference's planner loop
 * (pipeline.cpp:316-443: route -> account -> price every placement), with the
 * routes from the router GEMM instead of the synthetic sampler:
 *   LAYERS phase: zero the fused statistics buffer; routers (grouped launches
 *     of router_group layers, mpb_router_topk_layers) on the main stream with
 *     an SM budget of device_sms - side_sms; each chunk's statistics tails
 *     (mpb_dispatch_layout: demand / demand2 / tag histograms + permutation,
 *     and one mpb_coactivation over the whole chunk) on the side stream,
 *     beside the next chunk's router.
 *     One layer: the router on every SM; on one GPU with score_per_chunk it
 *     counts demand / demand2 itself (mpb_router_topk_demand) and the score
 *     jobs follow it on main while the layout (a third stream) and the
 *     co-activation (side) run beside them; otherwise the layout on main with
 *     the co-activation beside it, then the SCORE phase.
 *   SCORE phase: mpb_score_placements_finalize of score_jobs[0] on the main
 *     stream, the other jobs on the side stream beside it.
 * Multi-GPU: the plan issues its own NCCL collectives (mpb_step_attach_comm),
 * or the caller all-reduces the statistics between the two phases. Both
 * phases are asynchronous and ordered after / before the work already on
 * ctx's stream. mpb_step_capture replays them from CUDA graphs (captured
 * after one eager run that sizes every workspace). Per-chunk router times
 * (device events around every router launch, also inside the graphs) feed
 * the roofline. */
typedef struct mpb_step mpb_step;
typedef struct {
    const uint64_t *demand;    /* [B][rows][E] */
    uint32_t B, rows;
    const uint8_t *row_node;   /* [rows] */
    const uint8_t *luts;       /* [P][nodes][E] */
    uint32_t P;
    const uint8_t *group_to_node; /* [D] device */
    uint32_t D, nodes, E;
    uint64_t *inter, *intra, *rank_pairs;
    double cost[6];
    uint32_t tp_exp;
    int spans_nodes;
    double *out, *payload;     /* [P*B][6], [P*B][D] */
} mpb_score_job;

typedef struct {
    uint32_t layers;
    uint64_t T;
    uint32_t H, E, k;
    int score_fn, renorm;
    const void *const *X;      /* host array [layers] of device bf16 [T,H] */
    const void *const *W;      /* host array [layers] of device bf16 [E,H] */
    int32_t *idx;              /* [layers][T][k] */
    float *weights;            /* [layers][T][k] */
    const mpb_placement *deployed;
    const uint8_t *src_group;  /* [T] */
    const uint8_t *src_group2; /* [T] or NULL */
    const uint16_t *tag;       /* [T] or NULL */
    uint32_t n_tags;
    uint64_t *demand;          /* [layers][D][E] */
    uint64_t *demand2;         /* [layers][D][E] or NULL */
    uint64_t *tag_pop;         /* [n_tags][E] or NULL */
    uint64_t *coact;           /* [E][E] or NULL (no co-activation) */
    int32_t *sorted_pairs;     /* [T*k] or NULL (no permutation) */
    int32_t *pair_pos;
    int64_t *key_offsets;
    void *zero_base;           /* zeroed at the start of every LAYERS phase */
    uint64_t zero_bytes;
    const mpb_score_job *score_jobs; /* copied */
    uint32_t n_score_jobs;
    uint32_t side_sms;         /* 0: 20 when layers > 1 */
    uint32_t router_group;     /* 0: 8 */
    /* 1 (single GPU: the demand is final once a layer's tail is in): every
     * score job with B == layers is priced chunk by chunk right after the
     * chunk's statistics tails, beside the next routers, and the last chunk's
     * tails run on the main stream's grids after the last router; the SCORE
     * phase is then empty. 0: all scoring in the SCORE phase (multi-GPU: after
     * the caller's all-reduce). */
    uint32_t score_per_chunk;
} mpb_step_desc;

/* Multi-GPU collectives issued by the plan itself (NCCL over NVLink): after
 * each chunk's statistics tails, one grouped in-place all-reduce (sum, uint64)
 * of that chunk's per-layer demand / demand2 slices on the side stream —
 * beside the next routers — so every chunk is priced on the GLOBAL demand
 * right away (score jobs with B == layers, each rank its own candidate slice);
 * after the last chunk, the all-reduce of tag_pop / coact and an in-place
 * all-gather of the `gather` buffers (rank r's slice at r * bytes_per_rank).
 * Everything stays inside the step's CUDA graphs. The caller broadcasts rank
 * 0's id (mpb_nccl_get_unique_id) to every rank before mpb_step_attach_comm.
 * NCCL is resolved at run time (dlopen of libnccl.so.2: the copy already
 * loaded in the process, e.g. torch's, else the system one). */
typedef struct {
    void *buf;                  /* device buffer holding every rank's slice */
    uint64_t bytes_per_rank;    /* slice size (bytes) */
} mpb_gather_spec;
MPB_API mpb_status mpb_nccl_get_unique_id(uint8_t id[128]);
MPB_API mpb_status mpb_step_attach_comm(mpb_step *step, const uint8_t id[128], int world, int rank,
                                        const mpb_gather_spec *gather, uint32_t n_gather);

#define MPB_STEP_LAYERS 1u
#define MPB_STEP_SCORE 2u
MPB_API mpb_status mpb_step_create(mpb_context *ctx, const mpb_step_desc *desc, mpb_step **out);
MPB_API mpb_status mpb_step_destroy(mpb_step *step);
MPB_API mpb_status mpb_step_run(mpb_step *step, uint32_t phases);
MPB_API mpb_status mpb_step_capture(mpb_step *step);
/* Waits for both streams; reports kernel-flagged input errors of either. */
MPB_API mpb_status mpb_step_sync(mpb_step *step);
/* Per-layer router ms (a grouped launch's time divided over its layers) into
 * ms[layers], averaged over the runs since mpb_step_timing_reset (at most the
 * last 64; the last run when none); *n_runs = runs averaged. After sync. */
MPB_API mpb_status mpb_step_timing_reset(mpb_step *step);
MPB_API mpb_status mpb_step_router_ms(const mpb_step *step, float *ms, uint32_t *n_runs);
/* Kernels one run of `phases` launches; the chunking (layers per router
 * launch) into chunks[] (capacity layers), *n_chunks. */
MPB_API mpb_status mpb_step_info(const mpb_step *step, uint32_t phases, uint64_t *launches,
                                 uint32_t *chunks, uint32_t *n_chunks);
/* Tests / experiments. mpb_debug_step_fused: 1 when the plan's single-layer
 * step counts the demand in the router (mpb_router_topk_demand) and prices it
 * beside the layout (one layer, one GPU, MPB_ROUTER_DEMAND != 0).
 * mpb_debug_step_probe (plan created with MPB_STEP_PROBE=1, eager runs): the
 * last run's timeline in ms from its start — out[c] = router chunk c done,
 * out[nc + c] = chunk c's statistics tails + pricing done, out[2 nc] = step
 * end; returns the count written (2 nc + 1) or -1. */
MPB_API int mpb_debug_step_fused(const mpb_step *step);
MPB_API int mpb_debug_step_probe(const mpb_step *step, float *out, size_t n);

/* ---- host placement / grouping policies (no device needed) ----------------
 * Restatements of the reference policies with the same std::mt19937_64 /
 * libstdc++ distribution calls (bit-identical results):
 *   placement.cpp:296-313 linear, :315-350 eplb (LPT), :127-161 phase 1,
 *   :163-189 phase 2, :191-281 balance, :283-294 data_based, :96-125
 *   aggregate_usage; clustering.cpp:28-35 l2_normalize_rows, :54-230 kmeans,
 *   :232-320 cluster sizes + assign_clusters_to_groups.
 * Groups are returned flattened (group d's experts follow group d-1's); fixed
 * size M per group unless a sizes array is returned. Matrices are row-major
 * double. */
MPB_API mpb_status mpb_linear_placement(uint32_t E, uint32_t D, uint32_t *groups_out /* E */);
MPB_API mpb_status mpb_eplb_placement(const double *load /* E */, uint32_t E, uint32_t D,
                                      uint32_t *groups_out /* E */);
MPB_API mpb_status mpb_phase1_unique_distribution(const double *usage /* D*E */, uint32_t D,
                                                  uint32_t E, uint32_t *groups_out /* E */,
                                                  uint32_t *sizes_out /* D */);
MPB_API mpb_status mpb_phase2_redundant_addition(const uint32_t *groups_in, const uint32_t *sizes_in,
                                                 const double *usage, uint32_t D, uint32_t E,
                                                 uint32_t M, uint32_t *groups_out /* D*M */);
MPB_API mpb_status mpb_balance_and_verify(const uint32_t *groups_in, const uint32_t *sizes_in,
                                          uint32_t D, uint32_t E, uint32_t M, uint64_t seed,
                                          uint32_t *groups_out /* D*M */);
MPB_API mpb_status mpb_data_based_placement(const double *usage /* D*E */, uint32_t D, uint32_t E,
                                            uint32_t R, uint64_t seed,
                                            uint32_t *groups_out /* E+R */);
MPB_API mpb_status mpb_aggregate_usage(const uint32_t *labels /* rows */, const double *matrix,
                                       uint64_t rows, uint32_t E, uint32_t K,
                                       const uint32_t *assign_flat, const uint32_t *assign_sizes,
                                       uint32_t D, double *usage_out /* D*E */);
MPB_API mpb_status mpb_l2_normalize_rows(const double *matrix, uint64_t rows, uint32_t cols,
                                         double *out);
/* objective_history (nullable, capacity max_iterations): the objective after
 * each Lloyd iteration (ClusterModel::objective_history, clustering.cpp:207). */
MPB_API mpb_status mpb_kmeans(const double *rows, uint64_t n, uint32_t dim, uint32_t K,
                              uint64_t seed, uint32_t max_iterations, double tolerance,
                              uint32_t *labels_out /* n */, double *centroids_out /* K*dim */,
                              double *objective_out, uint32_t *iterations_out,
                              double *objective_history /* host */);
/* Device k-means (K7): same algorithm, order of operations and RNG draws as
 * kmeans / l2_normalize_rows (clustering.cpp:15-230) — bit-identical labels,
 * centroids and objective — on caller-owned device buffers, in ctx's stream
 * (returns after the stream has drained: the Lloyd loop is host-driven). */
MPB_API mpb_status mpb_l2_normalize_rows_device(mpb_context *ctx, const double *matrix /* dev */,
                                                uint64_t rows, uint32_t cols,
                                                double *out /* dev */);
MPB_API mpb_status mpb_kmeans_device(mpb_context *ctx, const double *rows /* dev n*dim */,
                                     uint64_t n, uint32_t dim, uint32_t K, uint64_t seed,
                                     uint32_t max_iterations, double tolerance,
                                     uint32_t *labels /* dev n */, double *centroids /* dev K*dim */,
                                     double *objective_out /* host */,
                                     uint32_t *iterations_out /* host */,
                                     double *objective_history /* host, nullable */);
/* Placement::verify (placement.cpp:35-56): exact group sizes M, no expert
 * twice within a group, ids < E, every expert placed -> MPB_VALIDATION_ERROR. */
MPB_API mpb_status mpb_placement_verify(const uint32_t *groups_flat, const uint32_t *group_sizes,
                                        uint32_t D, uint32_t E, uint32_t M);
MPB_API mpb_status mpb_assign_clusters_to_groups(const uint32_t *labels, uint64_t n, uint32_t K,
                                                 const double *raw, uint32_t dim, uint32_t D,
                                                 uint64_t seed, uint32_t *assign_flat /* <= K*D */,
                                                 uint32_t *assign_sizes /* K */,
                                                 double *cluster_sizes_out /* K */);

/* ---- characterisation metrics (metrics.cpp:11-132) -------------------------
 * mpb_label_row_sums: sums[l][c] = sum of matrix[r][c] over rows r with
 * labels[r] == l (labels NULL: one label, all rows) — the per-dataset
 * popularity vectors and the all-row sums of the prefill->decode correlation
 * (metrics.cpp:72-91), as exact uint64 histograms on the device (matrix, labels,
 * sums device; sums overwritten; synchronous). Entries must be non-negative
 * integers < 2^53 — then every sequential double sum of the reference is exact
 * and equals these — else MPB_VALIDATION_ERROR.
 * mpb_expert_load / mpb_pearson: host finalisation in the reference's order
 * (metrics.cpp:11-34, 42-68), same errors. */
MPB_API mpb_status mpb_label_row_sums(mpb_context *ctx, const double *matrix, uint64_t rows,
                                      uint32_t cols, const uint32_t *labels, uint32_t n_labels,
                                      uint64_t *sums);
MPB_API mpb_status mpb_expert_load(const double *counts, uint32_t E, uint32_t top_k,
                                   double *loads, uint64_t *total_tokens);
MPB_API mpb_status mpb_pearson(const double *x, const double *y, uint64_t n, double *r);

/* ---- host trace model (no device needed) -----------------------------------
 * trace.cpp:73-297: JSONL loader / writer (byte-identical to the reference's
 * nlohmann dump), activation-matrix builder, layers_present, and the
 * synthetic generator (same std:: RNG calls) with an optional per-token tap
 * (every token's k picks, in pick order, for the device kernels). */
typedef struct mpb_trace mpb_trace;
MPB_API mpb_status mpb_trace_parse(const char *text, uint64_t len, uint32_t E, uint32_t top_k,
                                   uint32_t layers, mpb_trace **out);
MPB_API mpb_status mpb_trace_read_file(const char *path, uint32_t E, uint32_t top_k,
                                       uint32_t layers, mpb_trace **out);
MPB_API mpb_status mpb_trace_write_file(const mpb_trace *t, const char *path);
MPB_API mpb_status mpb_trace_generate(uint32_t num_domains, uint32_t requests_per_domain,
                                      uint32_t preferred, double affinity,
                                      double decode_tokens_mean, uint64_t seed, uint32_t E,
                                      uint32_t top_k, uint32_t layers, int keep_picks,
                                      mpb_trace **out);
/* write_trace (trace.cpp:117-131) into buf: *len = bytes of the JSONL text,
 * copied when buf != NULL and cap >= *len. */
MPB_API mpb_status mpb_trace_dump(const mpb_trace *t, char *buf, uint64_t cap, uint64_t *len);
/* A trace from caller records (inverse of mpb_trace_export; pairs of record i
 * in [pair_offset[i], pair_offset[i+1]), ascending expert ids, label index into
 * labels[n_labels]). Used by the C++ drop-in to hand std::vector<ActivationRecord>
 * to the builders and the writer. */
MPB_API mpb_status mpb_trace_import(uint64_t n_records, const uint64_t *request_id,
                                    const uint32_t *layer, const uint8_t *stage,
                                    const uint64_t *input_len, const uint64_t *gen_tokens,
                                    const uint32_t *label, const uint64_t *pair_offset,
                                    const uint32_t *expert, const uint64_t *count,
                                    uint64_t n_labels, const char *const *labels, mpb_trace **out);
MPB_API mpb_status mpb_trace_destroy(mpb_trace *t);
MPB_API mpb_status mpb_trace_sizes(const mpb_trace *t, uint64_t *n_records, uint64_t *n_pairs,
                                   uint64_t *n_labels, uint64_t *n_picks);
MPB_API mpb_status mpb_trace_export(const mpb_trace *t, uint64_t *request_id, uint32_t *layer,
                                    uint8_t *stage, uint64_t *input_len, uint64_t *gen_tokens,
                                    uint32_t *label, uint64_t *pair_offset, uint32_t *expert,
                                    uint64_t *count, int32_t *picks, uint64_t *pick_offset);
MPB_API const char *mpb_trace_label(const mpb_trace *t, uint64_t i);
/* layer < 0: summed over layers; stage 0 prefill / 1 decode; values == NULL
 * queries *rows only. */
MPB_API mpb_status mpb_trace_matrix(const mpb_trace *t, uint32_t E, int64_t layer, int stage,
                                    uint64_t *rows, double *values, uint64_t *request_ids,
                                    uint32_t *labels);
MPB_API mpb_status mpb_trace_layers_present(const mpb_trace *t, int stage, uint32_t *layers,
                                            uint64_t *n);

#ifdef __cplusplus
}
#endif
#endif /* MOEPLACE_B200_H */
