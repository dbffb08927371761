// Drop-in replacement for the reference's cost evaluator translation unit
// (/root/reference/proj/core/src/simulator.cpp) that runs on the B200 through
// the C ABI of libmoeplace_b200.so (include/moeplace_b200.h).
//
// It is compiled against the reference's own public header
// moeplace/simulator.hpp (the boundary, proj/core/include/moeplace/
// simulator.hpp:17-138) and defines exactly the functions that header
// declares, so a maintainer swaps `src/simulator.cpp` for this file in
// core/CMakeLists.txt and links libmoeplace_b200.so. Every
// caller — run_pipeline, the CLI, the reference's unit and acceptance suites —
// then prices batches on the GPU:
//   simulate_layer      -> mpb_batch_demand + mpb_score_placements +
//                          mpb_finalize_layer_sims (bit-identical LayerSim)
//   compare_strategies  -> mpb_sample_batches (mt19937_64/seed_seq/Lemire on
//                          device) + mpb_route_sources + the same three kernels
//                          for every strategy and batch at once
// Input validation happens on the host before any launch, throwing the same
// exception classes at the same conditions as the reference (simulator.cpp:
// 14-25, 45-50, 66-71, 128-140). Token counts must be integers (they always
// are for trace-derived batches); a fractional count raises ValidationError
// instead of silently losing bit-exactness.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "moeplace/simulator.hpp"
#include "moeplace/stats.hpp"
#include "moeplace_b200.h"
#include "shim_common.hpp"

namespace moeplace {
namespace {

using namespace b200;

std::vector<uint8_t> dest_lut(const Placement &p, const Topology &t, uint32_t nodes) {
    const uint32_t D = p.D();
    std::vector<uint32_t> flat, sizes(D);
    for (uint32_t d = 0; d < D; ++d) {
        sizes[d] = static_cast<uint32_t>(p.groups[d].size());
        flat.insert(flat.end(), p.groups[d].begin(), p.groups[d].end());
    }
    if (flat.empty()) flat.push_back(0);
    std::vector<uint8_t> lut(size_t(nodes) * p.E);
    check(mpb_build_dest_lut(flat.data(), sizes.data(), D, p.E, t.group_to_node.data(),
                             lut.data()));
    return lut;
}

uint32_t node_count(const Topology &t, uint32_t D) {
    uint32_t n = 0;
    for (uint32_t d = 0; d < D; ++d) n = std::max(n, t.group_to_node[d] + 1);
    return n;
}

bool spans_nodes(const Topology &t) {
    for (std::size_t g = 1; g < t.group_to_node.size(); ++g)
        if (t.group_to_node[g] != t.group_to_node[0]) return true;
    return false;
}

uint32_t integral_count(double c) {
    if (!(c >= 0.0) || c != std::floor(c) || c >= 4294967296.0)
        throw ValidationError("simulate_layer (B200): token counts must be non-negative integers "
                              "below 2^32");
    return static_cast<uint32_t>(c);
}

LayerSim to_sim(const double *o, const double *payload, uint32_t D) {
    LayerSim s;
    s.inter_node_bytes = o[0];
    s.intra_node_bytes = o[1];
    s.dispatch_time = o[2];
    s.expert_compute_time = o[3];
    s.combine_time = o[4];
    s.layer_time = o[5];
    s.per_rank_payload.assign(payload, payload + D);
    return s;
}

std::array<double, 6> cost_array(const CostModelParams &c) {
    return {static_cast<double>(c.hidden_dim), static_cast<double>(c.bytes_per_element),
            c.inter_node_bandwidth, c.intra_node_bandwidth, c.expert_time_per_token,
            c.fixed_layer_overhead};
}

// Scores P placements (LUTs) on B node-level demand tables already on device.
void score_and_finalize(Device &dev, const uint64_t *d_demand, uint32_t B,
                        const std::vector<uint8_t> &luts, uint32_t P, const Topology &t,
                        uint32_t D, uint32_t nodes, uint32_t E, const CostModelParams &cost,
                        std::vector<double> &out, std::vector<double> &payload) {
    std::vector<uint8_t> g2n(D), row_node(nodes);
    for (uint32_t d = 0; d < D; ++d) g2n[d] = static_cast<uint8_t>(t.group_to_node[d]);
    for (uint32_t n = 0; n < nodes; ++n) row_node[n] = static_cast<uint8_t>(n);
    auto *d_g2n = dev.up(kG2n, g2n);
    auto *d_rn = dev.up(kRowNode, row_node);
    auto *d_luts = dev.up(kLuts, luts);
    const size_t N = size_t(P) * B;
    auto *d_inter = static_cast<uint64_t *>(dev.buf(kInter, N * 8));
    auto *d_intra = static_cast<uint64_t *>(dev.buf(kIntra, N * 8));
    auto *d_rank = static_cast<uint64_t *>(dev.buf(kRank, N * D * 8));
    check(mpb_score_placements(dev.ctx, d_demand, B, nodes, d_rn, d_luts, P, d_g2n, D, nodes, E,
                               d_inter, d_intra, d_rank));
    auto c = cost_array(cost);
    auto *d_out = dev.buf(kOut, N * 6 * 8);
    auto *d_pay = dev.buf(kPayload, N * D * 8);
    check(mpb_finalize_layer_sims(dev.ctx, d_inter, d_intra, d_rank, N, D, c.data(), t.tp_exp,
                                  spans_nodes(t) ? 1 : 0, static_cast<double *>(d_out),
                                  static_cast<double *>(d_pay)));
    check(mpb_context_sync(dev.ctx));
    out.resize(N * 6);
    payload.resize(N * D);
    dev.down(out, d_out);
    dev.down(payload, d_pay);
}

}  // namespace

void CostModelParams::validate() const {
    if (hidden_dim == 0 || bytes_per_element == 0)
        throw ConfigError("cost model: hidden_dim and bytes_per_element must be >= 1");
    if (inter_node_bandwidth <= 0.0 || intra_node_bandwidth <= 0.0)
        throw ConfigError("cost model: bandwidths must be positive");
    if (intra_node_bandwidth < inter_node_bandwidth)
        throw ConfigError("cost model: intra_node_bandwidth must be >= inter_node_bandwidth");
    if (expert_time_per_token <= 0.0)
        throw ConfigError("cost model: expert_time_per_token must be positive");
    if (fixed_layer_overhead < 0.0)
        throw ConfigError("cost model: fixed_layer_overhead must be >= 0");
}

double padded_all_to_all_time(std::span<const double> per_rank_payload_bytes,
                              const Topology &topology, const CostModelParams &cost) {
    if (per_rank_payload_bytes.empty()) return 0.0;
    const double mx = *std::max_element(per_rank_payload_bytes.begin(), per_rank_payload_bytes.end());
    const double bw = spans_nodes(topology) ? cost.inter_node_bandwidth : cost.intra_node_bandwidth;
    return mx / static_cast<double>(topology.tp_exp) / bw;
}

LayerSim simulate_layer(const BatchAssignment &batch, const Placement &placement,
                        const Topology &topology, const CostModelParams &cost) {
    cost.validate();
    topology.validate();
    const uint32_t D = placement.D();
    if (topology.ep != D)
        throw ConfigError("simulate_layer: topology.ep (" + std::to_string(topology.ep) +
                          ") != placement group count (" + std::to_string(D) + ")");
    std::vector<char> covered(placement.E, 0);
    for (const auto &g : placement.groups)
        for (uint32_t e : g)
            if (e < placement.E) covered[e] = 1;
    const uint32_t R = static_cast<uint32_t>(batch.requests.size());
    std::vector<uint32_t> row_ptr(R + 1, 0), cols, vals, rows(R);
    std::vector<uint8_t> src(R);
    for (uint32_t r = 0; r < R; ++r) {
        const auto &req = batch.requests[r];
        if (req.source_group >= D) throw ValidationError("simulate_layer: source group out of range");
        for (const auto &[expert, count] : req.expert_counts) {
            if (expert >= placement.E || !covered[expert])
                throw ValidationError("simulate_layer: expert " + std::to_string(expert) +
                                      " is not covered by the placement");
            cols.push_back(expert);
            vals.push_back(integral_count(count));
        }
        row_ptr[r + 1] = static_cast<uint32_t>(cols.size());
        rows[r] = r;
        src[r] = static_cast<uint8_t>(req.source_group);
    }
    const uint32_t nodes = node_count(topology, D), E = placement.E;
    Device &dev = device();
    std::lock_guard<std::recursive_mutex> lock(dev.mu);
    std::vector<uint8_t> g2n(D);
    for (uint32_t d = 0; d < D; ++d) g2n[d] = static_cast<uint8_t>(topology.group_to_node[d]);
    auto *d_demand = static_cast<uint64_t *>(dev.buf(kDemand, size_t(nodes) * E * 8));
    check(mpb_batch_demand(dev.ctx, dev.up(kRowPtr, row_ptr), dev.up(kCols, cols),
                           dev.up(kVals, vals), std::max(R, 1u), dev.up(kRows, rows),
                           dev.up(kSrc, src), 1, R, dev.up(kG2n, g2n), D, nodes, E, d_demand));
    std::vector<double> out, payload;
    score_and_finalize(dev, d_demand, 1, dest_lut(placement, topology, nodes), 1, topology, D,
                       nodes, E, cost, out, payload);
    return to_sim(out.data(), payload.data(), D);
}

std::vector<std::vector<std::uint32_t>> routing_table(const ClusterModel &model,
                                                      const GroupMap &group_map) {
    if (group_map.K != model.K)
        throw ValidationError("routing_table: group map K does not match model K");
    std::vector<std::vector<std::uint32_t>> table(model.labels.size());
    for (std::size_t r = 0; r < model.labels.size(); ++r) table[r] = group_map.assignment[model.labels[r]];
    return table;
}

ComparisonTable compare_strategies(const ActivationMatrix &decode_matrix,
                                   const std::vector<StrategyEntry> &strategies,
                                   const std::vector<std::vector<std::uint32_t>> &route_groups,
                                   const Topology &topology, const CostModelParams &cost,
                                   std::uint32_t num_batches, std::uint32_t batch_size,
                                   std::uint64_t seed) {
    if (decode_matrix.rows == 0) throw ValidationError("compare_strategies: empty decode matrix");
    if (strategies.empty()) throw ValidationError("compare_strategies: no strategies");
    if (num_batches == 0 || batch_size == 0)
        throw ConfigError("compare_strategies: batches and batch size must be >= 1");
    const std::uint32_t D = strategies[0].placement.D();
    bool any_cluster = false, any_base = false;
    for (const auto &entry : strategies) {
        if (entry.placement.D() != D)
            throw ValidationError("compare_strategies: strategies disagree on group count");
        if (entry.cluster_routed && route_groups.size() != decode_matrix.rows)
            throw ValidationError("compare_strategies: routing table does not cover the matrix");
        (entry.cluster_routed ? any_cluster : any_base) = true;
    }
    // simulate_layer's own validation, once for every batch it would run
    cost.validate();
    topology.validate();
    if (topology.ep != D)
        throw ConfigError("simulate_layer: topology.ep (" + std::to_string(topology.ep) +
                          ") != placement group count (" + std::to_string(D) + ")");
    const uint32_t R = static_cast<uint32_t>(decode_matrix.rows);
    const uint32_t E = static_cast<uint32_t>(decode_matrix.cols);
    std::vector<uint32_t> row_ptr(R + 1, 0), cols, vals;
    for (uint32_t r = 0; r < R; ++r) {
        auto row = decode_matrix.row(r);
        for (uint32_t e = 0; e < E; ++e)
            if (row[e] > 0.0) {
                cols.push_back(e);
                vals.push_back(integral_count(row[e]));
            }
        row_ptr[r + 1] = static_cast<uint32_t>(cols.size());
    }
    // Uncovered experts / out-of-range source groups are flagged by the kernels
    // only for pairs a sampled batch actually routes — where the reference's
    // per-batch simulate_layer would throw — and surface as ValidationError.
    std::vector<uint32_t> set_size, set_off(1, 0), groups;
    if (any_cluster) {
        for (const auto &g : route_groups) {
            if (g.empty()) throw ValidationError("compare_strategies: empty routing group set");
            set_size.push_back(static_cast<uint32_t>(g.size()));
            groups.insert(groups.end(), g.begin(), g.end());
            set_off.push_back(static_cast<uint32_t>(groups.size()));
        }
    }
    const uint32_t nodes = node_count(topology, D);
    Device &dev = device();
    std::lock_guard<std::recursive_mutex> lock(dev.mu);
    const size_t BS = size_t(num_batches) * batch_size;
    auto *d_rows = static_cast<uint32_t *>(dev.buf(kRows, BS * 4));
    auto *d_picks = static_cast<uint32_t *>(dev.buf(kPicks, BS * 4));
    check(mpb_sample_batches(dev.ctx, seed, num_batches, R, batch_size,
                             any_cluster ? dev.up(kSetSize, set_size) : nullptr, d_rows, d_picks));
    auto *d_rp = dev.up(kRowPtr, row_ptr);
    auto *d_cols = dev.up(kCols, cols);
    auto *d_vals = dev.up(kVals, vals);
    auto *d_setoff = any_cluster ? dev.up(kSetOff, set_off) : nullptr;
    auto *d_groups = any_cluster ? dev.up(kGroups, groups) : nullptr;
    std::vector<uint8_t> g2n(D);
    for (uint32_t d = 0; d < D; ++d) g2n[d] = static_cast<uint8_t>(topology.group_to_node[d]);

    ComparisonTable table;
    table.rows.resize(BS ? size_t(num_batches) * strategies.size() : 0);
    for (int mode = 0; mode < 2; ++mode) {
        if ((mode == 1 && !any_cluster) || (mode == 0 && !any_base)) continue;
        std::vector<uint32_t> ids;
        std::vector<uint8_t> luts;
        for (uint32_t s = 0; s < strategies.size(); ++s)
            if (strategies[s].cluster_routed == (mode == 1)) {
                ids.push_back(s);
                auto l = dest_lut(strategies[s].placement, topology, nodes);
                luts.insert(luts.end(), l.begin(), l.end());
            }
        auto *d_src = static_cast<uint8_t *>(dev.buf(kSrc, BS));
        check(mpb_route_sources(dev.ctx, d_rows, d_picks, num_batches, batch_size, d_setoff,
                                d_groups, D, mode, d_src));
        auto *d_demand =
            static_cast<uint64_t *>(dev.buf(kDemand, size_t(num_batches) * nodes * E * 8));
        check(mpb_batch_demand(dev.ctx, d_rp, d_cols, d_vals, R, d_rows, d_src, num_batches,
                               batch_size, dev.up(kG2n, g2n), D, nodes, E, d_demand));
        std::vector<double> out, payload;
        score_and_finalize(dev, d_demand, num_batches, luts, static_cast<uint32_t>(ids.size()),
                           topology, D, nodes, E, cost, out, payload);
        for (size_t j = 0; j < ids.size(); ++j)
            for (uint32_t b = 0; b < num_batches; ++b) {
                const size_t cell = j * num_batches + b;
                ComparisonRow &row = table.rows[size_t(b) * strategies.size() + ids[j]];
                row.batch = b;
                row.strategy = strategies[ids[j]].label;
                row.sim = to_sim(out.data() + cell * 6, payload.data() + cell * D, D);
            }
    }

    // normalisation and summaries: host arithmetic in the reference's order
    std::vector<double> linear_bytes;
    for (const auto &row : table.rows)
        if (row.strategy == "linear") linear_bytes.push_back(row.sim.inter_node_bytes);
    table.linear_median_bytes =
        linear_bytes.empty() ? std::numeric_limits<double>::quiet_NaN() : median(linear_bytes);
    for (auto &row : table.rows) {
        if (table.linear_median_bytes > 0.0)
            row.normalized = row.sim.inter_node_bytes / table.linear_median_bytes;
        else if (table.linear_median_bytes == 0.0)
            row.normalized =
                row.sim.inter_node_bytes == 0.0 ? 1.0 : std::numeric_limits<double>::infinity();
        else
            row.normalized = std::numeric_limits<double>::quiet_NaN();
    }
    for (const auto &entry : strategies) {
        std::vector<double> bytes, normalized, dispatch, compute, combine, layer;
        for (const auto &row : table.rows) {
            if (row.strategy != entry.label) continue;
            bytes.push_back(row.sim.inter_node_bytes);
            normalized.push_back(row.normalized);
            dispatch.push_back(row.sim.dispatch_time);
            compute.push_back(row.sim.expert_compute_time);
            combine.push_back(row.sim.combine_time);
            layer.push_back(row.sim.layer_time);
        }
        StrategySummary s;
        s.strategy = entry.label;
        s.median_inter_node_bytes = median(bytes);
        s.q25_inter_node_bytes = quantile(bytes, 0.25);
        s.q75_inter_node_bytes = quantile(bytes, 0.75);
        if (table.linear_median_bytes > 0.0)
            s.normalized_median = s.median_inter_node_bytes / table.linear_median_bytes;
        else if (table.linear_median_bytes == 0.0)
            s.normalized_median = s.median_inter_node_bytes == 0.0
                                      ? 1.0
                                      : std::numeric_limits<double>::infinity();
        else
            s.normalized_median = median(normalized);
        s.median_dispatch_time = median(dispatch);
        s.median_expert_compute_time = median(compute);
        s.median_combine_time = median(combine);
        s.median_layer_time = median(layer);
        table.summary.push_back(std::move(s));
    }
    return table;
}

ComparisonTable compare_default_strategies(const ActivationMatrix &decode_matrix,
                                           const ClusterModel &model, const GroupMap &group_map,
                                           const Topology &topology, const CostModelParams &cost,
                                           std::uint32_t num_batches, std::uint32_t batch_size,
                                           std::uint64_t seed, std::uint32_t R_redundancy) {
    const std::uint32_t E = static_cast<std::uint32_t>(decode_matrix.cols);
    const std::uint32_t D = group_map.D;
    std::vector<double> load(E, 0.0);
    for (std::size_t r = 0; r < decode_matrix.rows; ++r) {
        auto row = decode_matrix.row(r);
        for (std::size_t e = 0; e < E; ++e) load[e] += row[e];
    }
    UsageMatrix usage = aggregate_usage(group_map, decode_matrix, model, D);
    std::vector<StrategyEntry> strategies;
    strategies.push_back({"linear", linear_placement(E, D), false});
    strategies.push_back({"eplb", eplb_placement(load, E, D), false});
    strategies.push_back({"data_based", data_based_placement(usage, R_redundancy, seed), true});
    return compare_strategies(decode_matrix, strategies, routing_table(model, group_map), topology,
                              cost, num_batches, batch_size, seed);
}

std::vector<BreakdownRow> latency_breakdown_report(const ComparisonTable &table,
                                                   const CostModelParams &cost) {
    std::vector<BreakdownRow> report;
    for (const auto &s : table.summary) {
        BreakdownRow row;
        row.strategy = s.strategy;
        const double total = s.median_dispatch_time + s.median_expert_compute_time +
                             s.median_combine_time + cost.fixed_layer_overhead;
        if (total > 0.0) {
            row.dispatch_fraction = s.median_dispatch_time / total;
            row.compute_fraction = s.median_expert_compute_time / total;
            row.combine_fraction = s.median_combine_time / total;
            row.overhead_fraction = cost.fixed_layer_overhead / total;
        }
        row.median_layer_time = s.median_layer_time;
        report.push_back(std::move(row));
    }
    return report;
}

}  // namespace moeplace
