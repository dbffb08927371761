// ORACLE / TEST INFRASTRUCTURE — not product code.
//
// extern "C" driver around the UNMODIFIED reference core
// (/root/reference/proj/core, compiled by oracle/Makefile into
// oracle/_ref/libmoeplace_ref.so). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load it, and only as the
// checker or the timed CPU baseline.
//
// Entry points follow the reference's public API:
//   ref_simulate_tokens / ref_simulate_requests -> moeplace::simulate_layer
//       (proj/core/include/moeplace/simulator.hpp:63, src/simulator.cpp:43-99)
//   ref_generate_trace  -> moeplace::generate_synthetic_trace + write_trace_file
//       (trace.hpp:112, trace.cpp:263-297)
//   ref_compare_scenario -> run_cluster_stage / build_placements /
//       routing_for_matrix / compare_strategies (pipeline.cpp:128-260,
//       simulator.cpp:122-243), dumped as a JSON fixture
//   ref_expert_load / ref_pearson / ref_placement_* -> metrics.cpp, placement.cpp
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "moeplace/config.hpp"
#include "moeplace/metrics.hpp"
#include "moeplace/pipeline.hpp"
#include "moeplace/placement.hpp"
#include "moeplace/simulator.hpp"
#include "moeplace/trace.hpp"

using namespace moeplace;
using nlohmann::json;

namespace {

thread_local std::string g_error;

int status_of(const std::exception &e) {
    if (dynamic_cast<const ParseError *>(&e)) return 2;
    if (dynamic_cast<const ValidationError *>(&e)) return 3;
    if (dynamic_cast<const ConfigError *>(&e)) return 4;
    if (dynamic_cast<const EmptySelectionError *>(&e)) return 5;
    if (dynamic_cast<const UndefinedCorrelationError *>(&e)) return 6;
    if (dynamic_cast<const InfeasibleError *>(&e)) return 7;
    if (dynamic_cast<const LookupError *>(&e)) return 8;
    return 1;
}

template <typename F> int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const std::exception &e) {
        g_error = e.what();
        return status_of(e);
    }
}

// topo = {dp, tp, ep, tp_exp, nodes, gpus_per_node}; group_to_node[ep]
Topology make_topology(const std::uint32_t *topo, const std::uint32_t *g2n) {
    Topology t;
    t.dp = topo[0];
    t.tp = topo[1];
    t.ep = topo[2];
    t.tp_exp = topo[3];
    t.nodes = topo[4];
    t.gpus_per_node = topo[5];
    t.group_to_node.assign(g2n, g2n + t.ep);
    return t;
}

// cost = {hidden_dim, bytes_per_element, inter_bw, intra_bw, expert_time_per_token, overhead}
CostModelParams make_cost(const double *c) {
    CostModelParams p;
    p.hidden_dim = static_cast<std::uint32_t>(c[0]);
    p.bytes_per_element = static_cast<std::uint32_t>(c[1]);
    p.inter_node_bandwidth = c[2];
    p.intra_node_bandwidth = c[3];
    p.expert_time_per_token = c[4];
    p.fixed_layer_overhead = c[5];
    return p;
}

// groups_flat concatenates D groups; group_sizes[d] gives each length.
Placement make_placement(const std::uint32_t *groups_flat, const std::uint32_t *group_sizes,
                         std::uint32_t D, std::uint32_t E) {
    Placement p;
    p.E = E;
    p.groups.resize(D);
    std::size_t off = 0;
    for (std::uint32_t d = 0; d < D; ++d) {
        p.groups[d].assign(groups_flat + off, groups_flat + off + group_sizes[d]);
        off += group_sizes[d];
    }
    p.M = D ? group_sizes[0] : 0;
    p.R_redundancy = static_cast<std::uint32_t>(off) - E;
    return p;
}

void write_sim(const LayerSim &sim, double *out, double *payload) {
    out[0] = sim.inter_node_bytes;
    out[1] = sim.intra_node_bytes;
    out[2] = sim.dispatch_time;
    out[3] = sim.expert_compute_time;
    out[4] = sim.combine_time;
    out[5] = sim.layer_time;
    for (std::size_t d = 0; d < sim.per_rank_payload.size(); ++d)
        payload[d] = sim.per_rank_payload[d];
}

// Token-level batch exactly like benchmarks/simulator_bench.cpp:12-29 but
// with count 1 per (token, expert): each token is one BatchRequest.
BatchAssignment token_batch(const std::int32_t *idx, std::uint64_t T, std::uint32_t k,
                            const std::uint32_t *src) {
    BatchAssignment batch;
    batch.requests.resize(T);
    for (std::uint64_t t = 0; t < T; ++t) {
        auto &r = batch.requests[t];
        r.request_id = t;
        r.source_group = src[t];
        r.expert_counts.reserve(k);
        for (std::uint32_t j = 0; j < k; ++j)
            r.expert_counts.emplace_back(static_cast<std::uint32_t>(idx[t * k + j]), 1.0);
    }
    return batch;
}

json matrix_json(const ActivationMatrix &m) {
    json j;
    j["rows"] = m.rows;
    j["cols"] = m.cols;
    std::vector<std::uint64_t> v(m.values.size());
    for (std::size_t i = 0; i < v.size(); ++i)
        v[i] = static_cast<std::uint64_t>(m.values[i]);
    j["values"] = v;
    j["row_labels"] = m.row_labels;
    j["request_ids"] = m.request_ids;
    return j;
}

json sim_json(const LayerSim &s) {
    return json{{"inter_node_bytes", s.inter_node_bytes},
                {"intra_node_bytes", s.intra_node_bytes},
                {"dispatch_time", s.dispatch_time},
                {"expert_compute_time", s.expert_compute_time},
                {"combine_time", s.combine_time},
                {"layer_time", s.layer_time},
                {"per_rank_payload", s.per_rank_payload}};
}

} // namespace

extern "C" {

const char *ref_last_error() { return g_error.c_str(); }

int ref_simulate_tokens(const std::int32_t *idx, std::uint64_t T, std::uint32_t k,
                        const std::uint32_t *src, const std::uint32_t *groups_flat,
                        const std::uint32_t *group_sizes, std::uint32_t D, std::uint32_t E,
                        const std::uint32_t *topo, const std::uint32_t *g2n, const double *cost,
                        double *out, double *payload) {
    return guarded([&] {
        auto batch = token_batch(idx, T, k, src);
        auto sim = simulate_layer(batch, make_placement(groups_flat, group_sizes, D, E),
                                  make_topology(topo, g2n), make_cost(cost));
        write_sim(sim, out, payload);
    });
}

// Times `reps` simulate_layer calls on a prebuilt token-level batch (the
// BatchAssignment is the reference API's input format, built untimed).
int ref_bench_simulate_tokens(const std::int32_t *idx, std::uint64_t T, std::uint32_t k,
                              const std::uint32_t *src, const std::uint32_t *groups_flat,
                              const std::uint32_t *group_sizes, std::uint32_t D, std::uint32_t E,
                              const std::uint32_t *topo, const std::uint32_t *g2n,
                              const double *cost, std::uint32_t reps, double *seconds,
                              double *out, double *payload) {
    return guarded([&] {
        auto batch = token_batch(idx, T, k, src);
        auto placement = make_placement(groups_flat, group_sizes, D, E);
        auto topology = make_topology(topo, g2n);
        auto c = make_cost(cost);
        LayerSim sim;
        auto t0 = std::chrono::steady_clock::now();
        for (std::uint32_t r = 0; r < reps; ++r)
            sim = simulate_layer(batch, placement, topology, c);
        auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        write_sim(sim, out, payload);
    });
}

int ref_simulate_requests(std::uint64_t R, const std::uint32_t *src, const std::uint64_t *row_ptr,
                          const std::uint32_t *experts, const double *counts,
                          const std::uint32_t *groups_flat, const std::uint32_t *group_sizes,
                          std::uint32_t D, std::uint32_t E, const std::uint32_t *topo,
                          const std::uint32_t *g2n, const double *cost, double *out,
                          double *payload) {
    return guarded([&] {
        BatchAssignment batch;
        batch.requests.resize(R);
        for (std::uint64_t r = 0; r < R; ++r) {
            batch.requests[r].request_id = r;
            batch.requests[r].source_group = src[r];
            for (std::uint64_t i = row_ptr[r]; i < row_ptr[r + 1]; ++i)
                batch.requests[r].expert_counts.emplace_back(experts[i], counts[i]);
        }
        auto sim = simulate_layer(batch, make_placement(groups_flat, group_sizes, D, E),
                                  make_topology(topo, g2n), make_cost(cost));
        write_sim(sim, out, payload);
    });
}

int ref_padded_all_to_all_time(const double *payload, std::uint32_t n, const std::uint32_t *topo,
                               const std::uint32_t *g2n, const double *cost, double *out) {
    return guarded([&] {
        *out = padded_all_to_all_time(std::span<const double>(payload, n),
                                      make_topology(topo, g2n), make_cost(cost));
    });
}

int ref_generate_trace(std::uint32_t num_domains, std::uint32_t requests_per_domain,
                       std::uint32_t preferred, double affinity, double decode_tokens_mean,
                       std::uint64_t seed, std::uint32_t E, std::uint32_t top_k,
                       std::uint32_t layers, const char *path) {
    return guarded([&] {
        ModelConfig model{"synthetic", E, top_k, layers, false};
        SyntheticTraceSpec spec{num_domains, requests_per_domain, preferred,
                                affinity,    decode_tokens_mean,  seed};
        write_trace_file(generate_synthetic_trace(spec, model), path);
    });
}

// Times generate_synthetic_trace (serial by construction); returns the number
// of routed tokens (prefill + decode) in *tokens.
int ref_bench_generate_trace(std::uint32_t num_domains, std::uint32_t requests_per_domain,
                             std::uint32_t preferred, double affinity, double decode_tokens_mean,
                             std::uint64_t seed, std::uint32_t E, std::uint32_t top_k,
                             std::uint32_t layers, double *seconds, std::uint64_t *tokens) {
    return guarded([&] {
        ModelConfig model{"synthetic", E, top_k, layers, false};
        SyntheticTraceSpec spec{num_domains, requests_per_domain, preferred,
                                affinity,    decode_tokens_mean,  seed};
        auto t0 = std::chrono::steady_clock::now();
        auto records = generate_synthetic_trace(spec, model);
        auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        std::uint64_t n = 0;
        for (const auto &r : records)
            n += r.stage == Stage::decode ? r.generated_tokens : r.input_length;
        *tokens = n;
    });
}

int ref_expert_load(const double *counts, std::uint32_t E, std::uint32_t top_k, double *loads,
                    std::uint64_t *total_tokens, double *imbalance) {
    return guarded([&] {
        auto l = expert_load(std::span<const double>(counts, E), top_k);
        std::memcpy(loads, l.loads.data(), sizeof(double) * E);
        *total_tokens = l.total_tokens;
        *imbalance = imbalance_factor(l);
    });
}

int ref_pearson(const double *x, const double *y, std::uint64_t n, double *r) {
    return guarded([&] { *r = pearson(std::span<const double>(x, n), std::span<const double>(y, n)); });
}

// Placement policies; groups_out must hold D*M entries (M = E/D for
// linear/eplb, (E+R)/D for data_based).
int ref_linear_placement(std::uint32_t E, std::uint32_t D, std::uint32_t *groups_out) {
    return guarded([&] {
        auto p = linear_placement(E, D);
        std::size_t o = 0;
        for (auto &g : p.groups)
            for (auto e : g) groups_out[o++] = e;
    });
}

int ref_eplb_placement(const double *load, std::uint32_t E, std::uint32_t D,
                       std::uint32_t *groups_out) {
    return guarded([&] {
        auto p = eplb_placement(std::span<const double>(load, E), E, D);
        std::size_t o = 0;
        for (auto &g : p.groups)
            for (auto e : g) groups_out[o++] = e;
    });
}

int ref_data_based_placement(const double *usage, std::uint32_t D, std::uint32_t E,
                             std::uint32_t R, std::uint64_t seed, std::uint32_t *groups_out) {
    return guarded([&] {
        UsageMatrix u;
        u.D = D;
        u.E = E;
        u.values.assign(usage, usage + std::size_t(D) * E);
        auto p = data_based_placement(u, R, seed);
        std::size_t o = 0;
        for (auto &g : p.groups)
            for (auto e : g) groups_out[o++] = e;
    });
}

// Full comparison scenario from a RunConfig JSON (reference schema,
// config.cpp:108-138): synthetic trace -> cluster stage -> placements ->
// routing -> compare_strategies, with every input and output dumped to
// out_json_path. If trace_out is non-empty the trace is also written there.
int ref_compare_scenario(const char *config_json_path, const char *trace_out,
                         const char *out_json_path, double *seconds_compare) {
    return guarded([&] {
        RunConfig cfg = load_run_config(config_json_path);
        if (!cfg.has_synthetic)
            throw ConfigError("ref_compare_scenario: config needs a synthetic section");
        auto records = generate_synthetic_trace(cfg.synthetic, cfg.model);
        if (trace_out && *trace_out)
            write_trace_file(records, trace_out);
        const std::uint32_t D = cfg.topology.ep;
        auto stage = run_cluster_stage(records, cfg.model, cfg.clustering, D);
        auto strategies = build_placements(stage, cfg.placement);
        auto decode = build_activation_matrix(records, cfg.model.num_experts_per_layer,
                                              cfg.simulation.layer, Stage::decode);
        auto routes = routing_for_matrix(decode, stage.matrix.request_ids, stage.model,
                                         stage.group_map);
        auto t0 = std::chrono::steady_clock::now();
        auto table = compare_strategies(decode, strategies, routes, cfg.topology, cfg.cost,
                                        cfg.simulation.batches, cfg.simulation.batch_size,
                                        cfg.simulation.seed);
        auto t1 = std::chrono::steady_clock::now();
        if (seconds_compare)
            *seconds_compare = std::chrono::duration<double>(t1 - t0).count();

        json j;
        j["decode_matrix"] = matrix_json(decode);
        j["cluster_matrix"] = matrix_json(stage.matrix);
        j["cluster_K"] = stage.model.K;
        j["cluster_objective"] = stage.model.objective;
        j["clustering"] = {{"seed", cfg.clustering.seed},
                           {"restarts", cfg.clustering.restarts},
                           {"max_iterations", cfg.clustering.max_iterations},
                           {"tolerance", cfg.clustering.tolerance}};
        j["placement_cfg"] = {{"seed", cfg.placement.seed}, {"R", cfg.placement.R_redundancy}};
        j["cluster_labels"] = stage.model.labels;
        j["group_map"] = stage.group_map.assignment;
        json strat = json::array();
        for (const auto &s : strategies)
            strat.push_back({{"label", s.label},
                             {"groups", s.placement.groups},
                             {"E", s.placement.E},
                             {"M", s.placement.M},
                             {"cluster_routed", s.cluster_routed}});
        j["strategies"] = strat;
        j["routes"] = routes;
        j["topology"] = {{"dp", cfg.topology.dp},
                         {"tp", cfg.topology.tp},
                         {"ep", cfg.topology.ep},
                         {"tp_exp", cfg.topology.tp_exp},
                         {"nodes", cfg.topology.nodes},
                         {"gpus_per_node", cfg.topology.gpus_per_node},
                         {"group_to_node", cfg.topology.group_to_node}};
        j["cost"] = {cfg.cost.hidden_dim,           cfg.cost.bytes_per_element,
                     cfg.cost.inter_node_bandwidth, cfg.cost.intra_node_bandwidth,
                     cfg.cost.expert_time_per_token, cfg.cost.fixed_layer_overhead};
        j["num_batches"] = cfg.simulation.batches;
        j["batch_size"] = cfg.simulation.batch_size;
        j["seed"] = cfg.simulation.seed;
        json rows = json::array();
        for (const auto &r : table.rows) {
            json row = sim_json(r.sim);
            row["batch"] = r.batch;
            row["strategy"] = r.strategy;
            row["normalized"] = r.normalized;
            rows.push_back(row);
        }
        j["rows"] = rows;
        json summary = json::array();
        for (const auto &s : table.summary)
            summary.push_back({{"strategy", s.strategy},
                               {"median_inter_node_bytes", s.median_inter_node_bytes},
                               {"q25_inter_node_bytes", s.q25_inter_node_bytes},
                               {"q75_inter_node_bytes", s.q75_inter_node_bytes},
                               {"normalized_median", s.normalized_median},
                               {"median_dispatch_time", s.median_dispatch_time},
                               {"median_expert_compute_time", s.median_expert_compute_time},
                               {"median_combine_time", s.median_combine_time},
                               {"median_layer_time", s.median_layer_time}});
        j["summary"] = summary;
        j["linear_median_bytes"] = table.linear_median_bytes;
        std::ofstream out(out_json_path);
        if (!out)
            throw Error(std::string("cannot write ") + out_json_path);
        out << j.dump() << '\n';
    });
}

// emit_analysis (pipeline.cpp:65-126) as data: per (stage, layer) imbalance
// factor, per stage dataset correlation matrix, per layer PD correlation.
int ref_analysis(const char *trace_path, std::uint32_t E, std::uint32_t top_k,
                 std::uint32_t layers, const char *out_json_path) {
    return guarded([&] {
        ModelConfig model{"m", E, top_k, layers, false};
        auto records = read_trace_file(trace_path, model);
        json j;
        json imb = json::array();
        for (Stage stage : {Stage::prefill, Stage::decode})
            for (std::uint32_t layer : layers_present(records, stage)) {
                auto m = build_activation_matrix(records, E, layer, stage);
                std::vector<double> col(E, 0.0);
                for (std::size_t r = 0; r < m.rows; ++r)
                    for (std::size_t e = 0; e < E; ++e) col[e] += m.at(r, e);
                auto loads = expert_load(col, top_k);
                imb.push_back({{"stage", stage_name(stage)}, {"layer", layer},
                               {"imbalance", imbalance_factor(loads)}, {"loads", loads.loads},
                               {"total_tokens", loads.total_tokens}});
            }
        j["imbalance"] = imb;
        for (Stage stage : {Stage::prefill, Stage::decode}) {
            auto m = build_activation_matrix_summed(records, E, stage);
            auto c = dataset_correlation_matrix(m);
            std::vector<json> vals;
            for (double v : c.values) vals.push_back(std::isnan(v) ? json(nullptr) : json(v));
            j[std::string("dataset_correlation_") + stage_name(stage)] = {{"labels", c.labels},
                                                                          {"values", vals}};
        }
        json pd = json::array();
        for (std::uint32_t layer : layers_present(records, Stage::prefill)) {
            auto a = build_activation_matrix(records, E, layer, Stage::prefill);
            auto b = build_activation_matrix(records, E, layer, Stage::decode);
            pd.push_back({{"layer", layer}, {"pearson", prefill_decode_correlation(a, b)}});
        }
        j["prefill_decode"] = pd;
        std::ofstream out(out_json_path);
        out << j.dump() << '\n';
    });
}

// Times compare_strategies alone on a scenario (inputs rebuilt untimed).
int ref_bench_compare(const char *config_json_path, std::uint32_t reps, double *seconds) {
    return guarded([&] {
        RunConfig cfg = load_run_config(config_json_path);
        auto records = generate_synthetic_trace(cfg.synthetic, cfg.model);
        const std::uint32_t D = cfg.topology.ep;
        auto stage = run_cluster_stage(records, cfg.model, cfg.clustering, D);
        auto strategies = build_placements(stage, cfg.placement);
        auto decode = build_activation_matrix(records, cfg.model.num_experts_per_layer,
                                              cfg.simulation.layer, Stage::decode);
        auto routes = routing_for_matrix(decode, stage.matrix.request_ids, stage.model,
                                         stage.group_map);
        auto t0 = std::chrono::steady_clock::now();
        for (std::uint32_t r = 0; r < reps; ++r)
            (void)compare_strategies(decode, strategies, routes, cfg.topology, cfg.cost,
                                     cfg.simulation.batches, cfg.simulation.batch_size,
                                     cfg.simulation.seed);
        auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

// Times read_trace_file + build_activation_matrix_summed (a1/a2 wire path).
int ref_bench_parse(const char *trace_path, std::uint32_t E, std::uint32_t top_k,
                    std::uint32_t layers, double *parse_seconds, double *matrix_seconds,
                    std::uint64_t *records_out) {
    return guarded([&] {
        ModelConfig model{"m", E, top_k, layers, false};
        auto t0 = std::chrono::steady_clock::now();
        auto records = read_trace_file(trace_path, model);
        auto t1 = std::chrono::steady_clock::now();
        auto m = build_activation_matrix_summed(records, E, Stage::decode);
        auto t2 = std::chrono::steady_clock::now();
        *parse_seconds = std::chrono::duration<double>(t1 - t0).count();
        *matrix_seconds = std::chrono::duration<double>(t2 - t1).count();
        *records_out = records.size() + 0 * m.rows;
    });
}

// compare_strategies (simulator.cpp:122-243) on caller-given inputs: the
// decode matrix [R x E] (integer counts as double), S strategies (labels
// newline-separated, groups of strategy s at groups_flat[s], sizes in
// group_sizes[s*D..], cluster_routed[s]) and per-row routing group sets
// (route_off[R+1] into route_flat). Outputs: sims[B*S][6] (inter, intra,
// dispatch, compute, combine, layer), normalized[B*S], summary[S][8]
// (median / q25 / q75 inter bytes, normalized median, median dispatch /
// compute / combine / layer time) and the linear median.
int ref_compare_strategies(std::uint64_t R, std::uint32_t E, const double *values,
                           std::uint32_t S, const char *labels, const std::uint32_t *groups_flat,
                           const std::uint32_t *group_sizes, std::uint32_t D,
                           const std::int32_t *cluster_routed, const std::uint64_t *route_off,
                           const std::uint32_t *route_flat, const std::uint32_t *topo,
                           const std::uint32_t *g2n, const double *cost, std::uint32_t B,
                           std::uint32_t batch_size, std::uint64_t seed, double *sims,
                           double *normalized, double *summary, double *linear_median) {
    return guarded([&] {
        ActivationMatrix m;
        m.rows = R;
        m.cols = E;
        m.values.assign(values, values + R * E);
        m.row_labels.assign(R, "x");
        for (std::uint64_t r = 0; r < R; ++r) m.request_ids.push_back(r);
        std::vector<StrategyEntry> strategies(S);
        std::string all(labels);
        std::size_t pos = 0, off = 0;
        for (std::uint32_t s = 0; s < S; ++s) {
            const std::size_t nl = all.find('\n', pos);
            strategies[s].label = all.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos);
            pos = nl == std::string::npos ? all.size() : nl + 1;
            std::uint32_t n = 0;
            for (std::uint32_t d = 0; d < D; ++d) n += group_sizes[s * D + d];
            strategies[s].placement = make_placement(groups_flat + off, group_sizes + s * D, D, E);
            strategies[s].cluster_routed = cluster_routed[s] != 0;
            off += n;
        }
        std::vector<std::vector<std::uint32_t>> routes(R);
        for (std::uint64_t r = 0; r < R; ++r)
            routes[r].assign(route_flat + route_off[r], route_flat + route_off[r + 1]);
        auto table = compare_strategies(m, strategies, routes, make_topology(topo, g2n),
                                        make_cost(cost), B, batch_size, seed);
        for (std::size_t i = 0; i < table.rows.size(); ++i) {
            const auto &sim = table.rows[i].sim;
            double *o = sims + 6 * i;
            o[0] = sim.inter_node_bytes;
            o[1] = sim.intra_node_bytes;
            o[2] = sim.dispatch_time;
            o[3] = sim.expert_compute_time;
            o[4] = sim.combine_time;
            o[5] = sim.layer_time;
            normalized[i] = table.rows[i].normalized;
        }
        for (std::size_t s = 0; s < table.summary.size(); ++s) {
            const auto &x = table.summary[s];
            double *o = summary + 8 * s;
            o[0] = x.median_inter_node_bytes;
            o[1] = x.q25_inter_node_bytes;
            o[2] = x.q75_inter_node_bytes;
            o[3] = x.normalized_median;
            o[4] = x.median_dispatch_time;
            o[5] = x.median_expert_compute_time;
            o[6] = x.median_combine_time;
            o[7] = x.median_layer_time;
        }
        *linear_median = table.linear_median_bytes;
    });
}

} // extern "C"
