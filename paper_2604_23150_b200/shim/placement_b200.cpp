// Drop-in replacement for the reference's placement-policy translation unit
// (/root/reference/proj/core/src/placement.cpp), compiled against its public
// header moeplace/placement.hpp (:14-113). The policies are the library's
// host restatements behind the C ABI (csrc/host_policies.cpp: the same
// std::stable_sort orders, tie rules and std::mt19937_64 / libstdc++
// distribution calls, hence bit-identical placements):
//   aggregate_usage            -> mpb_aggregate_usage
//   phase1 / phase2 / balance  -> mpb_phase1_unique_distribution /
//                                 mpb_phase2_redundant_addition /
//                                 mpb_balance_and_verify
//   data_based / linear / eplb -> mpb_data_based_placement / mpb_linear_placement
//                                 / mpb_eplb_placement
//   Placement::verify          -> mpb_placement_verify
// The placements they produce are what the B200 scorer prices
// (mpb_score_placements); topology arithmetic, routing lookup and the
// placement text format are host code below.
#include <algorithm>
#include <fstream>
#include <istream>
#include <ostream>
#include <sstream>
#include <string>
#include <vector>

#include "moeplace/placement.hpp"
#include "shim_common.hpp"

namespace moeplace {
namespace {

using namespace b200;
using GroupList = std::vector<std::vector<std::uint32_t>>;

GroupList unflatten(const std::vector<uint32_t> &flat, const std::vector<uint32_t> &sizes) {
    GroupList g(sizes.size());
    std::size_t o = 0;
    for (std::size_t d = 0; d < sizes.size(); ++d) {
        g[d].assign(flat.begin() + o, flat.begin() + o + sizes[d]);
        o += sizes[d];
    }
    return g;
}

GroupList fixed_groups(const std::vector<uint32_t> &flat, std::uint32_t D, std::uint32_t M) {
    return unflatten(flat, std::vector<uint32_t>(D, M));
}

Placement make(GroupList groups, std::uint32_t E, std::uint32_t M, PlacementStrategy s) {
    Placement p;
    p.groups = std::move(groups);
    p.E = E;
    p.M = M;
    p.R_redundancy = M * p.D() - E;
    p.strategy = s;
    return p;
}

}  // namespace

const char *strategy_name(PlacementStrategy s) {
    switch (s) {
    case PlacementStrategy::linear: return "linear";
    case PlacementStrategy::eplb: return "eplb";
    case PlacementStrategy::data_based: return "data_based";
    }
    return "unknown";
}

PlacementStrategy strategy_from_name(const std::string &name) {
    for (auto s : {PlacementStrategy::linear, PlacementStrategy::eplb, PlacementStrategy::data_based})
        if (name == strategy_name(s)) return s;
    throw LookupError("unknown placement strategy '" + name + "'");
}

void Placement::verify() const {
    const FlatGroups f = flatten(groups);
    check(mpb_placement_verify(f.flat.data(), f.sizes.data(), D(), E, M));
}

void Topology::validate() const {
    if (!dp || !tp || !ep || !tp_exp || !nodes || !gpus_per_node)
        throw ConfigError("topology: all rank counts must be >= 1");
    const std::uint32_t ranks = dp * tp;
    if (ep * tp_exp != ranks)
        throw ConfigError("topology: ep*tp_exp (" + std::to_string(ep * tp_exp) + ") != dp*tp (" +
                          std::to_string(ranks) + ")");
    if (gpus_per_node * nodes != ranks)
        throw ConfigError("topology: gpus_per_node*nodes (" + std::to_string(gpus_per_node * nodes) +
                          ") != dp*tp (" + std::to_string(ranks) + ")");
    if (group_to_node.size() != ep)
        throw ConfigError("topology: group_to_node must list one node per EP group");
    if (std::any_of(group_to_node.begin(), group_to_node.end(),
                    [&](std::uint32_t n) { return n >= nodes; }))
        throw ConfigError("topology: node id out of range in group_to_node");
}

Topology Topology::contiguous(std::uint32_t dp, std::uint32_t tp, std::uint32_t ep,
                              std::uint32_t tp_exp, std::uint32_t nodes) {
    if (nodes == 0 || (dp * tp) % nodes != 0) throw ConfigError("topology: nodes must divide dp*tp");
    if (ep % nodes != 0)
        throw ConfigError("topology: nodes must divide ep for contiguous group layout");
    Topology t;
    t.dp = dp;
    t.tp = tp;
    t.ep = ep;
    t.tp_exp = tp_exp;
    t.nodes = nodes;
    t.gpus_per_node = dp * tp / nodes;
    const std::uint32_t per_node = ep / nodes;
    for (std::uint32_t g = 0; g < ep; ++g) t.group_to_node.push_back(g / per_node);
    t.validate();
    return t;
}

UsageMatrix aggregate_usage(const GroupMap &group_map, const ActivationMatrix &raw_matrix,
                            const ClusterModel &model, std::uint32_t D) {
    if (group_map.K != model.K)
        throw ValidationError("aggregate_usage: group map K does not match model K");
    if (group_map.D != D) throw ValidationError("aggregate_usage: group map D does not match D");
    if (raw_matrix.rows != model.labels.size())
        throw ValidationError("aggregate_usage: matrix rows do not match labels");
    UsageMatrix u;
    u.D = D;
    u.E = static_cast<std::uint32_t>(raw_matrix.cols);
    u.values.resize(std::size_t(D) * u.E);
    const FlatGroups a = flatten(group_map.assignment);
    check(mpb_aggregate_usage(model.labels.data(), raw_matrix.values.data(), raw_matrix.rows, u.E,
                              model.K, a.flat.data(), a.sizes.data(), D, u.values.data()));
    return u;
}

std::vector<std::vector<std::uint32_t>> phase1_unique_distribution(const UsageMatrix &usage) {
    std::vector<uint32_t> flat(std::max<std::uint32_t>(usage.E, 1)), sizes(usage.D);
    check(mpb_phase1_unique_distribution(usage.values.data(), usage.D, usage.E, flat.data(),
                                         sizes.data()));
    return unflatten(flat, sizes);
}

void phase2_redundant_addition(std::vector<std::vector<std::uint32_t>> &groups,
                               const UsageMatrix &usage, std::uint32_t M) {
    const FlatGroups f = flatten(groups);
    const std::uint32_t D = static_cast<std::uint32_t>(groups.size());
    std::vector<uint32_t> out(std::size_t(D) * M + 1);
    check(mpb_phase2_redundant_addition(f.flat.data(), f.sizes.data(), usage.values.data(), D,
                                        usage.E, M, out.data()));
    groups = fixed_groups(out, D, M);
}

Placement balance_and_verify(std::vector<std::vector<std::uint32_t>> groups, std::uint32_t E,
                             std::uint32_t M, std::uint64_t seed) {
    const FlatGroups f = flatten(groups);
    const std::uint32_t D = static_cast<std::uint32_t>(groups.size());
    std::vector<uint32_t> out(std::size_t(D) * M + 1);
    check(mpb_balance_and_verify(f.flat.data(), f.sizes.data(), D, E, M, seed, out.data()));
    return make(fixed_groups(out, D, M), E, M, PlacementStrategy::data_based);
}

Placement data_based_placement(const UsageMatrix &usage, std::uint32_t R_redundancy,
                               std::uint64_t seed) {
    const std::uint32_t D = usage.D, E = usage.E;
    std::vector<uint32_t> out(std::size_t(E) + R_redundancy + 1);
    check(mpb_data_based_placement(usage.values.data(), D, E, R_redundancy, seed, out.data()));
    const std::uint32_t M = (E + R_redundancy) / D;
    return make(fixed_groups(out, D, M), E, M, PlacementStrategy::data_based);
}

Placement linear_placement(std::uint32_t E, std::uint32_t D) {
    std::vector<uint32_t> out(std::max<std::uint32_t>(E, 1));
    check(mpb_linear_placement(E, D, out.data()));
    return make(fixed_groups(out, D, E / D), E, E / D, PlacementStrategy::linear);
}

Placement eplb_placement(std::span<const double> historical_per_expert_load, std::uint32_t E,
                         std::uint32_t D) {
    if (historical_per_expert_load.size() != E)
        throw ValidationError("eplb_placement: load vector length != E");
    std::vector<uint32_t> out(std::max<std::uint32_t>(E, 1));
    check(mpb_eplb_placement(historical_per_expert_load.data(), E, D, out.data()));
    return make(fixed_groups(out, D, E / D), E, E / D, PlacementStrategy::eplb);
}

std::vector<std::uint32_t> route_request(std::uint64_t request_id,
                                         std::span<const std::uint64_t> request_ids,
                                         const ClusterModel &model, const GroupMap &group_map) {
    if (request_ids.size() != model.labels.size())
        throw ValidationError("route_request: request id list does not match labels");
    const auto it = std::lower_bound(request_ids.begin(), request_ids.end(), request_id);
    if (it == request_ids.end() || *it != request_id)
        throw LookupError("route_request: unknown request id " + std::to_string(request_id));
    return group_map.assignment[model.labels[static_cast<std::size_t>(it - request_ids.begin())]];
}

void write_placement(const Placement &placement, std::ostream &out) {
    for (std::uint32_t d = 0; d < placement.D(); ++d) {
        out << d << ':';
        for (std::uint32_t e : placement.groups[d]) out << ' ' << e;
        out << '\n';
    }
}

Placement parse_placement(std::istream &in, PlacementStrategy strategy) {
    GroupList groups;
    std::uint32_t top = 0;
    std::size_t line_no = 0;
    for (std::string line; std::getline(in, line);) {
        ++line_no;
        if (line.empty()) continue;
        const std::size_t colon = line.find(':');
        if (colon == std::string::npos) throw ParseError(line_no, "expected 'group_id: e1 e2 ...'");
        unsigned long id = 0;
        try {
            id = std::stoul(line.substr(0, colon));
        } catch (const std::exception &) {
            throw ParseError(line_no, "bad group id");
        }
        if (static_cast<std::uint32_t>(id) != groups.size())
            throw ParseError(line_no, "group ids must be consecutive from 0");
        std::istringstream body(line.substr(colon + 1));
        std::vector<std::uint32_t> experts;
        for (std::uint32_t e; body >> e;) {
            experts.push_back(e);
            top = std::max(top, e);
        }
        if (body.fail() && !body.eof()) throw ParseError(line_no, "bad expert id");
        if (experts.empty()) throw ParseError(line_no, "empty group");
        groups.push_back(std::move(experts));
    }
    if (groups.empty()) throw ValidationError("placement file contains no groups");
    const std::uint32_t M = static_cast<std::uint32_t>(groups[0].size());
    Placement p = make(std::move(groups), top + 1, M, strategy);
    p.verify();
    return p;
}

void write_placement_file(const Placement &placement, const std::string &path) {
    std::ofstream out(path);
    if (!out) throw Error("cannot open placement file for writing: " + path);
    write_placement(placement, out);
}

Placement read_placement_file(const std::string &path, PlacementStrategy strategy) {
    std::ifstream in(path);
    if (!in) throw Error("cannot open placement file: " + path);
    return parse_placement(in, strategy);
}

}  // namespace moeplace
