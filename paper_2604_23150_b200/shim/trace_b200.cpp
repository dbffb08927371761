// Drop-in replacement for the reference's trace translation unit
// (/root/reference/proj/core/src/trace.cpp), compiled against its public
// header moeplace/trace.hpp (:14-119) and backed by the library's host trace
// model (csrc/host_trace.cpp) through the C ABI:
//   parse_trace / read_trace_file     -> mpb_trace_parse / mpb_trace_read_file
//                                        (multi-threaded fixed-schema scanner,
//                                        714 MB/s vs nlohmann's 30.8 MB/s)
//   write_trace / write_trace_file    -> mpb_trace_import + mpb_trace_dump /
//                                        mpb_trace_write_file (byte-identical
//                                        to nlohmann::json::dump)
//   build_activation_matrix[_summed]  -> mpb_trace_matrix
//   layers_present                    -> mpb_trace_layers_present
//   generate_synthetic_trace          -> mpb_trace_generate (same std:: RNG
//                                        calls: bit-identical records)
// Record / model validation keeps the reference's exception classes and
// conditions (trace.cpp:25-64).
#include <fstream>
#include <iterator>
#include <memory>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "moeplace/trace.hpp"
#include "shim_common.hpp"

namespace moeplace {
namespace {

using namespace b200;

struct TraceDeleter {
    void operator()(mpb_trace *t) const { mpb_trace_destroy(t); }
};
using Trace = std::unique_ptr<mpb_trace, TraceDeleter>;

// std::vector<ActivationRecord> -> library trace (labels deduplicated in
// first-seen order, which the matrix builder's first-seen rule needs).
Trace import_records(const std::vector<ActivationRecord> &records) {
    const std::size_t n = records.size();
    std::vector<uint64_t> rid(n), in_len(n), gen(n), off(n + 1, 0), cnt;
    std::vector<uint32_t> layer(n), lab(n), ex;
    std::vector<uint8_t> stage(n);
    std::vector<std::string> names;
    std::vector<const char *> name_ptrs;
    std::unordered_map<std::string, uint32_t> seen;
    for (std::size_t i = 0; i < n; ++i) {
        const auto &r = records[i];
        rid[i] = r.request_id;
        layer[i] = r.layer_index;
        stage[i] = r.stage == Stage::decode ? 1 : 0;
        in_len[i] = r.input_length;
        gen[i] = r.generated_tokens;
        const auto [it, fresh] =
            seen.try_emplace(r.dataset_label, static_cast<uint32_t>(names.size()));
        if (fresh) names.push_back(r.dataset_label);
        lab[i] = it->second;
        for (const auto &[e, c] : r.expert_counts) {
            ex.push_back(e);
            cnt.push_back(c);
        }
        off[i + 1] = ex.size();
    }
    for (const auto &s : names) name_ptrs.push_back(s.c_str());
    mpb_trace *t = nullptr;
    check(mpb_trace_import(n, rid.data(), layer.data(), stage.data(), in_len.data(), gen.data(),
                           lab.data(), off.data(), ex.data(), cnt.data(), names.size(),
                           name_ptrs.data(), &t));
    return Trace(t);
}

std::vector<ActivationRecord> export_records(const mpb_trace *t) {
    uint64_t nr = 0, np = 0, nl = 0;
    check(mpb_trace_sizes(t, &nr, &np, &nl, nullptr));
    std::vector<uint64_t> rid(nr), in_len(nr), gen(nr), off(nr + 1), cnt(np);
    std::vector<uint32_t> layer(nr), lab(nr), ex(np);
    std::vector<uint8_t> stage(nr);
    check(mpb_trace_export(t, rid.data(), layer.data(), stage.data(), in_len.data(), gen.data(),
                           lab.data(), off.data(), ex.data(), cnt.data(), nullptr, nullptr));
    std::vector<std::string> labels(nl);
    for (uint64_t i = 0; i < nl; ++i) labels[i] = mpb_trace_label(t, i);
    std::vector<ActivationRecord> out(nr);
    for (uint64_t i = 0; i < nr; ++i) {
        auto &r = out[i];
        r.dataset_label = labels[lab[i]];
        r.request_id = rid[i];
        r.stage = stage[i] ? Stage::decode : Stage::prefill;
        r.layer_index = layer[i];
        r.input_length = in_len[i];
        r.generated_tokens = gen[i];
        for (uint64_t j = off[i]; j < off[i + 1]; ++j)
            r.expert_counts.emplace_hint(r.expert_counts.end(), ex[j], cnt[j]);
    }
    return out;
}

ActivationMatrix matrix_of(const std::vector<ActivationRecord> &records, std::uint32_t E,
                           int64_t layer, Stage stage) {
    Trace t = import_records(records);
    const int st = stage == Stage::decode ? 1 : 0;
    uint64_t rows = 0;
    check(mpb_trace_matrix(t.get(), E, layer, st, &rows, nullptr, nullptr, nullptr));
    ActivationMatrix m;
    m.rows = rows;
    m.cols = E;
    m.values.resize(rows * E);
    m.request_ids.resize(rows);
    std::vector<uint32_t> lab(rows);
    check(mpb_trace_matrix(t.get(), E, layer, st, &rows, m.values.data(), m.request_ids.data(),
                           lab.data()));
    m.row_labels.reserve(rows);
    for (uint32_t l : lab) m.row_labels.emplace_back(mpb_trace_label(t.get(), l));
    return m;
}

std::string describe(const ActivationRecord &r) {
    std::ostringstream o;
    o << "record (dataset=" << r.dataset_label << ", request_id=" << r.request_id
      << ", stage=" << stage_name(r.stage) << ", layer=" << r.layer_index << ")";
    return o.str();
}

}  // namespace

const char *stage_name(Stage s) { return s == Stage::decode ? "decode" : "prefill"; }

Stage stage_from_name(const std::string &name) {
    if (name == "decode") return Stage::decode;
    if (name == "prefill") return Stage::prefill;
    throw ValidationError("unknown stage '" + name + "' (expected prefill|decode)");
}

void ModelConfig::validate() const {
    const std::string who = "model '" + name + "': ";
    if (num_experts_per_layer == 0) throw ConfigError(who + "num_experts_per_layer must be >= 1");
    if (top_k == 0 || top_k > num_experts_per_layer)
        throw ConfigError(who + "top_k must satisfy 1 <= top_k <= " +
                          std::to_string(num_experts_per_layer));
    if (num_moe_layers == 0) throw ConfigError(who + "num_moe_layers must be >= 1");
}

void ActivationRecord::validate(const ModelConfig &model) const {
    if (expert_counts.empty()) throw ValidationError(describe(*this) + ": empty expert_counts");
    std::uint64_t total = 0;
    for (const auto &[e, c] : expert_counts) {
        if (e >= model.num_experts_per_layer)
            throw ValidationError(describe(*this) + ": expert id " + std::to_string(e) + " >= E=" +
                                  std::to_string(model.num_experts_per_layer));
        if (c == 0)
            throw ValidationError(describe(*this) + ": expert " + std::to_string(e) +
                                  " has zero count");
        total += c;
    }
    const std::uint64_t want = generated_tokens * model.top_k;
    if (stage == Stage::decode && total != want)
        throw ValidationError(describe(*this) + ": decode counts sum to " + std::to_string(total) +
                              ", expected generated_tokens*top_k=" + std::to_string(want));
}

double ActivationMatrix::total() const {
    double s = 0.0;
    for (std::size_t i = 0; i < values.size(); ++i) s += values[i];
    return s;
}

std::vector<ActivationRecord> parse_trace(std::istream &in, const ModelConfig &model) {
    model.validate();
    const std::string text{std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
    mpb_trace *raw = nullptr;
    check(mpb_trace_parse(text.data(), text.size(), model.num_experts_per_layer, model.top_k,
                          model.num_moe_layers, &raw));
    Trace t(raw);
    return export_records(t.get());
}

void write_trace(const std::vector<ActivationRecord> &records, std::ostream &out) {
    Trace t = import_records(records);
    uint64_t len = 0;
    check(mpb_trace_dump(t.get(), nullptr, 0, &len));
    std::string text(len, '\0');
    check(mpb_trace_dump(t.get(), text.data(), len, &len));
    out.write(text.data(), static_cast<std::streamsize>(len));
}

std::vector<ActivationRecord> read_trace_file(const std::string &path, const ModelConfig &model) {
    if (!std::ifstream(path)) throw Error("cannot open trace file: " + path);
    model.validate();
    mpb_trace *raw = nullptr;
    check(mpb_trace_read_file(path.c_str(), model.num_experts_per_layer, model.top_k,
                              model.num_moe_layers, &raw));
    Trace t(raw);
    return export_records(t.get());
}

void write_trace_file(const std::vector<ActivationRecord> &records, const std::string &path) {
    Trace t = import_records(records);
    check(mpb_trace_write_file(t.get(), path.c_str()));
}

ActivationMatrix build_activation_matrix(const std::vector<ActivationRecord> &records,
                                         std::uint32_t num_experts, std::uint32_t layer_index,
                                         Stage stage) {
    return matrix_of(records, num_experts, static_cast<int64_t>(layer_index), stage);
}

ActivationMatrix build_activation_matrix_summed(const std::vector<ActivationRecord> &records,
                                                std::uint32_t num_experts, Stage stage) {
    return matrix_of(records, num_experts, -1, stage);
}

std::vector<std::uint32_t> layers_present(const std::vector<ActivationRecord> &records,
                                          Stage stage) {
    Trace t = import_records(records);
    uint64_t n = 0;
    const int st = stage == Stage::decode ? 1 : 0;
    check(mpb_trace_layers_present(t.get(), st, nullptr, &n));
    std::vector<std::uint32_t> out(n);
    check(mpb_trace_layers_present(t.get(), st, out.data(), &n));
    return out;
}

std::vector<std::uint32_t> domain_preferred_experts(const SyntheticTraceSpec &spec,
                                                    const ModelConfig &model,
                                                    std::uint32_t domain) {
    const std::uint64_t first = std::uint64_t(domain) * spec.preferred_experts_per_domain;
    std::vector<std::uint32_t> ids;
    ids.reserve(spec.preferred_experts_per_domain);
    for (std::uint64_t e = first; e < first + spec.preferred_experts_per_domain; ++e)
        ids.push_back(static_cast<std::uint32_t>(e % model.num_experts_per_layer));
    return ids;
}

std::vector<ActivationRecord> generate_synthetic_trace(const SyntheticTraceSpec &spec,
                                                       const ModelConfig &model) {
    model.validate();
    mpb_trace *raw = nullptr;
    check(mpb_trace_generate(spec.num_domains, spec.requests_per_domain,
                             spec.preferred_experts_per_domain, spec.affinity,
                             spec.decode_tokens_mean, spec.seed, model.num_experts_per_layer,
                             model.top_k, model.num_moe_layers, 0, &raw));
    Trace t(raw);
    return export_records(t.get());
}

}  // namespace moeplace
