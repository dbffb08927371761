// Drop-in replacement for the reference's metrics translation unit
// (/root/reference/proj/core/src/metrics.cpp), compiled against its public
// header moeplace/metrics.hpp (:14-49):
//   expert_load / pearson          -> mpb_expert_load / mpb_pearson (host
//                                     finalisation in the reference's order)
//   dataset_correlation_matrix /   -> per-dataset and all-row column sums as
//   prefill_decode_correlation        exact uint64 histograms on the B200
//                                     (mpb_label_row_sums), then pearson
// Trace-derived matrices hold integer token counts, for which the device sums
// equal the reference's sequential double sums exactly (metrics.cu). A matrix
// with a non-integral or negative entry is summed on the host in the
// reference's row order instead (mpb_label_row_sums refuses it), so the result
// is the reference's in every case.
#include <algorithm>
#include <limits>
#include <map>
#include <string>
#include <vector>

#include "moeplace/metrics.hpp"
#include "shim_common.hpp"

namespace moeplace {
namespace {

using namespace b200;

// Column sums of the rows carrying each label id (label ids in [0, n)).
std::vector<std::vector<double>> column_sums(const ActivationMatrix &m,
                                             const std::vector<uint32_t> &label_of_row,
                                             uint32_t n) {
    std::vector<std::vector<double>> out(n, std::vector<double>(m.cols, 0.0));
    if (m.rows == 0 || m.cols == 0) return out;
    Device &dev = device();
    std::lock_guard<std::recursive_mutex> lock(dev.mu);
    const double *d_m = dev.up(kMetMatrix, m.values.data(), m.rows * m.cols);
    const uint32_t *d_l = dev.up(kMetLabels, label_of_row);
    auto *d_s = static_cast<uint64_t *>(dev.buf(kMetSums, size_t(n) * m.cols * 8));
    const mpb_status st = mpb_label_row_sums(dev.ctx, d_m, m.rows, static_cast<uint32_t>(m.cols),
                                             d_l, n, d_s);
    if (st == MPB_OK) {
        std::vector<uint64_t> h(size_t(n) * m.cols);
        dev.down(h, d_s);
        for (uint32_t l = 0; l < n; ++l)
            for (std::size_t c = 0; c < m.cols; ++c)
                out[l][c] = static_cast<double>(h[size_t(l) * m.cols + c]);
        return out;
    }
    if (st != MPB_VALIDATION_ERROR) check(st);
    // non-integral entries: sequential sums in row order (metrics.cpp:72-91)
    for (std::size_t r = 0; r < m.rows; ++r) {
        auto &acc = out[label_of_row[r]];
        for (std::size_t c = 0; c < m.cols; ++c) acc[c] += m.values[r * m.cols + c];
    }
    return out;
}

std::vector<double> all_row_sums(const ActivationMatrix &m) {
    return column_sums(m, std::vector<uint32_t>(m.rows, 0u), 1)[0];
}

}  // namespace

ExpertLoadVector expert_load(std::span<const double> per_expert_token_counts,
                             std::uint32_t top_k) {
    if (per_expert_token_counts.empty()) throw ValidationError("expert_load: empty count vector");
    ExpertLoadVector v;
    v.loads.resize(per_expert_token_counts.size());
    v.top_k = top_k;
    check(mpb_expert_load(per_expert_token_counts.data(),
                          static_cast<uint32_t>(per_expert_token_counts.size()), top_k,
                          v.loads.data(), &v.total_tokens));
    return v;
}

double imbalance_factor(const ExpertLoadVector &loads) {
    if (loads.loads.empty()) throw ValidationError("imbalance_factor: empty load vector");
    return *std::max_element(loads.loads.begin(), loads.loads.end());
}

double pearson(std::span<const double> x, std::span<const double> y) {
    if (x.size() != y.size()) throw ValidationError("pearson: length mismatch");
    double r = 0.0;
    check(mpb_pearson(x.data(), y.data(), x.size(), &r));
    return r;
}

CorrelationMatrix dataset_correlation_matrix(const ActivationMatrix &matrix) {
    // datasets in lexicographic order (the reference's std::map iteration)
    std::map<std::string, uint32_t> ids;
    for (const auto &l : matrix.row_labels) ids.emplace(l, 0u);
    if (ids.size() < 2)
        throw ValidationError("dataset_correlation_matrix: need >= 2 datasets, got " +
                              std::to_string(ids.size()));
    CorrelationMatrix out;
    uint32_t next = 0;
    for (auto &[label, id] : ids) {
        id = next++;
        out.labels.push_back(label);
    }
    std::vector<uint32_t> row_label(matrix.rows);
    for (std::size_t r = 0; r < matrix.rows; ++r) row_label[r] = ids.at(matrix.row_labels[r]);
    const auto sums = column_sums(matrix, row_label, next);
    const std::size_t n = next;
    out.values.assign(n * n, std::numeric_limits<double>::quiet_NaN());
    for (std::size_t i = 0; i < n; ++i) {
        out.values[i * n + i] = 1.0;
        for (std::size_t j = i + 1; j < n; ++j) {
            double r = 0.0;
            const mpb_status st = mpb_pearson(sums[i].data(), sums[j].data(), matrix.cols, &r);
            if (st == MPB_UNDEFINED_CORRELATION_ERROR) continue;  // missing, not zero
            check(st);
            out.values[i * n + j] = out.values[j * n + i] = r;
        }
    }
    return out;
}

double prefill_decode_correlation(const ActivationMatrix &prefill, const ActivationMatrix &decode) {
    if (prefill.rows == 0 || decode.rows == 0)
        throw ValidationError("prefill_decode_correlation: empty matrix");
    if (prefill.cols != decode.cols)
        throw ValidationError("prefill_decode_correlation: expert count mismatch");
    const auto a = all_row_sums(prefill), b = all_row_sums(decode);
    return pearson(a, b);
}

}  // namespace moeplace
