// Drop-in replacement for the reference's grouping-policy translation unit
// (/root/reference/proj/core/src/clustering.cpp), compiled against its public
// header moeplace/clustering.hpp (:14-79):
//   l2_normalize_rows          -> mpb_l2_normalize_rows_device (B200)
//   kmeans                     -> K7 mpb_kmeans_device (k-means++ seeding +
//                                 Lloyd on the B200 in the reference's order of
//                                 fp64 operations: bit-identical labels,
//                                 centroids, objective and objective history);
//                                 shapes past K7's shared-memory tiles (K > 32
//                                 or K*dim centroids > 160 KiB) run the
//                                 library's host restatement mpb_kmeans (same
//                                 results)
//   assign_clusters_to_groups  -> mpb_assign_clusters_to_groups
//   l2_normalize, cluster_sizes, cluster-model text I/O: host, below
// Exceptions and their conditions follow clustering.cpp.
#include <cmath>
#include <istream>
#include <ostream>
#include <sstream>
#include <string>
#include <vector>

#include "moeplace/clustering.hpp"
#include "moeplace/text.hpp"
#include "shim_common.hpp"

namespace moeplace {
namespace {

using namespace b200;

ClusterModel empty_model(std::uint32_t K, std::size_t n, std::size_t dim) {
    ClusterModel m;
    m.K = K;
    m.dim = dim;
    m.labels.resize(n);
    m.centroids.resize(std::size_t(K) * dim);
    return m;
}

}  // namespace

std::vector<double> l2_normalize(std::span<const double> a) {
    std::vector<double> out(a.size());
    check(mpb_l2_normalize_rows(a.data(), 1, static_cast<uint32_t>(a.size()), out.data()));
    return out;
}

ActivationMatrix l2_normalize_rows(const ActivationMatrix &matrix) {
    ActivationMatrix out = matrix;
    if (matrix.rows == 0 || matrix.cols == 0) return out;
    Device &dev = device();
    std::lock_guard<std::recursive_mutex> lock(dev.mu);
    const std::size_t n = matrix.rows * matrix.cols;
    const double *d_in = dev.up(kClRows, matrix.values.data(), n);
    auto *d_out = static_cast<double *>(dev.buf(kClNorm, n * 8));
    check(mpb_l2_normalize_rows_device(dev.ctx, d_in, matrix.rows,
                                       static_cast<uint32_t>(matrix.cols), d_out));
    dev.down(out.values.data(), d_out, n);
    return out;
}

ClusterModel kmeans(std::span<const double> rows, std::size_t n_rows, std::size_t dim,
                    std::uint32_t K, std::uint64_t seed, std::uint32_t max_iterations,
                    double tolerance) {
    if (K == 0) throw InfeasibleError("kmeans: K must be >= 1");
    if (n_rows < K)
        throw InfeasibleError("kmeans: " + std::to_string(n_rows) + " rows < K=" +
                              std::to_string(K));
    if (rows.size() != n_rows * dim)
        throw ValidationError("kmeans: rows span size does not match n_rows * dim");
    ClusterModel m = empty_model(K, n_rows, dim);
    std::vector<double> history(std::max<std::uint32_t>(max_iterations, 1));
    const uint32_t d32 = static_cast<uint32_t>(dim);
    Device &dev = device();
    std::lock_guard<std::recursive_mutex> lock(dev.mu);
    const double *d_x = dev.up(kClRows, rows.data(), rows.size());
    auto *d_lab = static_cast<uint32_t *>(dev.buf(kClLabels, n_rows * 4));
    auto *d_cen = static_cast<double *>(dev.buf(kClCentroids, m.centroids.size() * 8));
    const mpb_status st = mpb_kmeans_device(dev.ctx, d_x, n_rows, d32, K, seed, max_iterations,
                                            tolerance, d_lab, d_cen, &m.objective,
                                            &m.iterations_run, history.data());
    if (st == MPB_OK) {
        dev.down(m.labels, d_lab);
        dev.down(m.centroids, d_cen);
    } else if (st == MPB_CONFIG_ERROR) {  // beyond K7's tiles: the host restatement
        check(mpb_kmeans(rows.data(), n_rows, d32, K, seed, max_iterations, tolerance,
                         m.labels.data(), m.centroids.data(), &m.objective, &m.iterations_run,
                         history.data()));
    } else {
        check(st);
    }
    m.objective_history.assign(history.begin(), history.begin() + m.iterations_run);
    return m;
}

std::vector<double> cluster_sizes(const ClusterModel &model, const ActivationMatrix &raw_matrix) {
    if (raw_matrix.rows != model.labels.size())
        throw ValidationError("cluster_sizes: matrix row count does not match labels");
    std::vector<double> s(model.K, 0.0);
    for (std::size_t r = 0; r < raw_matrix.rows; ++r) {
        double norm1 = 0.0;
        const double *row = raw_matrix.values.data() + r * raw_matrix.cols;
        for (std::size_t c = 0; c < raw_matrix.cols; ++c) norm1 += std::abs(row[c]);
        s[model.labels[r]] += norm1;
    }
    return s;
}

GroupMap assign_clusters_to_groups(const ClusterModel &model, const ActivationMatrix &raw_matrix,
                                   std::uint32_t D, std::uint64_t seed) {
    if (D == 0) throw InfeasibleError("assign_clusters_to_groups: D must be >= 1");
    GroupMap g;
    g.K = model.K;
    g.D = D;
    g.cluster_sizes = cluster_sizes(model, raw_matrix);  // validates the row count
    std::vector<uint32_t> flat(std::size_t(model.K) * std::max(D, 1u) + 1), sizes(model.K);
    std::vector<double> cs(model.K);
    check(mpb_assign_clusters_to_groups(model.labels.data(), model.labels.size(), model.K,
                                        raw_matrix.values.data(),
                                        static_cast<uint32_t>(raw_matrix.cols), D, seed,
                                        flat.data(), sizes.data(), cs.data()));
    g.assignment.resize(model.K);
    std::size_t o = 0;
    for (std::uint32_t k = 0; k < model.K; ++k) {
        g.assignment[k].assign(flat.begin() + o, flat.begin() + o + sizes[k]);
        o += sizes[k];
    }
    return g;
}

void write_cluster_model(const ClusterModel &model, std::span<const std::uint64_t> request_ids,
                         std::ostream &out) {
    out << "K " << model.K << "\nE " << model.dim << "\nR " << model.labels.size() << '\n';
    for (std::uint32_t k = 0; k < model.K; ++k) {
        out << "centroid " << k;
        for (std::size_t c = 0; c < model.dim; ++c)
            out << ' ' << fmt_double(model.centroids[std::size_t(k) * model.dim + c], 17);
        out << '\n';
    }
    out << "labels";
    for (std::uint32_t l : model.labels) out << ' ' << l;
    out << "\nrequest_ids";
    for (std::uint64_t id : request_ids) out << ' ' << id;
    out << '\n';
}

StoredClusterModel parse_cluster_model(std::istream &in) {
    StoredClusterModel s;
    ClusterModel &m = s.model;
    std::size_t R = 0, line_no = 0;
    for (std::string line; std::getline(in, line);) {
        ++line_no;
        if (line.empty()) continue;
        std::istringstream ls(line);
        std::string key;
        ls >> key;
        if (key == "K") {
            ls >> m.K;
        } else if (key == "E") {
            ls >> m.dim;
        } else if (key == "R") {
            ls >> R;
        } else if (key == "centroid") {
            std::uint32_t k = 0;
            ls >> k;
            if (m.dim == 0 || k >= m.K)
                throw ParseError(line_no, "centroid line before header or k out of range");
            m.centroids.resize(std::max(m.centroids.size(), std::size_t(m.K) * m.dim), 0.0);
            double *row = m.centroids.data() + std::size_t(k) * m.dim;
            for (std::size_t c = 0; c < m.dim; ++c)
                if (!(ls >> row[c])) throw ParseError(line_no, "short centroid row");
        } else if (key == "labels") {
            for (std::uint32_t l; ls >> l;) m.labels.push_back(l);
        } else if (key == "request_ids") {
            for (std::uint64_t id; ls >> id;) s.request_ids.push_back(id);
        } else {
            throw ParseError(line_no, "unknown key '" + key + "'");
        }
        if (ls.fail() && !ls.eof())
            throw ParseError(line_no, "malformed value for key '" + key + "'");
    }
    if (m.K == 0 || m.dim == 0) throw ValidationError("cluster model: missing K/E header");
    if (m.labels.size() != R || s.request_ids.size() != R)
        throw ValidationError("cluster model: labels/request_ids length does not match R");
    for (std::uint32_t l : m.labels)
        if (l >= m.K) throw ValidationError("cluster model: label out of range");
    return s;
}

}  // namespace moeplace
