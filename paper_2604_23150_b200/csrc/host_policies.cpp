// Host-side placement and grouping policies behind the C ABI.
//
// These are the reference's policy interfaces (µs-to-ms host work that feeds
// the device scorer), restated in this library so every caller — the Python
// mirror, the C++ moeplace:: shim and bench.py — gets one implementation:
//   placement  linear / EPLB (LPT) / data-based (phase 1, phase 2, balance)
//              /root/reference/proj/core/src/placement.cpp:96-350
//   grouping   l2-normalised k-means++ / Lloyd, cluster sizes, cluster ->
//              group assignment  clustering.cpp:15-320
// Randomness uses std::mt19937_64 and the libstdc++ distributions exactly as
// the reference calls them, so results are bit-identical with the same
// standard library. Built with -ffp-contract=off (no FMA contraction), like
// the reference's default x86-64 build.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "internal.cuh"

namespace mpb {
namespace {

using Groups = std::vector<std::vector<uint32_t>>;

struct HostError {
    mpb_status code;
    std::string what;
};

[[noreturn]] void raise(mpb_status code, const std::string &what) { throw HostError{code, what}; }

template <typename F>
mpb_status guard(F &&f) {
    try {
        f();
        return MPB_OK;
    } catch (const HostError &e) {
        return fail(e.code, e.what);
    } catch (const std::exception &e) {
        return fail(MPB_ERROR, e.what());
    }
}

void verify_placement(const Groups &groups, uint32_t E, uint32_t M) {
    std::vector<char> covered(E, 0);
    for (size_t d = 0; d < groups.size(); ++d) {
        if (groups[d].size() != M)
            raise(MPB_VALIDATION_ERROR, "placement: group " + std::to_string(d) + " has " +
                                            std::to_string(groups[d].size()) +
                                            " experts, expected M=" + std::to_string(M));
        std::set<uint32_t> uniq(groups[d].begin(), groups[d].end());
        if (uniq.size() != groups[d].size())
            raise(MPB_VALIDATION_ERROR, "placement: duplicate expert within group " + std::to_string(d));
        for (uint32_t e : groups[d]) {
            if (e >= E) raise(MPB_VALIDATION_ERROR, "placement: expert id " + std::to_string(e) + " >= E");
            covered[e] = 1;
        }
    }
    for (uint32_t e = 0; e < E; ++e)
        if (!covered[e])
            raise(MPB_VALIDATION_ERROR, "placement: expert " + std::to_string(e) +
                                            " is not placed in any group");
}

void write_groups(const Groups &g, uint32_t *flat, uint32_t *sizes) {
    size_t o = 0;
    for (size_t d = 0; d < g.size(); ++d) {
        if (sizes) sizes[d] = static_cast<uint32_t>(g[d].size());
        for (uint32_t e : g[d]) flat[o++] = e;
    }
}

Groups read_groups(const uint32_t *flat, const uint32_t *sizes, uint32_t D) {
    Groups g(D);
    size_t o = 0;
    for (uint32_t d = 0; d < D; ++d) {
        g[d].assign(flat + o, flat + o + sizes[d]);
        o += sizes[d];
    }
    return g;
}

// ---- placement policies (placement.cpp:127-350) -------------------------------

Groups phase1(const double *U, uint32_t D, uint32_t E) {
    if (D < 1 || E < D) raise(MPB_INFEASIBLE_ERROR, "phase1: requires E >= D >= 1");
    const uint32_t cap = (E + D - 1) / D;
    std::vector<double> imp(E, 0.0);
    for (uint32_t e = 0; e < E; ++e)
        for (uint32_t d = 0; d < D; ++d) imp[e] = std::max(imp[e], U[size_t(d) * E + e]);
    std::vector<uint32_t> order(E);
    std::iota(order.begin(), order.end(), 0u);
    std::stable_sort(order.begin(), order.end(),
                     [&](uint32_t a, uint32_t b) { return imp[a] > imp[b]; });
    Groups groups(D);
    std::vector<uint32_t> pref(D);
    for (uint32_t e : order) {
        std::iota(pref.begin(), pref.end(), 0u);
        std::stable_sort(pref.begin(), pref.end(), [&](uint32_t a, uint32_t b) {
            return U[size_t(a) * E + e] > U[size_t(b) * E + e];
        });
        for (uint32_t d : pref)
            if (groups[d].size() < cap) {
                groups[d].push_back(e);
                break;
            }
    }
    return groups;
}

void phase2(Groups &groups, const double *U, uint32_t E, uint32_t M) {
    for (size_t d = 0; d < groups.size(); ++d) {
        auto &g = groups[d];
        if (g.size() > M) raise(MPB_INFEASIBLE_ERROR, "phase2: group " + std::to_string(d) + " already above M");
        const size_t need = M - g.size();
        if (!need) continue;
        std::vector<char> in(E, 0);
        for (uint32_t e : g)
            if (e < E) in[e] = 1;  // ids >= E are never candidates anyway
        std::vector<uint32_t> cand;
        for (uint32_t e = 0; e < E; ++e)
            if (!in[e]) cand.push_back(e);
        if (need > cand.size())
            raise(MPB_INFEASIBLE_ERROR, "phase2: group " + std::to_string(d) + " needs " +
                                            std::to_string(need) + " experts but only " +
                                            std::to_string(cand.size()) + " candidates (M > E)");
        std::stable_sort(cand.begin(), cand.end(), [&](uint32_t a, uint32_t b) {
            return U[d * E + a] > U[d * E + b];
        });
        g.insert(g.end(), cand.begin(), cand.begin() + static_cast<std::ptrdiff_t>(need));
    }
}

Groups balance(Groups groups, uint32_t E, uint32_t M, uint64_t seed) {
    const uint32_t D = static_cast<uint32_t>(groups.size());
    if (D == 0) raise(MPB_INFEASIBLE_ERROR, "balance_and_verify: no groups");
    std::mt19937_64 rng(seed);
    std::vector<uint32_t> copies(E, 0);
    for (const auto &g : groups)
        for (uint32_t e : g) {
            if (e >= E) raise(MPB_VALIDATION_ERROR, "balance_and_verify: expert id out of range");
            ++copies[e];
        }
    for (auto &g : groups) {
        std::vector<char> seen(E, 0);
        std::vector<uint32_t> kept;
        kept.reserve(g.size());
        for (uint32_t e : g) {  // later duplicates inside a group go first
            if (seen[e]) {
                --copies[e];
                continue;
            }
            seen[e] = 1;
            kept.push_back(e);
        }
        g.swap(kept);
        while (g.size() > M) {  // trim the least-used tail, never a sole copy
            size_t i = g.size();
            while (i > 0 && copies[g[i - 1]] <= 1) --i;
            if (i == 0)
                raise(MPB_VALIDATION_ERROR, "balance_and_verify: oversized group holds only sole-copy experts");
            --copies[g[i - 1]];
            g.erase(g.begin() + static_cast<std::ptrdiff_t>(i - 1));
        }
    }
    for (uint32_t e = 0; e < E; ++e) {
        if (copies[e]) continue;
        std::vector<uint32_t> open;
        for (uint32_t d = 0; d < D; ++d)
            if (groups[d].size() < M) open.push_back(d);
        if (open.empty())
            raise(MPB_VALIDATION_ERROR, "balance_and_verify: expert " + std::to_string(e) +
                                            " missing but no group has a free slot");
        const uint32_t d = open[std::uniform_int_distribution<std::size_t>(0, open.size() - 1)(rng)];
        groups[d].push_back(e);
        ++copies[e];
    }
    for (uint32_t d = 0; d < D; ++d) {
        auto &g = groups[d];
        while (g.size() < M) {
            std::vector<char> in(E, 0);
            for (uint32_t e : g) in[e] = 1;
            std::vector<uint32_t> cand;
            for (uint32_t e = 0; e < E; ++e)
                if (!in[e]) cand.push_back(e);
            if (cand.empty())
                raise(MPB_INFEASIBLE_ERROR, "balance_and_verify: M > E, cannot fill group " + std::to_string(d));
            const uint32_t e = cand[std::uniform_int_distribution<std::size_t>(0, cand.size() - 1)(rng)];
            g.push_back(e);
            ++copies[e];
        }
    }
    verify_placement(groups, E, M);
    return groups;
}

// ---- k-means grouping (clustering.cpp:15-230) -----------------------------------

double sqdist(const double *a, const double *b, size_t dim) {
    double s = 0.0;
    for (size_t i = 0; i < dim; ++i) {
        const double d = a[i] - b[i];
        s += d * d;
    }
    return s;
}

struct KMeans {
    std::vector<uint32_t> labels;
    std::vector<double> centroids;
    double objective = 0.0;
    uint32_t iterations = 0;
    std::vector<double> history;  // objective after each Lloyd iteration
};

void assign(const double *X, size_t n, size_t dim, const std::vector<double> &C, uint32_t K,
            std::vector<uint32_t> &labels) {
    for (size_t i = 0; i < n; ++i) {
        double best = std::numeric_limits<double>::infinity();
        uint32_t bk = 0;
        for (uint32_t k = 0; k < K; ++k) {
            const double d = sqdist(X + i * dim, C.data() + size_t(k) * dim, dim);
            if (d < best) {
                best = d;
                bk = k;
            }
        }
        labels[i] = bk;
    }
}

void repair(const double *X, size_t n, size_t dim, std::vector<double> &C, uint32_t K,
            std::vector<uint32_t> &labels) {
    std::vector<size_t> size(K, 0);
    for (uint32_t l : labels) ++size[l];
    for (uint32_t k = 0; k < K; ++k) {
        if (size[k]) continue;
        double worst = -1.0;
        size_t victim = n;
        for (size_t i = 0; i < n; ++i) {
            if (size[labels[i]] <= 1) continue;
            const double d = sqdist(X + i * dim, C.data() + size_t(labels[i]) * dim, dim);
            if (d > worst) {
                worst = d;
                victim = i;
            }
        }
        if (victim == n) raise(MPB_INFEASIBLE_ERROR, "kmeans: cannot repair empty cluster");
        --size[labels[victim]];
        labels[victim] = k;
        size[k] = 1;
        std::copy(X + victim * dim, X + (victim + 1) * dim, C.begin() + size_t(k) * dim);
    }
}

double objective(const double *X, size_t n, size_t dim, const std::vector<double> &C,
                 const std::vector<uint32_t> &labels) {
    double t = 0.0;
    for (size_t i = 0; i < n; ++i) t += sqdist(X + i * dim, C.data() + size_t(labels[i]) * dim, dim);
    return t;
}

KMeans kmeans(const double *X, size_t n, size_t dim, uint32_t K, uint64_t seed, uint32_t max_iter,
              double tol) {
    if (K < 1) raise(MPB_INFEASIBLE_ERROR, "kmeans: K must be >= 1");
    if (n < K)
        raise(MPB_INFEASIBLE_ERROR, "kmeans: " + std::to_string(n) + " rows < K=" + std::to_string(K));
    std::mt19937_64 rng(seed);
    KMeans m;
    // k-means++ seeding
    std::vector<char> used(n, 0);
    const size_t first = std::uniform_int_distribution<std::size_t>(0, n - 1)(rng);
    used[first] = 1;
    m.centroids.assign(X + first * dim, X + (first + 1) * dim);
    std::vector<double> dmin(n);
    for (size_t i = 0; i < n; ++i) dmin[i] = sqdist(X + i * dim, X + first * dim, dim);
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    for (uint32_t k = 1; k < K; ++k) {
        double total = 0.0;
        for (double v : dmin) total += v;
        size_t pick = n;
        if (total > 0.0) {
            const double target = unit(rng) * total;
            double cum = 0.0;
            for (size_t i = 0; i < n; ++i) {
                cum += dmin[i];
                if (cum >= target) {
                    pick = i;
                    break;
                }
            }
            if (pick == n) pick = n - 1;
        } else {
            for (size_t i = 0; i < n && pick == n; ++i)
                if (!used[i]) pick = i;
            if (pick == n) pick = 0;
        }
        used[pick] = 1;
        m.centroids.insert(m.centroids.end(), X + pick * dim, X + (pick + 1) * dim);
        for (size_t i = 0; i < n; ++i)
            dmin[i] = std::min(dmin[i], sqdist(X + i * dim, X + pick * dim, dim));
    }
    m.labels.assign(n, 0);
    std::vector<double> prev, sums(size_t(K) * dim);
    std::vector<size_t> cnt(K);
    uint32_t it = 0;
    for (; it < max_iter; ++it) {
        assign(X, n, dim, m.centroids, K, m.labels);
        repair(X, n, dim, m.centroids, K, m.labels);
        prev = m.centroids;
        std::fill(sums.begin(), sums.end(), 0.0);
        std::fill(cnt.begin(), cnt.end(), 0);
        for (size_t i = 0; i < n; ++i) {
            double *acc = sums.data() + size_t(m.labels[i]) * dim;
            for (size_t c = 0; c < dim; ++c) acc[c] += X[i * dim + c];
            ++cnt[m.labels[i]];
        }
        for (uint32_t k = 0; k < K; ++k)
            for (size_t c = 0; c < dim; ++c)
                m.centroids[size_t(k) * dim + c] = sums[size_t(k) * dim + c] / static_cast<double>(cnt[k]);
        m.history.push_back(objective(X, n, dim, m.centroids, m.labels));
        double move = 0.0;
        for (uint32_t k = 0; k < K; ++k)
            move = std::max(move, std::sqrt(sqdist(m.centroids.data() + size_t(k) * dim,
                                                   prev.data() + size_t(k) * dim, dim)));
        if (move < tol) {
            ++it;
            break;
        }
    }
    m.iterations = it;
    assign(X, n, dim, m.centroids, K, m.labels);
    repair(X, n, dim, m.centroids, K, m.labels);
    m.objective = objective(X, n, dim, m.centroids, m.labels);
    return m;
}

std::vector<double> cluster_sizes(const uint32_t *labels, size_t n, const double *raw, size_t dim,
                                  uint32_t K) {
    std::vector<double> s(K, 0.0);
    for (size_t r = 0; r < n; ++r) {
        double l1 = 0.0;
        for (size_t c = 0; c < dim; ++c) l1 += std::abs(raw[r * dim + c]);
        s[labels[r]] += l1;
    }
    return s;
}

Groups assign_groups(const uint32_t *labels, size_t n, uint32_t K, const double *raw, size_t dim,
                     uint32_t D, uint64_t seed) {
    if (D < 1) raise(MPB_INFEASIBLE_ERROR, "assign_clusters_to_groups: D must be >= 1");
    const auto size = cluster_sizes(labels, n, raw, dim, K);
    Groups a(K);
    if (K == D) {
        for (uint32_t k = 0; k < K; ++k) a[k] = {k};
        return a;
    }
    if (D > K) {
        std::vector<uint32_t> order(K);
        std::iota(order.begin(), order.end(), 0u);
        std::stable_sort(order.begin(), order.end(),
                         [&](uint32_t x, uint32_t y) { return size[x] > size[y]; });
        for (uint32_t g = 0; g < D; ++g) a[order[g % K]].push_back(g);
        for (auto &v : a) std::sort(v.begin(), v.end());
        return a;
    }
    std::vector<double> u(size_t(K) * dim, 0.0);
    for (size_t r = 0; r < n; ++r)
        for (size_t c = 0; c < dim; ++c) u[size_t(labels[r]) * dim + c] += raw[r * dim + c];
    const KMeans meta = kmeans(u.data(), K, dim, D, seed, 100, 1e-6);
    std::vector<std::vector<uint32_t>> members(D);
    for (uint32_t k = 0; k < K; ++k) {
        a[k] = {meta.labels[k]};
        members[meta.labels[k]].push_back(k);
    }
    for (uint32_t g = 0; g < D; ++g) {
        if (!members[g].empty()) continue;
        uint32_t donor = 0;
        for (uint32_t d = 1; d < D; ++d)
            if (members[d].size() > members[donor].size()) donor = d;
        if (members[donor].size() < 2)
            raise(MPB_INFEASIBLE_ERROR, "assign_clusters_to_groups: cannot repair empty group");
        uint32_t stolen = members[donor][0];
        for (uint32_t k : members[donor])
            if (size[k] > size[stolen]) stolen = k;
        members[donor].erase(std::find(members[donor].begin(), members[donor].end(), stolen));
        members[g].push_back(stolen);
        a[stolen] = {g};
    }
    return a;
}

}  // namespace
}  // namespace mpb

using namespace mpb;

extern "C" {

mpb_status mpb_linear_placement(uint32_t E, uint32_t D, uint32_t *groups_out) {
    return guard([&] {
        if (D == 0 || E % D != 0)
            raise(MPB_CONFIG_ERROR, "linear_placement: D must divide E (E=" + std::to_string(E) +
                                        ", D=" + std::to_string(D) + ")");
        for (uint32_t e = 0; e < E; ++e) groups_out[e] = e;
    });
}

mpb_status mpb_eplb_placement(const double *load, uint32_t E, uint32_t D, uint32_t *groups_out) {
    return guard([&] {
        if (D == 0 || E % D != 0)
            raise(MPB_CONFIG_ERROR, "eplb_placement: D must divide E (E=" + std::to_string(E) +
                                        ", D=" + std::to_string(D) + ")");
        const uint32_t per = E / D;
        std::vector<uint32_t> order(E);
        std::iota(order.begin(), order.end(), 0u);
        std::stable_sort(order.begin(), order.end(),
                         [&](uint32_t a, uint32_t b) { return load[a] > load[b]; });
        Groups g(D);
        std::vector<double> gl(D, 0.0);
        for (uint32_t e : order) {
            uint32_t best = D;
            for (uint32_t d = 0; d < D; ++d)
                if (g[d].size() < per && (best == D || gl[d] < gl[best])) best = d;
            g[best].push_back(e);
            gl[best] += load[e];
        }
        verify_placement(g, E, per);
        write_groups(g, groups_out, nullptr);
    });
}

mpb_status mpb_phase1_unique_distribution(const double *usage, uint32_t D, uint32_t E,
                                          uint32_t *groups_out, uint32_t *sizes_out) {
    return guard([&] { write_groups(phase1(usage, D, E), groups_out, sizes_out); });
}

mpb_status mpb_phase2_redundant_addition(const uint32_t *groups_in, const uint32_t *sizes_in,
                                         const double *usage, uint32_t D, uint32_t E, uint32_t M,
                                         uint32_t *groups_out) {
    return guard([&] {
        Groups g = read_groups(groups_in, sizes_in, D);
        phase2(g, usage, E, M);
        write_groups(g, groups_out, nullptr);
    });
}

mpb_status mpb_balance_and_verify(const uint32_t *groups_in, const uint32_t *sizes_in, uint32_t D,
                                  uint32_t E, uint32_t M, uint64_t seed, uint32_t *groups_out) {
    return guard([&] {
        write_groups(balance(read_groups(groups_in, sizes_in, D), E, M, seed), groups_out, nullptr);
    });
}

mpb_status mpb_data_based_placement(const double *usage, uint32_t D, uint32_t E, uint32_t R,
                                    uint64_t seed, uint32_t *groups_out) {
    return guard([&] {
        if (D == 0 || (E + R) % D != 0)
            raise(MPB_CONFIG_ERROR, "data_based_placement: (E + R) = " + std::to_string(E + R) +
                                        " not divisible by D = " + std::to_string(D));
        const uint32_t M = (E + R) / D;
        Groups g = phase1(usage, D, E);
        phase2(g, usage, E, M);
        write_groups(balance(std::move(g), E, M, seed), groups_out, nullptr);
    });
}

mpb_status mpb_aggregate_usage(const uint32_t *labels, const double *matrix, uint64_t rows,
                               uint32_t E, uint32_t K, const uint32_t *assign_flat,
                               const uint32_t *assign_sizes, uint32_t D, double *usage_out) {
    return guard([&] {
        std::vector<double> tot(size_t(K) * E, 0.0);
        for (uint64_t r = 0; r < rows; ++r) {
            if (labels[r] >= K) raise(MPB_VALIDATION_ERROR, "aggregate_usage: label out of range");
            double *acc = tot.data() + size_t(labels[r]) * E;
            for (uint32_t e = 0; e < E; ++e) acc[e] += matrix[r * E + e];
        }
        std::fill(usage_out, usage_out + size_t(D) * E, 0.0);
        size_t o = 0;
        for (uint32_t k = 0; k < K; ++k) {
            for (uint32_t i = 0; i < assign_sizes[k]; ++i) {
                const uint32_t d = assign_flat[o + i];
                if (d >= D) raise(MPB_VALIDATION_ERROR, "aggregate_usage: group id out of range");
                for (uint32_t e = 0; e < E; ++e) usage_out[size_t(d) * E + e] += tot[size_t(k) * E + e];
            }
            o += assign_sizes[k];
        }
    });
}

mpb_status mpb_l2_normalize_rows(const double *matrix, uint64_t rows, uint32_t cols, double *out) {
    return guard([&] {
        for (uint64_t r = 0; r < rows; ++r) {
            const double *a = matrix + r * cols;
            double ss = 0.0;
            for (uint32_t c = 0; c < cols; ++c) ss += a[c] * a[c];
            if (ss == 0.0) raise(MPB_VALIDATION_ERROR, "l2_normalize: zero vector");
            const double inv = 1.0 / std::sqrt(ss);
            for (uint32_t c = 0; c < cols; ++c) out[r * cols + c] = a[c] * inv;
        }
    });
}

mpb_status mpb_kmeans(const double *rows, uint64_t n, uint32_t dim, uint32_t K, uint64_t seed,
                      uint32_t max_iterations, double tolerance, uint32_t *labels_out,
                      double *centroids_out, double *objective_out, uint32_t *iterations_out,
                      double *objective_history) {
    return guard([&] {
        KMeans m = kmeans(rows, n, dim, K, seed, max_iterations, tolerance);
        std::copy(m.labels.begin(), m.labels.end(), labels_out);
        if (centroids_out) std::copy(m.centroids.begin(), m.centroids.end(), centroids_out);
        if (objective_out) *objective_out = m.objective;
        if (iterations_out) *iterations_out = m.iterations;
        if (objective_history) std::copy(m.history.begin(), m.history.end(), objective_history);
    });
}

mpb_status mpb_placement_verify(const uint32_t *groups_flat, const uint32_t *group_sizes,
                                uint32_t D, uint32_t E, uint32_t M) {
    return guard([&] {
        if (D && (!groups_flat || !group_sizes))
            raise(MPB_VALIDATION_ERROR, "mpb_placement_verify: NULL argument");
        verify_placement(D ? read_groups(groups_flat, group_sizes, D) : Groups{}, E, M);
    });
}

mpb_status mpb_assign_clusters_to_groups(const uint32_t *labels, uint64_t n, uint32_t K,
                                         const double *raw, uint32_t dim, uint32_t D,
                                         uint64_t seed, uint32_t *assign_flat,
                                         uint32_t *assign_sizes, double *cluster_sizes_out) {
    return guard([&] {
        for (uint64_t r = 0; r < n; ++r)
            if (labels[r] >= K) raise(MPB_VALIDATION_ERROR, "assign_clusters_to_groups: label out of range");
        Groups a = assign_groups(labels, n, K, raw, dim, D, seed);
        write_groups(a, assign_flat, assign_sizes);
        if (cluster_sizes_out) {
            auto s = cluster_sizes(labels, n, raw, dim, K);
            std::copy(s.begin(), s.end(), cluster_sizes_out);
        }
    });
}

}  // extern "C"
