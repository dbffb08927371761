// Host finalisation of the characterisation metrics (metrics.cpp:11-68 of the
// reference) in its exact order of floating-point operations; compiled with
// -ffp-contract=off like the other host restatements. The column sums that
// feed them come from the device (metrics.cu, mpb_label_row_sums).
#include <cmath>
#include <cstdint>

#include "internal.cuh"

using namespace mpb;

extern "C" {

// expert_load (metrics.cpp:11-34): load_e = c_e / (sum / E) in that order;
// total = llround(sum / top_k).
mpb_status mpb_expert_load(const double *counts, uint32_t E, uint32_t top_k, double *loads,
                           uint64_t *total_tokens) {
    if (E == 0 || !counts) return fail(MPB_VALIDATION_ERROR, "expert_load: empty count vector");
    if (top_k == 0) return fail(MPB_VALIDATION_ERROR, "expert_load: top_k must be >= 1");
    double sum = 0.0;
    for (uint32_t e = 0; e < E; ++e) {
        if (counts[e] < 0.0) return fail(MPB_VALIDATION_ERROR, "expert_load: negative count");
        sum += counts[e];
    }
    if (sum == 0.0) return fail(MPB_VALIDATION_ERROR, "expert_load: all-zero counts, load undefined");
    const double share = sum / static_cast<double>(E);
    if (loads)
        for (uint32_t e = 0; e < E; ++e) loads[e] = counts[e] / share;
    if (total_tokens) *total_tokens = static_cast<uint64_t>(std::llround(sum / top_k));
    return MPB_OK;
}

// pearson (metrics.cpp:42-68): means first, then centred sums in index order,
// sxy / sqrt(sxx * syy) clamped to [-1, 1]; a constant vector is
// MPB_UNDEFINED_CORRELATION_ERROR.
mpb_status mpb_pearson(const double *x, const double *y, uint64_t n, double *r) {
    if (n < 2) return fail(MPB_VALIDATION_ERROR, "pearson: need at least 2 samples");
    if (!x || !y || !r) return fail(MPB_VALIDATION_ERROR, "pearson: NULL argument");
    double sx = 0.0, sy = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        sx += x[i];
        sy += y[i];
    }
    const double mx = sx / static_cast<double>(n), my = sy / static_cast<double>(n);
    double cxy = 0.0, cxx = 0.0, cyy = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double a = x[i] - mx, b = y[i] - my;
        cxy += a * b;
        cxx += a * a;
        cyy += b * b;
    }
    if (cxx == 0.0 || cyy == 0.0)
        return fail(MPB_UNDEFINED_CORRELATION_ERROR, "pearson: constant input vector");
    const double v = cxy / std::sqrt(cxx * cyy);
    *r = v < -1.0 ? -1.0 : (1.0 < v ? 1.0 : v);  // std::clamp semantics (NaN passes)
    return MPB_OK;
}

}  // extern "C"
