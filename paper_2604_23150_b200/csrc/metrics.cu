// Characterisation metrics behind the C ABI (metrics.cpp:11-132 of the
// reference): the per-label / all-row column sums that feed the dataset and
// prefill->decode correlations run on the device as exact integer
// histograms; the doubles (expert load, Pearson) are finalised on the host in
// the reference's order of operations (host_metrics.cpp).
//
// Exactness: the reference sums rows with sequential double additions
// (metrics.cpp:72-91). For integer-valued rows whose sums stay below 2^53
// (every trace-derived matrix: token counts) each of those additions is
// exact, so the sequential sum equals the integer sum in any order — the
// device accumulates uint64 and the host converts once. A non-integral or
// negative entry is flagged and reported as MPB_VALIDATION_ERROR so the caller
// can sum in the reference's order instead (none of the reference's callers
// produce one).
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "internal.cuh"

namespace mpb {
namespace {

constexpr int kLsThreads = 256;

// Block-privatised column sums per label: smem [n_labels][cols] u64 when it
// fits, else global atomics. Columns are the fast index (coalesced rows).
__global__ void k_label_sums(const double *__restrict__ M, uint64_t rows, uint32_t cols,
                             const uint32_t *__restrict__ labels, uint32_t n_labels,
                             uint64_t *__restrict__ out, int use_smem, uint32_t *err) {
    extern __shared__ unsigned long long s_acc[];
    const uint64_t cells = uint64_t(n_labels) * cols;
    if (use_smem)
        for (uint64_t i = threadIdx.x; i < cells; i += blockDim.x) s_acc[i] = 0;
    __syncthreads();
    const uint64_t total = rows * cols;
    bool bad = false;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t r = i / cols;
        const uint32_t c = static_cast<uint32_t>(i - r * cols);
        const double v = M[i];
        const uint32_t lab = labels ? labels[r] : 0u;
        if (!(v >= 0.0 && v < 9007199254740992.0 && v == floor(v)) || lab >= n_labels) {
            bad = true;
            continue;
        }
        const unsigned long long x = static_cast<unsigned long long>(v);
        if (x == 0) continue;
        if (use_smem)
            atomicAdd(&s_acc[uint64_t(lab) * cols + c], x);
        else
            atomicAdd(reinterpret_cast<unsigned long long *>(out) + uint64_t(lab) * cols + c, x);
    }
    if (bad) atomicOr(err, 1u);
    if (!use_smem) return;
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < cells; i += blockDim.x)
        if (s_acc[i]) atomicAdd(reinterpret_cast<unsigned long long *>(out) + i, s_acc[i]);
}

}  // namespace
}  // namespace mpb

using namespace mpb;

extern "C" {

mpb_status mpb_label_row_sums(mpb_context *ctx, const double *matrix, uint64_t rows, uint32_t cols,
                              const uint32_t *labels, uint32_t n_labels, uint64_t *sums) {
    if (!ctx || (rows && cols && (!matrix || !sums)))
        return fail(MPB_VALIDATION_ERROR, "mpb_label_row_sums: NULL argument");
    if (n_labels == 0) return fail(MPB_VALIDATION_ERROR, "mpb_label_row_sums: n_labels == 0");
    cudaStream_t st = ctx->stream;
    MPB_CUDA(cudaMemsetAsync(sums, 0, size_t(n_labels) * cols * 8, st));
    if (rows == 0 || cols == 0) return MPB_OK;
    const size_t cells = size_t(n_labels) * cols;
    const int use_smem = cells * 8 <= 96 * 1024;
    const size_t smem = use_smem ? cells * 8 : 0;
    if (use_smem)
        MPB_CUDA(cudaFuncSetAttribute(k_label_sums, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    const uint64_t total = rows * cols;
    const uint64_t want = (total + kLsThreads * 16 - 1) / (kLsThreads * 16);
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(
        1, std::min<uint64_t>(want, uint64_t(ctx->num_sms) * (use_smem ? 4 : 8))));
    k_label_sums<<<grid, kLsThreads, smem, st>>>(matrix, rows, cols, labels, n_labels, sums,
                                                 use_smem, ctx->d_error);
    MPB_LAUNCHED(ctx);
    uint32_t flag = 0;
    MPB_CUDA(cudaMemcpyAsync(&flag, ctx->d_error, 4, cudaMemcpyDeviceToHost, st));
    MPB_CUDA(cudaStreamSynchronize(st));
    if (flag) {
        MPB_CUDA(cudaMemsetAsync(ctx->d_error, 0, 4, st));
        return fail(MPB_VALIDATION_ERROR,
                    "mpb_label_row_sums: entries must be non-negative integers below 2^53 "
                    "(exact sums); label index out of range");
    }
    return MPB_OK;
}

}  // extern "C"
