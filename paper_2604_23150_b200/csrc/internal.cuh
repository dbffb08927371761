// Internal declarations shared by the moeplace_b200 CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "moeplace_b200.h"

namespace mpb {

// Error bits raised by kernels into mpb_context::d_error.
enum : uint32_t {
    kErrExpertRange = 1u,  // expert id < 0 or >= E
    kErrSourceRange = 2u,  // source group >= D
    kErrUncovered = 4u,    // expert not held by any group of the placement
    kErrCapacity = 8u,     // a2a rows beyond a receive buffer's capacity
};

struct Status {
    mpb_status code;
    std::string what;
};

void set_error(const std::string &msg);
mpb_status fail(mpb_status code, const std::string &msg);
mpb_status cuda_fail(cudaError_t err, const char *where);

#define MPB_CUDA(call)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) return ::mpb::cuda_fail(e_, #call);                         \
    } while (0)

#define MPB_LAUNCHED(ctx)                                                                  \
    do {                                                                                   \
        (ctx)->launches++;                                                                 \
        cudaError_t e_ = cudaGetLastError();                                               \
        if (e_ != cudaSuccess) return ::mpb::cuda_fail(e_, "kernel launch");               \
    } while (0)

// Programmatic dependent launch: kernels launched with launch_pdl may start
// (prologue: smem zeroing, TMEM alloc, barrier init) while the previous kernel
// in the stream drains; each calls pdl_wait() before touching global data the
// previous kernels produce or read, and pdl_trigger() once every CTA is running.
// MPB_PDL=0 disables the attribute (the device calls are then no-ops).
bool pdl_enabled();

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace mpb

struct mpb_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;      // SM budget grids are sized for (<= device_sms)
    int device_sms = 148;
    // the stream's kernels are confined to num_sms SMs by the hardware (a
    // green-context partition): early (programmatic) launches cannot land on
    // SMs another context uses, so the router keeps PDL
    bool confined = false;
    uint32_t *d_error = nullptr;
    uint64_t launches = 0;
    // grow-only scratch (permutation block histograms, co-activation partials)
    void *scratch = nullptr;
    size_t scratch_bytes = 0;
    cudaError_t ensure_scratch(size_t bytes);
    // Grow-only workspace rule (scratch, router_ws): a CUDA graph captured
    // earlier may still reference the old buffer, so a grown buffer's
    // predecessor is retired (freed at mpb_context_destroy), never freed in
    // place; growing while the stream is capturing is refused
    // (cudaErrorStreamCaptureUnsupported): size the workspaces with one eager
    // call at the largest shape before capture.
    std::vector<void *> retired;
    cudaError_t grow(void **buf, size_t *bytes, size_t need, size_t min_bytes, size_t zero_bytes);
    // router split-K tail: fp32 partial accumulators + per-slot ready flags
    void *router_ws = nullptr;
    size_t router_ws_bytes = 0;
    void *pinned = nullptr;  // small pinned host area (k-means control values)
    size_t pinned_bytes = 0;
    // grouped router: device tables of TMA descriptors ([layer][X, W]), keyed by
    // (shape, tile width, X / W pointers); written once, reused by every later call
    std::map<std::vector<uint64_t>, void *> router_maps;
};

struct mpb_placement {
    mpb_context *ctx = nullptr;
    uint32_t D = 0, E = 0, nodes = 0, NS = 0;  // NS = number of (group, expert) slots
    uint8_t *d_dest_lut = nullptr;   // [nodes][E] destination group, 255 = uncovered
    uint16_t *d_slot_lut = nullptr;  // [nodes][E] slot id of (dest, e), 0xFFFF = uncovered
    uint16_t *d_key_lb = nullptr;    // [D*E + 1] first slot with key >= d*E+e
    uint16_t *d_cell_slot = nullptr; // [D][E] slot of a pair from source group s to expert e
    uint8_t *d_g2n = nullptr;        // [D]
    std::vector<uint8_t> h_dest_lut;
    std::vector<uint32_t> h_g2n;
};

namespace mpb {
// Kernel launchers (defined per .cu file); all async on ctx->stream.
mpb_status launch_layout(mpb_context *ctx, const mpb_tokens *tk, const mpb_placement *pl,
                         uint64_t *demand, uint64_t *demand2, uint64_t *tag_pop,
                         int32_t *sorted_pairs, int32_t *pair_pos, int64_t *key_offsets,
                         uint32_t layers = 1);
mpb_status score_finalize_range(mpb_context *ctx, const mpb_score_job &job, uint32_t b0, uint32_t nb);
mpb_status score_finalize_pair(mpb_context *ctx, const mpb_score_job &a, const mpb_score_job &b,
                               uint32_t b0, uint32_t nb);
mpb_status launch_layout_derive(mpb_context *ctx, const mpb_placement *pl, const uint64_t *demand,
                                uint64_t *expert_count, uint64_t *group_pairs,
                                uint64_t *node_demand, uint64_t *inter_intra);
}  // namespace mpb
