// Context, error plumbing and placement tables of the moeplace_b200 C ABI.
//
// Placement resolution restates simulate_layer's holder rule
// (/root/reference/proj/core/src/simulator.cpp:52-55, 74-80): holders of an
// expert ascend by group id; a token from node n goes to the first holder on
// node n, else to the lowest holder. The result is baked once per placement
// into a [nodes x E] destination table so every kernel resolves a pair with a
// single byte load.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"

namespace mpb {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string &msg) { g_last_error = msg; }

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("MPB_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

mpb_status fail(mpb_status code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

mpb_status cuda_fail(cudaError_t err, const char *where) {
    g_last_error = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(err);
    return MPB_CUDA_ERROR;
}

}  // namespace mpb

cudaError_t mpb_context::grow(void **buf, size_t *bytes, size_t need, size_t min_bytes,
                              size_t zero_bytes) {
    if (need <= *bytes) return cudaSuccess;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(stream, &cs);
    if (e != cudaSuccess) return e;
    if (cs != cudaStreamCaptureStatusNone) return cudaErrorStreamCaptureUnsupported;
    void *p = nullptr;
    const size_t want = std::max(need, min_bytes);
    e = cudaMalloc(&p, want);
    if (e != cudaSuccess) return e;
    if (zero_bytes) {
        e = cudaMemsetAsync(p, 0, std::min(zero_bytes, want), stream);
        if (e != cudaSuccess) {
            cudaFree(p);
            return e;
        }
    }
    if (*buf) retired.push_back(*buf);
    *buf = p;
    *bytes = want;
    return cudaSuccess;
}

cudaError_t mpb_context::ensure_scratch(size_t need) {
    return grow(&scratch, &scratch_bytes, need, size_t(1) << 20, 0);
}

using namespace mpb;

extern "C" {

int mpb_abi_version(void) { return MPB_ABI_VERSION; }

const char *mpb_last_error_message(void) { return g_last_error.c_str(); }

mpb_status mpb_context_create(int device, void *stream, mpb_context **out) {
    if (!out) return fail(MPB_VALIDATION_ERROR, "mpb_context_create: out is NULL");
    *out = nullptr;
    MPB_CUDA(cudaSetDevice(device));
    int major = 0, minor = 0;
    MPB_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    MPB_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (major != 10 || minor != 0)
        return fail(MPB_CONFIG_ERROR, "mpb_context_create: this build targets sm_100a (B200); "
                                      "device reports sm_" + std::to_string(major) +
                                          std::to_string(minor));
    auto *ctx = new mpb_context();
    ctx->device = device;
    ctx->stream = static_cast<cudaStream_t>(stream);
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    ctx->device_sms = ctx->num_sms;
    cudaError_t e = cudaMalloc(&ctx->d_error, sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(ctx->d_error, 0, sizeof(uint32_t));
    if (e != cudaSuccess) {
        delete ctx;
        return cuda_fail(e, "mpb_context_create");
    }
    *out = ctx;
    return MPB_OK;
}

mpb_status mpb_context_destroy(mpb_context *ctx) {
    if (!ctx) return MPB_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->d_error) cudaFree(ctx->d_error);
    if (ctx->scratch) cudaFree(ctx->scratch);
    if (ctx->router_ws) cudaFree(ctx->router_ws);
    for (void *p : ctx->retired) cudaFree(p);
    for (auto &kv : ctx->router_maps) cudaFree(kv.second);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    delete ctx;
    return MPB_OK;
}

mpb_status mpb_context_set_stream(mpb_context *ctx, void *stream) {
    if (!ctx) return fail(MPB_VALIDATION_ERROR, "mpb_context_set_stream: NULL context");
    ctx->stream = static_cast<cudaStream_t>(stream);
    return MPB_OK;
}

uint64_t mpb_context_launch_count(const mpb_context *ctx) { return ctx ? ctx->launches : 0; }

mpb_status mpb_context_set_sm_budget(mpb_context *ctx, uint32_t sms) {
    if (!ctx) return fail(MPB_VALIDATION_ERROR, "mpb_context_set_sm_budget: NULL context");
    ctx->confined = false;
    ctx->num_sms = sms == 0 ? ctx->device_sms
                            : static_cast<int>(std::min<uint32_t>(sms, ctx->device_sms));
    if (ctx->num_sms < 2) ctx->num_sms = 2;  // a router CTA pair
    return MPB_OK;
}

mpb_status mpb_context_sync(mpb_context *ctx) {
    if (!ctx) return fail(MPB_VALIDATION_ERROR, "mpb_context_sync: NULL context");
    uint32_t flags = 0;
    MPB_CUDA(cudaMemcpyAsync(&flags, ctx->d_error, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                             ctx->stream));
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (flags) {
        MPB_CUDA(cudaMemsetAsync(ctx->d_error, 0, sizeof(uint32_t), ctx->stream));
        MPB_CUDA(cudaStreamSynchronize(ctx->stream));
        std::string what = "simulate_layer:";
        if (flags & kErrSourceRange) what += " source group out of range;";
        if (flags & kErrExpertRange) what += " expert id out of range (>= E);";
        if (flags & kErrUncovered) what += " expert is not covered by the placement;";
        if (flags & kErrCapacity) what = "all-to-all: rows beyond the receive buffer capacity;";
        return fail(MPB_VALIDATION_ERROR, what);
    }
    return MPB_OK;
}

mpb_status mpb_build_dest_lut(const uint32_t *groups_flat, const uint32_t *group_sizes,
                              uint32_t D, uint32_t E, const uint32_t *group_to_node,
                              uint8_t *dest_lut) {
    if (!groups_flat || !group_sizes || !group_to_node || !dest_lut)
        return fail(MPB_VALIDATION_ERROR, "mpb_build_dest_lut: NULL argument");
    if (D == 0 || D > 255) return fail(MPB_CONFIG_ERROR, "placement: need 1 <= D <= 255");
    uint32_t nodes = 0;
    for (uint32_t d = 0; d < D; ++d) nodes = std::max(nodes, group_to_node[d] + 1);
    // holders[e] in ascending group order (simulator.cpp:52-55)
    std::vector<std::vector<uint32_t>> holders(E);
    size_t off = 0;
    for (uint32_t d = 0; d < D; ++d) {
        for (uint32_t i = 0; i < group_sizes[d]; ++i) {
            uint32_t e = groups_flat[off + i];
            if (e < E && (holders[e].empty() || holders[e].back() != d)) holders[e].push_back(d);
        }
        off += group_sizes[d];
    }
    for (uint32_t n = 0; n < nodes; ++n)
        for (uint32_t e = 0; e < E; ++e) {
            uint8_t dest = 255;
            if (!holders[e].empty()) {
                dest = static_cast<uint8_t>(holders[e][0]);
                for (uint32_t d : holders[e])
                    if (group_to_node[d] == n) {
                        dest = static_cast<uint8_t>(d);
                        break;
                    }
            }
            dest_lut[size_t(n) * E + e] = dest;
        }
    return MPB_OK;
}

mpb_status mpb_placement_create(mpb_context *ctx, const uint32_t *groups_flat,
                                const uint32_t *group_sizes, uint32_t D, uint32_t E,
                                const uint32_t *group_to_node, mpb_placement **out) {
    if (!ctx || !out) return fail(MPB_VALIDATION_ERROR, "mpb_placement_create: NULL argument");
    *out = nullptr;
    if (E == 0 || E > 65535) return fail(MPB_CONFIG_ERROR, "placement: need 1 <= E <= 65535");
    uint32_t nodes = 0;
    for (uint32_t d = 0; d < D; ++d) nodes = std::max(nodes, group_to_node[d] + 1);
    std::vector<uint8_t> lut(size_t(std::max(nodes, 1u)) * E);
    mpb_status st = mpb_build_dest_lut(groups_flat, group_sizes, D, E, group_to_node, lut.data());
    if (st != MPB_OK) return st;

    // Slots: one per (group, expert) held, ordered by (group, expert id): the
    // permutation's sort key. key_lb maps any key d*E+e to its first slot >= key.
    std::vector<std::vector<uint8_t>> held(D, std::vector<uint8_t>(E, 0));
    size_t off = 0;
    for (uint32_t d = 0; d < D; ++d) {
        for (uint32_t i = 0; i < group_sizes[d]; ++i)
            if (groups_flat[off + i] < E) held[d][groups_flat[off + i]] = 1;
        off += group_sizes[d];
    }
    std::vector<uint16_t> slot_of(size_t(D) * E, 0xFFFF), key_lb(size_t(D) * E + 1);
    uint32_t NS = 0;
    for (uint32_t d = 0; d < D; ++d)
        for (uint32_t e = 0; e < E; ++e) {
            key_lb[size_t(d) * E + e] = static_cast<uint16_t>(NS);
            if (held[d][e]) slot_of[size_t(d) * E + e] = static_cast<uint16_t>(NS++);
        }
    key_lb[size_t(D) * E] = static_cast<uint16_t>(NS);
    if (NS >= 0xFFFF) return fail(MPB_CONFIG_ERROR, "placement: too many (group, expert) slots");
    std::vector<uint16_t> slot_lut(lut.size());
    for (uint32_t n = 0; n < nodes; ++n)
        for (uint32_t e = 0; e < E; ++e) {
            uint8_t d = lut[size_t(n) * E + e];
            slot_lut[size_t(n) * E + e] = d == 255 ? 0xFFFF : slot_of[size_t(d) * E + e];
        }
    std::vector<uint8_t> g2n(D);
    for (uint32_t d = 0; d < D; ++d) g2n[d] = static_cast<uint8_t>(group_to_node[d]);
    std::vector<uint16_t> cell_slot(size_t(D) * E);
    for (uint32_t d = 0; d < D; ++d)
        for (uint32_t e = 0; e < E; ++e)
            cell_slot[size_t(d) * E + e] = slot_lut[size_t(group_to_node[d]) * E + e];

    auto *p = new mpb_placement();
    p->ctx = ctx;
    p->D = D;
    p->E = E;
    p->nodes = nodes;
    p->NS = NS;
    p->h_dest_lut = lut;
    p->h_g2n.assign(group_to_node, group_to_node + D);
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_dest_lut, lut.size());
    if (e == cudaSuccess) e = cudaMalloc(&p->d_slot_lut, slot_lut.size() * 2);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_key_lb, key_lb.size() * 2);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_g2n, D);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_cell_slot, cell_slot.size() * 2);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_cell_slot, cell_slot.data(), cell_slot.size() * 2,
                       cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_dest_lut, lut.data(), lut.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_slot_lut, slot_lut.data(), slot_lut.size() * 2, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_key_lb, key_lb.data(), key_lb.size() * 2, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(p->d_g2n, g2n.data(), D, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        mpb_placement_destroy(p);
        return cuda_fail(e, "mpb_placement_create");
    }
    *out = p;
    return MPB_OK;
}

mpb_status mpb_placement_destroy(mpb_placement *p) {
    if (!p) return MPB_OK;
    if (p->ctx) cudaSetDevice(p->ctx->device);
    cudaFree(p->d_dest_lut);
    cudaFree(p->d_slot_lut);
    cudaFree(p->d_key_lb);
    cudaFree(p->d_cell_slot);
    cudaFree(p->d_g2n);
    delete p;
    return MPB_OK;
}

const uint8_t *mpb_placement_dest_lut(const mpb_placement *p, uint32_t *nodes) {
    if (!p) return nullptr;
    if (nodes) *nodes = p->nodes;
    return p->d_dest_lut;
}

}  // extern "C"
