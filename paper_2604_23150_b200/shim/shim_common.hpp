// Shared plumbing of the C++ drop-in translation units (shim/*.cpp): status ->
// moeplace exception mapping, the process-wide device context and its
// grow-only device buffers. Every TU of the drop-in includes this header; the
// inline accessors give one context per process (C++17 inline-function
// statics are unique across translation units).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "moeplace/errors.hpp"
#include "moeplace_b200.h"

namespace moeplace::b200 {

// mpb_status -> the reference's exception class (errors.hpp:11-66). Parse
// errors arrive as "line N: what" and become ParseError(N, what).
[[noreturn]] inline void throw_status(mpb_status s, const std::string &what) {
    switch (s) {
    case MPB_PARSE_ERROR: {
        std::size_t line = 0, pos = 0;
        if (what.compare(0, 5, "line ") == 0) {
            pos = 5;
            while (pos < what.size() && what[pos] >= '0' && what[pos] <= '9')
                line = line * 10 + static_cast<std::size_t>(what[pos++] - '0');
            if (what.compare(pos, 2, ": ") == 0) throw ParseError(line, what.substr(pos + 2));
        }
        throw ParseError(line, what);
    }
    case MPB_VALIDATION_ERROR: throw ValidationError(what);
    case MPB_CONFIG_ERROR: throw ConfigError(what);
    case MPB_EMPTY_SELECTION_ERROR: throw EmptySelectionError(what);
    case MPB_UNDEFINED_CORRELATION_ERROR: throw UndefinedCorrelationError(what);
    case MPB_INFEASIBLE_ERROR: throw InfeasibleError(what);
    case MPB_LOOKUP_ERROR: throw LookupError(what);
    default: throw Error(what);
    }
}

inline void check(mpb_status s) {
    if (s != MPB_OK) throw_status(s, mpb_last_error_message());
}

inline void check_cuda(cudaError_t e, const char *where) {
    if (e != cudaSuccess) throw Error(std::string(where) + ": " + cudaGetErrorString(e));
}

// Process-wide device context + grow-only device buffers (slot-indexed). The
// drop-in's calls are synchronous (value semantics, like the reference), so
// the buffers are reused call to call; `mu` serialises callers that share the
// context from several threads.
struct Device {
    mpb_context *ctx = nullptr;
    std::vector<void *> bufs;
    std::vector<size_t> sizes;
    std::recursive_mutex mu;

    Device() { check(mpb_context_create(0, nullptr, &ctx)); }
    ~Device() {
        for (void *p : bufs) cudaFree(p);
        mpb_context_destroy(ctx);
    }
    void *buf(size_t slot, size_t bytes) {
        if (bufs.size() <= slot) {
            bufs.resize(slot + 1, nullptr);
            sizes.resize(slot + 1, 0);
        }
        bytes = std::max<size_t>(bytes, 64);
        if (sizes[slot] < bytes) {
            if (bufs[slot]) cudaFree(bufs[slot]);
            bufs[slot] = nullptr;
            check_cuda(cudaMalloc(&bufs[slot], bytes), "cudaMalloc");
            sizes[slot] = bytes;
        }
        return bufs[slot];
    }
    template <typename T> T *up(size_t slot, const T *h, size_t n) {
        auto *d = static_cast<T *>(buf(slot, n * sizeof(T)));
        if (n) check_cuda(cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice), "H2D");
        return d;
    }
    template <typename T> T *up(size_t slot, const std::vector<T> &h) {
        return up(slot, h.data(), h.size());
    }
    template <typename T> void down(T *h, const void *d, size_t n) {
        if (n) check_cuda(cudaMemcpy(h, d, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
    }
    template <typename T> void down(std::vector<T> &h, const void *d) { down(h.data(), d, h.size()); }
};

inline Device &device() {
    static Device d;
    return d;
}

// Buffer slots, disjoint per translation unit (the context is shared).
enum Slot : size_t {
    // simulator_b200.cpp
    kRowPtr, kCols, kVals, kRows, kPicks, kSrc, kG2n, kLuts, kDemand, kInter, kIntra, kRank, kOut,
    kPayload, kSetSize, kSetOff, kGroups, kRowNode,
    // metrics_b200.cpp
    kMetMatrix, kMetLabels, kMetSums,
    // clustering_b200.cpp
    kClRows, kClNorm, kClLabels, kClCentroids,
};

// Flattened groups (group d's ids follow group d-1's) + sizes, the C ABI form.
struct FlatGroups {
    std::vector<uint32_t> flat, sizes;
};

inline FlatGroups flatten(const std::vector<std::vector<uint32_t>> &groups) {
    FlatGroups f;
    f.sizes.reserve(groups.size());
    for (const auto &g : groups) {
        f.sizes.push_back(static_cast<uint32_t>(g.size()));
        f.flat.insert(f.flat.end(), g.begin(), g.end());
    }
    if (f.flat.empty()) f.flat.push_back(0);  // never dereferenced past the sizes
    return f;
}

}  // namespace moeplace::b200
