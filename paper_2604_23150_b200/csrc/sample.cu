// On-device compare_strategies Monte-Carlo sampler.
//
// Restates, per batch b, the reference's per-batch streams
// (/root/reference/proj/core/src/simulator.cpp:115-118):
//   std::mt19937_64(std::seed_seq{seed, b, purpose})
// and libstdc++-13's uniform_int_distribution (Lemire's nearly-divisionless
// downscale through a 128-bit product, /usr/include/c++/13/bits/
// uniform_int_dist.h:257-280) — integer-only algorithms, so the device draws
// are bit-identical to the host. One thread per batch; the 312-word engine
// state lives in local memory.
#include "internal.cuh"

namespace mpb {
namespace {

constexpr int kN = 312, kM = 156;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull;

struct Mt64 {
    uint64_t mt[kN];
    int i;

    // std::seed_seq{v0, v1, v2}.generate(624 words) -> engine.seed(seq)
    __device__ void seed_seq3(uint64_t v0, uint64_t v1, uint64_t v2) {
        constexpr uint32_t n = 2 * kN, t = 11, p = (n - t) / 2, q = p + t;
        uint32_t *b = reinterpret_cast<uint32_t *>(mt);  // 624 words alias the state
        const uint32_t v[3] = {static_cast<uint32_t>(v0), static_cast<uint32_t>(v1),
                               static_cast<uint32_t>(v2)};
        const uint32_t s = 3;
        for (uint32_t k = 0; k < n; ++k) b[k] = 0x8b8b8b8bu;
        for (uint32_t k = 0; k < n; ++k) {  // m = max(s + 1, n) = n
            const uint32_t arg = b[k % n] ^ b[(k + p) % n] ^ b[(k + n - 1) % n];
            const uint32_t r1 = 1664525u * (arg ^ (arg >> 27));
            uint32_t r2;
            if (k == 0)
                r2 = r1 + s;
            else if (k <= s)
                r2 = r1 + k % n + v[k - 1];
            else
                r2 = r1 + k % n;
            b[(k + p) % n] += r1;
            b[(k + q) % n] += r2;
            b[k % n] = r2;
        }
        for (uint32_t k = n; k < 2 * n; ++k) {
            const uint32_t arg = b[k % n] + b[(k + p) % n] + b[(k + n - 1) % n];
            const uint32_t r3 = 1566083941u * (arg ^ (arg >> 27));
            const uint32_t r4 = r3 - k % n;
            b[(k + p) % n] ^= r3;
            b[(k + q) % n] ^= r4;
            b[k % n] = r4;
        }
        // little-endian aliasing already gives mt[i] = b[2i] | b[2i+1] << 32
        bool zero = (mt[0] & kUpper) == 0;
        for (int j = 1; zero && j < kN; ++j) zero = mt[j] == 0;
        if (zero) mt[0] = 1ull << 63;
        i = kN;
    }

    __device__ uint64_t next() {
        if (i >= kN) {
            for (int j = 0; j < kN; ++j) {
                const uint64_t y = (mt[j] & kUpper) | (mt[(j + 1) % kN] & kLower);
                uint64_t v = mt[(j + kM) % kN] ^ (y >> 1);
                if (y & 1ull) v ^= 0xB5026F5AA96619E9ull;
                mt[j] = v;
            }
            i = 0;
        }
        uint64_t z = mt[i++];
        z ^= (z >> 29) & 0x5555555555555555ull;
        z ^= (z << 17) & 0x71D67FFFEDA60000ull;
        z ^= (z << 37) & 0xFFF7EEE000000000ull;
        z ^= z >> 43;
        return z;
    }

    // uniform_int_distribution<>(0, range - 1) for a 64-bit engine (Lemire)
    __device__ uint64_t below(uint64_t range) {
        uint64_t x = next();
        uint64_t low = x * range;
        uint64_t high = __umul64hi(x, range);
        if (low < range) {
            const uint64_t threshold = (0ull - range) % range;
            while (low < threshold) {
                x = next();
                low = x * range;
                high = __umul64hi(x, range);
            }
        }
        return high;
    }
};

__global__ void k_sample(uint64_t seed, uint32_t B, uint32_t R, uint32_t S,
                         const uint32_t *set_size, uint32_t *rows, uint32_t *picks) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    Mt64 g;
    g.seed_seq3(seed, b, 1);
    uint32_t *rb = rows + static_cast<size_t>(b) * S;
    for (uint32_t i = 0; i < S; ++i) rb[i] = static_cast<uint32_t>(g.below(R));
    g.seed_seq3(seed, b, 2);
    uint32_t *pb = picks + static_cast<size_t>(b) * S;
    for (uint32_t i = 0; i < S; ++i) {
        const uint32_t n = set_size ? set_size[rb[i]] : 1u;
        pb[i] = n > 1 ? static_cast<uint32_t>(g.below(n)) : 0u;
    }
}

__global__ void k_route_sources(const uint32_t *rows, const uint32_t *picks, uint32_t B,
                                uint32_t S, const uint32_t *set_off, const uint32_t *groups,
                                uint32_t D, int cluster, uint8_t *src, uint32_t *err) {
    const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= static_cast<uint64_t>(B) * S) return;
    const uint32_t i = static_cast<uint32_t>(c % S);
    uint32_t g;
    if (cluster) {
        const uint32_t r = rows[c];
        const uint32_t lo = set_off[r], hi = set_off[r + 1];
        g = hi - lo == 1 ? groups[lo] : groups[lo + picks[c]];
    } else {
        g = i % D;  // baselines have no grouping notion (simulator.cpp:179)
    }
    if (g >= D) {
        atomicOr(err, kErrSourceRange);
        g = 0;
    }
    src[c] = static_cast<uint8_t>(g);
}

}  // namespace
}  // namespace mpb

using namespace mpb;

extern "C" {

mpb_status mpb_sample_batches(mpb_context *ctx, uint64_t seed, uint32_t B, uint32_t R, uint32_t S,
                              const uint32_t *set_size, uint32_t *rows, uint32_t *picks) {
    if (!ctx || !rows || !picks) return fail(MPB_VALIDATION_ERROR, "mpb_sample_batches: NULL argument");
    if (R == 0) return fail(MPB_VALIDATION_ERROR, "compare_strategies: empty decode matrix");
    if (B == 0 || S == 0)
        return fail(MPB_CONFIG_ERROR, "compare_strategies: batches and batch size must be >= 1");
    k_sample<<<(B + 63) / 64, 64, 0, ctx->stream>>>(seed, B, R, S, set_size, rows, picks);
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

mpb_status mpb_route_sources(mpb_context *ctx, const uint32_t *rows, const uint32_t *picks,
                             uint32_t B, uint32_t S, const uint32_t *set_off,
                             const uint32_t *groups, uint32_t D, int cluster_routed,
                             uint8_t *src) {
    if (!ctx || !rows || !src || (cluster_routed && (!picks || !set_off || !groups)))
        return fail(MPB_VALIDATION_ERROR, "mpb_route_sources: NULL argument");
    if (D == 0 || D > 255) return fail(MPB_CONFIG_ERROR, "mpb_route_sources: need 1 <= D <= 255");
    const uint64_t n = uint64_t(B) * S;
    if (n == 0) return MPB_OK;
    k_route_sources<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(
        rows, picks, B, S, set_off, groups, D, cluster_routed, src, ctx->d_error);
    MPB_LAUNCHED(ctx);
    return MPB_OK;
}

}  // extern "C"
