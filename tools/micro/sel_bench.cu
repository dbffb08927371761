// Micro-benchmark of the cluster tail's top-k (router.cu tail_select) in isolation: 148 CTAs x
// 384 threads, warps 4-11 select top-8 of 32 rows x 128 fp32 logits from shared memory
// (one warp per row, presorted lane lists, redux.sync max + ballot per round); compare
// tools/micro/epi_bench.cu (the per-thread insertion + shuffle merge it replaced).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/sel_bench tools/micro/sel_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int N = 128, KMAX = 8, RPS = 32, RS = N + 4, R = 4, V = N / 32;
__device__ __forceinline__ uint32_t rank_key(float v) {
    uint32_t b = __float_as_uint(v);
    b = b == 0x80000000u ? 0u : b;
    const uint32_t k = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return v != v ? 1u : k;
}
__device__ __forceinline__ float key_value(uint32_t key) {
    return key == 1u ? __uint_as_float(0x7FC00000u) : __uint_as_float((key & 0x80000000u) ? (key & 0x7FFFFFFFu) : ~key);
}
// compare-exchange on (key, slot) descending; equal keys keep the lower slot first
__device__ __forceinline__ void cx(uint32_t &ka, uint32_t &sa, uint32_t &kb, uint32_t &sb) {
    const bool sw = kb > ka || (kb == ka && sb < sa);
    const uint32_t k0 = sw ? kb : ka, k1 = sw ? ka : kb, s0 = sw ? sb : sa, s1 = sw ? sa : sb;
    ka = k0; kb = k1; sa = s0; sb = s1;
}
template <int MODE>
__global__ void __launch_bounds__(384, 1) k(const float *src, int *out_i, float *out_w, long long *cyc, uint32_t E, uint32_t kk, int renorm) {
    __shared__ __align__(16) float tile[RPS * RS];
    for (int i = threadIdx.x; i < RPS * N; i += blockDim.x) tile[(i / N) * RS + i % N] = src[blockIdx.x * RPS * N + i];
    __syncthreads();
    if (threadIdx.x < 128) return;
    const uint32_t t = threadIdx.x - 128, ew = t / 32, lane = t % 32;
    long long c0 = clock64();
    uint32_t key[R][V], sl[R][V];
    float x[R][V];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int i = 0; i < V; ++i) {
            x[r][i] = tile[(ew + 8 * r) * RS + lane + 32 * i];
            key[r][i] = lane + 32u * i < E ? rank_key(x[r][i]) : 0u;
            sl[r][i] = i;
        }
    // presort each lane's V keys descending (V = 4: 5 compare-exchanges)
#pragma unroll
    for (int r = 0; r < R; ++r) {
        cx(key[r][0], sl[r][0], key[r][1], sl[r][1]);
        cx(key[r][2], sl[r][2], key[r][3], sl[r][3]);
        cx(key[r][0], sl[r][0], key[r][2], sl[r][2]);
        cx(key[r][1], sl[r][1], key[r][3], sl[r][3]);
        cx(key[r][1], sl[r][1], key[r][2], sl[r][2]);
    }
    long long c1 = clock64();
    uint32_t skey[R], sid[R], mkey[R];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        if ((uint32_t)j >= kk) break;
        uint32_t km[R], b[R];
#pragma unroll
        for (int r = 0; r < R; ++r) km[r] = __reduce_max_sync(0xffffffffu, key[r][0]);
        bool tie = false;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            b[r] = __ballot_sync(0xffffffffu, key[r][0] == km[r]);
            tie |= __popc(b[r]) != 1;
        }
        if (tie) {  // equal keys at several lane heads: the lowest column id (slot first, then lane)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t ms = __reduce_min_sync(0xffffffffu, key[r][0] == km[r] ? sl[r][0] : 0xffu);
                b[r] = __ballot_sync(0xffffffffu, key[r][0] == km[r] && sl[r][0] == ms);
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t wl = __ffs(b[r]) - 1;
            const uint32_t id = __shfl_sync(0xffffffffu, lane + 32u * sl[r][0], wl);
            if (j == 0) mkey[r] = km[r];
            skey[r] = lane == (uint32_t)j ? km[r] : skey[r];
            sid[r] = lane == (uint32_t)j ? id : sid[r];
            const bool pop = lane == wl;
#pragma unroll
            for (int i = 0; i < V - 1; ++i) {
                key[r][i] = pop ? key[r][i + 1] : key[r][i];
                sl[r][i] = pop ? sl[r][i + 1] : sl[r][i];
            }
            key[r][V - 1] = pop ? 0u : key[r][V - 1];
        }
    }
    long long c2 = clock64();
    float ssum[R], tsum[R], e[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const float m = mkey[r] <= 1u ? -INFINITY : key_value(mkey[r]);
        const float mlog = m * 1.4426950408889634f;
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < V; ++i) { const float v = x[r][i]; s += (lane + 32u * i < E && v == v) ? exp2f(fmaf(v, 1.4426950408889634f, -mlog)) : 0.f; }
        ssum[r] = s;
        const float v = key_value(skey[r]);
        e[r] = (lane < kk && !isnan(v)) ? exp2f(fmaf(v, 1.4426950408889634f, -mlog)) : 0.f;
        tsum[r] = e[r];
    }
#pragma unroll
    for (uint32_t o = 16; o >= 1; o >>= 1)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            ssum[r] += __shfl_xor_sync(0xffffffffu, ssum[r], o);
            tsum[r] += __shfl_xor_sync(0xffffffffu, tsum[r], o);
        }
#pragma unroll
    for (int r = 0; r < R; ++r)
        if (lane < kk) {
            const uint32_t o = (blockIdx.x * RPS + ew + 8 * r) * kk + lane;
            out_i[o] = sid[r];
            out_w[o] = renorm ? (tsum[r] > 0.f ? e[r] / tsum[r] : 0.f) : e[r] / ssum[r];
        }
    long long c3 = clock64();
    if (blockIdx.x == 0 && t == 0) { cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; }
}
template <int MODE> void run(const float *src, int *oi, float *ow, long long *cyc, const float *h) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int it = 0; it < 3; ++it) k<MODE><<<148, 384>>>(src, oi, ow, cyc, N, KMAX, 1);
    cudaEventRecord(a);
    for (int it = 0; it < 20; ++it) k<MODE><<<148, 384>>>(src, oi, ow, cyc, N, KMAX, 1);
    cudaEventRecord(b); cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, a, b);
    int *hi = new int[148 * RPS * KMAX]; cudaMemcpy(hi, oi, 148 * RPS * KMAX * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int row = 0; row < 148 * RPS; ++row) {
        const float *x = h + row * N; int sel[KMAX]; bool used[N] = {};
        for (int j = 0; j < KMAX; ++j) { int bi = -1; for (int c = 0; c < N; ++c) if (!used[c] && (bi < 0 || x[c] > x[bi])) bi = c; used[bi] = true; sel[j] = bi; }
        for (int j = 0; j < KMAX; ++j) bad += sel[j] != hi[row * KMAX + j];
    }
    printf("sel mode %d: kernel %.2f us/launch; cycles load+presort %lld select %lld weights %lld; mismatches %d (%s)\n", MODE, ms / 20 * 1e3, cyc[0], cyc[1], cyc[2], bad, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    const int B = 148; float *src; int *oi; float *ow; long long *cyc;
    cudaMalloc(&src, B * RPS * N * 4); cudaMalloc(&oi, B * RPS * KMAX * 4); cudaMalloc(&ow, B * RPS * KMAX * 4);
    cudaMallocManaged(&cyc, 8 * 8);
    float *h = new float[B * RPS * N]; unsigned s = 1;
    for (int i = 0; i < B * RPS * N; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) * (1.0f / 16777216.0f) - 0.5f; }
    cudaMemcpy(src, h, B * RPS * N * 4, cudaMemcpyHostToDevice);
    run<0>(src, oi, ow, cyc, h);
}
