// Micro-benchmark of the router's shared-memory top-k epilogue (cluster tail,
// passes 1-4) in isolation: 148 CTAs x 384 threads, warps 4-11 select top-8
// of 32 rows x 128 fp32 logits from shared memory (TPR = 8 threads per row).
// Prints per-phase SM cycles (clock64) of thread 128 of CTA 0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/epi_bench tools/micro/epi_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 128, KMAX = 8, RPS = 32, RS = N + 4, TPR = 8;

__device__ __forceinline__ bool rb(float v, int id, float w, int jd) { return v > w || (v == w && id < jd); }
__device__ __forceinline__ float pick16(const unsigned (&r)[16], int i) {
    unsigned a[8], b[4], c[2];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = (i & 1) ? r[2 * j + 1] : r[2 * j];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = (i & 2) ? a[2 * j + 1] : a[2 * j];
#pragma unroll
    for (int j = 0; j < 2; ++j) c[j] = (i & 4) ? b[2 * j + 1] : b[2 * j];
    return __uint_as_float((i & 8) ? c[1] : c[0]);
}

__global__ void __launch_bounds__(384, 1) k(const float *src, int *out_i, float *out_w, long long *cyc, int E) {
    __shared__ __align__(16) float tile[RPS * RS];
    for (int i = threadIdx.x; i < RPS * N; i += blockDim.x) tile[(i / N) * RS + i % N] = src[blockIdx.x * RPS * N + i];
    __syncthreads();
    if (threadIdx.x < 128) return;
    const unsigned t = threadIdx.x - 128, r = t / TPR, sub = t % TPR, CW = N / TPR, c0 = sub * CW;
    const float *row = tile + r * RS;
    long long c_0 = clock64();
    float m = -INFINITY, t0 = INFINITY;
    {
        float gm = -INFINITY;
        for (unsigned c = c0; c < c0 + CW; c += 4) {
            const float4 v = *reinterpret_cast<const float4 *>(row + c);
            gm = fmaxf(fmaxf(gm, v.x), fmaxf(v.y, fmaxf(v.z, v.w)));
        }
        t0 = fminf(t0, gm);
        m = fmaxf(m, gm);
    }
    for (unsigned o = 1; o < TPR; o <<= 1) {
        t0 = fminf(t0, __shfl_xor_sync(0xffffffffu, t0, o));
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    long long c_1 = clock64();
    float tv[KMAX];
    int ti[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) { tv[j] = -INFINITY; ti[j] = 0x7FFFFFFF; }
    for (unsigned c = c0; c < c0 + CW; c += 8) {
        unsigned rr[16];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float4 v = *reinterpret_cast<const float4 *>(row + c + 4 * j);
            rr[4 * j] = __float_as_uint(v.x); rr[4 * j + 1] = __float_as_uint(v.y);
            rr[4 * j + 2] = __float_as_uint(v.z); rr[4 * j + 3] = __float_as_uint(v.w);
        }
#pragma unroll
        for (int j = 8; j < 16; ++j) rr[j] = __float_as_uint(-INFINITY);
        unsigned hit = 0;
        const float thr = fmaxf(tv[KMAX - 1], t0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float v = __uint_as_float(rr[i]);
            hit |= (unsigned)((c + i) < (unsigned)E && (v > thr || (v == t0 && v > tv[KMAX - 1]))) << i;
        }
        while (hit) {
            const int i = __ffs(hit) - 1;
            hit &= hit - 1;
            const float v = pick16(rr, i);
            const int e = c + i;
#pragma unroll
            for (int j = KMAX - 1; j >= 0; --j) {
                const bool here = v > tv[j];
                const bool above = j > 0 && v > tv[j > 0 ? j - 1 : 0];
                tv[j] = above ? tv[j > 0 ? j - 1 : 0] : (here ? v : tv[j]);
                ti[j] = above ? ti[j > 0 ? j - 1 : 0] : (here ? e : ti[j]);
            }
        }
    }
    long long c_2 = clock64();
    for (unsigned o = 1; o < TPR; o <<= 1) {
        float bv[KMAX]; int bi[KMAX];
#pragma unroll
        for (int j = 0; j < KMAX; ++j) { bv[j] = __shfl_xor_sync(0xffffffffu, tv[j], o); bi[j] = __shfl_xor_sync(0xffffffffu, ti[j], o); }
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            const bool a = rb(tv[j], ti[j], bv[KMAX - 1 - j], bi[KMAX - 1 - j]);
            tv[j] = a ? tv[j] : bv[KMAX - 1 - j]; ti[j] = a ? ti[j] : bi[KMAX - 1 - j];
        }
#pragma unroll
        for (int d = KMAX / 2; d >= 1; d >>= 1)
#pragma unroll
            for (int j = 0; j < KMAX; ++j)
                if ((j & d) == 0) {
                    const bool a = rb(tv[j], ti[j], tv[j + d], ti[j + d]);
                    const float xv = a ? tv[j] : tv[j + d], yv = a ? tv[j + d] : tv[j];
                    const int xi = a ? ti[j] : ti[j + d], yi = a ? ti[j + d] : ti[j];
                    tv[j] = xv; tv[j + d] = yv; ti[j] = xi; ti[j + d] = yi;
                }
    }
    long long c_3 = clock64();
    float ssum = 0.f;
    const float mlog = m * 1.4426950408889634f;
    for (unsigned c = c0; c < c0 + CW; ++c) ssum += exp2f(fmaf(row[c], 1.4426950408889634f, -mlog));
    for (unsigned o = 1; o < TPR; o <<= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
    long long c_4 = clock64();
    if (sub == 0) {
        const unsigned orow = blockIdx.x * RPS + r;
        for (int j = 0; j < KMAX; ++j) { out_i[orow * KMAX + j] = ti[j]; out_w[orow * KMAX + j] = exp2f(fmaf(tv[j], 1.4426950408889634f, -mlog)) / ssum; }
    }
    long long c_5 = clock64();
    if (blockIdx.x == 0 && t == 0) { cyc[0] = c_1 - c_0; cyc[1] = c_2 - c_1; cyc[2] = c_3 - c_2; cyc[3] = c_4 - c_3; cyc[4] = c_5 - c_4; }
}

int main() {
    const int B = 148;
    float *src; int *oi; float *ow; long long *cyc;
    cudaMalloc(&src, B * RPS * N * 4); cudaMalloc(&oi, B * RPS * KMAX * 4); cudaMalloc(&ow, B * RPS * KMAX * 4);
    cudaMallocManaged(&cyc, 8 * 8);
    float *h = new float[B * RPS * N];
    unsigned s = 1;
    for (int i = 0; i < B * RPS * N; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) * (1.0f / 16777216.0f); }
    cudaMemcpy(src, h, B * RPS * N * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int it = 0; it < 3; ++it) k<<<B, 384>>>(src, oi, ow, cyc, N);
    cudaEventRecord(a);
    for (int it = 0; it < 20; ++it) k<<<B, 384>>>(src, oi, ow, cyc, N);
    cudaEventRecord(b);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("kernel %.2f us/launch; cycles: pass1 %lld pass2 %lld merge %lld softmax %lld out %lld (%s)\n", ms / 20 * 1e3,
           cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cudaGetErrorString(cudaGetLastError()));
}
