// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/green/probe tools/green/probe.cu -lcuda
// Run:   tools/green/probe <side SMs>   (on a B200, e.g. under gpurun)
// Feasibility probe: SM partitions through green contexts, runtime-API launches
// into their streams, and events shared with the primary context.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>

__global__ void k_smid(unsigned *out) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    if (threadIdx.x == 0) out[blockIdx.x] = s;
    // keep the SM busy a little
    long long t0 = clock64();
    while (clock64() - t0 < 200000) {}
}

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char *m; cuGetErrorString(r, &m); printf("FAIL %s: %s\n", #x, m); return 1; } } while (0)
#define RK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main(int argc, char **argv) {
    int side = argc > 1 ? atoi(argv[1]) : 20;
    RK(cudaSetDevice(0));
    RK(cudaFree(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUdevResource all;
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("SMs %u\n", all.sm.smCount);
    CUdevResource grp[1], rest;
    unsigned n = 1;
    CK(cuDevSmResourceSplitByCount(grp, &n, &all, &rest, 0, side));
    printf("split: side group %u SMs, remaining %u SMs\n", grp[0].sm.smCount, rest.sm.smCount);
    CUdevResourceDesc dside, dmain;
    CK(cuDevResourceGenerateDesc(&dside, &grp[0], 1));
    CK(cuDevResourceGenerateDesc(&dmain, &rest, 1));
    CUgreenCtx gside, gmain;
    CK(cuGreenCtxCreate(&gside, dside, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxCreate(&gmain, dmain, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream sside, smain;
    CK(cuGreenCtxStreamCreate(&sside, gside, CU_STREAM_NON_BLOCKING, 0));
    CK(cuGreenCtxStreamCreate(&smain, gmain, CU_STREAM_NON_BLOCKING, 0));
    unsigned *d;
    RK(cudaMalloc(&d, 4096 * 4));  // primary-context allocation
    // runtime launches into the green streams with the PRIMARY context current
    k_smid<<<1024, 128, 0, (cudaStream_t)sside>>>(d);
    RK(cudaGetLastError());
    k_smid<<<1024, 128, 0, (cudaStream_t)smain>>>(d + 1024);
    RK(cudaGetLastError());
    cudaEvent_t ev;
    RK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    RK(cudaEventRecord(ev, (cudaStream_t)sside));
    RK(cudaStreamWaitEvent((cudaStream_t)smain, ev, 0));
    cudaStream_t prim;
    RK(cudaStreamCreate(&prim));
    RK(cudaStreamWaitEvent(prim, ev, 0));
    RK(cudaDeviceSynchronize());
    unsigned h[2048];
    RK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
    std::set<unsigned> a(h, h + 1024), b(h + 1024, h + 2048);
    int overlap = 0;
    for (unsigned x : a) overlap += b.count(x);
    printf("side stream used %zu distinct SMs, main stream %zu, overlap %d\n", a.size(), b.size(), overlap);
    printf("OK\n");
    return 0;
}
