// Max co-resident clusters for a persistent kernel shaped like the router
// (384 threads, ~227 KB dynamic smem, 1 CTA/SM): how many SMs a cluster size
// can actually use on this part (GPC granularity).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/micro/cluster_occ tools/micro/cluster_occ.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k() { extern __shared__ char s[]; s[threadIdx.x] = 0; }
int main() {
    const int smem = 227 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute a[1];
        cfg.gridDim = dim3(cs * 64);
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = smem;
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        int n = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
        printf("cluster %2d: %3d clusters = %3d SMs (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
    }
}
