// How many clusters of each size fit on the device with one 200 KB-smem CTA per SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* o) { extern __shared__ int s[]; if (threadIdx.x == 0 && o) o[blockIdx.x] = s[0]; }
int main() {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs = 1; cs <= 16; ++cs) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(cs); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = 200 * 1024; cfg.attrs = a; cfg.numAttrs = 1;
        int n = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
        printf("cs=%2d clusters=%3d SMs=%3d %s\n", cs, n, n * cs, e ? cudaGetErrorString(e) : "");
    }
}
