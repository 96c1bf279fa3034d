// Query co-resident cluster capacity for a 1-CTA/SM kernel at several cluster sizes.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int *p) { if (p) p[blockIdx.x] = 1; }
int main() {
  cudaDeviceProp pr; cudaGetDeviceProperties(&pr, 0);
  printf("SMs %d\n", pr.multiProcessorCount);
  for (int smem : {200 * 1024, 224 * 1024}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {4, 6, 7, 8}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 16); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a; a.id = cudaLaunchAttributeClusterDimension; a.val.clusterDim.x = cs; a.val.clusterDim.y = 1; a.val.clusterDim.z = 1;
      cfg.attrs = &a; cfg.numAttrs = 1;
      int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %dK cluster %2d -> %d clusters (%d CTAs) %s\n", smem / 1024, cs, n, n * cs, cudaGetErrorString(e));
    }
  }
}
