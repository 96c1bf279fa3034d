// Max co-resident clusters for cluster sizes 1..16 at ~223 KB dynamic smem, 512 threads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int *p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int smem : {100 * 1024, 200 * 1024, 223 * 1024}) {
    for (int cs = 1; cs <= 16; ++cs) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 16);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a;
      a.id = cudaLaunchAttributeClusterDimension;
      a.val.clusterDim.x = cs; a.val.clusterDim.y = 1; a.val.clusterDim.z = 1;
      cfg.attrs = &a; cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %dKB cluster %2d: %3d clusters = %3d CTAs %s\n", smem / 1024, cs, n, n * cs, e ? cudaGetErrorString(e) : "");
    }
  }
  cudaDeviceProp pr; cudaGetDeviceProperties(&pr, 0);
  printf("SMs %d\n", pr.multiProcessorCount);
}
