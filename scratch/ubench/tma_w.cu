// Per-SM TMA throughput of 16 KB weight boxes vs ring depth (bytes in flight),
// from an L2-resident (16 MB) or HBM-resident (2 GB, streamed once) buffer.
#include <cstdio>
#include <vector>
#include "../../paper_2509_09560_b200/csrc/tc_util.cuh"
using namespace auras;
namespace auras {
void set_error(const char *fmt, ...) {}
int cuda_check(cudaError_t e, const char *what) { return e ? -1 : 0; }
}
__global__ void bench(const __grid_constant__ CUtensorMap tm, int stages, int iters, long long rows_total, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *buf = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  uint64_t *full = reinterpret_cast<uint64_t *>(buf + stages * 16384);
  if (threadIdx.x == 0) { for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  long long t0 = clock64();
  const long long nbox = rows_total / 128;
  for (int i = 0; i < iters + stages; ++i) {
    const int st = i % stages;
    if (i >= stages) mbar_wait(&full[st], ((i / stages) - 1) & 1);
    if (i < iters) {
      const long long box = ((long long)blockIdx.x * iters + i) % nbox;
      tma_load_2d_warp(buf + st * 16384, &tm, &full[st], 16384, 0, (int)(box * 128));
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
  long long *out; cudaMalloc(&out, 148 * 8);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (long long mb : {16LL, 2048LL}) {
    void *w; cudaMalloc(&w, mb << 20); cudaMemset(w, 0, mb << 20);
    const long long rows = (mb << 20) / 128;
    CUtensorMap tm;
    EncodeTiledFn enc = encode_fn();
    cuuint64_t dims[2] = {64, (cuuint64_t)rows}; cuuint64_t str[1] = {128}; cuuint32_t box[2] = {64, 128}; cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int stages : {4, 8, 12}) {
      const size_t smem = 1024 + stages * 16384 + 256;
      cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int grid : {1, 16, 64, 112, 148}) {
        const int iters = mb == 16 ? 2000 : (int)std::min<long long>(2000, (mb << 20) / 16384 / grid);
        bench<<<grid, 64, smem>>>(tm, stages, iters, rows, out);
        cudaDeviceSynchronize();
        bench<<<grid, 64, smem>>>(tm, stages, iters, rows, out);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost);
        long long mx = 0; for (auto v : h) mx = v > mx ? v : mx;
        const double us = mx / (clk * 1e-3);
        printf("%5lld MB stages %2d grid %3d: %.1f GB/s per SM, %.0f GB/s total %s\n", mb, stages, grid,
               16384.0 * iters / us * 1e-3, 16384.0 * iters * grid / us * 1e-3, cudaGetErrorString(e));
      }
    }
    cudaFree(w);
  }
}
