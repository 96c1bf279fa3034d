// Per-SM ingest: tensor TMA 16 KB boxes (1 or 2 issuing warps) vs 1-D bulk
// copies (cp.async.bulk) of 4/16/32 KB, L2- (16 MB) or HBM-resident (2 GB).
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../../paper_2509_09560_b200/csrc/tc_util.cuh"
using namespace auras;
namespace auras {
void set_error(const char *fmt, ...) {}
int cuda_check(cudaError_t e, const char *what) { return e ? -1 : 0; }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// mode 0: tensor box, issuers = nw warps (each its own ring slice); mode 1: bulk chunk of `chunk` bytes
__device__ __forceinline__ void wait_mode(uint64_t *bar, uint32_t parity, int wm) {
  if (wm == 0) { mbar_wait(bar, parity); return; }
  if (wm == 1) {
    asm volatile("{\n.reg .pred P1;\nW1:\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W1;\n}\n"
                 ::"r"(smem_u32(bar)), "r"(parity) : "memory");
    return;
  }
  asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n@!P1 bra W2;\n}\n"
               ::"r"(smem_u32(bar)), "r"(parity), "r"(wm == 2 ? 20 : 200) : "memory");
}
__global__ void bench(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm2, const uint8_t *g, long long gbytes, int mode, int nw,
                      int chunk, int ring_bytes, long long per_cta, long long *out, int wm) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *buf = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  const int stages_total = ring_bytes / chunk;
  const int stages = stages_total / nw;
  uint64_t *full = reinterpret_cast<uint64_t *>(buf + ring_bytes);
  if (threadIdx.x == 0) { for (int i = 0; i < stages_total; ++i) mbar_init(&full[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if (w >= nw) return;
  const long long n = per_cta / chunk / nw;
  long long t0 = clock64();
  for (long long i = 0; i < n + stages; ++i) {
    const int st = w * stages + (int)(i % stages);
    if (i >= stages) wait_mode(&full[st], ((i / stages) - 1) & 1, wm);
    if (i < n) {
      const long long off = ((long long)blockIdx.x * per_cta + (i * nw + w) * (long long)chunk) % gbytes;
      if (mode == 0) tma_load_2d_warp(buf + (size_t)st * chunk, &tm, &full[st], chunk, 0, (int)(off / 128));
      else if (mode == 2) tma_load_2d_warp(buf + (size_t)st * chunk, &tm2, &full[st], chunk, 0, (int)(off / 128));
      else {
        if ((threadIdx.x & 31) == 0) {
          mbar_expect_tx(&full[st], chunk);
          bulk_g2s(buf + (size_t)st * chunk, g + off, chunk, &full[st]);
        }
        __syncwarp();
      }
    }
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long *)&out[blockIdx.x], (unsigned long long)(t1 - t0));
}
int main() {
  long long *out; cudaMalloc(&out, 148 * 8);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (long long mb : {16LL, 2048LL}) {
    uint8_t *w; cudaMalloc(&w, mb << 20); cudaMemset(w, 0, mb << 20);
    const long long rows = (mb << 20) / 128;
    CUtensorMap tm;
    EncodeTiledFn enc = encode_fn();
    cuuint64_t dims[2] = {64, (cuuint64_t)rows}; cuuint64_t str[1] = {128}; cuuint32_t box[2] = {64, 128}; cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap tm2; cuuint32_t box2[2] = {64, 256};
    enc(&tm2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    struct C { int mode, nw, chunk; const char *name; };
    for (int wm : {0})
    for (C c : {C{2, 1, 32768, "tensor 32K x1"}, C{2, 4, 32768, "tensor 32K x4"}, C{0, 8, 16384, "tensor 16K x8"}, C{2, 2, 32768, "tensor 32K x2"}}) {
      const int ring = 131072;
      const size_t smem = 1024 + ring + 8 * 64;
      cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int grid : {1, 64, 112}) {
        const long long per_cta = mb == 16 ? (32LL << 20) : std::min<long long>(32LL << 20, ((mb << 20) / grid) & ~65535LL);
        cudaMemset(out, 0, 148 * 8);
        bench<<<grid, 256, smem>>>(tm, tm2, w, mb << 20, c.mode, c.nw, c.chunk, ring, per_cta, out, wm);
        cudaDeviceSynchronize();
        cudaMemset(out, 0, 148 * 8);
        bench<<<grid, 256, smem>>>(tm, tm2, w, mb << 20, c.mode, c.nw, c.chunk, ring, per_cta, out, wm);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost);
        long long mx = 0; for (auto v : h) mx = v > mx ? v : mx;
        const double us = mx / (clk * 1e-3);
        printf("wait%d %5lld MB %-14s grid %3d: %6.1f GB/s per SM, %6.0f GB/s total %s\n", wm, mb, c.name, grid,
               per_cta / us * 1e-3, (double)per_cta * grid / us * 1e-3, cudaGetErrorString(e));
      }
    }
    cudaFree(w);
  }
}
