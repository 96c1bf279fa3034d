// Activation B-operand boxes: per-box TMA cost for the im2col views of a
// channel-blocked activation (C=2048, T=4, S=8): s-major 5-D (kernel today),
// t-major 5-D, and one contiguous 2-D run; 1 or 3 issuing warps.
#include <cstdio>
#include <vector>
#include "../../paper_2509_09560_b200/csrc/tc_util.cuh"
using namespace auras;
namespace auras {
void set_error(const char *fmt, ...) {}
int cuda_check(cudaError_t e, const char *what) { return e ? -1 : 0; }
}
__device__ __forceinline__ void tma5(void *dst, const CUtensorMap *tm, uint64_t *bar, uint32_t bytes, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, 0xffffffff;\n"
               "@px mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n"
               "@px cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%4, %5, %6, %7, %8}], [%2];\n}\n"
               ::"r"(smem_u32(dst)), "l"(tm), "r"(smem_u32(bar)), "r"(bytes), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4) : "memory");
}
__device__ __forceinline__ void tma3(void *dst, const CUtensorMap *tm, uint64_t *bar, uint32_t bytes, int c0, int c1, int c2) {
  asm volatile("{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, 0xffffffff;\n"
               "@px mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n"
               "@px cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%4, %5, %6}], [%2];\n}\n"
               ::"r"(smem_u32(dst)), "l"(tm), "r"(smem_u32(bar)), "r"(bytes), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
constexpr int ST = 12;  // 4 KB stages (mode 3 uses two 20 KB halves of the same 48 KB)
__global__ void bench(const __grid_constant__ CUtensorMap tm, int mode, int nw, int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *buf = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  uint64_t *full = reinterpret_cast<uint64_t *>(buf + ST * 4096);
  if (threadIdx.x == 0) { for (int i = 0; i < ST; ++i) mbar_init(&full[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if (w >= nw) return;
  const int per = ST / nw;
  long long t0 = clock64();
  for (int i = 0; i < iters + per; ++i) {
    const int st = w * per + i % per;
    if (i >= per) mbar_wait(&full[st], ((i / per) - 1) & 1);
    if (i < iters) {
      const int kb = (i * nw + w + blockIdx.x) % 160, tap = kb / 32, cb = kb % 32;
      if (mode == 0) tma5(buf + st * 4096, &tm, &full[st], 4096, 0, 0, tap - 2, 0, cb);          // {64,1,Wo,s,cb}
      else if (mode == 3) tma5(buf + (st % 2) * 20480, &tm, &full[st], 20480, 0, 0, tap - 2, 0, cb & ~7);  // 5 cbs per box
      else if (mode == 1) tma5(buf + st * 4096, &tm, &full[st], 4096, 0, 0, 0, tap - 2, cb);     // {64,s,1,Wo,cb}
      else tma3(buf + st * 4096, &tm, &full[st], 4096, 0, (tap - 2) * 8, cb);                     // {64, T*S, cb}
    }
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long *)&out[blockIdx.x], (unsigned long long)(t1 - t0));
}
int main() {
  const int C = 2048, T = 4, S = 8, CB = C / 64;
  void *act; cudaMalloc(&act, (size_t)CB * T * S * 128); cudaMemset(act, 0, (size_t)CB * T * S * 128);
  long long *out; cudaMalloc(&out, 148 * 8);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  EncodeTiledFn enc = encode_fn();
  for (int mode = 0; mode < 4; ++mode) {
    CUtensorMap tm;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r;
    if (mode == 0 || mode == 3) {   // s-major buffer [cb][s][t][64]: dims {64, stride=1, T, S, CB}
      cuuint64_t d[5] = {64, 1, (cuuint64_t)T, (cuuint64_t)S, (cuuint64_t)CB};
      cuuint64_t st[4] = {128, 128, 128 * T, (cuuint64_t)128 * T * S};
      cuuint32_t b[5] = {64, 1, 4, 8, (cuuint32_t)(mode == 3 ? 5 : 1)};
      r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, act, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else if (mode == 1) {   // t-major buffer [cb][t][s][64]: dims {64, S, stride=1, T, CB}
      cuuint64_t d[5] = {64, (cuuint64_t)S, 1, (cuuint64_t)T, (cuuint64_t)CB};
      cuuint64_t st[4] = {128, 128 * S, 128 * S, (cuuint64_t)128 * T * S};
      cuuint32_t b[5] = {64, 8, 1, 4, 1};
      r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, act, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {                   // t-major, 3-D {64, T*S, CB}
      cuuint64_t d[3] = {64, (cuuint64_t)T * S, (cuuint64_t)CB};
      cuuint64_t st[2] = {128, (cuuint64_t)128 * T * S};
      cuuint32_t b[3] = {64, 32, 1};
      r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, act, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r) { printf("encode %d failed %d\n", mode, (int)r); continue; }
    const size_t smem = 1024 + ST * 4096 + 256;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int nw : {1, 3}) for (int grid : {1, 64}) {
      const int iters = 600;
      cudaMemset(out, 0, 148 * 8);
      bench<<<grid, 128, smem>>>(tm, mode, nw, iters, out); cudaDeviceSynchronize();
      cudaMemset(out, 0, 148 * 8);
      bench<<<grid, 128, smem>>>(tm, mode, nw, iters, out);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<long long> h(grid); cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost);
      long long mx = 0; for (auto v : h) mx = v > mx ? v : mx;
      const double us = mx / (clk * 1e-3);
      const double bb = mode == 3 ? 20480.0 : 4096.0;
      printf("%-22s warps %d grid %3d: %.3f us per box (%.0f KB), %.1f GB/s per SM %s\n",
             mode == 0 ? "s-major 5D (today)" : mode == 1 ? "t-major 5D" : mode == 2 ? "t-major 3D contiguous" : "s-major 5D x5 cb", nw, grid,
             us / iters, bb / 1024, bb * iters / us * 1e-3, cudaGetErrorString(e));
    }
  }
}
