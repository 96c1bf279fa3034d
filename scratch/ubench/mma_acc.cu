// Microbenchmark: UMMA (tcgen05.mma cta_group::1 kind::f16, SS operands, 128B swizzle)
// issue cost per instruction vs N, M and the number of independent accumulators
// the instruction stream rotates over (8 MMAs per asm block).
#include <cstdio>
#include "../../paper_2509_09560_b200/csrc/tc_util.cuh"
using namespace auras;
namespace auras { void set_error(const char *, ...) {} int cuda_check(cudaError_t, const char *) { return 0; } }

template <int NACC>
__device__ __forceinline__ void issue8(uint32_t tmem, int stride, uint64_t ad, uint64_t bd, uint32_t idesc) {
  // 8 K=16 steps; step i accumulates into accumulator i % NACC (columns i % NACC * stride)
  asm volatile(
      "{\n"
      ".reg .b32 rx, d0, d1, d2, d3;\n"
      ".reg .pred px;\n"
      ".reg .b64 a1, a2, a3, b1, b2, b3;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "add.s64 a1, %1, 2;\n add.s64 a2, %1, 4;\n add.s64 a3, %1, 6;\n"
      "add.s64 b1, %2, 2;\n add.s64 b2, %2, 4;\n add.s64 b3, %2, 6;\n"
      "mov.b32 d0, %0;\n"
      "add.s32 d1, %0, %4;\n"
      "add.s32 d2, d1, %4;\n"
      "add.s32 d3, d2, %4;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [d0], %1, %2, %3, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%5], a1, b1, %3, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%6], a2, b2, %3, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%7], a3, b3, %3, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [d0], %1, %2, %3, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%5], a1, b1, %3, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%6], a2, b2, %3, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%7], a3, b3, %3, 1;\n"
      "}\n" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(stride), "r"(tmem + (1 % NACC) * stride), "r"(tmem + (2 % NACC) * stride),
      "r"(tmem + (3 % NACC) * stride));
}

__global__ void __launch_bounds__(128, 1) bench(int iters, int n, int m, int nacc, long long *out) {
  extern __shared__ uint8_t raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = sm, *sB = sm + 32768;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sB + 32768);
  uint32_t *slot = reinterpret_cast<uint32_t *>(bars + 4);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bars[0], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  if (warp == 1) {
    uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
    const uint64_t ad = umma_desc(smem_u32(sA)), bd = umma_desc(smem_u32(sB));
    const int stride = n;     // accumulator column stride
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (nacc == 1) issue8<1>(tmem, stride, ad, bd, idesc);
      else if (nacc == 2) issue8<2>(tmem, stride, ad, bd, idesc);
      else issue8<4>(tmem, stride, ad, bd, idesc);
    }
    umma_commit_warp(&bars[0]);
    mbar_wait(&bars[0], 0);
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
  long long *d;
  cudaMalloc(&d, 8 * 148);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000);
  const int iters = 1000;
  for (int m : {128, 64})
    for (int n : {16, 32, 64, 128, 256})
      for (int nacc : {1, 2, 4}) {
        if (n * nacc > 512) continue;
        bench<<<148, 128, 80000>>>(iters, n, m, nacc, d);
        long long h = 0;
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        const double per = (double)h / (iters * 8);
        printf("M=%3d N=%3d nacc=%d: %.1f cyc/MMA  %.0f MAC/cyc %s\n", m, n, nacc, per, m * n * 16 / per,
               e ? cudaGetErrorString(e) : "");
        if (e) return 1;
      }
  return 0;
}
