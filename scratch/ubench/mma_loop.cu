// Microbenchmark: per-k-block cost of the megakernel's MMA-issue loop with resident operands.
#include <cstdio>
#include "../../paper_2509_09560_b200/csrc/tc_util.cuh"
using namespace auras;
namespace auras { void set_error(const char *, ...) {} int cuda_check(cudaError_t, const char *) { return 0; } }

__global__ void __launch_bounds__(128, 1) bench(int nkb, int bn, int mode, long long *out) {
  extern __shared__ uint8_t raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = sm, *sB = sm + 10 * 16384;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sB + 4 * 16384);
  uint32_t *slot = reinterpret_cast<uint32_t *>(bars + 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (10 * 16384 + 4 * 16384) / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 1) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(256)); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  if (warp == 1) {
    const uint32_t idesc = umma_idesc(bn);
    long long t0 = clock64();
    for (int kb = 0; kb < nkb; ++kb) {
      const int sa = kb % 10, sb = kb % 4;
      if (mode >= 1) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = smem_u32(sA + sa * 16384), b0 = smem_u32(sB + sb * 16384);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) umma_bf16_warp(tmem, umma_desc(a0 + kk * 32), umma_desc(b0 + kk * 32), idesc, (kb > 0 || kk > 0) ? 1u : 0u);
      if (mode >= 2) { umma_commit_warp(&bars[sa % 8]); umma_commit_warp(&bars[8 + sb]); }
      __syncwarp();
    }
    umma_commit_warp(&bars[15]);
    mbar_wait(&bars[15], 0);
    long long t1 = clock64();
    if (lane == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
  long long *d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 232000);
  for (int bn : {32, 128}) for (int mode = 0; mode < 3; ++mode) for (int nkb : {20, 200}) {
    bench<<<1, 128, 232000>>>(nkb, bn, mode, d);
    long long h = 0; cudaError_t e = cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("bn=%3d mode=%d nkb=%3d: %lld cycles, %.1f cyc/kb %s\n", bn, mode, nkb, h, (double)h / nkb, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
