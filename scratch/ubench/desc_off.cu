// Does a tcgen05 smem descriptor whose start is shifted by r 128-byte rows
// (r not a multiple of 8) read a SWIZZLE_128B operand that was written with
// the absolute-address swizzle?  Tries base_offset = 0 and = (addr>>7)&7.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include "../../paper_2509_09560_b200/csrc/tc_util.cuh"
using namespace auras;
namespace auras {
void set_error(const char *fmt, ...) {}
int cuda_check(cudaError_t e, const char *what) { return e ? -1 : 0; }
}
__device__ uint64_t desc_bo(uint32_t saddr, int mode) {
  uint64_t d = umma_desc(saddr);
  if (mode == 1) d |= (uint64_t)((saddr >> 7) & 7) << 49;
  return d;
}
__global__ void k(const __nv_bfloat16 *A, const __nv_bfloat16 *B, float *out, int shift, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *s = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  uint8_t *sA = s, *sB = s + 16384;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * 8; e += blockDim.x) {   // A: 128 rows x 8 chunks
    const int m = e >> 3, c = e & 7;
    *reinterpret_cast<uint4 *>(sA + m * 128 + ((c ^ (m & 7)) * 16)) = *reinterpret_cast<const uint4 *>(A + m * 64 + c * 8);
  }
  for (int e = tid; e < 40 * 8; e += blockDim.x) {    // B: 40 rows, absolute swizzle
    const int r = e >> 3, c = e & 7;
    const uint32_t a = smem_u32(sB + r * 128);
    *reinterpret_cast<uint4 *>(sB + r * 128 + ((c ^ ((a >> 7) & 7)) * 16)) = *reinterpret_cast<const uint4 *>(B + r * 64 + c * 8);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t idesc = umma_idesc(16);
    const uint32_t b0 = smem_u32(sB + shift * 128);
    for (int kk = 0; kk < 4; ++kk)
      umma_bf16_warp(tmem, umma_desc(smem_u32(sA) + kk * 32), desc_bo(b0 + kk * 32, mode), idesc, kk > 0);
    umma_commit_warp(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float v[16];
  tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
  const int m = warp * 32 + (tid & 31);
  for (int n = 0; n < 16; ++n) out[m * 16 + n] = v[n];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}
int main() {
  std::vector<__nv_bfloat16> hA(128 * 64), hB(40 * 64);
  std::vector<float> fA(128 * 64), fB(40 * 64);
  srand(1);
  for (int i = 0; i < 128 * 64; ++i) { hA[i] = __float2bfloat16((rand() % 17 - 8) / 8.f); fA[i] = __bfloat162float(hA[i]); }
  for (int i = 0; i < 40 * 64; ++i) { hB[i] = __float2bfloat16((rand() % 17 - 8) / 8.f); fB[i] = __bfloat162float(hB[i]); }
  __nv_bfloat16 *dA, *dB; float *dO;
  cudaMalloc(&dA, hA.size() * 2); cudaMalloc(&dB, hB.size() * 2); cudaMalloc(&dO, 128 * 16 * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  for (int shift : {0, 1, 2, 4, 8, 12}) for (int mode : {0, 1}) {
    k<<<1, 128, 32768>>>(dA, dB, dO, shift, mode);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> o(128 * 16);
    cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int m = 0; m < 128; ++m) for (int n = 0; n < 16; ++n) {
      double r = 0; for (int kk = 0; kk < 64; ++kk) r += fA[m * 64 + kk] * fB[(shift + n) * 64 + kk];
      mx = fmax(mx, fabs(r - o[m * 16 + n]));
    }
    printf("shift %2d rows, base_offset mode %d: max err %g (%s)\n", shift, mode, mx, cudaGetErrorString(e));
  }
}
