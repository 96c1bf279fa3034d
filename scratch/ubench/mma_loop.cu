// Microbenchmark: per-k-block cost of the megakernel's MMA-issue loop with resident operands.
#include <cstdio>
#include "../../paper_2509_09560_b200/csrc/tc_util.cuh"
using namespace auras;
namespace auras { void set_error(const char *, ...) {} int cuda_check(cudaError_t, const char *) { return 0; } }

__global__ void __launch_bounds__(128, 1) bench(int nkb, int bn, int mode, long long *out, const __grid_constant__ CUtensorMap tm, int *flag) {
  extern __shared__ uint8_t raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = sm, *sB = sm + 10 * 16384;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sB + 4 * 16384);
  uint32_t *slot = reinterpret_cast<uint32_t *>(bars + 32);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (10 * 16384 + 4 * 16384) / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = (mode & 8) ? (0x3c003c00u ^ ((i * 2654435761u) & 0x83ff83ffu)) : 0x3c003c00u;
  if (threadIdx.x == 0) { for (int i = 0; i < 32; ++i) mbar_init(&bars[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 1) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(256)); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) { mbar_arrive(&bars[20]); }
  __syncthreads();
  if (warp >= 2 && mode >= 5) {
    volatile int *stop = flag + 1;
    if (mode == 5 && warp == 2) {          // TMA stream into A regions 6..9 until the MMA loop ends
      for (int i = 0; *stop == 0; ++i) {
        const int st = i & 3;
        if (i >= 4) mbar_wait(&bars[16 + st], ((i >> 2) - 1) & 1);
        tma_load_2d_warp(sA + (6 + st) * 16384, &tm, &bars[16 + st], 16384, 0, (int)(((long long)(blockIdx.x * 5000 + i) * 128) % (1ll << 23)));
      }
    }
    if (mode == 6 && (threadIdx.x & 31) == 0) {
      while (*stop == 0) { int v; asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory"); }
    }
  }
  const int nissue = mode == 50 ? 2 : mode == 51 ? 3 : 1;
  if (warp >= 1 && warp <= nissue) {
    const int iw = warp - 1;
    const uint32_t idesc = umma_idesc(bn);
    long long t0 = clock64();
    for (int kb = 0; kb < nkb; ++kb) {
      const int sa = kb % 10, sb = kb % 4;
      if (mode >= 1) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = smem_u32(sA + sa * 16384), b0 = smem_u32(sB + sb * 16384);
      if (mode == 14) {                               // descriptor bases from global memory (non-uniform)
        const int o = __ldcg(flag + 4 + (kb & 3));
        umma_kblock2_warp(tmem, tmem + 64, umma_desc(a0 + o), umma_desc(b0 + o), idesc, kb > 0);
        umma_commit_warp(&bars[sa % 8]); umma_commit_warp(&bars[8 + sb]);
        __syncwarp();
        continue;
      }
      if (mode == 7 || mode == 13) {                  // + wait on an already-completed barrier (+ the stage commit path)
        mbar_wait(&bars[20], 0);
        umma_kblock2_warp(tmem, tmem + 64, umma_desc(a0), umma_desc(b0), idesc, kb > 0);
        umma_commit_warp(&bars[sa % 8]); umma_commit_warp(&bars[8 + sb]);
        __syncwarp();
        continue;
      }
      if (mode == 50 || mode == 51) {
        umma_kblock_warp(tmem + iw * 64, umma_desc(a0), umma_desc(b0), idesc, kb > 0);
        umma_commit_warp(&bars[sa % 8]); umma_commit_warp(&bars[8 + sb]);
        __syncwarp();
        continue;
      }
      if (mode >= 40 && mode < 50) {                  // operand-major / M variants of the K=64 block
        uint32_t id = idesc;
        uint64_t ad = umma_desc(a0), bd = umma_desc(b0);
        if (mode == 40 || mode == 43) { id |= 1u << 15; ad = (ad & ~(0x3FFFull << 16)) | ((uint64_t)(8192 >> 4) << 16); }
        if (mode == 41) id = (id & ~(0x1Fu << 24)) | ((uint32_t)(64 >> 4) << 24);
        if (mode == 42 || mode == 43) { id |= 1u << 16; bd = (bd & ~(0x3FFFull << 16)) | ((uint64_t)(8192 >> 4) << 16); }
        if (mode == 44) id = (id & ~(0x1Fu << 24)) | ((uint32_t)(256 >> 4) << 24);
        umma_kblock_warp(tmem, ad, bd, id, kb > 0);
        umma_commit_warp(&bars[sa % 8]); umma_commit_warp(&bars[8 + sb]);
        __syncwarp();
        continue;
      }
      if (mode >= 20 && mode < 30) {                  // 4 K=16 steps into `nacc` accumulators (round robin)
        const int nacc = mode - 20;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16_warp(tmem + (kk % nacc) * 64, umma_desc(a0 + kk * 32), umma_desc(b0 + kk * 32), idesc, (kb > 0) ? 1u : 0u);
        umma_commit_warp(&bars[sa % 8]); umma_commit_warp(&bars[8 + sb]);
        __syncwarp();
        continue;
      }
      if (mode >= 30 && mode < 40) {                  // 8 K=16 steps (two k-blocks) into `nacc` accumulators
        const int nacc = mode - 30;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_warp(tmem + (kk % nacc) * 32, umma_desc(a0 + (kk & 3) * 32 + (kk >> 2) * 16384), umma_desc(b0 + (kk & 3) * 32), idesc, (kb > 0) ? 1u : 0u);
        umma_commit_warp(&bars[sa % 8]); umma_commit_warp(&bars[8 + sb]);
        __syncwarp();
        continue;
      }
      if ((mode & 7) == 3) {
        umma_kblock2_warp(tmem, tmem + 64, umma_desc(a0), umma_desc(b0), idesc, kb > 0);
        umma_commit_warp(&bars[sa % 8]); umma_commit_warp(&bars[8 + sb]);
        __syncwarp();
        continue;
      }
      if ((mode & 7) == 4) {
        umma_kblock_warp(tmem, umma_desc(a0), umma_desc(b0), idesc, kb > 0);
        umma_commit_warp(&bars[sa % 8]); umma_commit_warp(&bars[8 + sb]);
        __syncwarp();
        continue;
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) umma_bf16_warp(tmem, umma_desc(a0 + kk * 32), umma_desc(b0 + kk * 32), idesc, (kb > 0 || kk > 0) ? 1u : 0u);
      if (mode >= 2) { umma_commit_warp(&bars[sa % 8]); umma_commit_warp(&bars[8 + sb]); }
      __syncwarp();
    }
    umma_commit_warp(&bars[24 + iw]);
    mbar_wait(&bars[24 + iw], 0);
    long long t1 = clock64();
    if (lane == 0 && iw == 0) { out[0] = t1 - t0; *(volatile int *)(flag + 1) = 1; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
  long long *d; cudaMalloc(&d, 8);
  int *flag; cudaMalloc(&flag, 64); cudaMemset(flag, 0, 64);
  void *w; cudaMalloc(&w, 1ull << 30); cudaMemset(w, 0, 1ull << 30);
  CUtensorMap tm;
  { EncodeTiledFn enc = encode_fn();
    cuuint64_t dims[2] = {64, 1ull << 23}; cuuint64_t str[1] = {128}; cuuint32_t box[2] = {64, 128}; cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); }
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 232000);
  for (int bn : {16, 32, 64, 128, 256}) for (int grid : {1, 148}) for (int mode : {0, 4, 8, 12}) for (int nkb : {2000}) {
    cudaMemset(flag, 0, 64);
    bench<<<grid, 128, 232000>>>(nkb, bn, mode, d, tm, flag);
    long long h = 0; cudaError_t e = cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("grid %3d bn=%3d mode=%d nkb=%3d: %lld cycles, %.1f cyc/kb %s\n", grid, bn, mode, nkb, h, (double)h / nkb, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
