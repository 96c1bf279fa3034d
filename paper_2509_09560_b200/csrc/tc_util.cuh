// tcgen05 / TMA / mbarrier helpers shared by the sm_100a engines.
#pragma once
#include <cuda.h>

#include "conv.cuh"

namespace auras {

// ---------------------------------------------------------------- host: tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}


// Tensor map of a [M][Kp] bf16 weight matrix, 128 x 64 boxes, 128B swizzle.
inline int make_weight_map(CUtensorMap *tm, const void *w, int M, int Kp) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return AURAS_E_CUDA; }
  cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)M};
  cuuint64_t strides[1] = {(cuuint64_t)Kp * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(w), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("weight tensor map: CUresult %d", (int)r); return AURAS_E_CUDA; }
  return AURAS_OK;
}

// Tensor map of a 1-D conv input viewed as {channel, phase, time/stride, sample}
// (see gemm_sm100.cu): box {64, 1, Wo, s_box}.
inline int make_act_map(CUtensorMap *tm, const void *in, int coff, int Cin, int pitch, int W, int stride, int S,
                        int Wo, int s_box) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return AURAS_E_CUDA; }
  const uint8_t *base = static_cast<const uint8_t *>(in) + (size_t)coff * 2;
  cuuint64_t dims[4] = {(cuuint64_t)Cin, (cuuint64_t)stride, (cuuint64_t)(W / stride), (cuuint64_t)S};
  cuuint64_t strides[3] = {(cuuint64_t)pitch * 2, (cuuint64_t)pitch * 2 * stride, (cuuint64_t)pitch * 2 * W};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)Wo, (cuuint32_t)s_box};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint8_t *>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("activation tensor map: CUresult %d", (int)r); return AURAS_E_CUDA; }
  return AURAS_OK;
}

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Wait for an mbarrier phase, backing off between probes: for warps whose
// wait is not latency critical, so they do not take issue slots from a warp
// on the same scheduler that is (the MMA issuer).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity, int ns = 128) {
  uint32_t ok;
  while (true) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(ns);
  }
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *tm, uint64_t *bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *tm, uint64_t *bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// UMMA shared-memory descriptor: K-major operand, 128B swizzle, 8-row atoms
// 1024 B apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);          // start address
  d |= (uint64_t)(16 >> 4) << 16;                   // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                 // SBO
  d |= (uint64_t)1 << 46;                           // descriptor version
  d |= (uint64_t)2 << 61;                           // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D f32, A/B bf16, both K-major, M = 128, N = n.
__device__ __forceinline__ uint32_t umma_idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}


// ---- warp-uniform variants: every lane executes the call with identical
// operands; one lane is elected inside the PTX, so descriptors and addresses
// stay in uniform registers (no per-instruction R2UR/ELECT loops).
__device__ __forceinline__ void umma_bf16_warp(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                               uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px, p;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit_warp(uint64_t *bar) {
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "@px tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_2d_warp(void *dst, const CUtensorMap *tm, uint64_t *bar, uint32_t bytes,
                                                 int c0, int c1) {
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "@px mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n"
      "@px cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%4, %5}], [%2];\n"
      "}\n" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(bytes), "r"(c0), "r"(c1)
      : "memory");
}

// expect_tx(bytes) once, then one or two 2-D boxes (rows c1a and c1b) into
// consecutive 16 KB halves of dst.
__device__ __forceinline__ void tma_load_2d_pair_warp(void *dst, const CUtensorMap *tm, uint64_t *bar, uint32_t bytes,
                                                      int c0, int c1a, int c1b, int two) {
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px, p2;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "setp.ne.and.b32 p2, %7, 0, px;\n"
      "@px mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n"
      "@px cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%4, %5}], [%2];\n"
      "@p2 cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%8], [%1, {%4, %6}], [%2];\n"
      "}\n" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(bytes), "r"(c0), "r"(c1a), "r"(c1b), "r"(two),
      "r"(smem_u32(dst) + 16384)
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx_warp(uint64_t *bar, uint32_t bytes) {
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "@px mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

// TMA only (the barrier's expect_tx was armed separately).
__device__ __forceinline__ void tma_4d_warp(void *dst, const CUtensorMap *tm, uint64_t *bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "@px cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2];\n"
      "}\n" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d_warp(void *dst, const CUtensorMap *tm, uint64_t *bar, uint32_t bytes,
                                                 int c0, int c1, int c2, int c3) {
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "@px mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n"
      "@px cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%4, %5, %6, "
      "%7}], [%2];\n"
      "}\n" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(bytes), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ int ld_acquire_i32(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void spin_until(const int *ctr, int target) {
  while (ld_acquire_i32(ctr) < target) {
  }
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}


// One k-block (K = 64) of UMMAs from one elected lane: four K=16 steps along
// the 128-byte swizzled rows (descriptor start address +32 B = +2 per step).
// acc = 0 overwrites the accumulator on the first step.  nmt = 2 adds a second
// M=128 tile whose A rows sit 16 KB (+1024 in descriptor units) further and
// whose accumulator is `dt2`.
__device__ __forceinline__ void umma_kblock_warp(uint32_t dt, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px, p;\n"
      ".reg .b64 a1, a2, a3, b1, b2, b3;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "add.s64 a1, %1, 2;\n add.s64 a2, %1, 4;\n add.s64 a3, %1, 6;\n"
      "add.s64 b1, %2, 2;\n add.s64 b2, %2, 4;\n add.s64 b3, %2, 6;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n"
      "}\n" ::"r"(dt),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_kblock2_warp(uint32_t dt, uint32_t dt2, uint64_t ad, uint64_t bd, uint32_t idesc,
                                                  uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px, p;\n"
      ".reg .b64 a1, a2, a3, c0, c1, c2, c3, b1, b2, b3;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "setp.ne.b32 p, %5, 0;\n"
      "add.s64 a1, %2, 2;\n add.s64 a2, %2, 4;\n add.s64 a3, %2, 6;\n"
      "add.s64 c0, %2, 1024;\n add.s64 c1, %2, 1026;\n add.s64 c2, %2, 1028;\n add.s64 c3, %2, 1030;\n"
      "add.s64 b1, %3, 2;\n add.s64 b2, %3, 4;\n add.s64 b3, %3, 6;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %4, p;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%1], c0, %3, %4, p;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %4, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%1], c1, b1, %4, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %4, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%1], c2, b2, %4, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %4, 1;\n"
      "@px tcgen05.mma.cta_group::1.kind::f16 [%1], c3, b3, %4, 1;\n"
      "}\n" ::"r"(dt),
      "r"(dt2), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
}  // namespace auras
