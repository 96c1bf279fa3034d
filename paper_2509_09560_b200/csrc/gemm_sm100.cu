// tcgen05 / TMA implicit-GEMM engine for the weight-streaming convolutions of
// the denoise chain, sm_100a only.
//
//   D[m, n] = sum_k W[m, k] * B[n, k]      (swap-AB: M = C_out, N = samples x time)
//
// * A (weights, [M][Kp] bf16, K-major) streams through a multi-stage TMA ring
//   (128 x 64 tiles, 128B swizzle) -- this is the HBM stream the kernel exists
//   for; every weight byte is read exactly once per denoise step.
// * B (activations) is the implicit im2col of a 1-D conv, loaded by TMA from a
//   4-D view {channel, phase, time/stride, sample}: k-block (tap, c0) of output
//   row t reads input row t*stride - pad + tap = (t + q)*stride + h, i.e. box
//   {64, 1, Wo, S_box} at coordinate {c0, h, q, s0}.  Out-of-range rows
//   (padding) and samples come back as zeros from the TMA unit.
// * One elected thread issues tcgen05.mma (M=128, N=S_box*Wo rounded to 16,
//   K=16) into a TMEM accumulator; tcgen05.commit frees smem stages.
// * Split-K across CTAs so one wave covers the 148 SMs; the epilogue warps
//   drain TMEM with tcgen05.ld and write fp32 partials [split][n][m] that the
//   fused GroupNorm/Mish/FiLM epilogue kernel reduces in a fixed order.
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "conv.cuh"

namespace auras {

// ---------------------------------------------------------------- host: tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
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

constexpr int TC_BM = 128, TC_BK = 64;
constexpr int TC_THREADS = 128;
constexpr int TC_SMS = 148;

struct TcPlan {
  int m_tiles, n_tiles, splits, kb_total, kb_per_split, s_box, rows, bn, stages, tmem_cols;
  size_t smem;
};

static TcPlan tc_plan(const ConvGemmArgs &g) {
  TcPlan p;
  p.m_tiles = (g.M + TC_BM - 1) / TC_BM;
  const int S = g.N / g.Wo;
  p.s_box = std::min(S, 256 / g.Wo);
  p.n_tiles = (S + p.s_box - 1) / p.s_box;
  p.rows = p.s_box * g.Wo;
  p.bn = (p.rows + 15) / 16 * 16;
  p.kb_total = g.Kp / TC_BK;
  int want = std::max(1, TC_SMS / (p.m_tiles * p.n_tiles));
  want = std::min(want, p.kb_total);
  p.kb_per_split = (p.kb_total + want - 1) / want;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  const int stage_bytes = TC_BM * TC_BK * 2 + p.bn * TC_BK * 2;
  p.stages = std::max(2, std::min(8, (200 * 1024) / stage_bytes));
  p.stages = std::min(p.stages, std::max(2, p.kb_per_split));
  p.tmem_cols = 32;
  while (p.tmem_cols < p.bn) p.tmem_cols <<= 1;
  p.smem = 1024 + (size_t)p.stages * stage_bytes + 256;
  return p;
}

bool gemm_sm100_supported(const ConvGemmArgs &g) {
  if (!encode_fn()) return false;
  if (g.H != 1 || g.kh != 1 || g.Ho != 1) return false;     // 1-D (time) convolutions
  if (g.Cin % TC_BK || g.Kp % TC_BK || g.Kp < g.Kreal) return false;
  if (g.stride < 1 || g.stride > 2 || g.W % g.stride) return false;
  if (g.Wo > 256 || g.Wo < 1) return false;
  if (g.in_pitch % 8 || g.in_coff % 8) return false;
  if ((reinterpret_cast<uintptr_t>(g.w) & 15) || (reinterpret_cast<uintptr_t>(g.in) & 15)) return false;
  return true;
}

int gemm_sm100_splits(const ConvGemmArgs &g) { return tc_plan(g).splits; }

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

struct TcArgs {
  float *partial;
  int M, N, Cin, Wo, stride, pad, S, s_box, rows, bn, kb_per_split, kb_total, stages, tmem_cols;
};

__global__ void __launch_bounds__(TC_THREADS, 1)
    conv_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int a_bytes = TC_BM * TC_BK * 2;
  const int b_bytes = a.bn * TC_BK * 2;
  const int stage_bytes = a_bytes + b_bytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)a.stages * stage_bytes);
  uint64_t *empty = full + a.stages;
  uint64_t *done = empty + a.stages;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * TC_BM;
  const int s0 = blockIdx.y * a.s_box;
  const int split = blockIdx.z;
  const int kb0 = split * a.kb_per_split;
  const int kb1 = min(a.kb_total, kb0 + a.kb_per_split);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (lane 0 issues)
    for (int i = 0; i < nkb && lane == 0; ++i) {
      const int st = i % a.stages;
      const uint32_t ph = (i / a.stages) & 1;
      mbar_wait(&empty[st], ph ^ 1);
      uint8_t *sa = smem + (size_t)st * stage_bytes;
      uint8_t *sb = sa + a_bytes;
      const int kb = kb0 + i;
      const int k = kb * TC_BK;
      const int tap = k / a.Cin, c0 = k - tap * a.Cin;
      const int off = tap - a.pad;                       // input row = t*stride + off
      const int q = off >= 0 ? off / a.stride : -((-off + a.stride - 1) / a.stride);
      const int h = off - q * a.stride;
      mbar_expect_tx(&full[st], a_bytes + a.rows * TC_BK * 2);
      tma_load_2d(sa, &tmA, &full[st], k, m0);
      tma_load_4d(sb, &tmB, &full[st], c0, h, q, s0);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (one elected lane)
    const uint32_t idesc = umma_idesc(a.bn);
    for (int i = 0; i < nkb; ++i) {
      const int st = i % a.stages;
      const uint32_t ph = (i / a.stages) & 1;
      mbar_wait(&full[st], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t sa = smem_u32(smem + (size_t)st * stage_bytes);
        const uint32_t sb = sa + a_bytes;
#pragma unroll
        for (int kk = 0; kk < TC_BK / 16; ++kk)
          umma_bf16(tmem, umma_desc(sa + kk * 32), umma_desc(sb + kk * 32), idesc, (i > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&empty[st]);
        if (i == nkb - 1) umma_commit(done);
      }
      __syncwarp();
    }
    if (nkb == 0 && lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(done)) : "memory");
  }

  // ---------------- epilogue: TMEM -> fp32 partials [split][n][m]
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int m = m0 + warp * 32 + lane;
  float *out = a.partial + (int64_t)split * a.N * a.M;
  const int nbase = s0 * a.Wo;
  const int nvalid = min(a.rows, (a.S - s0) * a.Wo);
  for (int c = 0; c < a.bn; c += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    if (m < a.M) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = c + j;
        if (n < nvalid) out[(int64_t)(nbase + n) * a.M + m] = nkb > 0 ? v[j] : 0.f;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
}

int launch_gemm_sm100(const ConvGemmArgs &g, cudaStream_t st) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return AURAS_E_CUDA; }
  const TcPlan p = tc_plan(g);
  CUtensorMap tmA, tmB;
  {
    cuuint64_t dims[2] = {(cuuint64_t)g.Kp, (cuuint64_t)g.M};
    cuuint64_t strides[1] = {(cuuint64_t)g.Kp * 2};
    cuuint32_t box[2] = {TC_BK, TC_BM};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(g.w), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { set_error("tensor map A: CUresult %d", (int)r); return AURAS_E_CUDA; }
  }
  {
    const int S = g.N / g.Wo;
    const uint8_t *base = static_cast<const uint8_t *>(g.in) + (size_t)g.in_coff * 2;
    cuuint64_t dims[4] = {(cuuint64_t)g.Cin, (cuuint64_t)g.stride, (cuuint64_t)(g.W / g.stride), (cuuint64_t)S};
    cuuint64_t strides[3] = {(cuuint64_t)g.in_pitch * 2, (cuuint64_t)g.in_pitch * 2 * g.stride,
                             (cuuint64_t)g.in_pitch * 2 * g.W};
    cuuint32_t box[4] = {TC_BK, 1, (cuuint32_t)g.Wo, (cuuint32_t)p.s_box};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint8_t *>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { set_error("tensor map B: CUresult %d", (int)r); return AURAS_E_CUDA; }
  }
  static size_t configured = 0;
  if (p.smem > configured) {
    AURAS_CUDA(cudaFuncSetAttribute(conv_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    configured = 227 * 1024;
  }
  TcArgs a;
  a.partial = g.partial;
  a.M = g.M; a.N = g.N; a.Cin = g.Cin; a.Wo = g.Wo; a.stride = g.stride; a.pad = g.pad_w;
  a.S = g.N / g.Wo; a.s_box = p.s_box; a.rows = p.rows; a.bn = p.bn;
  a.kb_per_split = p.kb_per_split; a.kb_total = p.kb_total; a.stages = p.stages; a.tmem_cols = p.tmem_cols;
  dim3 grid(p.m_tiles, p.n_tiles, p.splits);
  conv_gemm_tc<<<grid, TC_THREADS, p.smem, st>>>(tmA, tmB, a);
  AURAS_LAUNCHED("conv_gemm_tc");
  return AURAS_OK;
}

}  // namespace auras

extern "C" int auras_tc_available(void) { return auras::encode_fn() != nullptr; }
