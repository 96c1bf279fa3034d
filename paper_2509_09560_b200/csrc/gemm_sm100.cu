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

#include "tc_util.cuh"

namespace auras {

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
  if (g.Wo % 4) return false;                               // epilogue stores 4 positions at a time
  if (g.in_pitch % 8 || g.in_coff % 8) return false;
  if ((reinterpret_cast<uintptr_t>(g.w) & 15) || (reinterpret_cast<uintptr_t>(g.in) & 15)) return false;
  return true;
}

int gemm_sm100_splits(const ConvGemmArgs &g) { return tc_plan(g).splits; }

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
      float *row = out + (int64_t)m * a.N + nbase + c;          // partial[split][m][n]
#pragma unroll
      for (int j = 0; j < 16; j += 4)
        if (c + j < nvalid)
          *reinterpret_cast<float4 *>(row + j) = nkb > 0 ? make_float4(v[j], v[j + 1], v[j + 2], v[j + 3])
                                                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
}

int launch_gemm_sm100(const ConvGemmArgs &g, cudaStream_t st) {
  const TcPlan p = tc_plan(g);
  CUtensorMap tmA, tmB;
  int rc = make_weight_map(&tmA, g.w, g.M, g.Kp);
  if (rc) return rc;
  rc = make_act_map(&tmB, g.in, g.in_coff, g.Cin, g.in_pitch, g.W, g.stride, g.N / g.Wo, g.Wo, p.s_box);
  if (rc) return rc;
  if (int rc2 = ensure_smem_attr(conv_gemm_tc, 227 * 1024)) return rc2;
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

