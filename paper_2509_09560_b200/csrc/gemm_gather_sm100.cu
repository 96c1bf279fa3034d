// tcgen05 implicit-GEMM convolution with a thread-gathered im2col operand
// (the ResNet-18-GN perception encoder), sm_100a only.
//
//   D[m, n] = sum_k W[m, k] * B[n, k],  n = (sample, oy, ox),  k = (ky, kx, c)
//
// * A (weights [M][Kp] bf16) streams through TMA (128 x 64 boxes, 128B swizzle).
// * B is gathered by 4 warps straight into the UMMA K-major 128B-swizzled
//   layout: each thread moves 16-byte chunks (8 channels of one filter tap) of
//   8 output pixels, zero-filling padding, then fences the generic-proxy
//   stores for the async proxy and arrives on the stage's mbarrier.  This
//   handles any stride / padding / tap count (the 7x7/s2 stem, 3x3/s1 and
//   3x3/s2 bodies, 1x1/s2 downsamples) without an im2col buffer in HBM.
// * One elected lane issues tcgen05.mma (M=128, N=128, K=16) into TMEM; the
//   gather warps drain TMEM into split-K partials [split][m][n] that the fused
//   GroupNorm/ReLU/residual epilogue reduces.
#include <algorithm>

#include "tc_util.cuh"

namespace auras {

constexpr int GG_BM = 128, GG_BN = 128, GG_BK = 64;
constexpr int GG_THREADS = 192;          // warp 0 TMA, warp 1 MMA, warps 2-5 gather + epilogue
constexpr int GG_STAGES = 4;
constexpr int GG_A_BYTES = GG_BM * GG_BK * 2;
constexpr int GG_B_BYTES = GG_BN * GG_BK * 2;
constexpr size_t GG_SMEM = 1024 + (size_t)GG_STAGES * (GG_A_BYTES + GG_B_BYTES) + 256;

struct GatherArgs {
  const __nv_bfloat16 *in;
  float *partial;
  int M, N, Kreal, Cin, H, W, pitch, coff, kw, stride, ph, pw, Ho, Wo;
  int kb_total, kb_per_split;
};

struct GatherPlan {
  int m_tiles, n_tiles, splits, kb_total, kb_per_split;
};

static GatherPlan gather_plan(const ConvGemmArgs &g) {
  GatherPlan p;
  p.m_tiles = (g.M + GG_BM - 1) / GG_BM;
  p.n_tiles = (g.N + GG_BN - 1) / GG_BN;
  p.kb_total = g.Kp / GG_BK;
  // enough CTAs to occupy a slice of the GPU (or the op's cta_target when the
  // caller runs it alone), but keep >= 4 k-blocks per CTA
  const int target = g.cta_target > 0 ? g.cta_target : 32;
  int want = std::max(1, target / (p.m_tiles * p.n_tiles));
  want = std::min(want, std::max(1, p.kb_total / 4));
  p.kb_per_split = (p.kb_total + want - 1) / want;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  return p;
}

bool gemm_gather_supported(const ConvGemmArgs &g) {
  if (!encode_fn()) return false;
  if (g.Cin % 8 || g.Kp % GG_BK || g.Kp < g.Kreal) return false;
  if (g.in_pitch % 8 || g.in_coff % 8) return false;
  if ((reinterpret_cast<uintptr_t>(g.w) & 15) || (reinterpret_cast<uintptr_t>(g.in) & 15)) return false;
  return true;
}

int gemm_gather_splits(const ConvGemmArgs &g) { return gather_plan(g).splits; }

__global__ void __launch_bounds__(GG_THREADS, 1)
    conv_gemm_tc_gather(const __grid_constant__ CUtensorMap tmA, GatherArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = sA + GG_STAGES * GG_A_BYTES;
  uint64_t *fullA = reinterpret_cast<uint64_t *>(sB + GG_STAGES * GG_B_BYTES);
  uint64_t *fullB = fullA + GG_STAGES;
  uint64_t *empty = fullB + GG_STAGES;
  uint64_t *done = empty + GG_STAGES;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * GG_BM, n0 = blockIdx.y * GG_BN, split = blockIdx.z;
  const int kb0 = split * a.kb_per_split, kb1 = min(a.kb_total, kb0 + a.kb_per_split);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    for (int i = 0; i < GG_STAGES; ++i) {
      mbar_init(&fullA[i], 1);
      mbar_init(&fullB[i], 128);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- weights via TMA
    for (int i = 0; i < nkb; ++i) {
      const int st = i % GG_STAGES;
      mbar_wait(&empty[st], ((i / GG_STAGES) & 1) ^ 1);
      tma_load_2d_warp(sA + st * GG_A_BYTES, &tmA, &fullA[st], GG_A_BYTES, (kb0 + i) * GG_BK, m0);
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    const uint32_t idesc = umma_idesc(GG_BN);
    for (int i = 0; i < nkb; ++i) {
      const int st = i % GG_STAGES;
      const uint32_t ph = (i / GG_STAGES) & 1;
      mbar_wait(&fullA[st], ph);
      mbar_wait(&fullB[st], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = smem_u32(sA + st * GG_A_BYTES), b0 = smem_u32(sB + st * GG_B_BYTES);
#pragma unroll
      for (int kk = 0; kk < GG_BK / 16; ++kk)
        umma_bf16_warp(tmem, umma_desc(a0 + kk * 32), umma_desc(b0 + kk * 32), idesc, (i > 0 || kk > 0) ? 1u : 0u);
      umma_commit_warp(&empty[st]);
      __syncwarp();
    }
    if (nkb > 0) umma_commit_warp(done);
    else if (lane == 0) mbar_arrive(done);
  } else {
    // ---------------- im2col gather: 16-byte chunk j of rows r_i = gt/8 + 16 i
    const int gt = threadIdx.x - 64;
    const int j = gt & 7;
    const int P = a.Ho * a.Wo;
    int sbase[8], iy0[8], ix0[8];
    bool nok[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int n = n0 + (gt >> 3) + 16 * i;
      nok[i] = n < a.N;
      const int nn = nok[i] ? n : 0;
      const int s = nn / P, p = nn - s * P;
      const int oy = p / a.Wo, ox = p - oy * a.Wo;
      sbase[i] = s * a.H;
      iy0[i] = oy * a.stride - a.ph;
      ix0[i] = ox * a.stride - a.pw;
    }
    for (int i = 0; i < nkb; ++i) {
      const int st = i % GG_STAGES;
      mbar_wait(&empty[st], ((i / GG_STAGES) & 1) ^ 1);
      const int kk = (kb0 + i) * GG_BK + 8 * j;
      const int tap = kk / a.Cin, c = kk - tap * a.Cin;
      const int ky = tap / a.kw, kx = tap - ky * a.kw;
      const bool kok = kk < a.Kreal;
      uint4 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int iy = iy0[q] + ky, ix = ix0[q] + kx;
        v[q] = make_uint4(0, 0, 0, 0);
        if (kok && nok[q] && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W)
          v[q] = __ldg(reinterpret_cast<const uint4 *>(a.in + ((int64_t)(sbase[q] + iy) * a.W + ix) * a.pitch +
                                                       a.coff + c));
      }
      uint8_t *tile = sB + st * GG_B_BYTES;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int r = (gt >> 3) + 16 * q;
        *reinterpret_cast<uint4 *>(tile + r * 128 + ((j ^ (r & 7)) << 4)) = v[q];
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&fullB[st]);
    }
    // ---------------- epilogue: TMEM -> fp32 partials [split][m][n]
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quad = warp & 3;                     // TMEM lane quadrant of this warp
    const int m = m0 + quad * 32 + lane;
    float *out = a.partial + (int64_t)split * a.N * a.M;
    for (int c = 0; c < GG_BN; c += 16) {
      float vals[16];
      tmem_ld16(tmem + ((uint32_t)(quad * 32) << 16) + c, vals);
      if (m < a.M) {
        float *row = out + (int64_t)m * a.N + n0 + c;
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (n0 + c + q < a.N) row[q] = nkb > 0 ? vals[q] : 0.f;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

int launch_gemm_gather(const ConvGemmArgs &g, cudaStream_t st) {
  const GatherPlan p = gather_plan(g);
  CUtensorMap tmA;
  int rc = make_weight_map(&tmA, g.w, g.M, g.Kp);
  if (rc) return rc;
  if (int rc2 = ensure_smem_attr(conv_gemm_tc_gather, (int)GG_SMEM)) return rc2;
  GatherArgs a;
  a.in = static_cast<const __nv_bfloat16 *>(g.in);
  a.partial = g.partial;
  a.M = g.M; a.N = g.N; a.Kreal = g.Kreal; a.Cin = g.Cin; a.H = g.H; a.W = g.W; a.pitch = g.in_pitch;
  a.coff = g.in_coff; a.kw = g.kw; a.stride = g.stride; a.ph = g.pad_h; a.pw = g.pad_w; a.Ho = g.Ho; a.Wo = g.Wo;
  a.kb_total = p.kb_total; a.kb_per_split = p.kb_per_split;
  dim3 grid(p.m_tiles, p.n_tiles, p.splits);
  conv_gemm_tc_gather<<<grid, GG_THREADS, GG_SMEM, st>>>(tmA, a);
  AURAS_LAUNCHED("conv_gemm_tc_gather");
  return AURAS_OK;
}

}  // namespace auras
