// Persistent DP-T denoise iteration (Diffusion Policy's TransformerForDiffusion,
// BASELINE configs[3]), sm_100a.
//
// The launch-per-layer program (dpt.cu + the conv engine, ~110 launches per
// iteration) spends ~6 us per launch on 128 x 256 GEMMs that take well under a
// microsecond of tensor time: at one frame of eight samples the iteration is
// launch- and latency-bound, not FLOP- or byte-bound (its 18 MB of bf16 weights
// stay L2-resident).  Here ONE launch of ONE 8-CTA cluster runs the whole
// iteration for up to 8 samples (128 action tokens) as a fixed program of
// phases separated by cluster barriers:
//
//   GEMM  : D[128 tokens][N] = A[128][K] W[N][K]^T (+ bias, GELU, residual).
//           CTA r owns columns [r N/8, (r+1) N/8): its weight slice streams
//           through a 4-stage TMA ring next to the activation k-blocks (both
//           128B-swizzled), one elected lane issues tcgen05.mma (M = 128
//           tokens, N = N/8, K = 16) into TMEM, warps 4-7 drain the
//           accumulator (tcgen05.ld), apply the epilogue and store bf16 rows.
//   LN    : LayerNorm of the residual stream, a warp per token row.
//   ATTN  : softmax(q k^T / sqrt(dh) + mask) v, a warp per (sample, head, query)
//           (causal self-attention over the 16 action tokens; cross-attention
//           over the 3 cond tokens whose K|V rows dpt_kv_gather staged).
//   UPDATE: the DDPM / DDIM step of every sample into its request lane.
//
// Activations live in global memory (L2): a phase's generic stores are made
// visible to the next phase's TMA reads by fence.proxy.async + the cluster
// barrier (release / acquire at cluster scope).  The arithmetic matches the
// launch-per-layer program (bf16 operands and stored activations, fp32
// accumulation, fp32 LayerNorm statistics, exact-erf GELU), so the two paths
// agree to bf16 rounding flips (tests/test_gpu_dpt.py).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "cluster.cuh"
#include "common.cuh"
#include "tc_util.cuh"

namespace auras {

#ifndef DP_CLUSTER
#define DP_CLUSTER 16
#endif
constexpr int DP_CL = DP_CLUSTER;             // CTAs in the cluster (16: non-portable cluster size)
constexpr int DP_THREADS = 256;               // warps 0 TMA, 1 MMA, 4-7 epilogue; all 8 in SIMT phases
constexpr int DP_STAGES = 4;
constexpr int DP_A_BYTES = 128 * 64 * 2;      // one 128-token x 64-channel activation k-block
constexpr int DP_B_MAX = 128 * 64 * 2;        // weight slice k-block, <= 128 rows
constexpr int DP_STAGE = DP_A_BYTES + DP_B_MAX;
constexpr int DP_TMEM_COLS = 128;
constexpr size_t DP_SMEM = 1024 + (size_t)DP_STAGES * DP_STAGE + 4 * DP_A_BYTES + 256;   // ring + LayerNorm'd A
constexpr int DP_MAXK = 16;                   // keys per query (horizon <= 16; 3 cond tokens)
constexpr int DP_E = 256;                     // embedding width (LayerNorm row)

enum { DP_GEMM = 0, DP_LN = 1, DP_ATTN = 2, DP_UPDATE = 3, DP_NOP = 4 };

struct alignas(64) DpGemmDev {
  CUtensorMap tmA;           // activation [128][K] bf16, box {64, 128} (unless ln_g: A = LN(ln_src))
  CUtensorMap tmB;           // weight [N][K] bf16, box {64, ncta}
  const float *bias;
  const __nv_bfloat16 *res;  // residual (may alias out: each element is read, then written, by one thread)
  __nv_bfloat16 *out;
  float *out_f32;
  int K, N, ncta, ldo, ldr, ldf, act, ctas;
  const __nv_bfloat16 *ln_src;   // optional: A = LayerNorm(ln_src [128][256]) (K = 256), computed in the phase
  const float *ln_g, *ln_b;
};

struct DpOpDev {
  int type, gemm;
  const __nv_bfloat16 *in;   // LN input / attention q
  __nv_bfloat16 *out;        // LN output / attention output
  const float *g, *b;        // LN affine
  const __nv_bfloat16 *k, *v;
  int ldi, ldo, ldk, ldv, nk, mask_off, heads, dh;
};

struct DpParams {
  long long *trace;          // optional: globaltimer after every phase barrier (CTA 0, thread 0)
  const DpOpDev *ops;
  const DpGemmDev *gemms;
  int n_ops, S, T;
  // update
  const float *eps;
  int eps_pitch;
  const int *agents, *lanes, *steps;
  float *x_lanes;
  const float *noise_lanes;
  int lanes_per_agent, horizon, adim;
  auras_sched sched;
};

__device__ __forceinline__ float dp_wsum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// LayerNorm of one 256-wide bf16 row (fp32 statistics), bf16 out.
__device__ __forceinline__ void dp_ln_row(const __nv_bfloat16 *xr, __nv_bfloat16 *yr, const float *g, const float *b,
                                          int lane) {
  float xv[DP_E / 32];
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < DP_E / 32; ++u) {
    xv[u] = __bfloat162float(xr[lane + 32 * u]);
    s += xv[u];
  }
  const float mu = dp_wsum(s) * (1.f / DP_E);
  float q = 0.f;
#pragma unroll
  for (int u = 0; u < DP_E / 32; ++u) {
    const float d = xv[u] - mu;
    q += d * d;
  }
  const float rstd = rsqrtf(dp_wsum(q) * (1.f / DP_E) + 1e-5f);
#pragma unroll
  for (int u = 0; u < DP_E / 32; ++u) {
    const int c = lane + 32 * u;
    yr[c] = __float2bfloat16_rn((xv[u] - mu) * rstd * g[c] + b[c]);
  }
}

// Attention queries [q0, q1) of the flattened (sample, head, query) space by
// one warp (dh = 64, nk <= 16 keys; key j visible to query n iff
// j <= n + mask_off), four queries at a time with their reductions
// interleaved.  Every load is issued up front (a phase runs on 16 SMs, so
// latency must not serialise): lane j holds key row j (scores), lane l holds
// value columns 2l, 2l+1 of every key (output); K / V are reloaded only when
// the (sample, head) unit changes.
constexpr int DP_QB = 4;

__device__ __forceinline__ void dp_attn_block(const DpOpDev &o, int q0, int q1, int T, int lane) {
  const int nk = o.nk, dh = 64;
  const float scale = rsqrtf((float)dh);
  int unit = -1;
  uint4 kr[8];
  float2 vc[DP_MAXK];
  for (int qi = q0; qi < q1;) {
    const int n0 = qi % T, u = qi / T, h = u % o.heads, s = u / o.heads;
    const int nq = min(min(DP_QB, q1 - qi), T - n0);    // queries of this unit in the batch
    uint32_t qw[DP_QB];
#pragma unroll
    for (int b = 0; b < DP_QB; ++b)
      qw[b] = b < nq ? *reinterpret_cast<const uint32_t *>(o.in + ((int64_t)s * T + n0 + b) * o.ldi + h * dh + 2 * lane)
                     : 0u;
    if (u != unit) {
      unit = u;
      if (lane < nk) {
        const uint4 *kp = reinterpret_cast<const uint4 *>(o.k + ((int64_t)s * nk + lane) * o.ldk + h * dh);
#pragma unroll
        for (int i = 0; i < 8; ++i) kr[i] = kp[i];
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) kr[i] = make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < DP_MAXK; ++j)
        vc[j] = j < nk ? __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(
                             o.v + ((int64_t)s * nk + j) * o.ldv + h * dh + 2 * lane))
                       : make_float2(0.f, 0.f);
    }
    // scores of key `lane` for the batch's queries
    float sc[DP_QB];
#pragma unroll
    for (int b = 0; b < DP_QB; ++b) sc[b] = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t kw[4] = {kr[i].x, kr[i].y, kr[i].z, kr[i].w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float2 kf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&kw[c]));
#pragma unroll
        for (int b = 0; b < DP_QB; ++b) {
          const uint32_t qq = __shfl_sync(0xffffffffu, qw[b], 4 * i + c);   // columns 8 i + 2 c, +1
          const float2 qf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&qq));
          sc[b] = fmaf(qf.x, kf.x, sc[b]);
          sc[b] = fmaf(qf.y, kf.y, sc[b]);
        }
      }
    }
    float mx[DP_QB], pe[DP_QB], sm[DP_QB];
#pragma unroll
    for (int b = 0; b < DP_QB; ++b) {
      sc[b] *= scale;
      mx[b] = lane < min(nk, n0 + b + o.mask_off + 1) ? sc[b] : -INFINITY;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1)
#pragma unroll
      for (int b = 0; b < DP_QB; ++b) mx[b] = fmaxf(mx[b], __shfl_xor_sync(0xffffffffu, mx[b], off));
#pragma unroll
    for (int b = 0; b < DP_QB; ++b) {
      pe[b] = lane < min(nk, n0 + b + o.mask_off + 1) ? __expf(sc[b] - mx[b]) : 0.f;
      sm[b] = pe[b];
    }
#pragma unroll
    for (int off = 16; off; off >>= 1)
#pragma unroll
      for (int b = 0; b < DP_QB; ++b) sm[b] += __shfl_xor_sync(0xffffffffu, sm[b], off);
    float ox[DP_QB], oy[DP_QB];
#pragma unroll
    for (int b = 0; b < DP_QB; ++b) { ox[b] = 0.f; oy[b] = 0.f; }
#pragma unroll
    for (int j = 0; j < DP_MAXK; ++j) {
      if (j >= nk) break;
#pragma unroll
      for (int b = 0; b < DP_QB; ++b) {
        const float pj = __shfl_sync(0xffffffffu, pe[b], j);
        ox[b] = fmaf(pj, vc[j].x, ox[b]);
        oy[b] = fmaf(pj, vc[j].y, oy[b]);
      }
    }
#pragma unroll
    for (int b = 0; b < DP_QB; ++b) {
      if (b >= nq) break;
      const float inv = 1.f / sm[b];
      *reinterpret_cast<__nv_bfloat162 *>(o.out + ((int64_t)s * T + n0 + b) * o.ldo + h * dh + 2 * lane) =
          __floats2bfloat162_rn(ox[b] * inv, oy[b] * inv);
    }
    qi += nq;
  }
}

__global__ void __launch_bounds__(DP_THREADS, 1) dpt_persist(const __grid_constant__ DpParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + DP_STAGES * DP_STAGE + 4 * DP_A_BYTES);
  uint64_t *empty = full + DP_STAGES;
  uint64_t *done = empty + DP_STAGES;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_ctarank();
  const int rows = P.S * P.T;
  if (P.trace && rank == 0 && threadIdx.x == 0) {
    long long tn;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
    P.trace[0] = tn;
  }

  if (threadIdx.x == 0) {
    for (int i = 0; i < DP_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(DP_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  int ip = 0, ic = 0, ng = 0;     // producer / consumer ring positions, GEMMs done by this CTA
  for (int oi = 0; oi < P.n_ops; ++oi) {
    const DpOpDev &o = P.ops[oi];
    if (o.type == DP_GEMM) {
      const DpGemmDev &g = P.gemms[o.gemm];
      if (rank < g.ctas) {
        const int nkb = g.K / 64, ncta = g.ncta;
        const bool lnA = g.ln_g != nullptr;                // A = LayerNorm(src) computed here, not loaded
        uint8_t *sAln = smem + DP_STAGES * DP_STAGE;       // 128 x 256 bf16, four 128B-swizzled k-blocks
        if (warp == 0 && lane == 0) {
          // ---- TMA producer: weight slice k-block (+ activation k-block) per stage
          if (!lnA) asm volatile("prefetch.tensormap [%0];" ::"l"(&g.tmA) : "memory");
          asm volatile("prefetch.tensormap [%0];" ::"l"(&g.tmB) : "memory");
          for (int kb = 0; kb < nkb; ++kb, ++ip) {
            const int st = ip % DP_STAGES;
            mbar_wait(&empty[st], ((ip / DP_STAGES) & 1) ^ 1);
            uint8_t *sa = smem + st * DP_STAGE;
            mbar_expect_tx(&full[st], (lnA ? 0 : DP_A_BYTES) + ncta * 128);
            if (!lnA) tma_load_2d(sa, &g.tmA, &full[st], kb * 64, 0);
            tma_load_2d(sa + DP_A_BYTES, &g.tmB, &full[st], kb * 64, rank * ncta);
          }
        }
        __syncwarp();
        if (lnA) {
          // ---- the A operand: LayerNorm of every token row of the residual stream, written
          //      straight into the UMMA layout (K-major, 128B swizzle: 16-byte chunk j of row r
          //      at chunk j ^ (r & 7)); lane l owns columns 8 l .. 8 l + 7
          // this warp's 16 rows in two batches of 8: a batch's loads are issued together and its
          // warp reductions interleaved (independent chains)
          const float4 g0 = *reinterpret_cast<const float4 *>(g.ln_g + 8 * lane);
          const float4 g1 = *reinterpret_cast<const float4 *>(g.ln_g + 8 * lane + 4);
          const float4 b0 = *reinterpret_cast<const float4 *>(g.ln_b + 8 * lane);
          const float4 b1 = *reinterpret_cast<const float4 *>(g.ln_b + 8 * lane + 4);
          const float ga[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
          const float ba[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
          for (int hb = 0; hb < 2; ++hb) {
          uint4 xin4[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = warp + 8 * (8 * hb + i);
            xin4[i] = r < rows ? *reinterpret_cast<const uint4 *>(g.ln_src + (int64_t)r * DP_E + 8 * lane)
                               : make_uint4(0, 0, 0, 0);
          }
          // statistics of the 16 rows with their warp reductions interleaved (independent chains)
          float mu[8], rs[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t xw[4] = {xin4[i].x, xin4[i].y, xin4[i].z, xin4[i].w};
            float sm = 0.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&xw[k]));
              sm += f.x + f.y;
            }
            mu[i] = sm;
          }
#pragma unroll
          for (int off = 16; off; off >>= 1)
#pragma unroll
            for (int i = 0; i < 8; ++i) mu[i] += __shfl_xor_sync(0xffffffffu, mu[i], off);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            mu[i] *= 1.f / DP_E;
            const uint32_t xw[4] = {xin4[i].x, xin4[i].y, xin4[i].z, xin4[i].w};
            float q = 0.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&xw[k]));
              q += (f.x - mu[i]) * (f.x - mu[i]) + (f.y - mu[i]) * (f.y - mu[i]);
            }
            rs[i] = q;
          }
#pragma unroll
          for (int off = 16; off; off >>= 1)
#pragma unroll
            for (int i = 0; i < 8; ++i) rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], off);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = warp + 8 * (8 * hb + i);
            if (r >= rows) break;
            const float rstd = rsqrtf(rs[i] * (1.f / DP_E) + 1e-5f);
            const uint32_t xw[4] = {xin4[i].x, xin4[i].y, xin4[i].z, xin4[i].w};
            uint32_t yw[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&xw[k]));
              const __nv_bfloat162 h2 = __floats2bfloat162_rn((f.x - mu[i]) * rstd * ga[2 * k] + ba[2 * k],
                                                              (f.y - mu[i]) * rstd * ga[2 * k + 1] + ba[2 * k + 1]);
              yw[k] = *reinterpret_cast<const uint32_t *>(&h2);
            }
            const int kb = lane >> 3, ch = lane & 7;          // k-block of these 8 columns, chunk within the row
            *reinterpret_cast<uint4 *>(sAln + kb * DP_A_BYTES + r * 128 + ((ch ^ (r & 7)) << 4)) =
                make_uint4(yw[0], yw[1], yw[2], yw[3]);
          }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncthreads();
        }
        if (warp == 1) {
          // ---- MMA issuer
          const uint32_t idesc = umma_idesc(ncta);
          for (int kb = 0; kb < nkb; ++kb, ++ic) {
            const int st = ic % DP_STAGES;
            mbar_wait(&full[st], (ic / DP_STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = lnA ? smem_u32(sAln + kb * DP_A_BYTES) : smem_u32(smem + st * DP_STAGE);
            const uint32_t sb = smem_u32(smem + st * DP_STAGE) + DP_A_BYTES;
            umma_kblock_warp(tmem, umma_desc(sa), umma_desc(sb), idesc, kb > 0 ? 1u : 0u);
            umma_commit_warp(&empty[st]);
            if (kb == nkb - 1) umma_commit_warp(done);
            __syncwarp();
          }
        }
        {
          // ---- epilogue, all 8 warps: token row = TMEM lane (warp % 4 quadrant), warps
          //      0-3 / 4-7 take alternate 16-column chunks
          const int row = (warp & 3) * 32 + lane, grp = warp >> 2;
          const int n0 = rank * ncta;
          // residual of this warp's first two chunks while the MMAs run
          uint4 rpre[4];
          const bool pre = g.res && row < rows && n0 + ncta <= g.N;
          if (pre) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int c = 16 * (grp + 2 * k);
              const uint4 *rp = reinterpret_cast<const uint4 *>(g.res + (int64_t)row * g.ldr + n0 + c);
              rpre[2 * k] = c < ncta ? rp[0] : make_uint4(0, 0, 0, 0);
              rpre[2 * k + 1] = c < ncta ? rp[1] : make_uint4(0, 0, 0, 0);
            }
          }
          mbar_wait(done, ng & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          for (int c = 16 * grp, k = 0; c < ncta; c += 32, ++k) {
            float v[16];
            tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + c, v);
            if (row >= rows) continue;
            const int nb = n0 + c;
            if (nb + 16 <= g.N) {
#pragma unroll
              for (int i = 0; i < 16; i += 4) {
                const float4 bb = *reinterpret_cast<const float4 *>(g.bias + nb + i);
                v[i] += bb.x; v[i + 1] += bb.y; v[i + 2] += bb.z; v[i + 3] += bb.w;
              }
              if (g.act)
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = activate(v[i], g.act);
              if (g.res) {
                uint4 r0, r1;
                if (pre && k < 2) {
                  r0 = k == 0 ? rpre[0] : rpre[2];
                  r1 = k == 0 ? rpre[1] : rpre[3];
                } else {
                  const uint4 *rp = reinterpret_cast<const uint4 *>(g.res + (int64_t)row * g.ldr + nb);
                  r0 = rp[0];
                  r1 = rp[1];
                }
                const uint32_t rw[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&rw[i]));
                  v[2 * i] += f.x;
                  v[2 * i + 1] += f.y;
                }
              }
              if (g.out) {
                uint32_t ow[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
                  ow[i] = *reinterpret_cast<const uint32_t *>(&h2);
                }
                uint4 *op = reinterpret_cast<uint4 *>(g.out + (int64_t)row * g.ldo + nb);
                op[0] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
                op[1] = make_uint4(ow[4], ow[5], ow[6], ow[7]);
              }
              if (g.out_f32)
#pragma unroll
                for (int i = 0; i < 16; ++i) g.out_f32[(int64_t)row * g.ldf + nb + i] = v[i];
            } else {
              // ragged tail (the 7-wide action head): scalar, columns < N only
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const int n = nb + i;
                if (n >= g.N) continue;
                float x = activate(v[i] + g.bias[n], g.act);
                if (g.res) x += __bfloat162float(g.res[(int64_t)row * g.ldr + n]);
                if (g.out) g.out[(int64_t)row * g.ldo + n] = __float2bfloat16_rn(x);
                if (g.out_f32) g.out_f32[(int64_t)row * g.ldf + n] = x;
              }
            }
          }
        }
        ++ng;
      }
    } else if (o.type == DP_LN) {
      for (int r = rank * 8 + warp; r < rows; r += DP_CL * 8)
        dp_ln_row(o.in + (int64_t)r * o.ldi, o.out + (int64_t)r * o.ldo, o.g, o.b, lane);
    } else if (o.type == DP_ATTN) {
      // contiguous query ranges over the 64 warps of the cluster
      const int items = P.S * o.heads * P.T, per = (items + DP_CL * 8 - 1) / (DP_CL * 8);
      const int gw = rank * 8 + warp;
      dp_attn_block(o, min(items, gw * per), min(items, (gw + 1) * per), P.T, lane);
    } else if (o.type == DP_NOP) {
      // timing probe: a phase with no work (the cost of the phase boundary alone)
    } else {
      // ---- DDPM / DDIM update of sample s (dpt.cu dpt_update_kernel arithmetic)
      const auras_sched &sch = P.sched;
      for (int s = rank; s < P.S; s += DP_CL) {
        const int agent = P.agents[s], ln = P.lanes[s], i = P.steps[s];
        float *x = P.x_lanes + ((int64_t)agent * P.lanes_per_agent + ln) * P.horizon * P.adim;
        const float *z = P.noise_lanes ? P.noise_lanes + (((int64_t)agent * P.lanes_per_agent + ln) * sch.n_steps + i) *
                                                             P.horizon * P.adim
                                       : nullptr;
        const float sab = sch.sqrt_ab[i], s1m = sch.sqrt_1mab[i];
        const float cx0 = sch.c_x0[i], cxt = sch.c_xt[i], ceps = sch.c_eps[i], sig = sch.sigma[i];
        for (int e = threadIdx.x; e < P.horizon * P.adim; e += DP_THREADS) {
          const int t = e / P.adim, a = e % P.adim;
          const float xt = x[e], ep = P.eps[((int64_t)s * P.horizon + t) * P.eps_pitch + a];
          float x0 = (xt - s1m * ep) / sab;
          if (sch.clip_sample) x0 = fminf(fmaxf(x0, -1.f), 1.f);
          float nx = cx0 * x0 + cxt * xt + ceps * ep;
          if (sch.ddpm && z) nx += sig * z[e];
          x[e] = nx;
        }
      }
    }
    // phase boundary: generic stores visible to the next phase's TMA reads, TMEM drained
    fence_proxy_async();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (P.trace && rank == 0 && threadIdx.x == 0) {
      long long tn;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
      P.trace[oi + 1] = tn;
    }
  }
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(DP_TMEM_COLS));
}

struct DpPlan {
  DpOpDev *ops = nullptr;
  DpGemmDev *gemms = nullptr;
  long long *trace = nullptr;          // AURAS_DPT_TRACE: per-phase timestamps of the last run
  int n_ops = 0, n_gemms = 0, T = 16;
};

static int dp_map(CUtensorMap *tm, const void *base, int K, int rows, int box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return AURAS_E_CUDA; }
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("dpt_persist map: CUresult %d", (int)r); return AURAS_E_CUDA; }
  return AURAS_OK;
}

}  // namespace auras

using namespace auras;

extern "C" {

int auras_dpt_persist_build(const auras_dpt_gemm *gemms, int n_gemms, const auras_dpt_op *ops, int n_ops, int T,
                            void **plan_out) {
  if (!gemms || !ops || n_gemms < 1 || n_ops < 1 || !plan_out || T < 1 || T > DP_MAXK || T * 8 > 128) {
    // (T = horizon <= 16 keys of the causal self-attention)
    set_error("dpt_persist_build: bad arguments");
    return AURAS_E_ARG;
  }
  std::vector<DpGemmDev> hg(n_gemms);
  for (int i = 0; i < n_gemms; ++i) {
    const auras_dpt_gemm &s = gemms[i];
    DpGemmDev &d = hg[i];
    memset(&d, 0, sizeof(d));
    const int ctas = s.N <= 16 ? 1 : DP_CL;
    const int ncta = ctas == 1 ? 16 : s.N / DP_CL;
    if (s.K % 64 || s.act_rows != 128 || (ctas > 1 && (s.N % DP_CL || ncta % 16 || ncta > 128)) ||
        (s.out && s.ldo % 8) || (s.res && s.ldr % 8)) {
      set_error("dpt_persist_build: gemm %d shape K=%d N=%d rows=%d", i, s.K, s.N, s.act_rows);
      return AURAS_E_ARG;
    }
    if (s.ln_g && (s.K != DP_E || !s.ln_src || !s.ln_b)) {
      set_error("dpt_persist_build: gemm %d LayerNorm'd A needs K = 256", i);
      return AURAS_E_ARG;
    }
    if (!s.ln_g)
      if (int rc = dp_map(&d.tmA, s.act, s.K, s.act_rows, 128)) return rc;
    d.ln_src = static_cast<const __nv_bfloat16 *>(s.ln_src);
    d.ln_g = s.ln_g;
    d.ln_b = s.ln_b;
    if (int rc = dp_map(&d.tmB, s.w, s.K, s.N, ncta)) return rc;
    d.bias = s.bias;
    d.res = static_cast<const __nv_bfloat16 *>(s.res);
    d.out = static_cast<__nv_bfloat16 *>(s.out);
    d.out_f32 = s.out_f32;
    d.K = s.K; d.N = s.N; d.ncta = ncta; d.ctas = ctas;
    d.ldo = s.ldo; d.ldr = s.ldr; d.ldf = s.ldf; d.act = s.act_fn;
  }
  std::vector<DpOpDev> ho(n_ops);
  for (int i = 0; i < n_ops; ++i) {
    const auras_dpt_op &s = ops[i];
    DpOpDev &d = ho[i];
    memset(&d, 0, sizeof(d));
    d.type = s.type; d.gemm = s.gemm;
    d.in = static_cast<const __nv_bfloat16 *>(s.in);
    d.out = static_cast<__nv_bfloat16 *>(s.out);
    d.g = s.g; d.b = s.b;
    d.k = static_cast<const __nv_bfloat16 *>(s.k);
    d.v = static_cast<const __nv_bfloat16 *>(s.v);
    d.ldi = s.ldi; d.ldo = s.ldo; d.ldk = s.ldk; d.ldv = s.ldv;
    d.nk = s.nk; d.mask_off = s.mask_off; d.heads = s.heads; d.dh = s.dh;
    if ((s.type == DP_GEMM && (s.gemm < 0 || s.gemm >= n_gemms)) || (s.type == DP_ATTN && (s.nk > DP_MAXK || s.dh != 64)) ||
        s.type < 0 || s.type > DP_NOP) {
      set_error("dpt_persist_build: op %d", i);
      return AURAS_E_ARG;
    }
  }
  DpPlan *p = new DpPlan;
  p->n_ops = n_ops;
  p->n_gemms = n_gemms;
  p->T = T;
  if (cudaMalloc(&p->ops, sizeof(DpOpDev) * n_ops) != cudaSuccess ||
      cudaMalloc(&p->gemms, sizeof(DpGemmDev) * n_gemms) != cudaSuccess) {
    cudaFree(p->ops);
    delete p;
    return cuda_check(cudaGetLastError(), "dpt_persist alloc");
  }
  cudaMemcpy(p->ops, ho.data(), sizeof(DpOpDev) * n_ops, cudaMemcpyHostToDevice);
  cudaMemcpy(p->gemms, hg.data(), sizeof(DpGemmDev) * n_gemms, cudaMemcpyHostToDevice);
  if (getenv("AURAS_DPT_TRACE")) cudaMalloc(&p->trace, sizeof(long long) * (n_ops + 1));
  *plan_out = p;
  return cuda_check(cudaGetLastError(), "dpt_persist_build");
}

int auras_dpt_persist_run(void *plan, int S, const float *eps, int eps_pitch, const int *agents, const int *lanes,
                          const int *steps, float *x_lanes, const float *noise_lanes, int lanes_per_agent,
                          int horizon, int adim, const auras_sched *sched, void *stream) {
  DpPlan *p = static_cast<DpPlan *>(plan);
  if (!p || !sched || S < 1 || S * p->T > 128 || horizon != p->T) {
    set_error("dpt_persist_run: bad arguments (S=%d)", S);
    return AURAS_E_ARG;
  }
  if (int rc = ensure_smem_attr(dpt_persist, (int)DP_SMEM)) return rc;
  if (DP_CL > 8) {
    static bool np = false;
    if (!np) {
      AURAS_CUDA(cudaFuncSetAttribute(dpt_persist, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      np = true;
    }
  }
  DpParams P;
  memset(&P, 0, sizeof(P));
  P.trace = p->trace;
  P.ops = p->ops; P.gemms = p->gemms; P.n_ops = p->n_ops; P.S = S; P.T = p->T;
  P.eps = eps; P.eps_pitch = eps_pitch;
  P.agents = agents; P.lanes = lanes; P.steps = steps;
  P.x_lanes = x_lanes; P.noise_lanes = noise_lanes;
  P.lanes_per_agent = lanes_per_agent; P.horizon = horizon; P.adim = adim;
  P.sched = *sched;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(DP_CL);
  cfg.blockDim = dim3(DP_THREADS);
  cfg.dynamicSmemBytes = DP_SMEM;
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = DP_CL;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  AURAS_CUDA(cudaLaunchKernelEx(&cfg, dpt_persist, P));
  return AURAS_OK;
}

// Diagnostics (AURAS_DPT_TRACE set at build): per-phase globaltimer stamps of
// the last run, n_ops + 1 values.  Returns the count copied.
int auras_dpt_persist_trace(void *plan, long long *out, int n) {
  DpPlan *p = static_cast<DpPlan *>(plan);
  if (!p || !p->trace || !out) return 0;
  const int m = std::min(n, p->n_ops + 1);
  cudaMemcpy(out, p->trace, sizeof(long long) * m, cudaMemcpyDeviceToHost);
  return m;
}

void auras_dpt_persist_free(void *plan) {
  DpPlan *p = static_cast<DpPlan *>(plan);
  if (!p) return;
  cudaFree(p->trace);
  cudaFree(p->ops);
  cudaFree(p->gemms);
  delete p;
}

}  // extern "C"
