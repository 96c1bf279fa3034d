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
constexpr int DP_CT = 256;                    // compute warps 0-7: LN / epilogue / SIMT phases; warp 1 issues the MMAs
constexpr int DP_THREADS = DP_CT + 32;        // + warp 8: the TMA producer (never writes generic memory, so it
                                              //   never executes a proxy fence behind its own bulk loads)
constexpr int DP_STAGES = 8;                  // ring depth: the K = 1024 GEMM streams 16 k-blocks
constexpr int DP_A_BYTES = 128 * 64 * 2;      // one 128-token x 64-channel activation k-block
constexpr int DP_B_BYTES = 64 * 64 * 2;       // weight slice k-block, <= 64 rows (N <= 64 x 16)
constexpr int DP_R_BYTES = 128 * 16 * 2;      // residual slice (TMA'd when the slice is 16 columns)
// shared memory: A ring [8][16 KB] | B ring [8][8 KB] | residual slice | barriers | metadata.  The
// LayerNorm'd A tile (4 k-blocks) aliases A-ring stages 0-3: a LayerNorm GEMM loads no A blocks, and
// the previous GEMM's MMAs completed before the phase barrier.
constexpr size_t DP_B_OFF = (size_t)DP_STAGES * DP_A_BYTES;
constexpr size_t DP_R_OFF = DP_B_OFF + (size_t)DP_STAGES * DP_B_BYTES;
constexpr size_t DP_BAR_OFF = DP_R_OFF + DP_R_BYTES;
constexpr int DP_TMEM_COLS = 128;
// Program metadata and this CTA's bias slices are staged in shared memory at launch: every
// phase barrier (barrier.cluster acquire) invalidates L1, so a per-phase read of the op
// table from global memory would be an L2 round trip (~1 us) on the critical path of
// every one of the ~67 phases.
constexpr int DP_MAX_OPS = 88, DP_MAX_GEMMS = 56, DP_BIAS_SLAB = 3072;
constexpr size_t DP_STAT_OFF = DP_BAR_OFF + 256;  // per-row (mean, rstd) of the tile a LayerNorm phase applies
constexpr size_t DP_SAMP_OFF = DP_STAT_OFF + 128 * 8;   // agents / lanes / steps of the launch (<= 128 each)
constexpr size_t DP_META_OFF = DP_SAMP_OFF + 3 * 128 * 4;
constexpr size_t DP_META_BYTES = (size_t)DP_MAX_OPS * 112 + DP_MAX_GEMMS * 96 + DP_BIAS_SLAB * 4;
constexpr size_t DP_SMEM = 1024 + DP_META_OFF + DP_META_BYTES;   // ring + LayerNorm'd A + barriers + metadata
static_assert(DP_SMEM <= 232448, "dpt_persist shared memory");
constexpr int DP_MAXK = 16;                   // keys per query (horizon <= 16; 3 cond tokens)
constexpr int DP_E = 256;                     // embedding width (LayerNorm row)

enum { DP_GEMM = 0, DP_LN = 1, DP_ATTN = 2, DP_UPDATE = 3, DP_NOP = 4, DP_PREP = 5, DP_XATTN = 6 };
constexpr int DP_XK = 4, DP_XH = 4;           // folded cross-attention: memory tokens / heads (at most)

struct alignas(64) DpGemmDev {
  CUtensorMap tmA;           // activation [128][K] bf16, box {64, 128} (unless ln_g: A = LN(ln_src))
  CUtensorMap tmB;           // weight [N][K] bf16, box {64, ncta}
  CUtensorMap tmR;           // residual [128][N] bf16 (pitch ldr), box {ncta, 128}, unswizzled (when rtma)
  const float *bias;
  const __nv_bfloat16 *res;  // residual (may alias out: each element is read, then written, by one thread)
  __nv_bfloat16 *out;
  float *out_f32;
  int K, N, ncta, ldo, ldr, ldf, act, ctas;
  const __nv_bfloat16 *ln_src;   // optional: A = LayerNorm(ln_src [128][256]) (K = 256), computed in the phase
  const float *ln_g, *ln_b;
  int boff;                  // this GEMM's bias slice in the shared-memory slab
  int rtma;                  // the residual slice is TMA'd into shared memory (16-column slices)
  int stats_out;             // epilogue writes per-row (mean, M2) of its 16 stored columns to P.stats
  int stats_in;              // the LayerNorm'd A uses the row statistics the previous writer left in P.stats
};

// The GEMM fields the phases read (no tensor maps: those stay in global memory for the TMA unit).
struct DpGemmMeta {
  const __nv_bfloat16 *res;
  __nv_bfloat16 *out;
  float *out_f32;
  const __nv_bfloat16 *ln_src;
  const float *ln_g, *ln_b;
  int K, N, ncta, ldo, ldr, ldf, act, ctas, boff, rtma, stats_out, stats_in;
};
static_assert(sizeof(DpGemmMeta) <= 96, "DpGemmMeta");

struct DpOpDev {
  int type, gemm;
  const __nv_bfloat16 *in;   // LN input / attention q
  __nv_bfloat16 *out;        // LN output / attention output
  const float *g, *b;        // LN affine
  const __nv_bfloat16 *k, *v;
  int ldi, ldo, ldk, ldv, nk, mask_off, heads, dh;
  // GEMM ops: parities of this op's lnbar (bit 0) / resbar (bit 1) / done (bit 2) phase and its
  // first ring job, [0] for CTAs 1.., [1] for CTA 0 (which also runs the single-CTA GEMMs);
  // host-computed so that no counter lives across phases (168 registers: it would be spilled)
  int par[2], job[2];
  int gather;                // attention: k / v row 0 from the time table (by the sample's step), rows
                             // 1 .. nk - 1 from the frame's observation rows (by its agent);
                             // GEMM: 2 = scheduler update in the epilogue (fuse_update), 3 = A tile
                             // built from the request lanes (a_from_lanes)
  int ksplit;                // GEMM: K split over the cluster halves (auras_dpt_gemm.ksplit)
};
static_assert(sizeof(DpOpDev) == 112, "DpOpDev");

// Attention operand maps (128B-swizzled boxes {64, rows}: q {dh, T}, k / v {dh, nk}).
struct alignas(64) DpAttnDev {
  CUtensorMap tq, tk, tv;
  CUtensorMap tk2, tv2;      // gather mode: the observation rows (tk / tv: the time table, 1-row boxes)
};
constexpr int DP_ATT_UNIT = 3 * 2048;         // q, k, v tiles of one (sample, head) unit, <= 16 rows each
constexpr int DP_ATT_SLOTS = 4;               // units per CTA (S * heads <= 4 * DP_CL)
constexpr size_t DP_ATT_OFF = 4 * (size_t)DP_A_BYTES;   // A-ring stages 4-5: idle outside GEMM phases

struct DpParams {
  long long *trace;          // optional: globaltimer after every phase barrier (CTA 0, thread 0)
  const DpOpDev *ops;
  const DpGemmDev *gemms;
  const DpAttnDev *attns;    // per attention op (DpOpDev::gemm indexes it)
  int n_ops, n_gemms, S, T;
  int dbg;                   // AURAS_DPT_DBG timing variants (0 in production)
  int pf;                    // weight prefetch across phase barriers (0: only in the GEMM's own phase)
  int mslices;               // CTAs that load (and multicast) a slice of each activation block
  float2 *stats;             // [128 rows][DP_CL slices] (mean, M2) of the residual stream's last writer
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

// (noinline: its ~130 live registers must not push the persistent loop's state into local memory)
__device__ __noinline__ void dp_attn_block(const DpOpDev &o, int q0, int q1, int T, int lane, long long *stamp) {
  const int nk = o.nk, dh = 64;
  const float scale = rsqrtf((float)dh);
  int unit = -1;
  uint4 kr[8];
  __nv_bfloat162 vc[DP_MAXK];    // value columns 2 lane, 2 lane + 1 of every key (bf16 pairs: half the registers)
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
        vc[j] = j < nk ? *reinterpret_cast<const __nv_bfloat162 *>(o.v + ((int64_t)s * nk + j) * o.ldv + h * dh + 2 * lane)
                       : __floats2bfloat162_rn(0.f, 0.f);
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
    if (stamp && qi == q0) stamp[0] = clock64();
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
      const float2 vf = __bfloat1622float2(vc[j]);
#pragma unroll
      for (int b = 0; b < DP_QB; ++b) {
        const float pj = __shfl_sync(0xffffffffu, pe[b], j);
        ox[b] = fmaf(pj, vf.x, ox[b]);
        oy[b] = fmaf(pj, vf.y, oy[b]);
      }
    }
#pragma unroll
    for (int b = 0; b < DP_QB; ++b) {
      if (b >= nq) break;
      const float inv = __fdividef(1.f, sm[b]);     // sm >= 1 (the row max contributes exp(0))
      *reinterpret_cast<__nv_bfloat162 *>(o.out + ((int64_t)s * T + n0 + b) * o.ldo + h * dh + 2 * lane) =
          __floats2bfloat162_rn(ox[b] * inv, oy[b] * inv);
    }
    qi += nq;
  }
  if (stamp) stamp[1] = clock64();
}

// ---- folded cross-attention block (DP_XATTN; tables from auras_dpt_xfold).
// The decoder's memory is 1 + n_obs tokens, so the query projection folds into
// the keys (score[h][j] = xhat . a'[h][j] + c'[h][j], the LayerNorm affine
// included) and the output projection into the values (ca_out(attn) =
// sum_{h,j} p[h][j] U'[h][j], ca_out's bias spread over U'): the ca_in GEMM,
// the attention and the ca_out GEMM become one SIMT phase of 4 NK dot products
// and 4 NK axpys per token row (4 heads).  The CTA's 8 rows (one warp each)
// belong to one sample (T % 8 == 0, checked at build): its NK table blocks are
// staged into shared memory once (every load in flight at once: one L2 round
// trip after the phase barrier).  Lane l owns columns 4l..4l+3 and 128+4l..+3,
// so every float4 table read of a warp is one contiguous 512-byte run (no bank
// conflicts: 8 warps x the whole table is the phase's shared-memory traffic).
// The 4 NK partial scores are summed by a transposing butterfly (16 shuffles:
// lane l ends with the score of (j, h) = ((l >> 1) / 4, (l >> 1) % 4)), the
// softmax over j runs across lanes l, l ^ 8, l ^ 16, l ^ 24, and the
// probabilities are broadcast back for the combination.  The row is updated in
// place; either (mean, M2) slice partials go to a following LayerNorm'd GEMM
// (stats_in), or (o.g set) the warp, which holds the whole updated row, writes
// its LayerNorm to o.out for a plain-A GEMM.
template <int NK>
__device__ __noinline__ void dp_xattn(const DpOpDev &o, int r0, int rows, int T, const int *s_agent,
                                      const int *s_step, float *stab, float2 *stats, int warp, int lane,
                                      long long *stamp, uint64_t *tbar) {
  constexpr int H = DP_XH;                                     // (checked at build)
  constexpr int SB = 2 * H * DP_E + 4;                         // staged floats per memory token (a', U', c', pad)
  const int tid = warp * 32 + lane;
  const int sidx = r0 / T;
  const int step = s_step[sidx], obs0 = s_agent[sidx] * (NK - 1);
  const int r = r0 + warp;
  const bool live = r < rows;
  const int q0 = 4 * lane, q1 = 128 + 4 * lane;
  // optional: the next LayerNorm (o.g, o.b) of the updated row into o.out -- the following GEMM
  // then takes a plain A operand instead of normalising its tile in its own phase (affine loads
  // issued now, off the critical path)
  const bool lnout = o.g != nullptr;
  float4 lg0 = make_float4(0.f, 0.f, 0.f, 0.f), lg1 = lg0, lb0 = lg0, lb1 = lg0;
  if (lnout && live) {
    lg0 = *reinterpret_cast<const float4 *>(o.g + q0);
    lg1 = *reinterpret_cast<const float4 *>(o.g + q1);
    lb0 = *reinterpret_cast<const float4 *>(o.b + q0);
    lb1 = *reinterpret_cast<const float4 *>(o.b + q1);
  }
  uint2 xa = make_uint2(0, 0), xb = make_uint2(0, 0);
  if (live) {
    xa = *reinterpret_cast<const uint2 *>(o.in + (int64_t)r * o.ldi + q0);
    xb = *reinterpret_cast<const uint2 *>(o.in + (int64_t)r * o.ldi + q1);
  }
  if (tbar) {
    // the tables were prefetched during the previous phase (producer warp, bulk copies)
    mbar_wait(tbar, o.par[0] & 1);
  } else {
    constexpr int Q4 = SB / 4, N4 = NK * Q4;
    constexpr int PER = (N4 + DP_CT - 1) / DP_CT;
    const float *tk = reinterpret_cast<const float *>(o.k) + (int64_t)step * o.ldk;
    const float *tv = reinterpret_cast<const float *>(o.v) + (int64_t)obs0 * o.ldv;
    float4 tmp[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = tid + k * DP_CT;
      if (i < N4) {
        const int j = i / Q4, c = i - j * Q4;
        const float *src = j == 0 ? tk : tv + (int64_t)(j - 1) * o.ldv;
        tmp[k] = reinterpret_cast<const float4 *>(src)[c];
      }
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = tid + k * DP_CT;
      if (i < N4) reinterpret_cast<float4 *>(stab)[i] = tmp[k];
    }
  }
  if (stamp && tid == 0) stamp[0] = clock64();
  if (!tbar) named_sync(1, DP_CT);
  if (stamp && tid == 0) stamp[1] = clock64();
  if (!live) return;
  const int t = r - sidx * T;
  float x[8], xh[8];
  {
    const uint32_t xw[4] = {xa.x, xa.y, xb.x, xb.y};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&xw[i]));
      x[2 * i] = f.x;
      x[2 * i + 1] = f.y;
    }
  }
  float sm = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) sm += x[i];
  const float mu = dp_wsum(sm) * (1.f / DP_E);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) q = fmaf(x[i] - mu, x[i] - mu, q);
  const float rstd = rsqrtf(dp_wsum(q) * (1.f / DP_E) + 1e-5f);
#pragma unroll
  for (int i = 0; i < 8; ++i) xh[i] = (x[i] - mu) * rstd;
  // partial scores of the 16 (j, h) slots (slots j >= NK stay 0)
  float v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int j = k >> 2, h = k & 3;
    float a = 0.f;
    if (j < NK) {
      const float *ap = stab + j * SB + h * DP_E;
      const float4 a0 = *reinterpret_cast<const float4 *>(ap + q0);
      const float4 a1 = *reinterpret_cast<const float4 *>(ap + q1);
      a = xh[0] * a0.x + xh[1] * a0.y + xh[2] * a0.z + xh[3] * a0.w + xh[4] * a1.x + xh[5] * a1.y + xh[6] * a1.z +
          xh[7] * a1.w;
    }
    v[k] = a;
  }
  // transposing butterfly: after the xor-16/8/4/2 halvings lane l holds slot l >> 1 summed over
  // its 16 lanes, the xor-1 step completes it
  {
    const bool b4 = lane & 16;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float send = b4 ? v[i] : v[i + 8];
      const float keep = b4 ? v[i + 8] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    const bool b3 = lane & 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float send = b3 ? v[i] : v[i + 4];
      const float keep = b3 ? v[i + 4] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    const bool b2 = lane & 4;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float send = b2 ? v[i] : v[i + 2];
      const float keep = b2 ? v[i + 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    const bool b1 = lane & 2;
    {
      const float send = b1 ? v[0] : v[1];
      const float keep = b1 ? v[1] : v[0];
      v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  }
  if (stamp && tid == 0) stamp[2] = clock64();
  // this lane's slot: memory token j = slot / 4 (visible iff j < NK and j <= t + mask_off), head slot % 4;
  // the head's NK slots sit on lanes l, l ^ 8, l ^ 16, l ^ 24
  const int slot = lane >> 1, jj = slot >> 2;
  const bool vis = jj < NK && jj <= t + o.mask_off;
  const float sc = vis ? v[0] + stab[jj * SB + 2 * H * DP_E + (slot & 3)] : -INFINITY;
  float mx = fmaxf(sc, __shfl_xor_sync(0xffffffffu, sc, 8));
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
  const float e = vis ? __expf(sc - mx) : 0.f;
  float den = e + __shfl_xor_sync(0xffffffffu, e, 8);
  den += __shfl_xor_sync(0xffffffffu, den, 16);
  const float pr = e * __fdividef(1.f, den);                   // (den >= 1: the max contributes exp(0))
  // h += sum p U' (bf16 residual stream, fp32 combination), in place
  float y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) y[i] = x[i];
#pragma unroll
  for (int k = 0; k < 4 * NK; ++k) {
    const float pk = __shfl_sync(0xffffffffu, pr, 2 * k);
    const float *up = stab + (k >> 2) * SB + H * DP_E + (k & 3) * DP_E;
    const float4 u0 = *reinterpret_cast<const float4 *>(up + q0);
    const float4 u1 = *reinterpret_cast<const float4 *>(up + q1);
    y[0] = fmaf(pk, u0.x, y[0]); y[1] = fmaf(pk, u0.y, y[1]); y[2] = fmaf(pk, u0.z, y[2]); y[3] = fmaf(pk, u0.w, y[3]);
    y[4] = fmaf(pk, u1.x, y[4]); y[5] = fmaf(pk, u1.y, y[5]); y[6] = fmaf(pk, u1.z, y[6]); y[7] = fmaf(pk, u1.w, y[7]);
  }
  uint32_t ow[4];
  float f[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 h2 = __floats2bfloat162_rn(y[2 * i], y[2 * i + 1]);
    ow[i] = *reinterpret_cast<const uint32_t *>(&h2);
    const float2 g2 = __bfloat1622float2(h2);
    f[2 * i] = g2.x;
    f[2 * i + 1] = g2.y;
  }
  if (lnout) {
    // the row back into the residual stream (in), its LayerNorm into out (fp32 statistics of the
    // stored bf16 values, as the LayerNorm'd GEMM path computes them)
    __nv_bfloat16 *hr = const_cast<__nv_bfloat16 *>(o.in) + (int64_t)r * o.ldi;
    *reinterpret_cast<uint2 *>(hr + q0) = make_uint2(ow[0], ow[1]);
    *reinterpret_cast<uint2 *>(hr + q1) = make_uint2(ow[2], ow[3]);
    float s2 = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s2 += f[i];
    const float m2 = dp_wsum(s2) * (1.f / DP_E);
    float v2 = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) v2 = fmaf(f[i] - m2, f[i] - m2, v2);
    const float rs2 = rsqrtf(dp_wsum(v2) * (1.f / DP_E) + 1e-5f);
    const float ga[8] = {lg0.x, lg0.y, lg0.z, lg0.w, lg1.x, lg1.y, lg1.z, lg1.w};
    const float ba[8] = {lb0.x, lb0.y, lb0.z, lb0.w, lb1.x, lb1.y, lb1.z, lb1.w};
    uint32_t lw[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 h2 = __floats2bfloat162_rn((f[2 * i] - m2) * rs2 * ga[2 * i] + ba[2 * i],
                                                      (f[2 * i + 1] - m2) * rs2 * ga[2 * i + 1] + ba[2 * i + 1]);
      lw[i] = *reinterpret_cast<const uint32_t *>(&h2);
    }
    *reinterpret_cast<uint2 *>(o.out + (int64_t)r * o.ldo + q0) = make_uint2(lw[0], lw[1]);
    *reinterpret_cast<uint2 *>(o.out + (int64_t)r * o.ldo + q1) = make_uint2(lw[2], lw[3]);
    if (stamp && tid == 0) stamp[3] = clock64();
    return;
  }
  *reinterpret_cast<uint2 *>(o.out + (int64_t)r * o.ldo + q0) = make_uint2(ow[0], ow[1]);
  *reinterpret_cast<uint2 *>(o.out + (int64_t)r * o.ldo + q1) = make_uint2(ow[2], ow[3]);
  if (stamp && tid == 0) stamp[3] = clock64();
  // (mean, M2) of each 16-column slice of the stored row: slice lane / 4 from the first quads of
  // lanes 4k..4k+3, slice 8 + lane / 4 from their second quads (equal-count Chan combinations)
  float mq[2], qq[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const float m4 = 0.25f * (f[4 * u] + f[4 * u + 1] + f[4 * u + 2] + f[4 * u + 3]);
    float q4 = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) q4 = fmaf(f[4 * u + i] - m4, f[4 * u + i] - m4, q4);
    float mo = __shfl_xor_sync(0xffffffffu, m4, 1), qo = __shfl_xor_sync(0xffffffffu, q4, 1);
    float d = mo - m4;
    const float m8 = 0.5f * (m4 + mo), q8 = q4 + qo + 2.f * d * d;
    mo = __shfl_xor_sync(0xffffffffu, m8, 2);
    qo = __shfl_xor_sync(0xffffffffu, q8, 2);
    d = mo - m8;
    mq[u] = 0.5f * (m8 + mo);
    qq[u] = q8 + qo + 4.f * d * d;
  }
  if (!(lane & 3)) {
    stats[r * DP_CL + (lane >> 2)] = make_float2(mq[0], qq[0]);
    stats[r * DP_CL + 8 + (lane >> 2)] = make_float2(mq[1], qq[1]);
  }
}

// Every CTA of the cluster needs the same activation block: each loads 128 / DP_CL of its rows and
// multicasts them to all (16 SMs reading the same L2 lines at once serialise on those lines: a
// per-CTA 16 KB block took ~850 cycles, 19 B/cycle).
constexpr int DP_MROWS = 128 / DP_CL;
constexpr uint16_t DP_MASK = (uint16_t)((1u << DP_CL) - 1);
static_assert(128 % DP_CL == 0, "multicast slices");

__device__ __forceinline__ void dp_tma_mc(void *dst, const CUtensorMap *tm, uint64_t *bar, int c0, int c1,
                                          uint16_t mask = DP_MASK) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

// MMA completion arrives on the same barrier in every CTA (a ring stage is free only when all the
// CTAs its multicast fills have consumed it).
__device__ __forceinline__ void dp_commit_all(uint64_t *bar) {
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "@px tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
      "}\n" ::"r"(smem_u32(bar)), "h"(DP_MASK)
      : "memory");
}

__device__ __forceinline__ bool dp_stage_free(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Weight-slice cursor of the TMA producer.  Weights are constant for the whole
// launch, so the k-blocks of upcoming GEMMs are issued as soon as a ring stage
// frees up -- at the end of the previous GEMM phase, i.e. during the phase
// barrier and any SIMT phases in between -- and their L2 latency leaves the
// critical path.  Ring job j (in program order over the GEMMs this CTA takes
// part in) uses stage j % DP_STAGES; its full barrier expects two arrivals:
// the weight block (issued here, early) and the activation block (issued in
// the GEMM's own phase, or a plain arrive when A is the LayerNorm tile).
struct DpBCursor {
  int op = 0, kb = 0, job = 0;
};

// Issue the next weight k-block; false when the program has none left or
// (non-blocking) its stage is still held by the MMAs.
__device__ __forceinline__ bool dp_issue_b(const DpParams &P, const DpOpDev *ops, const DpGemmMeta *gm, DpBCursor &c,
                                           int rank, uint8_t *smem, uint64_t *full, uint64_t *empty, bool block) {
  while (c.op < P.n_ops) {
    const DpOpDev &o = ops[c.op];
    if (o.type != DP_GEMM || c.kb == (gm[o.gemm].K >> (o.ksplit ? 7 : 6))) {
      ++c.op;
      c.kb = 0;
      continue;
    }
    const DpGemmMeta &g = gm[o.gemm];
    const int st = c.job % DP_STAGES;
    const uint32_t par = ((c.job / DP_STAGES) & 1) ^ 1;
    if (block) {
      if (P.dbg & 2) { while (!dp_stage_free(&empty[st], par)) {} }
      else mbar_wait(&empty[st], par);
    }
    else if (!dp_stage_free(&empty[st], par)) return false;
    mbar_expect_tx(&full[st], g.ncta * 128);
    if (o.ksplit)      // K half rank / 8, columns of CTA rank % 8
      tma_load_2d(smem + DP_B_OFF + st * DP_B_BYTES, &P.gemms[o.gemm].tmB, &full[st],
                  ((rank >> 3) * (g.K >> 7) + c.kb) * 64, (rank & 7) * g.ncta);
    else
      tma_load_2d(smem + DP_B_OFF + st * DP_B_BYTES, &P.gemms[o.gemm].tmB, &full[st], c.kb * 64, rank * g.ncta);
    ++c.kb;
    ++c.job;
    return true;
  }
  return false;
}

// GELU with erf from Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7, far below the bf16 rounding of
// the stored activation): branch-free, so the 16 columns of a chunk evaluate with full ILP (erff
// branches per element and serialises).
__device__ __forceinline__ float dp_gelu(float x) {
  const float z = fabsf(x) * 0.70710678118654752f;
  const float t = __fdividef(1.f, fmaf(0.3275911f, z, 1.f));
  float p = fmaf(1.061405429f, t, -1.453152027f);
  p = fmaf(p, t, 1.421413741f);
  p = fmaf(p, t, -0.284496736f);
  p = fmaf(p, t, 0.254829592f);
  const float e = 1.f - p * t * __expf(-z * z);          // erf(|x| / sqrt 2)
  return 0.5f * x * (1.f + copysignf(e, x));
}

// Sub-phase stamps (SM clock, CTA 0) after the per-phase globaltimer stamps: diagnostics only.
#define DP_STAMP(k, cond)                                                                              \
  do {                                                                                                 \
    if (P.trace && rank == 0 && (cond)) P.trace[P.n_ops + 1 + 8 * oi + (k)] = clock64();              \
  } while (0)
#define DP_KSTAMP(k, cond)                                                                             \
  do {                                                                                                 \
    if (P.trace && rank == 0 && (cond) && (k) < 64) P.trace[9 * P.n_ops + 1 + 64 * oi + (k)] = clock64(); \
  } while (0)

// Attention of queries [n0, n0 + DP_QB) of unit (s, h) from its TMA'd tiles (128B-swizzled rows of
// 64 bf16: 16-byte chunk c of row r at chunk c ^ (r & 7)).  Lane j scores key j (its K row chunks
// against the broadcast q chunks), softmax over the lanes, lane l accumulates output dims 2l, 2l+1.
__device__ __forceinline__ const uint8_t *dp_sw(const uint8_t *t, int r, int chunk) {
  return t + r * 128 + ((chunk ^ (r & 7)) << 4);
}

__device__ __forceinline__ void dp_ldsm4(uint32_t (&r)[4], const void *p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void dp_ldsm4t(uint32_t (&r)[4], const void *p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
// D += A B, m16n8k16, bf16 in, fp32 accumulate
__device__ __forceinline__ void dp_mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
               "{%0, %1, %2, %3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t dp_pack(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t *>(&h);
}

// One (sample, head) unit by one warp on the tensor cores (the tiles are 16 x 64: far too small
// for tcgen05, one mma.sync m16n8k16 sequence is ~30 instructions): S = Q K^T (16 queries x 16
// key slots), masked softmax on the accumulator fragments, O = P V with P split into bf16 hi + lo
// parts (P V to ~2^-16, as the fp32 softmax of the launch-per-layer program).  Key slots >= nk
// hold finite neighbouring rows (or TMA zero fill) and are masked.
__device__ __noinline__ void dp_attn_tile(const DpOpDev &o, const uint8_t *t, int s, int h, int T, int lane,
                                          int dn0, int dn1) {
  const uint8_t *tq = t, *tk = t + 2048, *tv = t + 4096;
  const int g = lane >> 2, tq4 = lane & 3;
  const int lr = lane & 15, lc = lane >> 4;          // ldmatrix row / chunk-half of this lane
  float sc[2][4];                                    // [key n-tile][c0..c3]
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) sc[n][i] = 0.f;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {                   // head dims 16 ks .. 16 ks + 15
    uint32_t a[4], b[4];
    dp_ldsm4(a, dp_sw(tq, lr, 2 * ks + lc));
    // K: lanes 0-7 keys 0-7 dims +0, 8-15 keys 0-7 dims +8, 16-23 keys 8-15 +0, 24-31 keys 8-15 +8
    dp_ldsm4(b, dp_sw(tk, (lane & 7) + 8 * (lane >> 4), 2 * ks + ((lane >> 3) & 1)));
    dp_mma(sc[0], a, b[0], b[1]);
    dp_mma(sc[1], a, b[2], b[3]);
  }
  // masked softmax: this lane holds rows g (c0, c1) and g + 8 (c2, c3), key slots 8 n + 2 tq4 + {0, 1}
  const float scale = 0.125f;                         // 1 / sqrt(64)
  float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = g + 8 * (i >> 1), key = 8 * n + 2 * tq4 + (i & 1);
      const bool ok = key < o.nk && key <= row + o.mask_off;
      sc[n][i] = ok ? sc[n][i] * scale : -INFINITY;
      mx[i >> 1] = fmaxf(mx[i >> 1], sc[n][i]);
    }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
    mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
  }
  float sm[2] = {0.f, 0.f};
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      sc[n][i] = sc[n][i] == -INFINITY ? 0.f : __expf(sc[n][i] - mx[i >> 1]);
      sm[i >> 1] += sc[n][i];
    }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    sm[r] += __shfl_xor_sync(0xffffffffu, sm[r], 1);
    sm[r] += __shfl_xor_sync(0xffffffffu, sm[r], 2);
  }
  // P as the A operand (the m16n8 accumulator layout is the m16n8k16 A layout), hi + lo bf16
  uint32_t ph[4], pl[4];
  {
    const float p[8] = {sc[0][0], sc[0][1], sc[0][2], sc[0][3], sc[1][0], sc[1][1], sc[1][2], sc[1][3]};
    const int ord[4][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}};   // a0 (g, k 0-7) a1 (g+8, k 0-7) a2 (g, 8-15) a3
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float x0 = p[ord[i][0]], x1 = p[ord[i][1]];
      ph[i] = dp_pack(x0, x1);
      const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&ph[i]));
      pl[i] = dp_pack(x0 - hf.x, x1 - hf.y);
    }
  }
  const float inv[2] = {__fdividef(1.f, sm[0]), __fdividef(1.f, sm[1])};
#pragma unroll
  for (int dn = dn0; dn < dn1; ++dn) {               // head dims 16 dn .. 16 dn + 15: two n-tiles
    uint32_t b[4];
    // V^T fragments: lanes 0-7 keys 0-7 / 8-15 keys 8-15 at dims +0, 16-23 / 24-31 at dims +8
    dp_ldsm4t(b, dp_sw(tv, (lane & 7) + 8 * ((lane >> 3) & 1), 2 * dn + (lane >> 4)));
    float acc[2][4];
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[n][i] = 0.f;
    dp_mma(acc[0], ph, b[0], b[1]);
    dp_mma(acc[0], pl, b[0], b[1]);
    dp_mma(acc[1], ph, b[2], b[3]);
    dp_mma(acc[1], pl, b[2], b[3]);
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int row = g + 8 * r;
        if (row < T)
          *reinterpret_cast<uint32_t *>(o.out + ((int64_t)s * T + row) * o.ldo + h * 64 + 16 * dn + 8 * n + 2 * tq4) =
              dp_pack(acc[n][2 * r] * inv[r], acc[n][2 * r + 1] * inv[r]);
      }
  }
}

// LayerNorm of the 128 x 256 tile in sAln, in place (UMMA layout: K-major, 128B swizzle, 16-byte
// chunk j of row r at chunk j ^ (r & 7)); warp w normalises rows w, w + 8, ..., 8 at a time with
// their reductions interleaved; lane l owns columns 8 l .. 8 l + 7 (k-block l / 8, chunk l % 8).
// Rows >= S T hold stale finite activations: normalised too, never stored (a row of D depends
// only on its own row of A).  noinline for the same reason as dp_attn_block.
__device__ __noinline__ void dp_ln_tile(uint8_t *sAln, const float *ln_g, const float *ln_b, int warp, int lane) {
  const float4 g0 = *reinterpret_cast<const float4 *>(ln_g + 8 * lane);
  const float4 g1 = *reinterpret_cast<const float4 *>(ln_g + 8 * lane + 4);
  const float4 b0 = *reinterpret_cast<const float4 *>(ln_b + 8 * lane);
  const float4 b1 = *reinterpret_cast<const float4 *>(ln_b + 8 * lane + 4);
  const float ga[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
  const float ba[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
  const int kbl = lane >> 3, ch = lane & 7;
  for (int hb = 0; hb < 2; ++hb) {
    uint4 *px[8];
    uint4 xin4[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = warp + 8 * (8 * hb + i);
      px[i] = reinterpret_cast<uint4 *>(sAln + kbl * DP_A_BYTES + r * 128 + ((ch ^ (r & 7)) << 4));
      xin4[i] = *px[i];
    }
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
      // (rows >= S T hold stale finite activations: normalised too, never stored --
      //  a row of D depends only on its own row of A)
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
      *px[i] = make_uint4(yw[0], yw[1], yw[2], yw[3]);
    }
  }
}

// LayerNorm of the tile with the row statistics given (mean, rstd per row in shared memory): the
// normalisation pass only, no reductions.
__device__ __forceinline__ void dp_ln_apply(uint8_t *sAln, const float (&ga)[8], const float (&ba)[8],
                                            const float2 *srs, int warp, int lane) {
  const int kbl = lane >> 3, ch = lane & 7;
#pragma unroll 4
  for (int i = 0; i < 128 / 8; ++i) {
    const int r = warp + 8 * i;
    uint4 *px = reinterpret_cast<uint4 *>(sAln + kbl * DP_A_BYTES + r * 128 + ((ch ^ (r & 7)) << 4));
    const uint4 xv = *px;
    const float2 st = srs[r];
    const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
    uint32_t yw[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&xw[k]));
      const __nv_bfloat162 h2 = __floats2bfloat162_rn((f.x - st.x) * st.y * ga[2 * k] + ba[2 * k],
                                                      (f.y - st.x) * st.y * ga[2 * k + 1] + ba[2 * k + 1]);
      yw[k] = *reinterpret_cast<const uint32_t *>(&h2);
    }
    *px = make_uint4(yw[0], yw[1], yw[2], yw[3]);
  }
}

__global__ void __launch_bounds__(DP_THREADS, 1) dpt_persist(const __grid_constant__ DpParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + DP_BAR_OFF);
  uint64_t *empty = full + DP_STAGES;
  uint64_t *done = empty + DP_STAGES;
  uint64_t *lnbar = done + 1;     // the LayerNorm source tile landed in sAln
  uint64_t *resbar = lnbar + 1;   // the residual slice landed
  uint64_t *attbar = resbar + 1;  // the attention tiles landed
  uint64_t *rxbar = attbar + 1;   // K-split GEMM: the partner half's partial sums landed
  uint64_t *rdybar = rxbar + 1;   // K-split GEMM: the partner's MMAs are done (its A ring may be written)
  uint64_t *tbar = rdybar + 1;    // folded cross-attention: the sample's table blocks prefetched
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tbar + 1);
  DpOpDev *sops = reinterpret_cast<DpOpDev *>(smem + DP_META_OFF);
  DpGemmMeta *sgm = reinterpret_cast<DpGemmMeta *>(smem + DP_META_OFF + DP_MAX_OPS * 112);
  float *sbias = reinterpret_cast<float *>(smem + DP_META_OFF + DP_MAX_OPS * 112 + DP_MAX_GEMMS * 96);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_ctarank();
#define rows (P.S * P.T)      // (from the constant bank: not a register across the phase loop)
  {
    // ---- stage the program and this CTA's bias slices
    const uint64_t *src = reinterpret_cast<const uint64_t *>(P.ops);
    uint64_t *dst = reinterpret_cast<uint64_t *>(sops);
    for (int i = threadIdx.x; i < P.n_ops * 14; i += DP_THREADS) dst[i] = src[i];
    for (int i = threadIdx.x; i < P.n_gemms; i += DP_THREADS) {
      const DpGemmDev &g = P.gemms[i];
      DpGemmMeta m;
      m.res = g.res; m.out = g.out; m.out_f32 = g.out_f32;
      m.ln_src = g.ln_src; m.ln_g = g.ln_g; m.ln_b = g.ln_b;
      m.K = g.K; m.N = g.N; m.ncta = g.ncta; m.ldo = g.ldo; m.ldr = g.ldr; m.ldf = g.ldf;
      m.act = g.act; m.ctas = g.ctas; m.boff = g.boff; m.rtma = g.rtma;
      m.stats_out = g.stats_out; m.stats_in = g.stats_in;
      sgm[i] = m;
    }
    for (int i = warp; i < P.n_ops; i += DP_THREADS / 32) {
      const DpOpDev &op = P.ops[i];
      if (op.type != DP_GEMM) continue;
      const DpGemmDev &g = P.gemms[op.gemm];
      if (rank >= g.ctas) continue;
      const int cb = op.ksplit ? (rank & 7) : rank;        // K split: the half's CTAs share columns
      for (int c = lane; c < g.ncta; c += 32) {
        const int n = cb * g.ncta + c;
        sbias[g.boff + c] = n < g.N ? g.bias[n] : 0.f;
      }
    }
    // the launch's samples, and zeroed attention tiles (a gathered k / v tile fills only its
    // first nk rows; the masked rows must hold finite values for P V)
    int *ssamp = reinterpret_cast<int *>(smem + DP_SAMP_OFF);
    for (int i = threadIdx.x; i < P.S; i += DP_THREADS) {
      ssamp[i] = P.agents[i];
      ssamp[128 + i] = P.lanes[i];
      ssamp[256 + i] = P.steps[i];
    }
    for (int i = threadIdx.x; i < DP_ATT_SLOTS * DP_ATT_UNIT / 16; i += DP_THREADS)
      reinterpret_cast<uint4 *>(smem + DP_ATT_OFF)[i] = make_uint4(0, 0, 0, 0);
  }
  const int *s_agent = reinterpret_cast<const int *>(smem + DP_SAMP_OFF);
  const int *s_lane = s_agent + 128, *s_step = s_agent + 256;
  if (P.trace && rank == 0 && threadIdx.x == 0) {
    long long tn;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
    P.trace[0] = tn;
  }

  if (threadIdx.x == 0) {
    for (int i = 0; i < DP_STAGES; ++i) {
      mbar_init(&full[i], 2);      // weight block + activation block (see DpBCursor)
      mbar_init(&empty[i], DP_CL);   // one multicast commit from every CTA
    }
    mbar_init(done, 1);
    mbar_init(lnbar, 1);
    mbar_init(resbar, 1);
    mbar_init(attbar, 1);
    mbar_init(rxbar, 1);
    mbar_init(rdybar, 1);
    mbar_init(tbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(DP_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();      // (a CTA barrier first: the metadata staging and the mbarrier inits)
  // cluster-wide: no CTA may multicast into (or arrive on) a peer's barriers before the peer
  // initialised them
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == DP_CT / 32) {
    // ---- TMA producer warp (lane 0).  Per phase: the activation k-blocks of this phase's
    //      GEMM (they depend on the previous phase, so only after its barrier), then -- having
    //      arrived on the phase barrier already -- the weight blocks of the next GEMMs into the
    //      stages the ring frees up (DpBCursor), then the barrier wait.
    DpBCursor bc;
    int ip = 0;
    for (int oi = 0; oi < P.n_ops; ++oi) {
      const DpOpDev &o = sops[oi];
      if (lane == 0 && o.type == DP_GEMM) {     // (every CTA streams every GEMM: the multicast ring runs in lockstep)
        const DpGemmMeta &g = sgm[o.gemm];
        const int nkb = g.K / 64;
        const bool lnA = g.ln_g != nullptr;
        if (lnA) {
          // the residual-stream rows to normalise, straight into the A tile (normalised in place)
          mbar_expect_tx(lnbar, 4 * DP_A_BYTES);
#pragma unroll
          for (int kb = 0; kb < 4; ++kb)
            if (rank < P.mslices)
              dp_tma_mc(smem + kb * DP_A_BYTES + rank * (128 / P.mslices) * 128, &P.gemms[o.gemm].tmA, lnbar,
                        kb * 64, rank * (128 / P.mslices));
        }
        const int nkbx = o.ksplit ? nkb / 2 : nkb;
        for (int kb = 0; kb < nkbx; ++kb, ++ip) {
          while (bc.job <= ip) dp_issue_b(P, sops, sgm, bc, rank, smem, full, empty, true);
          DP_KSTAMP(kb, kb < 16);
          const int st = ip % DP_STAGES;
          if (lnA || o.gather == 3) {
            mbar_arrive(&full[st]);                   // A comes from the LayerNorm / action-token warps
          } else if (o.ksplit) {
            // this half's k-blocks: 16 rows from each of its 8 CTAs, multicast within the half
            mbar_expect_tx(&full[st], DP_A_BYTES);
            dp_tma_mc(smem + st * DP_A_BYTES + (rank & 7) * 16 * 128, &P.gemms[o.gemm].tmA, &full[st],
                      ((rank >> 3) * nkbx + kb) * 64, (rank & 7) * 16, (uint16_t)(0xFFu << (rank & 8)));
          } else {
            mbar_expect_tx(&full[st], DP_A_BYTES);     // (all DP_CL slices, from every CTA)
            if (rank < P.mslices)
              dp_tma_mc(smem + st * DP_A_BYTES + rank * (128 / P.mslices) * 128, &P.gemms[o.gemm].tmA, &full[st],
                        kb * 64, rank * (128 / P.mslices));
          }
          DP_KSTAMP(16 + kb, kb < 16);
        }
        if (g.rtma && rank < g.ctas) {
          mbar_expect_tx(resbar, 128 * g.ncta * 2);
          tma_load_2d(smem + DP_R_OFF, &P.gemms[o.gemm].tmR, resbar, rank * g.ncta, 0);
        }
        DP_STAMP(1, true);
      } else if (lane == 0 && o.type == DP_ATTN) {
        // this CTA's (sample, head) units u = rank + DP_CL k: q / k / v tiles in one transaction
        const DpAttnDev &a = P.attns[o.gemm];
        const int units = P.S * o.heads;
        int bytes = 0;
        for (int u = rank; u < units; u += DP_CL) bytes += (P.T + 2 * (o.gather ? o.nk : 16)) * 128;
        mbar_expect_tx(attbar, bytes);                     // (0 bytes: a plain arrive)
        for (int u = rank, k = 0; u < units; u += DP_CL, ++k) {
          const int sidx = u / o.heads, h = u % o.heads;
          uint8_t *t = smem + DP_ATT_OFF + k * DP_ATT_UNIT;
          tma_load_2d(t, &a.tq, attbar, h * 64, sidx * P.T);
          if (o.gather) {
            // row 0: the time token of the sample's inference step; rows 1 ..: its agent's
            // observation tokens (the 128B swizzle follows the shared-memory address)
            const int step = s_step[sidx], obs0 = s_agent[sidx] * (o.nk - 1);
            tma_load_2d(t + 2048, &a.tk, attbar, h * 64, step);
            tma_load_2d(t + 2048 + 128, &a.tk2, attbar, h * 64, obs0);
            tma_load_2d(t + 4096, &a.tv, attbar, h * 64, step);
            tma_load_2d(t + 4096 + 128, &a.tv2, attbar, h * 64, obs0);
          } else {
            tma_load_2d(t + 2048, &a.tk, attbar, h * 64, sidx * o.nk);
            tma_load_2d(t + 4096, &a.tv, attbar, h * 64, sidx * o.nk);
          }
        }
      }
      if (lane == 0 && oi + 1 < P.n_ops && sops[oi + 1].type == DP_XATTN && sops[oi + 1].job[0] >= 0 &&
          rank * (128 / DP_CL) < rows) {
        // the next phase's folded cross-attention tables (launch constants: by the CTA's sample's
        // step and agent) into two A-ring stages this phase's GEMM does not use (host-chosen);
        // issued after this phase's own loads so that they do not queue behind the tables
        const DpOpDev &x = sops[oi + 1];
        const int sidx = rank * (128 / DP_CL) / P.T, sb = 2 * x.heads * DP_E + 4;
        const uint32_t bytes = (uint32_t)sb * 4;
        uint8_t *dst = smem + x.job[0] * DP_A_BYTES;
        mbar_expect_tx(tbar, x.nk * bytes);
        for (int j = 0; j < x.nk; ++j) {
          const float *src = j == 0 ? reinterpret_cast<const float *>(x.k) + (int64_t)s_step[sidx] * x.ldk
                                    : reinterpret_cast<const float *>(x.v) +
                                          (int64_t)(s_agent[sidx] * (x.nk - 1) + j - 1) * x.ldv;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           smem_u32(dst + j * bytes)),
                       "l"(src), "r"(bytes), "r"(smem_u32(tbar))
                       : "memory");
        }
      }
      __syncwarp();
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
      if (lane == 0 && P.pf) {
        // weight blocks ahead: jobs < ip + DP_STAGES only wait for MMAs of this phase or
        // earlier ones, which complete without the producer
        while (bc.job < ip + DP_STAGES && dp_issue_b(P, sops, sgm, bc, rank, smem, full, empty, true)) {}
      }
      __syncwarp();
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
  } else {
  for (int oi = 0; oi < P.n_ops; ++oi) {
    const DpOpDev &o = sops[oi];
    DP_STAMP(0, threadIdx.x == 0);
    if (o.type == DP_GEMM) {
      const DpGemmMeta &g = sgm[o.gemm];
      {
        const int nkb = g.K >> (o.ksplit ? 7 : 6), ncta = g.ncta;
        const bool lnA = g.ln_g != nullptr;                // A = LayerNorm(src) computed here, not loaded
        uint8_t *sAln = smem;                              // 128 x 256 bf16, four 128B-swizzled k-blocks
        if (lnA) {
          // ---- the A operand: LayerNorm of every token row of the residual stream.  The
          //      producer TMA'd the rows into sAln in the UMMA layout (K-major, 128B swizzle:
          //      16-byte chunk j of row r at chunk j ^ (r & 7)); each warp normalises its 16 rows
          //      in place, 8 at a time with their reductions interleaved; lane l owns columns
          //      8 l .. 8 l + 7 (k-block l / 8, chunk l % 8)
          if (g.stats_in) {
            // row statistics from the 16 column-slice partials the residual GEMM's epilogue
            // left (equal-count Chan combination, a 4-level tree), one row per thread; the
            // loads overlap the tile's TMA
            float2 *srs = reinterpret_cast<float2 *>(smem + DP_STAT_OFF);
            // this lane's LayerNorm affine (columns 8 lane .. 8 lane + 7) first: an L2 round trip
            // that would otherwise stall the first normalised row
            const float4 g0 = *reinterpret_cast<const float4 *>(g.ln_g + 8 * lane);
            const float4 g1 = *reinterpret_cast<const float4 *>(g.ln_g + 8 * lane + 4);
            const float4 b0 = *reinterpret_cast<const float4 *>(g.ln_b + 8 * lane);
            const float4 b1 = *reinterpret_cast<const float4 *>(g.ln_b + 8 * lane + 4);
            if (threadIdx.x < 128) {
              const float4 *sp = reinterpret_cast<const float4 *>(P.stats + threadIdx.x * DP_CL);
              float mu[DP_CL], m2[DP_CL];
#pragma unroll
              for (int i = 0; i < DP_CL / 2; ++i) {
                const float4 q = sp[i];
                mu[2 * i] = q.x; m2[2 * i] = q.y; mu[2 * i + 1] = q.z; m2[2 * i + 1] = q.w;
              }
              float n = (float)(DP_E / DP_CL);
#pragma unroll
              for (int w = 1; w < DP_CL; w *= 2) {
#pragma unroll
                for (int i = 0; i < DP_CL; i += 2 * w) {
                  const float d = mu[i + w] - mu[i];
                  m2[i] = m2[i] + m2[i + w] + d * d * (0.5f * n);
                  mu[i] = 0.5f * (mu[i] + mu[i + w]);
                }
                n *= 2.f;
              }
              srs[threadIdx.x] = make_float2(mu[0], rsqrtf(m2[0] * (1.f / DP_E) + 1e-5f));
            }
            named_sync(1, DP_CT);
            mbar_wait(lnbar, o.par[rank == 0] & 1);
            DP_KSTAMP(57, threadIdx.x == 0);
            const float ga[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
            const float ba[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
            dp_ln_apply(sAln, ga, ba, srs, warp, lane);
          } else {
            mbar_wait(lnbar, o.par[rank == 0] & 1);
            DP_KSTAMP(57, threadIdx.x == 0);
            dp_ln_tile(sAln, g.ln_g, g.ln_b, warp, lane);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          named_sync(1, DP_CT);
          DP_STAMP(2, threadIdx.x == 0);
        } else if (o.gather == 3) {
          // ---- the input GEMM's A (K = 64): every sample's action tokens straight from its
          //      request lane into the UMMA tile (K-major, 128B swizzle: 16-byte chunk j of row r
          //      at chunk j ^ (r & 7)), bf16(x[t][a]) for a < adim, zeros elsewhere -- the
          //      separate prep phase (out[s T + t] = x[t]) and its L2 round trip are gone
          for (int i = threadIdx.x; i < 128 * 8; i += DP_CT) {
            const int r = i >> 3, j = i & 7;
            uint32_t w[4] = {0u, 0u, 0u, 0u};
            if (r < rows && 8 * j < P.adim) {
              const int sm = r / P.T, t = r - sm * P.T;
              const float *x = P.x_lanes +
                               ((int64_t)s_agent[sm] * P.lanes_per_agent + s_lane[sm]) * P.horizon * P.adim +
                               t * P.adim;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int a0 = 8 * j + 2 * k;
                w[k] = dp_pack(a0 < P.adim ? x[a0] : 0.f, a0 + 1 < P.adim ? x[a0 + 1] : 0.f);
              }
            }
            *reinterpret_cast<uint4 *>(sAln + r * 128 + ((j ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          named_sync(1, DP_CT);
          DP_STAMP(2, threadIdx.x == 0);
        }
        if (warp == 1) {
          // ---- MMA issuer
          // Each barrier probe is a round trip to the synchronisation unit (~200 cycles), more
          // than the four UMMAs of a k-block: after the blocking wait for stage kb, the next
          // stages are probed together (independent test_waits in flight at once) and every
          // k-block already landed is issued back to back.
          const uint32_t idesc = umma_idesc(ncta);
          const int j0 = o.job[rank == 0];
          for (int kb = 0; kb < nkb;) {
            const int ic = j0 + kb;
            mbar_wait(&full[ic % DP_STAGES], (ic / DP_STAGES) & 1);
            constexpr int PROBE = 4;
            bool t[PROBE - 1];
#pragma unroll
            for (int r = 1; r < PROBE; ++r)
              t[r - 1] = kb + r < nkb && dp_stage_free(&full[(ic + r) % DP_STAGES], ((ic + r) / DP_STAGES) & 1);
            int ready = 1;
#pragma unroll
            for (int r = 0; r < PROBE - 1; ++r) ready += (ready == r + 1 && t[r]) ? 1 : 0;
            if (kb == 0) DP_STAMP(3, lane == 0);
            DP_KSTAMP(32 + kb, lane == 0 && kb < 16);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int r = 0; r < ready; ++r, ++kb) {
              const int st = (j0 + kb) % DP_STAGES;
              const uint32_t sa =
                  smem_u32((lnA || o.gather == 3) ? sAln + kb * DP_A_BYTES : smem + st * DP_A_BYTES);
              const uint32_t sb = smem_u32(smem + DP_B_OFF + st * DP_B_BYTES);
              if (!(P.dbg & 8)) umma_kblock_warp(tmem, umma_desc(sa), umma_desc(sb), idesc, kb > 0 ? 1u : 0u);
              dp_commit_all(&empty[st]);
            }
            if (kb == nkb) DP_STAMP(4, lane == 0);
            __syncwarp();
          }
          umma_commit_warp(done);
          __syncwarp();
        }
        {
          // ---- epilogue, all 8 warps: token row = TMEM lane (warp % 4 quadrant), warps
          //      0-3 / 4-7 take alternate 16-column chunks
          const int row = (warp & 3) * 32 + lane, grp = warp >> 2;
          const int n0 = (o.ksplit ? (rank & 7) : rank) * ncta;
          // K split: this CTA owns 16-column chunk kh = rank / 8 of its 32 columns (warps with grp ==
          // kh); the other chunk's partials go to the partner CTA rank ^ 8 (which owns it) over DSMEM,
          // into its A-ring stage 0 once the partner's MMAs are done (rdybar)
          const bool ks = o.ksplit != 0;
          const int kh = rank >> 3;
          float *rx = reinterpret_cast<float *>(smem);      // [128 rows][16] fp32 partner partials
          if (ks && threadIdx.x == 0) mbar_expect_tx(rxbar, 128 * 16 * 4);
          const uint8_t *sres = smem + DP_R_OFF + row * ncta * 2;     // this row of the TMA'd residual slice
          // the GEMM's fields in registers: g lives in shared memory behind a generic pointer, so
          // every global store below would otherwise force it to be re-read
          const float *bias_s = sbias + g.boff;
          const __nv_bfloat16 *res = g.res;
          __nv_bfloat16 *out = g.out;
          float *outf = g.out_f32;
          const int ldo = g.ldo, ldr = g.ldr, ldf = g.ldf, act = g.act, N = g.N;
          const bool rtma = g.rtma != 0 && rank < g.ctas;
          const bool stats_out = g.stats_out != 0;
          const int ncols = rank < g.ctas ? ncta : 0;    // (the single-CTA head: only CTA 0 stores)
          if (P.dbg & 1) mbar_wait_sleep(done, (o.par[rank == 0] >> 2) & 1, 256);
          else mbar_wait(done, (o.par[rank == 0] >> 2) & 1);
          if (rtma) {
            mbar_wait(resbar, (o.par[rank == 0] >> 1) & 1);
          }
          if (ks && threadIdx.x == 0)       // my MMAs are done: the partner may write my A ring
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                             mapa_shared(smem_u32(rdybar), rank ^ 8))
                         : "memory");
          DP_STAMP(5, threadIdx.x == 0);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          for (int c = 16 * grp; c < ncols; c += 32) {
            float v[16];
            tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + c, v);
            if (ks) {
              const uint32_t kpar = (o.par[0] >> 3) & 1;
              if (grp != kh) {
                // the partner's chunk: wait until its A ring is free, then push the 16 partials
                mbar_wait_cluster(rdybar, kpar);
                const uint32_t dst = mapa_shared(smem_u32(rx + row * 16), rank ^ 8);
                const uint32_t rb = mapa_shared(smem_u32(rxbar), rank ^ 8);
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                  st_async_v4_b32(dst + 4 * i, __float_as_uint(v[i]), __float_as_uint(v[i + 1]),
                                  __float_as_uint(v[i + 2]), __float_as_uint(v[i + 3]), rb);
                continue;
              }
              mbar_wait_cluster(rxbar, kpar);
              const float4 *rp = reinterpret_cast<const float4 *>(rx + row * 16);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float4 q = rp[i];
                v[4 * i] += q.x; v[4 * i + 1] += q.y; v[4 * i + 2] += q.z; v[4 * i + 3] += q.w;
              }
            }
            DP_KSTAMP(48 + 3 * (c >> 5), threadIdx.x == 0 && c < 96);
            if (row >= rows) continue;
            const int nb = n0 + c;
            if (nb + 16 <= N) {
#pragma unroll
              for (int i = 0; i < 16; i += 4) {
                const float4 bb = *reinterpret_cast<const float4 *>(bias_s + c + i);
                v[i] += bb.x; v[i + 1] += bb.y; v[i + 2] += bb.z; v[i + 3] += bb.w;
              }
              if (act == AURAS_ACT_GELU) {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = dp_gelu(v[i]);
              } else if (act) {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = activate(v[i], act);
              }
              DP_KSTAMP(49 + 3 * (c >> 5), threadIdx.x == 0 && c < 96);
              if (res) {
                uint4 r0, r1;
                if (rtma) {
                  r0 = reinterpret_cast<const uint4 *>(sres + c * 2)[0];
                  r1 = reinterpret_cast<const uint4 *>(sres + c * 2)[1];
                } else {
                  const uint4 *rp = reinterpret_cast<const uint4 *>(res + (int64_t)row * ldr + nb);
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
              if (out) {
                uint32_t ow[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
                  ow[i] = *reinterpret_cast<const uint32_t *>(&h2);
                }
                uint4 *op = reinterpret_cast<uint4 *>(out + (int64_t)row * ldo + nb);
                op[0] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
                op[1] = make_uint4(ow[4], ow[5], ow[6], ow[7]);
                if (stats_out) {
                  // (mean, M2) of the 16 stored (bf16-rounded) values: the next LayerNorm's input
                  float x[16], sm = 0.f;
#pragma unroll
                  for (int i = 0; i < 8; ++i) {
                    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&ow[i]));
                    x[2 * i] = f.x;
                    x[2 * i + 1] = f.y;
                    sm += f.x + f.y;
                  }
                  const float mu = sm * (1.f / 16.f);
                  float m2 = 0.f;
#pragma unroll
                  for (int i = 0; i < 16; ++i) m2 = fmaf(x[i] - mu, x[i] - mu, m2);
                  P.stats[row * DP_CL + (nb >> 4)] = make_float2(mu, m2);
                }
              }
              if (outf) {
                float4 *fp = reinterpret_cast<float4 *>(outf + (int64_t)row * ldf + nb);
#pragma unroll
                for (int i = 0; i < 4; ++i) fp[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
              }
              DP_KSTAMP(50 + 3 * (c >> 5), threadIdx.x == 0 && c < 96);
            } else {
              // ragged tail (the 7-wide action head): columns < N only
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] += bias_s[c + i];
              if (act)
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = activate(v[i], act);
              if (res)
#pragma unroll
                for (int i = 0; i < 16; ++i)
                  if (nb + i < N) v[i] += __bfloat162float(res[(int64_t)row * ldr + nb + i]);
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                if (nb + i >= N) break;
                if (out) out[(int64_t)row * ldo + nb + i] = __float2bfloat16_rn(v[i]);
                if (outf) outf[(int64_t)row * ldf + nb + i] = v[i];
              }
              if (o.gather == 2) {
                // the scheduler update fused into the action head (auras_dpt_gemm.fuse_update): token
                // row = (sample, t), its adim eps values in v (the UPDATE phase's arithmetic)
                const auras_sched &sch = P.sched;
                const int sm = row / P.T, t = row - sm * P.T;
                const int agent = s_agent[sm], ln = s_lane[sm], i = s_step[sm];
                float *x = P.x_lanes + ((int64_t)agent * P.lanes_per_agent + ln) * P.horizon * P.adim + t * P.adim;
                const float *z = P.noise_lanes ? P.noise_lanes +
                                                     (((int64_t)agent * P.lanes_per_agent + ln) * sch.n_steps + i) *
                                                         P.horizon * P.adim + t * P.adim
                                               : nullptr;
                const float sab = sch.sqrt_ab[i], s1m = sch.sqrt_1mab[i];
                const float cx0 = sch.c_x0[i], cxt = sch.c_xt[i], ceps = sch.c_eps[i], sig = sch.sigma[i];
#pragma unroll
                for (int a = 0; a < 16; ++a) {
                  if (nb + a >= P.adim) break;
                  const float xt = x[nb + a], ep = v[a];
                  float x0 = (xt - s1m * ep) / sab;
                  if (sch.clip_sample) x0 = fminf(fmaxf(x0, -1.f), 1.f);
                  float nx = cx0 * x0 + cxt * xt + ceps * ep;
                  if (sch.ddpm && z) nx += sig * z[nb + a];
                  x[nb + a] = nx;
                }
              }
              DP_KSTAMP(50, threadIdx.x == 0);
            }
          }
        }
      }
    } else if (o.type == DP_LN) {
      for (int r = rank * 8 + warp; r < rows; r += DP_CL * 8)
        dp_ln_row(o.in + (int64_t)r * o.ldi, o.out + (int64_t)r * o.ldo, o.g, o.b, lane);
    } else if (o.type == DP_ATTN) {
      long long *stamp = P.trace && rank == 0 && threadIdx.x == 0 ? P.trace + 9 * P.n_ops + 1 + 64 * oi + 56 : nullptr;
      mbar_wait(attbar, (o.par[0] >> 3) & 1);
      if (stamp) stamp[0] = clock64();
      // unit slot k (u = rank + DP_CL k); the 8 warps split the CTA's units, each unit's P V by
      // head-dim blocks (the scores are recomputed per warp: 8 MMAs against the 16 of P V)
      const int units = P.S * o.heads;
      const int nu = units > rank ? (units - rank + DP_CL - 1) / DP_CL : 0;   // this CTA's units (<= 4)
      if (nu > 0) {
        const int wpu = nu == 1 ? 4 : (nu == 2 ? 4 : 2);                       // warps per unit
        const int k = warp / wpu, part = warp % wpu, nd = 4 / wpu;
        const int u = rank + DP_CL * k;
        if (k < nu && part * nd < 4)
          dp_attn_tile(o, smem + DP_ATT_OFF + k * DP_ATT_UNIT, u / o.heads, u % o.heads, P.T, lane, part * nd,
                       part * nd + nd);
      }
      if (stamp) stamp[1] = clock64();
    } else if (o.type == DP_PREP) {
      // ---- the action tokens of every sample from its request lane (dpt.cu dpt_prep_kernel):
      //      out[s T + t][a] = bf16(x[t][a]) for a < adim, 0 up to 64 (the input GEMM's A)
      const int items = P.S * P.T * 8;                     // (row, 8-column chunk)
      for (int i = rank * DP_CT + threadIdx.x; i < items; i += DP_CL * DP_CT) {
        const int r = i >> 3, c0 = (i & 7) * 8, sidx = r / P.T, t = r % P.T;
        const float *x = P.x_lanes + ((int64_t)s_agent[sidx] * P.lanes_per_agent + s_lane[sidx]) * P.horizon * P.adim +
                         t * P.adim;
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int a0 = c0 + 2 * k;
          w[k] = dp_pack(a0 < P.adim ? x[a0] : 0.f, a0 + 1 < P.adim ? x[a0 + 1] : 0.f);
        }
        *reinterpret_cast<uint4 *>(o.out + (int64_t)r * 64 + c0) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    } else if (o.type == DP_XATTN) {
      // table blocks staged in A-ring stages 4-5 (idle outside GEMM phases, like the attention tiles)
      const int r0 = rank * (128 / DP_CL);
      long long *stamp = P.trace && rank == 0 ? P.trace + 9 * P.n_ops + 1 + 64 * oi + 56 : nullptr;
      if (stamp && threadIdx.x == 0) stamp[4] = clock64();
      if (r0 < rows) {
        uint64_t *tb = o.job[0] >= 0 ? tbar : nullptr;
        float *stab = reinterpret_cast<float *>(smem + (tb ? o.job[0] * DP_A_BYTES : DP_ATT_OFF));
        if (o.nk == 3)
          dp_xattn<3>(o, r0, rows, P.T, s_agent, s_step, stab, P.stats, warp, lane, stamp, tb);
        else if (o.nk == 2)
          dp_xattn<2>(o, r0, rows, P.T, s_agent, s_step, stab, P.stats, warp, lane, stamp, tb);
        else if (o.nk == 4)
          dp_xattn<4>(o, r0, rows, P.T, s_agent, s_step, stab, P.stats, warp, lane, stamp, tb);
        else
          dp_xattn<1>(o, r0, rows, P.T, s_agent, s_step, stab, P.stats, warp, lane, stamp, tb);
      }
    } else if (o.type == DP_NOP) {
      // timing probe: a phase with no work (the cost of the phase boundary alone)
    } else {
      // ---- DDPM / DDIM update of sample s (dpt.cu dpt_update_kernel arithmetic)
      const auras_sched &sch = P.sched;
      for (int s = rank; s < P.S; s += DP_CL) {
        const int agent = s_agent[s], ln = s_lane[s], i = s_step[s];
        float *x = P.x_lanes + ((int64_t)agent * P.lanes_per_agent + ln) * P.horizon * P.adim;
        const float *z = P.noise_lanes ? P.noise_lanes + (((int64_t)agent * P.lanes_per_agent + ln) * sch.n_steps + i) *
                                                             P.horizon * P.adim
                                       : nullptr;
        const float sab = sch.sqrt_ab[i], s1m = sch.sqrt_1mab[i];
        const float cx0 = sch.c_x0[i], cxt = sch.c_xt[i], ceps = sch.c_eps[i], sig = sch.sigma[i];
        for (int e = threadIdx.x; e < P.horizon * P.adim; e += DP_CT) {
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
    // weight blocks of the next GEMMs into the stages this phase released
    DP_STAMP(6, threadIdx.x == 0);
    // phase boundary: generic global stores visible to the next phase's TMA reads, TMEM drained
    // (the residual reads of sAln completed into registers before this point; LayerNorm's
    // generic writes of sAln were proxy-fenced in their phase)
    fence_proxy_async();
    DP_STAMP(7, threadIdx.x == 0);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (P.trace && rank == 0 && threadIdx.x == 0) {
      long long tn;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
      P.trace[oi + 1] = tn;
    }
  }
  }
  // (every multicast commit / TMA into this CTA was consumed before the last phase barrier)
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(DP_TMEM_COLS));
}
#undef rows

// CTAs loading a multicast slice of each activation block (AURAS_DPT_MSLICES: 1, 2, 4, 8 or 16)
static int dp_mslices() {
  static int m = -1;
  if (m < 0) {
    const char *e = getenv("AURAS_DPT_MSLICES");
    m = e ? atoi(e) : DP_CL;
    if (m < 1 || m > DP_CL || (DP_CL % m) || (128 % m)) m = DP_CL;
  }
  return m;
}

// ---- auras_dpt_xfold: one block per (kv row, layer, head), one thread per
// embedding column e (coalesced reads of Wq's and Wo^T's rows).
__global__ void dpt_xfold_kernel(const __nv_bfloat16 *kv, int kv_ld, int L, int E, int H, const float *wq,
                                 const float *bq, const float *woT, const float *bo, const float *lng,
                                 const float *lnb, float *out, int xs) {
  extern __shared__ float xf_sh[];                 // k[dh], v[dh], warp partials[32]
  const int r = blockIdx.x, l = blockIdx.y, h = blockIdx.z, e = threadIdx.x;
  const int dh = E / H;
  const __nv_bfloat16 *kr = kv + (int64_t)r * kv_ld + (int64_t)l * 2 * E + h * dh;
  if (e < dh) {
    xf_sh[e] = __bfloat162float(kr[e]);
    xf_sh[dh + e] = __bfloat162float(kr[E + e]);
  }
  __syncthreads();
  const float scale = rsqrtf((float)dh);
  const float *wql = wq + (int64_t)l * E * E + (int64_t)h * dh * E;
  const float *wol = woT + (int64_t)l * E * E + (int64_t)h * dh * E;
  float a = 0.f, u = 0.f;
  for (int d = 0; d < dh; ++d) {
    a = fmaf(wql[(int64_t)d * E + e], xf_sh[d], a);
    u = fmaf(wol[(int64_t)d * E + e], xf_sh[dh + d], u);
  }
  a *= scale;
  float *o = out + ((int64_t)r * L + l) * xs;
  o[h * E + e] = lng[l * E + e] * a;
  o[H * E + h * E + e] = u + bo[l * E + e] / (float)H;
  float c = lnb[l * E + e] * a + (e < dh ? bq[l * E + h * dh + e] * xf_sh[e] * scale : 0.f);
  c = dp_wsum(c);
  float *red = xf_sh + 2 * dh;
  if ((e & 31) == 0) red[e >> 5] = c;
  __syncthreads();
  if (e == 0) {
    float t = 0.f;
    for (int w = 0; w < (E + 31) / 32; ++w) t += red[w];
    o[2 * H * E + h] = t;
  }
  if (h == 0)
    for (int i = 2 * H * E + H + e; i < xs; i += E) o[i] = 0.f;   // pad (read by the float4 staging)
}

struct DpPlan {
  float2 *stats = nullptr;             // [128][DP_CL] row-statistics partials
  DpAttnDev *attns = nullptr;          // attention operand maps, per attention op
  DpOpDev *ops = nullptr;
  DpGemmDev *gemms = nullptr;
  long long *trace = nullptr;          // AURAS_DPT_TRACE: per-phase timestamps of the last run
  int n_ops = 0, n_gemms = 0, T = 16, heads = 0;   // (heads: the most of any attention op)
};

// Residual slice map: [rows][N] bf16 with row pitch ld, box {ncta, 128}, no swizzle (row-major
// [128][ncta] in shared memory).
static int dp_map_res(CUtensorMap *tm, const void *base, int N, int ld, int rows, int ncta) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return AURAS_E_CUDA; }
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)ncta, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("dpt_persist residual map: CUresult %d", (int)r); return AURAS_E_CUDA; }
  return AURAS_OK;
}

// [rows][cols] bf16 with row pitch ld (elements), box {64, box_rows}, 128B swizzle.
static int dp_map_pitch(CUtensorMap *tm, const void *base, int cols, int ld, int rows, int box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return AURAS_E_CUDA; }
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * 2) % 16) {
    set_error("dpt_persist map: unaligned operand");
    return AURAS_E_ARG;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("dpt_persist map: CUresult %d", (int)r); return AURAS_E_CUDA; }
  return AURAS_OK;
}

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
  if (n_ops > DP_MAX_OPS || n_gemms > DP_MAX_GEMMS) {
    set_error("dpt_persist_build: %d ops / %d GEMMs (max %d / %d)", n_ops, n_gemms, DP_MAX_OPS, DP_MAX_GEMMS);
    return AURAS_E_ARG;
  }
  std::vector<DpGemmDev> hg(n_gemms);
  int boff = 0;
  for (int i = 0; i < n_gemms; ++i) {
    const auras_dpt_gemm &s = gemms[i];
    DpGemmDev &d = hg[i];
    memset(&d, 0, sizeof(d));
    const int ctas = s.N <= 16 ? 1 : DP_CL;
    const int ncta = ctas == 1 ? 16 : s.N / (s.ksplit ? DP_CL / 2 : DP_CL);
    if (s.ksplit && (DP_CL != 16 || ctas != DP_CL || s.ln_g || !s.out || s.out_f32 || s.N % 128 || ncta > 64 ||
                     ncta != 32 || s.K % 128)) {
      // (the epilogue exchanges one 16-column chunk with the partner half: 32 columns per CTA)
      set_error("dpt_persist_build: gemm %d K split needs a plain-A bf16 GEMM, N = 256, K %% 128 == 0", i);
      return AURAS_E_ARG;
    }
    if (s.K % 64 || s.act_rows != 128 || (ctas > 1 && (s.N % DP_CL || ncta % 16 || ncta * 128 > DP_B_BYTES)) ||
        (s.out && s.ldo % 8) || (s.res && s.ldr % 8) ||
        (ctas > 1 && s.out_f32 && (s.ldf % 4 || (reinterpret_cast<uintptr_t>(s.out_f32) & 15)))) {
      set_error("dpt_persist_build: gemm %d shape K=%d N=%d rows=%d", i, s.K, s.N, s.act_rows);
      return AURAS_E_ARG;
    }
    if (s.ln_g && (s.K != DP_E || !s.ln_src || !s.ln_b)) {
      set_error("dpt_persist_build: gemm %d LayerNorm'd A needs K = 256", i);
      return AURAS_E_ARG;
    }
    // A operand, or (LayerNorm'd A) the residual-stream rows the phase normalises in place
    if (int rc = dp_map(&d.tmA, s.ln_g ? s.ln_src : s.act, s.K, s.act_rows, s.ksplit ? 16 : 128 / dp_mslices()))
      return rc;
    d.ln_src = static_cast<const __nv_bfloat16 *>(s.ln_src);
    d.ln_g = s.ln_g;
    d.ln_b = s.ln_b;
    if (int rc = dp_map(&d.tmB, s.w, s.K, s.N, ncta)) return rc;
    d.bias = s.bias;
    d.res = static_cast<const __nv_bfloat16 *>(s.res);
    d.rtma = s.res && ctas > 1 && ncta * 128 * 2 <= DP_R_BYTES && (reinterpret_cast<uintptr_t>(s.res) & 15) == 0 ? 1 : 0;
    if (d.rtma)
      if (int rc = dp_map_res(&d.tmR, s.res, s.N, s.ldr, s.act_rows, ncta)) return rc;
    d.out = static_cast<__nv_bfloat16 *>(s.out);
    d.out_f32 = s.out_f32;
    d.K = s.K; d.N = s.N; d.ncta = ncta; d.ctas = ctas;
    d.boff = boff;
    boff += (ncta + 3) & ~3;           // float4-aligned slices
    if (boff > DP_BIAS_SLAB) {
      set_error("dpt_persist_build: bias slices exceed %d floats", DP_BIAS_SLAB);
      return AURAS_E_ARG;
    }
    d.ldo = s.ldo; d.ldr = s.ldr; d.ldf = s.ldf; d.act = s.act_fn;
  }
  std::vector<DpOpDev> ho(n_ops);
  int nln[2] = {0, 0}, nres[2] = {0, 0}, ng[2] = {0, 0}, nj[2] = {0, 0};   // [CTAs 1..] / [CTA 0]
  int nks = 0;                                                              // K-split GEMMs so far
  int ntp = 0;                                                              // prefetched cross-attention tables
  int natt = 0;
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
    d.gather = s.type == DP_ATTN && s.gather;
    if (s.type == DP_ATTN) {
      d.par[0] = d.par[1] = (natt & 1) << 3;
      ++natt;
    }
    if (s.type == DP_GEMM && s.gemm >= 0 && s.gemm < n_gemms) {
      const DpGemmDev &gg = hg[s.gemm];
      d.ksplit = gemms[s.gemm].ksplit ? 1 : 0;
      if (gemms[s.gemm].a_from_lanes) {
        const auras_dpt_gemm &gg3 = gemms[s.gemm];
        if (gg3.K != 64 || gg3.ln_g || gg3.ksplit || gg3.fuse_update) {
          set_error("dpt_persist_build: gemm %d A from the request lanes needs K = 64, plain A", s.gemm);
          return AURAS_E_ARG;
        }
        d.gather = 3;
      }
      if (gemms[s.gemm].fuse_update) {
        const auras_dpt_gemm &gg2 = gemms[s.gemm];
        if (gg2.N > 16 || !gg2.out_f32 || gg2.ksplit || gg2.res) {
          set_error("dpt_persist_build: gemm %d fused update needs the single-CTA fp32 action head", s.gemm);
          return AURAS_E_ARG;
        }
        d.gather = 2;
      }
      for (int c = 0; c < 2; ++c) {
        const bool runs = true;        // every CTA streams every GEMM (multicast ring)
        d.par[c] = (nln[c] & 1) | ((nres[c] & 1) << 1) | ((ng[c] & 1) << 2) | ((nks & 1) << 3);
        d.job[c] = nj[c];
        if (!runs) continue;
        if (gg.ln_g) ++nln[c];
        if (gg.rtma) ++nres[c];
        ++ng[c];
        nj[c] += gg.K / (d.ksplit ? 128 : 64);
      }
      nks += d.ksplit;
    }
    if (s.type == DP_XATTN) {
      // table prefetch during the previous phase: needs a plain-A GEMM there whose ring jobs leave
      // two adjacent A-ring stages free (the LayerNorm tile would hold stages 0-3)
      d.job[0] = d.job[1] = -1;
      if (i > 0 && ops[i - 1].type == DP_GEMM && !gemms[ops[i - 1].gemm].ln_g && !gemms[ops[i - 1].gemm].a_from_lanes &&
          !getenv("AURAS_DPT_NO_TPF")) {
        const auras_dpt_gemm &pg = gemms[ops[i - 1].gemm];
        const int j0 = ho[i - 1].job[0], nkb = pg.K / (pg.ksplit ? 128 : 64);
        auto used = [&](int st) {
          for (int k = 0; k < nkb; ++k)
            if ((j0 + k) % DP_STAGES == st) return true;
          return false;
        };
        for (int st = 0; st + 1 < DP_STAGES; ++st)
          if (!used(st) && !used(st + 1)) { d.job[0] = d.job[1] = st; break; }
        if (d.job[0] >= 0) {
          d.par[0] = d.par[1] = ntp & 1;
          ++ntp;
        }
      }
      // one sample per CTA (8 rows), table blocks within A-ring stages 4-5, float4-aligned rows
      const int SB = 2 * s.heads * DP_E + 4;
      if (T % (128 / DP_CL) || s.nk < 1 || s.nk > DP_XK || s.heads != DP_XH || s.mask_off < 0 ||
          s.nk * SB * 4 > 2 * DP_A_BYTES || s.ldk % 4 || s.ldv % 4 || s.ldk < SB || (s.nk > 1 && s.ldv < SB) ||
          s.ldi % 8 || s.ldo % 8 || !s.in || !s.out || !s.k || (s.nk > 1 && !s.v) || (s.g && (!s.b || s.out == s.in)) ||
          (!s.g && s.out != s.in) ||
          (reinterpret_cast<uintptr_t>(s.k) & 15) || (reinterpret_cast<uintptr_t>(s.v) & 15)) {
        set_error("dpt_persist_build: folded cross-attention op %d (T=%d nk=%d heads=%d)", i, T, s.nk, s.heads);
        return AURAS_E_ARG;
      }
    }
    if ((s.type == DP_GEMM && (s.gemm < 0 || s.gemm >= n_gemms)) || (s.type == DP_ATTN && (s.nk > DP_MAXK || s.dh != 64)) ||
        s.type < 0 || s.type > DP_XATTN) {
      set_error("dpt_persist_build: op %d", i);
      return AURAS_E_ARG;
    }
  }
  std::vector<DpAttnDev> ha;
  int max_heads = 0;
  for (int i = 0; i < n_ops; ++i) {
    if (ops[i].type != DP_ATTN) continue;
    const auras_dpt_op &s = ops[i];
    if (s.qrows < 1 || s.krows < 1 || s.heads * 64 > s.ldi || s.heads * 64 > s.ldk || s.ldk != s.ldv ||
        s.nk < 1 || s.nk > 16 || (s.gather && (s.nk < 2 || !s.k2 || !s.v2 || s.k2rows < 1))) {
      set_error("dpt_persist_build: attention op %d (qrows %d krows %d)", i, s.qrows, s.krows);
      return AURAS_E_ARG;
    }
    DpAttnDev a;
    memset(&a, 0, sizeof(a));
    if (int rc = dp_map_pitch(&a.tq, s.in, s.heads * 64, s.ldi, s.qrows, T)) return rc;
    if (s.gather) {
      // time table rows (one per sample, by inference step) + the agent's observation rows
      if (int rc = dp_map_pitch(&a.tk, s.k, s.heads * 64, s.ldk, s.krows, 1)) return rc;
      if (int rc = dp_map_pitch(&a.tv, s.v, s.heads * 64, s.ldv, s.krows, 1)) return rc;
      if (int rc = dp_map_pitch(&a.tk2, s.k2, s.heads * 64, s.ldk, s.k2rows, s.nk - 1)) return rc;
      if (int rc = dp_map_pitch(&a.tv2, s.v2, s.heads * 64, s.ldv, s.k2rows, s.nk - 1)) return rc;
    } else {
      // (k / v boxes of 16 rows: slots >= nk hold neighbouring rows or zero fill, masked in the kernel)
      if (int rc = dp_map_pitch(&a.tk, s.k, s.heads * 64, s.ldk, s.krows, 16)) return rc;
      if (int rc = dp_map_pitch(&a.tv, s.v, s.heads * 64, s.ldv, s.krows, 16)) return rc;
    }
    ho[i].gemm = (int)ha.size();
    max_heads = std::max(max_heads, s.heads);
    ha.push_back(a);
  }
  {
    // Row-statistics handoff: a GEMM whose epilogue writes 16-column slices of a 256-wide
    // activation (N = DP_E over the cluster) records per-slice (mean, M2); a later LayerNorm'd
    // GEMM reading that same activation, with no other writer in between, uses them.
    // (one statistics buffer: only writers of a LayerNorm source take part)
    std::vector<const void *> lsrc;
    for (int i = 0; i < n_gemms; ++i)
      if (hg[i].ln_g) lsrc.push_back(hg[i].ln_src);
    auto is_lsrc = [&](const void *q) { return std::find(lsrc.begin(), lsrc.end(), q) != lsrc.end(); };
    const void *valid = nullptr;
    for (int i = 0; i < n_ops; ++i) {
      if (ops[i].type == DP_XATTN) {
        // rewrites its residual rows: slice statistics only without the LayerNorm output
        if (ops[i].g || ops[i].in != valid) valid = nullptr;
        continue;
      }
      if (ops[i].type != DP_GEMM) continue;
      DpGemmDev &d = hg[ops[i].gemm];
      if (d.ln_g) d.stats_in = valid && d.ln_src == valid;
      if (d.out && is_lsrc(d.out)) {
        const bool ok = d.N == DP_E && d.ctas == DP_CL && (d.ncta == 16 || (gemms[ops[i].gemm].ksplit && d.ncta == 32));
        d.stats_out = ok;
        valid = ok ? d.out : nullptr;
      }
    }
  }
  DpPlan *p = new DpPlan;
  p->n_ops = n_ops;
  p->n_gemms = n_gemms;
  p->T = T;
  p->heads = max_heads;
  if (cudaMalloc(&p->ops, sizeof(DpOpDev) * n_ops) != cudaSuccess ||
      cudaMalloc(&p->gemms, sizeof(DpGemmDev) * n_gemms) != cudaSuccess ||
      cudaMalloc(&p->stats, sizeof(float2) * 128 * DP_CL) != cudaSuccess ||
      cudaMalloc(&p->attns, sizeof(DpAttnDev) * std::max<size_t>(1, ha.size())) != cudaSuccess) {
    cudaFree(p->ops);
    cudaFree(p->gemms);
    delete p;
    return cuda_check(cudaGetLastError(), "dpt_persist alloc");
  }
  cudaMemset(p->stats, 0, sizeof(float2) * 128 * DP_CL);
  if (!ha.empty()) cudaMemcpy(p->attns, ha.data(), sizeof(DpAttnDev) * ha.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(p->ops, ho.data(), sizeof(DpOpDev) * n_ops, cudaMemcpyHostToDevice);
  cudaMemcpy(p->gemms, hg.data(), sizeof(DpGemmDev) * n_gemms, cudaMemcpyHostToDevice);
  if (getenv("AURAS_DPT_TRACE")) {
    cudaMalloc(&p->trace, sizeof(long long) * (73 * n_ops + 1));
    cudaMemset(p->trace, 0, sizeof(long long) * (73 * n_ops + 1));
  }
  *plan_out = p;
  return cuda_check(cudaGetLastError(), "dpt_persist_build");
}

int auras_dpt_persist_run(void *plan, int S, const float *eps, int eps_pitch, const int *agents, const int *lanes,
                          const int *steps, float *x_lanes, const float *noise_lanes, int lanes_per_agent,
                          int horizon, int adim, const auras_sched *sched, void *stream) {
  DpPlan *p = static_cast<DpPlan *>(plan);
  if (!p || !sched || S < 1 || S * p->T > 128 || horizon != p->T || S * p->heads > DP_ATT_SLOTS * DP_CL) {
    set_error("dpt_persist_run: bad arguments (S=%d)", S);
    return AURAS_E_ARG;
  }
  if (int rc = ensure_smem_attr(dpt_persist, (int)DP_SMEM)) return rc;
  if (DP_CL > 8) {
    // (a function attribute is per device: a process-wide flag would miss a second GPU)
    static thread_local bool np[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cuda_check(cudaGetLastError(), "dpt device");
    if (!np[dev]) {
      AURAS_CUDA(cudaFuncSetAttribute(dpt_persist, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      np[dev] = true;
    }
  }
  DpParams P;
  memset(&P, 0, sizeof(P));
  P.trace = p->trace;
  P.stats = p->stats;
  P.attns = p->attns;
  P.ops = p->ops; P.gemms = p->gemms; P.n_ops = p->n_ops; P.n_gemms = p->n_gemms; P.S = S; P.T = p->T;
  P.eps = eps; P.eps_pitch = eps_pitch;
  P.agents = agents; P.lanes = lanes; P.steps = steps;
  P.x_lanes = x_lanes; P.noise_lanes = noise_lanes;
  P.lanes_per_agent = lanes_per_agent; P.horizon = horizon; P.adim = adim;
  P.sched = *sched;
  {
    static int pf = -1;
    if (pf < 0) pf = getenv("AURAS_DPT_PF") ? atoi(getenv("AURAS_DPT_PF")) : 1;
    P.pf = pf;
    P.mslices = dp_mslices();
    static int dbg = -1;
    if (dbg < 0) dbg = getenv("AURAS_DPT_DBG") ? atoi(getenv("AURAS_DPT_DBG")) : 0;
    P.dbg = dbg;
  }
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

int auras_dpt_xfold(const void *kv, int kv_ld, int rows, int L, int E, int H, const float *wq, const float *bq,
                    const float *woT, const float *bo, const float *ln_g, const float *ln_b, float *out, int xs,
                    void *stream) {
  if (rows < 0 || L < 1 || H < 1 || E < 32 || E > 1024 || E % 32 || E % H || (E / H) > E || kv_ld < 2 * L * E ||
      xs < 2 * H * E + 4 || xs % 4 || !kv || !wq || !bq || !woT || !bo || !ln_g || !ln_b || !out) {
    set_error("dpt_xfold: bad arguments (E=%d H=%d L=%d xs=%d)", E, H, L, xs);
    return AURAS_E_ARG;
  }
  if (rows == 0) return AURAS_OK;
  const size_t sh = sizeof(float) * (2 * (E / H) + 32);
  dpt_xfold_kernel<<<dim3(rows, L, H), E, sh, as_stream(stream)>>>(static_cast<const __nv_bfloat16 *>(kv), kv_ld, L,
                                                                   E, H, wq, bq, woT, bo, ln_g, ln_b, out, xs);
  return cuda_check(cudaGetLastError(), "dpt_xfold");
}


// Diagnostics (AURAS_DPT_TRACE set at build): per-phase globaltimer stamps of
// the last run, n_ops + 1 values.  Returns the count copied.
int auras_dpt_persist_trace(void *plan, long long *out, int n) {
  DpPlan *p = static_cast<DpPlan *>(plan);
  if (!p || !p->trace || !out) return 0;
  const int m = std::min(n, 73 * p->n_ops + 1);   // per-phase stamps, then 8 sub-phase clocks per op
  cudaMemcpy(out, p->trace, sizeof(long long) * m, cudaMemcpyDeviceToHost);
  return m;
}

void auras_dpt_persist_free(void *plan) {
  DpPlan *p = static_cast<DpPlan *>(plan);
  if (!p) return;
  cudaFree(p->trace);
  cudaFree(p->ops);
  cudaFree(p->gemms);
  cudaFree(p->stats);
  cudaFree(p->attns);
  delete p;
}

}  // extern "C"
