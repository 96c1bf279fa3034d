// Implicit-GEMM convolution (SIMT path), fused conv epilogue, GEMV and the
// perception helpers of the Diffusion Policy plugin.
//
// The SIMT GEMM is the fp32 "reference precision" engine and the fallback for
// shapes the tcgen05 engine (gemm_sm100.cu) does not take.  The epilogue is
// shared by both engines.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "conv.cuh"
#include "epi.cuh"

namespace auras {

// ------------------------------------------------------------------ GEMM (SIMT)
// partial[split][m][n] = sum_{k in split} W[m][k] * B[n][k]
// B[n][k] = in[s, oy*st-ph+ky, ox*st-pw+kx, c]; n=(s,oy,ox), k=((ky*kw+kx)*Cin + c)
constexpr int SB_M = 64, SB_N = 64, SB_K = 32;

template <typename T>
__global__ void __launch_bounds__(256) conv_gemm_simt(ConvGemmArgs a) {
  __shared__ float As[SB_K][SB_M + 4];
  __shared__ float Bs[SB_K][SB_N + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.x * SB_M, n0 = blockIdx.y * SB_N;
  const int kb = blockIdx.z * a.kchunk;
  const int ke = min(a.Kp, kb + a.kchunk);
  const T *W = static_cast<const T *>(a.w);
  const T *X = static_cast<const T *>(a.in);
  const int P = a.Ho * a.Wo;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k0 = kb; k0 < ke; k0 += SB_K) {
#pragma unroll
    for (int e = 0; e < (SB_M * SB_K) / 256; ++e) {
      const int idx = tid + e * 256;
      const int mm = idx / SB_K, kk = idx % SB_K;
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < a.M && k < ke) ? Elem<T>::load(W + (int64_t)m * a.Kp + k) : 0.f;
    }
#pragma unroll
    for (int e = 0; e < (SB_N * SB_K) / 256; ++e) {
      const int idx = tid + e * 256;
      const int nn = idx / SB_K, kk = idx % SB_K;
      const int n = n0 + nn, k = k0 + kk;
      float v = 0.f;
      if (n < a.N && k < ke && k < a.Kreal) {
        const int s = n / P, p = n - s * P;
        const int oy = p / a.Wo, ox = p - oy * a.Wo;
        const int tap = k / a.Cin, c = k - tap * a.Cin;
        const int ky = tap / a.kw, kx = tap - ky * a.kw;
        const int iy = oy * a.stride - a.pad_h + ky, ix = ox * a.stride - a.pad_w + kx;
        if (iy >= 0 && iy < a.H && ix >= 0 && ix < a.W)
          v = Elem<T>::load(X + ((int64_t)(s * a.H + iy) * a.W + ix) * a.in_pitch + a.in_coff + c);
      }
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < SB_K; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][tx * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][ty * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float *out = a.partial + (int64_t)blockIdx.z * a.N * a.M;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int n = n0 + ty * 4 + j;
    if (n >= a.N) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + tx * 4 + i;
      if (m < a.M) out[(int64_t)m * a.N + n] = acc[i][j];
    }
  }
}

template <typename T>
int launch_conv_gemm_simt(const ConvGemmArgs &a, cudaStream_t st) {
  dim3 grid((a.M + SB_M - 1) / SB_M, (a.N + SB_N - 1) / SB_N, a.splits);
  conv_gemm_simt<T><<<grid, 256, 0, st>>>(a);
  AURAS_LAUNCHED("conv_gemm_simt");
  return AURAS_OK;
}

// ------------------------------------------------------------------ epilogue
template <typename T>
__global__ void __launch_bounds__(512) conv_epilogue(EpiArgs a) {
  __shared__ float red[32];
  epi_unit<T>(a, blockIdx.x, blockIdx.y, threadIdx.x, blockDim.x, red, [] __device__() { __syncthreads(); });
}

template <typename T>
int launch_conv_epilogue(const EpiArgs &a, int S, cudaStream_t st) {
  const bool gn = a.gn_gamma != nullptr;
  if (gn && (a.groups <= 0 || a.M % a.groups)) { set_error("epilogue: M %% groups"); return AURAS_E_ARG; }
  if (a.pool_out && !a.out_f32) { set_error("epilogue: pool without out_f32"); return AURAS_E_ARG; }
  dim3 grid(S, gn ? a.groups : (a.M + 63) / 64);
  conv_epilogue<T><<<grid, 512, 0, st>>>(a);
  AURAS_LAUNCHED("conv_epilogue");
  return AURAS_OK;
}

// Token-wise epilogue for 1-row convolutions without GroupNorm / FiLM / pooling
// (the ViT linear layers, op.cta_target > 0): the split-K partials are
// [split][m][n] and the output rows [n][pitch], so a 32 x 32 tile is summed
// with n-contiguous reads, transposed through shared memory and stored with
// m-contiguous writes.  bias -> act -> + residual, as epi_unit.
template <typename T>
__global__ void __launch_bounds__(256) tok_epilogue(EpiArgs a) {
  __shared__ float tile[32][33];
  const int m0 = blockIdx.x * 32, n0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t NM = (int64_t)a.N * a.M;
  for (int i = ty; i < 32; i += 8) {
    const int m = m0 + i, n = n0 + tx;
    float v = 0.f;
    if (m < a.M && n < a.N) {
      v = a.bias ? a.bias[m] : 0.f;
      const float *pp = a.partial + (int64_t)m * a.N + n;
      int z = 0;
      for (; z + 4 <= a.splits; z += 4) {          // four split loads in flight
        const float t0 = pp[z * NM], t1 = pp[(z + 1) * NM], t2 = pp[(z + 2) * NM], t3 = pp[(z + 3) * NM];
        v += (t0 + t1) + (t2 + t3);
      }
      for (; z < a.splits; ++z) v += pp[z * NM];
      v = activate(v, a.act);
    }
    tile[i][tx] = v;
  }
  __syncthreads();
  const T *res = static_cast<const T *>(a.res);
  T *out = static_cast<T *>(a.out);
  for (int i = ty; i < 32; i += 8) {
    const int n = n0 + i, m = m0 + tx;
    if (m < a.M && n < a.N) {
      float v = tile[tx][i];
      if (res) v += Elem<T>::load(res + (int64_t)n * a.res_pitch + a.res_coff + m);
      Elem<T>::store(out + (int64_t)n * a.out_pitch + a.out_coff + m, v);
    }
  }
}

// Token epilogue fused with the LayerNorm that follows a residual add (the
// DP-T decoder, M <= 1024): one CTA per token (measured faster than 8 per
// CTA: more CTAs in flight), one thread per channel;
// out[n] = partials + bias + residual (bf16, stored), ln[n] = LayerNorm(out[n])
// with fp32 statistics of the stored (rounded) values, as a separate
// layernorm launch would compute them.
constexpr int TLN_TOK = 1;
__global__ void __launch_bounds__(1024) tok_epilogue_ln(EpiArgs a, const float *__restrict__ g,
                                                         const float *__restrict__ b, __nv_bfloat16 *__restrict__ ln,
                                                         int ln_pitch, float eps) {
  __shared__ float red[2][TLN_TOK][32];
  const int m = threadIdx.x, n0 = blockIdx.x * TLN_TOK;
  const int warp = m >> 5, lane = m & 31, nw = blockDim.x >> 5;
  const int64_t NM = (int64_t)a.N * a.M;
  const auto *res = static_cast<const __nv_bfloat16 *>(a.res);
  auto *out = static_cast<__nv_bfloat16 *>(a.out);
  float y[TLN_TOK];
#pragma unroll
  for (int t = 0; t < TLN_TOK; ++t) {
    const int n = n0 + t;
    float v = 0.f;
    if (n < a.N && m < a.M) {
      v = a.bias ? a.bias[m] : 0.f;
      for (int z = 0; z < a.splits; ++z) v += a.partial[z * NM + (int64_t)m * a.N + n];
      v = activate(v, a.act);
      if (res) v += __bfloat162float(res[(int64_t)n * a.res_pitch + a.res_coff + m]);
      const __nv_bfloat16 hv = __float2bfloat16_rn(v);
      out[(int64_t)n * a.out_pitch + a.out_coff + m] = hv;
      v = __bfloat162float(hv);
    }
    y[t] = v;
  }
  // mean, then biased variance, per token (block reductions over the channels)
  float part[TLN_TOK];
#pragma unroll
  for (int t = 0; t < TLN_TOK; ++t) {
    float v = y[t];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    part[t] = v;
  }
  if (lane == 0)
    for (int t = 0; t < TLN_TOK; ++t) red[0][t][warp] = part[t];
  __syncthreads();
  float mu[TLN_TOK];
#pragma unroll
  for (int t = 0; t < TLN_TOK; ++t) {
    float sum = 0.f;
    for (int w = 0; w < nw; ++w) sum += red[0][t][w];
    mu[t] = sum / a.M;
    float d = m < a.M ? y[t] - mu[t] : 0.f;
    d *= d;
    for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    part[t] = d;
  }
  if (lane == 0)
    for (int t = 0; t < TLN_TOK; ++t) red[1][t][warp] = part[t];
  __syncthreads();
#pragma unroll
  for (int t = 0; t < TLN_TOK; ++t) {
    const int n = n0 + t;
    float q = 0.f;
    for (int w = 0; w < nw; ++w) q += red[1][t][w];
    const float rstd = rsqrtf(q / a.M + eps);
    if (n < a.N && m < a.M)
      ln[(int64_t)n * ln_pitch + m] = __float2bfloat16_rn((y[t] - mu[t]) * rstd * g[m] + b[m]);
  }
}

// ------------------------------------------------------------------ linear / GEMV
// y[n][m] = sum_k W[m][k] * f(x[n][k]) + b[m]; one warp per output row m,
// x staged in shared memory; weights streamed once with 16-byte loads.
constexpr int LIN_NMAX = 8;

template <typename T>
__global__ void __launch_bounds__(256) linear_kernel(LinArgs a) {
  extern __shared__ float xs[];   // [N][Kp]
  const int Kp = a.ldw;
  for (int i = threadIdx.x; i < a.N * Kp; i += blockDim.x) {
    const int n = i / Kp, k = i - n * Kp;
    float v = k < a.K ? a.x[(int64_t)n * a.ldx + k] : 0.f;
    xs[i] = a.mish_in ? mish(v) : v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const T *W = static_cast<const T *>(a.w);
  for (int m = blockIdx.x * warps + (threadIdx.x >> 5); m < a.M; m += gridDim.x * warps) {
    float acc[LIN_NMAX];
#pragma unroll
    for (int n = 0; n < LIN_NMAX; ++n) acc[n] = 0.f;
    const T *wr = W + (int64_t)m * Kp;
    for (int k = lane * 8; k < Kp; k += 256) {
      float wv[8];
      if constexpr (sizeof(T) == 2) {
        const uint4 raw = *reinterpret_cast<const uint4 *>(wr + k);
        const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&raw);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(h[q]);
          wv[2 * q] = f.x;
          wv[2 * q + 1] = f.y;
        }
      } else {
        const float4 r0 = *reinterpret_cast<const float4 *>(wr + k);
        const float4 r1 = *reinterpret_cast<const float4 *>(wr + k + 4);
        wv[0] = r0.x; wv[1] = r0.y; wv[2] = r0.z; wv[3] = r0.w;
        wv[4] = r1.x; wv[5] = r1.y; wv[6] = r1.z; wv[7] = r1.w;
      }
#pragma unroll
      for (int n = 0; n < LIN_NMAX; ++n) {
        if (n < a.N) {
          const float *xr = xs + n * Kp + k;
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[n] = fmaf(wv[q], xr[q], acc[n]);
        }
      }
    }
#pragma unroll
    for (int n = 0; n < LIN_NMAX; ++n) {
      if (n < a.N) {
        const float v = warp_sum(acc[n]);
        if (lane == 0) a.y[(int64_t)n * a.ldy + m] = v + (a.bias ? a.bias[m] : 0.f);
      }
    }
  }
}

template <typename T>
int launch_linear(LinArgs a, cudaStream_t st) {
  if (a.ldw % 8) { set_error("linear: weight row stride must be a multiple of 8"); return AURAS_E_ARG; }
  const int N = a.N;
  for (int n0 = 0; n0 < N; n0 += LIN_NMAX) {
    LinArgs b = a;
    b.N = std::min(LIN_NMAX, N - n0);
    b.x = a.x + (int64_t)n0 * a.ldx;
    b.y = a.y + (int64_t)n0 * a.ldy;
    const size_t smem = sizeof(float) * b.N * a.ldw;
    if (smem > 200 * 1024) { set_error("linear: K too large"); return AURAS_E_ARG; }
    if (smem > 48 * 1024)
      if (int rc = ensure_smem_attr(linear_kernel<T>, (int)smem)) return rc;
    int blocks = (a.M + 7) / 8;
    blocks = std::min(blocks, 148 * 8);
    linear_kernel<T><<<blocks, 256, smem, st>>>(b);
    AURAS_LAUNCHED("linear_kernel");
  }
  return AURAS_OK;
}

// ------------------------------------------------------------------ perception helpers
template <typename T>
__global__ void image_to_nhwc_kernel(const uint8_t *img, int S, int C, int H, int W, T *out, int cpad) {
  const int64_t total = (int64_t)S * H * W * cpad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = i % cpad;
    const int64_t pix = i / cpad;
    const int x = pix % W;
    const int64_t t = pix / W;
    const int y = t % H;
    const int s = t / H;
    float v = 0.f;
    if (c < C) v = img[(((int64_t)s * C + c) * H + y) * W + x] * (2.f / 255.f) - 1.f;
    Elem<T>::store(out + i, v);
  }
}

template <typename T>
__global__ void maxpool3s2_kernel(const T *in, int S, int H, int W, int C, T *out) {
  const int Ho = (H + 2 - 3) / 2 + 1, Wo = (W + 2 - 3) / 2 + 1;
  const int64_t total = (int64_t)S * Ho * Wo * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = i % C;
    const int64_t pix = i / C;
    const int ox = pix % Wo;
    const int64_t t = pix / Wo;
    const int oy = t % Ho;
    const int s = t / Ho;
    float m = -INFINITY;
    for (int dy = 0; dy < 3; ++dy) {
      const int iy = oy * 2 - 1 + dy;
      if (iy < 0 || iy >= H) continue;
      for (int dx = 0; dx < 3; ++dx) {
        const int ix = ox * 2 - 1 + dx;
        if (ix < 0 || ix >= W) continue;
        m = fmaxf(m, Elem<T>::load(in + (((int64_t)s * H + iy) * W + ix) * C + c));
      }
    }
    Elem<T>::store(out + i, m);
  }
}

__global__ void assemble_cond_kernel(const float *feat, const float *pos, float *prev, int feat_dim,
                                     int pos_dim, int n_obs, int first, float *gc_out,
                                     int64_t row_stride) {
  const int a = blockIdx.x;
  const int d = feat_dim + pos_dim;
  float *dst = gc_out + a * row_stride;
  float *pv = prev + (int64_t)a * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float cur = i < feat_dim ? feat[(int64_t)a * feat_dim + i] : pos[(int64_t)a * pos_dim + i - feat_dim];
    if (n_obs == 2) {
      const float old = first ? cur : pv[i];
      dst[i] = old;
      dst[d + i] = cur;
    } else {
      dst[i] = cur;
    }
    pv[i] = cur;
  }
}

__global__ void sinusoidal_kernel(const int32_t *t, int n, int dim, float *out) {
  const int half = dim / 2;
  const float scale = logf(10000.f) / (half - 1);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * half; i += gridDim.x * blockDim.x) {
    const int r = i / half, j = i - r * half;
    const float arg = (float)t[r] * expf(-scale * j);
    out[(int64_t)r * dim + j] = sinf(arg);
    out[(int64_t)r * dim + half + j] = cosf(arg);
  }
}

__global__ void copy_f32_kernel(float *dst, const float *src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

struct FinishBatch {
  int agents[64];
  int lanes[64];
};

__global__ void dp_finish_kernel(const float *x, FinishBatch b, int n, int lanes_per_agent,
                                 int row_floats, float *out) {
  const int i = blockIdx.x;
  if (i >= n) return;
  const float *src = x + ((int64_t)b.agents[i] * lanes_per_agent + b.lanes[i]) * row_floats;
  for (int j = threadIdx.x; j < row_floats; j += blockDim.x) out[(int64_t)i * row_floats + j] = src[j];
}

// ------------------------------------------------------------------ dispatch helpers
int conv_op_to_args(const auras_conv_op &op, int S, int dtype, float *partial, ConvGemmArgs &g, EpiArgs &e) {
  if (op.M <= 0 || op.Cin <= 0 || op.Kp <= 0 || op.splits <= 0 || op.kh <= 0 || op.kw <= 0) {
    set_error("conv op: bad shape M=%d Cin=%d Kp=%d splits=%d", op.M, op.Cin, op.Kp, op.splits);
    return AURAS_E_ARG;
  }
  memset(&g, 0, sizeof(g));
  memset(&e, 0, sizeof(e));
  g.w = op.w; g.in = op.in; g.partial = partial;
  g.M = op.M; g.N = S * op.Ho * op.Wo; g.Kp = op.Kp; g.Kreal = op.kh * op.kw * op.Cin;
  g.Cin = op.Cin; g.H = op.H; g.W = op.W; g.in_pitch = op.in_pitch; g.in_coff = op.in_coff;
  g.kh = op.kh; g.kw = op.kw; g.stride = op.stride; g.pad_h = op.pad_h; g.pad_w = op.pad_w;
  g.Ho = op.Ho; g.Wo = op.Wo; g.splits = op.splits; g.cta_target = op.cta_target;
  if (dtype == AURAS_DT_BF16 && gemm_sm100_supported(g)) {
    g.engine = 1;
    g.splits = gemm_sm100_splits(g);
    g.kchunk = 0;
  } else if (dtype == AURAS_DT_BF16 && gemm_gather_supported(g) && !getenv("AURAS_NO_GATHER")) {
    g.engine = 2;
    g.splits = gemm_gather_splits(g);
    g.kchunk = 0;
  } else {
    int kc = (op.Kp + op.splits - 1) / op.splits;
    kc = (kc + 63) / 64 * 64;
    g.kchunk = kc;
    g.splits = (op.Kp + kc - 1) / kc;
  }
  e.partial = partial; e.bias = op.bias; e.gn_gamma = op.gn_gamma; e.gn_beta = op.gn_beta;
  e.res = op.res; e.res_f32 = op.res_f32; e.out = op.out; e.out_f32 = op.out_f32;
  e.M = op.M; e.N = g.N; e.Ho = op.Ho; e.Wo = op.Wo; e.splits = g.splits; e.groups = op.groups;
  e.act = op.act; e.res_before_act = op.res_before_act; e.film_off = op.film_off;
  e.out_pitch = op.out_pitch; e.out_coff = op.out_coff; e.res_pitch = op.res_pitch;
  e.res_coff = op.res_coff; e.out_stuff = op.out_stuff; e.pool_out = op.pool_out;
  return AURAS_OK;
}

int run_gemm(const ConvGemmArgs &g, int dtype, cudaStream_t st) {
  if (g.engine == 1) return launch_gemm_sm100(g, st);
  if (g.engine == 2) return launch_gemm_gather(g, st);
  if (dtype == AURAS_DT_BF16) return launch_conv_gemm_simt<__nv_bfloat16>(g, st);
  return launch_conv_gemm_simt<float>(g, st);
}

int run_epilogue(const EpiArgs &e, int S, int dtype, cudaStream_t st) {
  return dtype == AURAS_DT_BF16 ? launch_conv_epilogue<__nv_bfloat16>(e, S, st)
                                : launch_conv_epilogue<float>(e, S, st);
}

int64_t conv_scratch_floats(const auras_conv_op &op, int S, int dtype) {
  ConvGemmArgs g;
  EpiArgs e;
  if (conv_op_to_args(op, S, dtype, nullptr, g, e)) return 0;
  return (int64_t)g.splits * S * op.Ho * op.Wo * op.M;
}

}  // namespace auras

using namespace auras;

extern "C" int64_t auras_conv_scratch_floats(const auras_conv_op *op, int dtype, int S) {
  return op ? conv_scratch_floats(*op, S, dtype) : -1;
}

extern "C" {

int auras_conv_ln(const auras_conv_op *op, int dtype, int S, const float *ln_gamma, const float *ln_beta,
                  void *ln_out, int ln_pitch, float eps, float *scratch, int64_t scratch_floats, void *stream) {
  if (!op || !scratch || !ln_out || dtype != AURAS_DT_BF16) { set_error("conv_ln: bad args"); return AURAS_E_ARG; }
  if (op->gn_gamma || op->pool_out || op->film_off >= 0 || op->out_stuff || op->out_f32 || op->res_f32 ||
      op->Ho != 1 || op->M > 1024 || op->M % 32) {
    set_error("conv_ln: only plain 1-row token convolutions with M <= 1024, M %% 32 == 0");
    return AURAS_E_ARG;
  }
  if (conv_scratch_floats(*op, S, dtype) > scratch_floats) { set_error("conv_ln: scratch too small"); return AURAS_E_ARG; }
  ConvGemmArgs g;
  EpiArgs e;
  int rc = conv_op_to_args(*op, S, dtype, scratch, g, e);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  if ((rc = run_gemm(g, dtype, st))) return rc;
  tok_epilogue_ln<<<(e.N + TLN_TOK - 1) / TLN_TOK, e.M, 0, st>>>(e, ln_gamma, ln_beta,
                                                                static_cast<__nv_bfloat16 *>(ln_out), ln_pitch, eps);
  AURAS_LAUNCHED("tok_epilogue_ln");
  return AURAS_OK;
}

int auras_conv(const auras_conv_op *op, int dtype, int S, const float *film_rows, int film_stride,
               float *scratch, int64_t scratch_floats, void *stream) {
  if (!op || !scratch) { set_error("conv: null"); return AURAS_E_ARG; }
  if (conv_scratch_floats(*op, S, dtype) > scratch_floats) { set_error("conv: scratch too small"); return AURAS_E_ARG; }
  ConvGemmArgs g;
  EpiArgs e;
  int rc = conv_op_to_args(*op, S, dtype, scratch, g, e);
  if (rc) return rc;
  if (op->film_off >= 0) {
    if (!film_rows) { set_error("conv: FiLM op without film rows"); return AURAS_E_ARG; }
    e.film_a = film_rows;
    e.film_a_stride = film_stride;
  }
  cudaStream_t st = as_stream(stream);
  if ((rc = run_gemm(g, dtype, st))) return rc;
  // (any Ho: NHWC rows ((s * Ho + y) * Wo + x) are the GEMM's n in order)
  if (op->cta_target > 0 && !e.gn_gamma && !e.pool_out && e.film_off < 0 && !e.out_stuff && !e.out_f32 &&
      !e.res_f32 && e.out) {
    dim3 grid((e.M + 31) / 32, (e.N + 31) / 32);
    if (dtype == AURAS_DT_BF16) tok_epilogue<__nv_bfloat16><<<grid, 256, 0, st>>>(e);
    else tok_epilogue<float><<<grid, 256, 0, st>>>(e);
    AURAS_LAUNCHED("tok_epilogue");
    return AURAS_OK;
  }
  return run_epilogue(e, S, dtype, st);
}

int auras_linear(const auras_linear_op *op, int dtype, int N, const float *x, int ldx, float *y, int ldy,
                 void *stream) {
  if (!op || !x || !y || N <= 0) { set_error("linear: bad args"); return AURAS_E_ARG; }
  LinArgs a;
  memset(&a, 0, sizeof(a));
  a.w = op->w; a.bias = op->bias; a.M = op->M; a.K = op->K; a.ldw = op->ldw ? op->ldw : op->K;
  a.mish_in = op->mish_in; a.N = N; a.x = x; a.ldx = ldx; a.y = y; a.ldy = ldy;
  return dtype == AURAS_DT_BF16 ? launch_linear<__nv_bfloat16>(a, as_stream(stream))
                                : launch_linear<float>(a, as_stream(stream));
}

int auras_image_to_nhwc(const uint8_t *img, int S, int C, int H, int W, void *out, int cpad, int dtype,
                        void *stream) {
  const int64_t total = (int64_t)S * H * W * cpad;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  if (dtype == AURAS_DT_BF16)
    image_to_nhwc_kernel<__nv_bfloat16><<<blocks, 256, 0, as_stream(stream)>>>(
        img, S, C, H, W, static_cast<__nv_bfloat16 *>(out), cpad);
  else
    image_to_nhwc_kernel<float><<<blocks, 256, 0, as_stream(stream)>>>(img, S, C, H, W,
                                                                        static_cast<float *>(out), cpad);
  AURAS_LAUNCHED("image_to_nhwc");
  return AURAS_OK;
}

int auras_maxpool3s2(const void *in, int S, int H, int W, int C, void *out, int dtype, void *stream) {
  const int Ho = (H - 1) / 2 + 1, Wo = (W - 1) / 2 + 1;
  const int64_t total = (int64_t)S * Ho * Wo * C;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  if (dtype == AURAS_DT_BF16)
    maxpool3s2_kernel<__nv_bfloat16><<<blocks, 256, 0, as_stream(stream)>>>(
        static_cast<const __nv_bfloat16 *>(in), S, H, W, C, static_cast<__nv_bfloat16 *>(out));
  else
    maxpool3s2_kernel<float><<<blocks, 256, 0, as_stream(stream)>>>(static_cast<const float *>(in), S, H,
                                                                     W, C, static_cast<float *>(out));
  AURAS_LAUNCHED("maxpool3s2");
  return AURAS_OK;
}

int auras_dp_assemble_cond(const float *feat, const float *pos, float *prev_cache, int A, int feat_dim,
                           int pos_dim, int n_obs_steps, int first, float *gc_out, int64_t gc_row_stride,
                           void *stream) {
  if (A <= 0 || (n_obs_steps != 1 && n_obs_steps != 2)) { set_error("assemble_cond: bad args"); return AURAS_E_ARG; }
  assemble_cond_kernel<<<A, 256, 0, as_stream(stream)>>>(feat, pos, prev_cache, feat_dim, pos_dim,
                                                         n_obs_steps, first, gc_out, gc_row_stride);
  AURAS_LAUNCHED("assemble_cond");
  return AURAS_OK;
}

int auras_sinusoidal(const int32_t *t, int n, int dim, float *out, void *stream) {
  if (dim % 2 || dim < 4) { set_error("sinusoidal: dim"); return AURAS_E_ARG; }
  sinusoidal_kernel<<<std::max(1, (n * dim / 2 + 255) / 256), 256, 0, as_stream(stream)>>>(t, n, dim, out);
  AURAS_LAUNCHED("sinusoidal");
  return AURAS_OK;
}

int auras_dp_copy_rows(float *dst, const float *src, int64_t n_floats, void *stream) {
  const int blocks = (int)std::min<int64_t>((n_floats + 255) / 256, 148 * 4);
  copy_f32_kernel<<<std::max(blocks, 1), 256, 0, as_stream(stream)>>>(dst, src, n_floats);
  AURAS_LAUNCHED("copy_f32");
  return AURAS_OK;
}

int auras_dp_finish(const float *x_lanes, int A, const int *agents, const int *lanes, int n,
                    int lanes_per_agent, int row_floats, float *out, void *stream) {
  if (n <= 0) return AURAS_OK;
  if (n > 64) { set_error("dp_finish: n > 64"); return AURAS_E_ARG; }
  FinishBatch b;
  memset(&b, 0, sizeof(b));
  for (int i = 0; i < n; ++i) {
    if (agents[i] < 0 || agents[i] >= A) { set_error("dp_finish: agent"); return AURAS_E_ARG; }
    b.agents[i] = agents[i];
    b.lanes[i] = lanes[i];
  }
  dp_finish_kernel<<<n, 64, 0, as_stream(stream)>>>(x_lanes, b, n, lanes_per_agent, row_floats, out);
  AURAS_LAUNCHED("dp_finish");
  return AURAS_OK;
}

}  // extern "C"
