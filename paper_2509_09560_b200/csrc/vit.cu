// ViT-B/16 perception pieces that are not GEMMs (BASELINE configs[3], SURVEY.md
// §2.4 K7).  The patch embedding and every linear layer run on the tcgen05
// implicit-GEMM conv path (auras_conv with 16x16/s16 and 1x1 kernels over the
// token axis, bias / GELU / residual fused in its epilogue); these kernels
// cover the rest of a pre-norm block:
//
//   vit_tokens    : [CLS; patches] + position embedding -> residual stream
//   layernorm     : per-token LayerNorm (fp32 statistics), bf16 or fp32 out
//   vit_attention : softmax(q k^T / sqrt(dh)) v per (image, head), K and V of
//                   the head staged in shared memory (row pitch padded so lanes
//                   reading different keys hit different banks)
//
// Token rows are [S][N][C] bf16 with C = heads * dh, q | k | v packed as
// [S][N][3C] in the order timm's reshape(B, N, 3, heads, dh) produces.
#include <cmath>

#include "common.cuh"

namespace auras {
namespace {

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void vit_tokens_kernel(const __nv_bfloat16 *__restrict__ patches, const float *__restrict__ cls,
                                  const float *__restrict__ pos, __nv_bfloat16 *__restrict__ x, int S, int N,
                                  int nv, int C) {
  const int64_t total = (int64_t)S * N * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int64_t r = i / C;
    const int n = (int)(r % N);
    const int64_t s = r / N;
    if (n >= nv) {                                 // pad row
      x[i] = __float2bfloat16_rn(0.f);
      continue;
    }
    const float v = n == 0 ? cls[c] : __bfloat162float(patches[(s * (nv - 1) + (n - 1)) * C + c]);
    x[i] = __float2bfloat16_rn(v + pos[(int64_t)n * C + c]);
  }
}

// One warp per row: two-pass mean / biased variance in fp32 (torch's LayerNorm).
// Rows up to 32 * LN_MAXV elements stay in registers after one read.
constexpr int LN_MAXV = 32;
template <typename TO>
__global__ void layernorm_kernel(const __nv_bfloat16 *__restrict__ in, int64_t ldi, TO *__restrict__ out,
                                 int64_t ldo, const float *__restrict__ g, const float *__restrict__ b, int rows,
                                 int C, float eps) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const __nv_bfloat16 *xr = in + warp * ldi;
  float xv[LN_MAXV];
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < LN_MAXV; ++u) {
    const int c = lane + 32 * u;
    xv[u] = c < C ? __bfloat162float(xr[c]) : 0.f;
    s += xv[u];
  }
  const float mu = warp_sum_f(s) / C;
  float q = 0.f;
#pragma unroll
  for (int u = 0; u < LN_MAXV; ++u) {
    const int c = lane + 32 * u;
    const float d = c < C ? xv[u] - mu : 0.f;
    q += d * d;
  }
  const float rstd = rsqrtf(warp_sum_f(q) / C + eps);
  TO *yr = out + warp * ldo;
#pragma unroll
  for (int u = 0; u < LN_MAXV; ++u) {
    const int c = lane + 32 * u;
    if (c < C) {
      const float v = (xv[u] - mu) * rstd * g[c] + b[c];
      if constexpr (sizeof(TO) == 4) yr[c] = v;
      else yr[c] = __float2bfloat16_rn(v);
    }
  }
}

constexpr int ATT_THREADS = 256;
constexpr int ATT_QB = 16;          // queries per CTA (two per warp): measured best with the 16-byte K/V staging

// grid (S * heads, ceil(N / ATT_QB)); dh <= 64 (two head columns per lane).
__global__ void __launch_bounds__(ATT_THREADS) vit_attention_kernel(const __nv_bfloat16 *__restrict__ qkv,
                                                                    __nv_bfloat16 *__restrict__ out, int N,
                                                                    int nv, int H, int dh, float scale) {
  extern __shared__ float sm[];
  const int C = H * dh;
  const int kp = dh + 1;                          // padded row pitch (floats): conflict-free key reads
  float *ks = sm;                                 // [N][kp]
  float *vs = ks + (int64_t)N * kp;               // [N][dh]
  float *ps = vs + (int64_t)N * dh;               // [warps][N] probabilities
  float *qs = ps + (ATT_THREADS / 32) * N;        // [warps][dh]
  const int s = blockIdx.x / H, h = blockIdx.x % H;
  const __nv_bfloat16 *base = qkv + (int64_t)s * N * 3 * C;
  if ((dh & 7) == 0) {
    // 16-byte loads, 4 rows' worth in flight per thread: an L2 round trip is
    // long enough here that a scalar loop over 2 x 12.6 K elements costs tens of us
    const int cpr = dh >> 3;                      // 8-element chunks per row
    const int total = N * cpr;
    for (int i0 = threadIdx.x; i0 < total; i0 += 4 * ATT_THREADS) {
      uint4 kq[4], vq[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * ATT_THREADS;
        if (i < total) {
          const int n = i / cpr, j = i % cpr;
          const __nv_bfloat16 *row = base + (int64_t)n * 3 * C + h * dh + 8 * j;
          kq[u] = *reinterpret_cast<const uint4 *>(row + C);
          vq[u] = *reinterpret_cast<const uint4 *>(row + 2 * C);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * ATT_THREADS;
        if (i < total) {
          const int n = i / cpr, j = i % cpr;
          const __nv_bfloat16 *kb = reinterpret_cast<const __nv_bfloat16 *>(&kq[u]);
          const __nv_bfloat16 *vb = reinterpret_cast<const __nv_bfloat16 *>(&vq[u]);
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            ks[n * kp + 8 * j + t] = __bfloat162float(kb[t]);
            vs[n * dh + 8 * j + t] = __bfloat162float(vb[t]);
          }
        }
      }
    }
  } else {
    for (int i = threadIdx.x; i < N * dh; i += ATT_THREADS) {
      const int n = i / dh, e = i % dh;
      ks[n * kp + e] = __bfloat162float(base[(int64_t)n * 3 * C + C + h * dh + e]);
      vs[n * dh + e] = __bfloat162float(base[(int64_t)n * 3 * C + 2 * C + h * dh + e]);
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float *p = ps + warp * N;
  float *q = qs + warp * dh;
  for (int qi = warp; qi < ATT_QB; qi += ATT_THREADS / 32) {
    const int n = blockIdx.y * ATT_QB + qi;
    if (n >= nv) break;                           // warp-uniform; pad rows are not queries
    for (int e = lane; e < dh; e += 32) q[e] = __bfloat162float(base[(int64_t)n * 3 * C + h * dh + e]) * scale;
    __syncwarp();
    float mx = -INFINITY;
    for (int k = lane; k < nv; k += 32) {
      const float *kr = ks + k * kp;
      float a = 0.f;
      for (int e = 0; e < dh; ++e) a = fmaf(q[e], kr[e], a);
      p[k] = a;
      mx = fmaxf(mx, a);
    }
    mx = warp_max_f(mx);
    float sum = 0.f;
    for (int k = lane; k < nv; k += 32) {
      const float e = __expf(p[k] - mx);
      p[k] = e;
      sum += e;
    }
    sum = warp_sum_f(sum);
    const float inv = 1.f / sum;
    __syncwarp();
    for (int e = lane; e < dh; e += 32) {
      float a = 0.f;
      for (int k = 0; k < nv; ++k) a = fmaf(p[k], vs[k * dh + e], a);
      out[((int64_t)s * N + n) * C + h * dh + e] = __float2bfloat16_rn(a * inv);
    }
    __syncwarp();
  }
}

}  // namespace
}  // namespace auras

using namespace auras;

extern "C" int auras_vit_tokens(const void *patches, const float *cls, const float *pos, void *x, int S, int N,
                                int n_valid, int C, void *stream) {
  if (S < 1 || n_valid < 2 || N < n_valid || C < 1) {
    set_error("vit_tokens: bad sizes S=%d N=%d C=%d", S, N, C);
    return AURAS_E_ARG;
  }
  const int64_t total = (int64_t)S * N * C;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  vit_tokens_kernel<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const __nv_bfloat16 *>(patches), cls, pos,
                                                         static_cast<__nv_bfloat16 *>(x), S, N, n_valid, C);
  AURAS_LAUNCHED("vit_tokens");
  return AURAS_OK;
}

extern "C" int auras_layernorm(const void *in, int64_t ldi, void *out, int64_t ldo, int out_f32, const float *gamma,
                               const float *beta, int rows, int C, float eps, void *stream) {
  if (rows < 1 || C < 1 || C > 32 * LN_MAXV) {
    set_error("layernorm: bad sizes rows=%d C=%d (C <= %d)", rows, C, 32 * LN_MAXV);
    return AURAS_E_ARG;
  }
  const int grid = (rows * 32 + 255) / 256;
  const auto *x = static_cast<const __nv_bfloat16 *>(in);
  if (out_f32)
    layernorm_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(x, ldi, static_cast<float *>(out), ldo, gamma,
                                                                 beta, rows, C, eps);
  else
    layernorm_kernel<__nv_bfloat16><<<grid, 256, 0, as_stream(stream)>>>(
        x, ldi, static_cast<__nv_bfloat16 *>(out), ldo, gamma, beta, rows, C, eps);
  AURAS_LAUNCHED("layernorm");
  return AURAS_OK;
}

extern "C" int auras_vit_attention(const void *qkv, void *out, int S, int N, int n_valid, int heads, int dh,
                                   void *stream) {
  if (S < 1 || n_valid < 1 || N < n_valid || heads < 1 || dh < 1 || dh > 64) {
    set_error("vit_attention: bad sizes S=%d N=%d heads=%d dh=%d", S, N, heads, dh);
    return AURAS_E_ARG;
  }
  const size_t smem = sizeof(float) * ((size_t)N * (dh + 1) + (size_t)N * dh + (ATT_THREADS / 32) * (size_t)N +
                                       (ATT_THREADS / 32) * (size_t)dh);
  if (smem > 220 * 1024) {
    set_error("vit_attention: %d tokens need %zu B of shared memory", N, smem);
    return AURAS_E_ARG;
  }
  if (smem > 48 * 1024)
    if (int rc = ensure_smem_attr(vit_attention_kernel, (int)smem)) return rc;
  dim3 grid(S * heads, (n_valid + ATT_QB - 1) / ATT_QB);
  vit_attention_kernel<<<grid, ATT_THREADS, smem, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16 *>(qkv), static_cast<__nv_bfloat16 *>(out), N, n_valid, heads, dh,
      1.f / sqrtf((float)dh));
  AURAS_LAUNCHED("vit_attention");
  return AURAS_OK;
}
