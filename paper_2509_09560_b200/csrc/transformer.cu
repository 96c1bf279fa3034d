// Causal pre-norm transformer with a KV cache in HBM, fp64 (fp/transformer.py:69-211),
// the model behind the autoregressive merged prefill.
//
// One forward = rows [start, start + n) of a sequence whose rows [0, start)
// already sit in the KV cache: a prefill is start = 0, a decode is n = 1,
// start = cache length.  Per layer two row-parallel kernels:
//
//   tf_qkv   : (layer 0: token / embedding + position) -> LN1 -> q, k, v;
//              k, v go straight into the cache row, q into a scratch row
//   tf_block : causal attention of the row over cache rows 0..pos, out
//              projection + residual, LN2, GELU MLP + residual (and the final
//              LN after the last layer)
//
// Every row's arithmetic is the same sequence of operations whichever CTA,
// launch or prefill length computes it, and a row reads only cache rows at
// or before its own position.  So a merged prefill reproduces a separate
// shorter prefill (or prefill + decodes) bit for bit, and perturbing a later
// token leaves earlier rows bit-identical -- stronger than the reference's
// 1e-5 relative tolerance (t/test_transformer.py:8, :166-173).
//
// Sizes are tiny (d = 64, 4 heads, 4 layers, <= 256 positions): the kernels are
// latency bound.  Each CTA takes TF_R rows so a weight element loaded from L2
// feeds TF_R FMAs; weights are read with consecutive threads on consecutive
// output columns (coalesced).
#include <cmath>

#include "common.cuh"

namespace auras {
namespace {

constexpr int TF_R = 4;        // rows per CTA
constexpr int TF_THREADS = 256;

struct TfDims {
  int d, h, dh, layers, vocab, max_len;
};

// Parameter blob offsets (doubles); the host packs the blob in this order.
__host__ __device__ inline int64_t tf_layer_stride(int d) { return 12LL * d * d + 9LL * d; }
__host__ __device__ inline int64_t tf_layer_base(const TfDims &m, int l) {
  return (int64_t)m.vocab * m.d + (int64_t)m.max_len * m.d + l * tf_layer_stride(m.d);
}
struct TfLayer {
  const double *ln1_g, *ln1_b, *wq, *wk, *wv, *wo, *ln2_g, *ln2_b, *w1, *b1, *w2, *b2;
};
__device__ inline TfLayer tf_layer(const double *prm, const TfDims &m, int l) {
  const int d = m.d;
  const double *p = prm + tf_layer_base(m, l);
  TfLayer L;
  L.ln1_g = p; p += d;
  L.ln1_b = p; p += d;
  L.wq = p; p += (int64_t)d * d;
  L.wk = p; p += (int64_t)d * d;
  L.wv = p; p += (int64_t)d * d;
  L.wo = p; p += (int64_t)d * d;
  L.ln2_g = p; p += d;
  L.ln2_b = p; p += d;
  L.w1 = p; p += 4LL * d * d;
  L.b1 = p; p += 4LL * d;
  L.w2 = p; p += 4LL * d * d;
  L.b2 = p;
  return L;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// LayerNorm of `rows` rows of width d (fp/transformer.py:59-62): one warp per
// row, two-pass mean / biased variance, eps 1e-5.
__device__ void tf_layer_norm(const double *x, double *y, int rows, int d, const double *g,
                              const double *b) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < rows; r += TF_THREADS / 32) {
    const double *xr = x + r * d;
    double s = 0.0;
    for (int i = lane; i < d; i += 32) s += xr[i];
    const double mu = warp_sum_d(s) / d;
    double q = 0.0;
    for (int i = lane; i < d; i += 32) {
      const double c = xr[i] - mu;
      q += c * c;
    }
    const double var = warp_sum_d(q) / d;
    const double inv = sqrt(var + 1e-5);
    for (int i = lane; i < d; i += 32) y[r * d + i] = (xr[i] - mu) / inv * g[i] + b[i];
  }
}

__device__ __forceinline__ double tf_gelu(double x) {
  const double c = 0.7978845608028654;  // sqrt(2 / pi)
  return 0.5 * x * (1.0 + tanh(c * (x + 0.044715 * (x * x * x))));
}

// out[r][j] (+)= sum_i a[r][i] * W[i][j] for TF_R rows, columns j < ncols.
template <typename Emit>
__device__ __forceinline__ void tf_rows_gemv(const double *a, int lda, int rows, int k, const double *W,
                                             int ncols, Emit emit) {
  for (int j = threadIdx.x; j < ncols; j += TF_THREADS) {
    double acc[TF_R];
#pragma unroll
    for (int r = 0; r < TF_R; ++r) acc[r] = 0.0;
    for (int i = 0; i < k; ++i) {
      const double w = __ldg(W + (int64_t)i * ncols + j);
#pragma unroll
      for (int r = 0; r < TF_R; ++r) acc[r] = fma(a[r * lda + i], w, acc[r]);
    }
#pragma unroll
    for (int r = 0; r < TF_R; ++r)
      if (r < rows) emit(r, j, acc[r]);
  }
}

__global__ void __launch_bounds__(TF_THREADS) tf_qkv(const double *__restrict__ prm, TfDims m, int layer,
                                                     const int *__restrict__ ids,
                                                     const double *__restrict__ emb, int start, int n,
                                                     double *__restrict__ kv, double *__restrict__ resid,
                                                     double *__restrict__ qbuf) {
  extern __shared__ double sm[];
  const int d = m.d;
  double *xs = sm;                 // [TF_R][d]
  double *as = xs + TF_R * d;      // [TF_R][d]
  const int r0 = blockIdx.x * TF_R;
  const int rows = min(TF_R, n - r0);
  for (int idx = threadIdx.x; idx < TF_R * d; idx += TF_THREADS) {
    const int r = idx / d, c = idx % d;
    double v = 0.0;
    if (r < rows) {
      const int row = r0 + r;
      if (layer == 0) {
        // fp/transformer.py:104-109,126: token (or given) embedding + position
        const double e = ids ? prm[(int64_t)ids[row] * d + c] : emb[(int64_t)row * d + c];
        v = e + prm[(int64_t)m.vocab * d + (int64_t)(start + row) * d + c];
        resid[(int64_t)row * d + c] = v;
      } else {
        v = resid[(int64_t)row * d + c];
      }
    }
    xs[idx] = v;
  }
  __syncthreads();
  const TfLayer L = tf_layer(prm, m, layer);
  tf_layer_norm(xs, as, rows, d, L.ln1_g, L.ln1_b);
  __syncthreads();
  double *kc = kv + (int64_t)layer * 2 * m.max_len * d;
  double *vc = kc + (int64_t)m.max_len * d;
  tf_rows_gemv(as, d, rows, d, L.wq, d, [&](int r, int j, double v) { qbuf[(int64_t)(r0 + r) * d + j] = v; });
  tf_rows_gemv(as, d, rows, d, L.wk, d,
               [&](int r, int j, double v) { kc[(int64_t)(start + r0 + r) * d + j] = v; });
  tf_rows_gemv(as, d, rows, d, L.wv, d,
               [&](int r, int j, double v) { vc[(int64_t)(start + r0 + r) * d + j] = v; });
}

__global__ void __launch_bounds__(TF_THREADS) tf_block(const double *__restrict__ prm, TfDims m, int layer,
                                                       int start, int n, const double *__restrict__ kv,
                                                       double *__restrict__ resid,
                                                       const double *__restrict__ qbuf,
                                                       double *__restrict__ hidden) {
  extern __shared__ double sm[];
  const int d = m.d, H = m.h, dh = m.dh, P = m.max_len;
  double *xs = sm;                  // [TF_R][d]   residual rows
  double *at = xs + TF_R * d;       // [TF_R][d]   attention output / LN2 output
  double *hs = at + TF_R * d;       // [TF_R][4d]  MLP hidden
  double *sc = hs + TF_R * 4 * d;   // [TF_R][H][P] attention weights
  const int r0 = blockIdx.x * TF_R;
  const int rows = min(TF_R, n - r0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double *kc = kv + (int64_t)layer * 2 * P * d;
  const double *vc = kc + (int64_t)P * d;
  for (int idx = threadIdx.x; idx < TF_R * d; idx += TF_THREADS)
    xs[idx] = (idx / d < rows) ? resid[(int64_t)(r0 + idx / d) * d + idx % d] : 0.0;

  // causal attention, one warp per (row, head) (fp/transformer.py:134-141)
  const double scale = sqrt((double)dh);
  for (int pr = warp; pr < rows * H; pr += TF_THREADS / 32) {
    const int r = pr / H, hh = pr % H;
    const int pos = start + r0 + r;
    const double *q = qbuf + (int64_t)(r0 + r) * d + hh * dh;
    double *w = sc + ((int64_t)r * H + hh) * P;
    double mx = -INFINITY;
    for (int k = lane; k <= pos; k += 32) {
      const double *kr = kc + (int64_t)k * d + hh * dh;
      double s = 0.0;
      for (int e = 0; e < dh; ++e) s = fma(q[e], kr[e], s);
      s = s / scale;
      w[k] = s;
      mx = fmax(mx, s);
    }
    mx = warp_max_d(mx);
    double sum = 0.0;
    for (int k = lane; k <= pos; k += 32) {
      const double e = exp(w[k] - mx);
      w[k] = e;
      sum += e;
    }
    sum = warp_sum_d(sum);
    __syncwarp();
    for (int k = lane; k <= pos; k += 32) w[k] = w[k] / sum;
    __syncwarp();
    // out[e] = sum_k w[k] v[k][e]: lanes split dh columns x key groups
    const int groups = (dh <= 32 && 32 % dh == 0) ? 32 / dh : 1;
    for (int e0 = 0; e0 < dh; e0 += (groups > 1 ? dh : 32)) {
      const int e = (groups > 1) ? lane % dh : e0 + lane;
      const int g = (groups > 1) ? lane / dh : 0;
      double acc = 0.0;
      if (e < dh)
        for (int k = g; k <= pos; k += groups) acc = fma(w[k], vc[(int64_t)k * d + hh * dh + e], acc);
      for (int o = dh; o < 32 && groups > 1; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (e < dh && g == 0) at[r * d + hh * dh + e] = acc;
    }
  }
  __syncthreads();
  const TfLayer L = tf_layer(prm, m, layer);
  // x = x + attn @ wo
  tf_rows_gemv(at, d, rows, d, L.wo, d, [&](int r, int j, double v) { xs[r * d + j] = xs[r * d + j] + v; });
  __syncthreads();
  tf_layer_norm(xs, at, rows, d, L.ln2_g, L.ln2_b);
  __syncthreads();
  tf_rows_gemv(at, d, rows, d, L.w1, 4 * d,
               [&](int r, int j, double v) { hs[r * 4 * d + j] = tf_gelu(v + L.b1[j]); });
  __syncthreads();
  // x = x + gelu(..) @ w2 + b2   (left to right, as numpy evaluates it)
  tf_rows_gemv(hs, 4 * d, rows, 4 * d, L.w2, d,
               [&](int r, int j, double v) { xs[r * d + j] = (xs[r * d + j] + v) + L.b2[j]; });
  __syncthreads();
  if (layer == m.layers - 1) {
    const double *lnf = prm + tf_layer_base(m, m.layers);
    tf_layer_norm(xs, at, rows, d, lnf, lnf + d);
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * d; idx += TF_THREADS)
      hidden[(int64_t)(r0 + idx / d) * d + idx % d] = at[idx];
  } else {
    for (int idx = threadIdx.x; idx < rows * d; idx += TF_THREADS)
      resid[(int64_t)(r0 + idx / d) * d + idx % d] = xs[idx];
  }
}

// logits = hidden @ tok_emb^T, greedy = argmax (first maximum, as np.argmax)
__global__ void __launch_bounds__(TF_THREADS) tf_logits(const double *__restrict__ prm, int d, int vocab,
                                                        const double *__restrict__ hidden,
                                                        double *__restrict__ logits, int *__restrict__ best) {
  __shared__ double sv[TF_THREADS];
  __shared__ int si[TF_THREADS];
  const double *hrow = hidden + (int64_t)blockIdx.x * d;
  double bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int v = threadIdx.x; v < vocab; v += TF_THREADS) {
    const double *er = prm + (int64_t)v * d;
    double s = 0.0;
    for (int i = 0; i < d; ++i) s = fma(hrow[i], er[i], s);
    if (logits) logits[(int64_t)blockIdx.x * vocab + v] = s;
    if (s > bv) { bv = s; bi = v; }
  }
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = TF_THREADS / 2; o; o >>= 1) {
    if (threadIdx.x < o) {
      const double ov = sv[threadIdx.x + o];
      const int oi = si[threadIdx.x + o];
      if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
        sv[threadIdx.x] = ov;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && best) best[blockIdx.x] = si[0];
}

int tf_dims(TfDims &m, int d, int h, int layers, int vocab, int max_len) {
  if (d <= 0 || h <= 0 || layers <= 0 || vocab <= 0 || max_len <= 0 || d % h) {
    set_error("transformer: bad dimensions d=%d h=%d layers=%d vocab=%d max_len=%d", d, h, layers, vocab,
              max_len);
    return AURAS_E_ARG;
  }
  m = TfDims{d, h, d / h, layers, vocab, max_len};
  return AURAS_OK;
}

size_t tf_block_smem(const TfDims &m) {
  return sizeof(double) * ((size_t)TF_R * 6 * m.d + (size_t)TF_R * m.h * m.max_len);
}

}  // namespace
}  // namespace auras

using namespace auras;

extern "C" int64_t auras_tf_param_count(int d_model, int n_heads, int n_layers, int vocab, int max_len) {
  TfDims m;
  if (tf_dims(m, d_model, n_heads, n_layers, vocab, max_len)) return -1;
  return tf_layer_base(m, n_layers) + 2LL * d_model;
}

extern "C" int auras_tf_forward(const double *params, int d_model, int n_heads, int n_layers, int vocab,
                                int max_len, const int *token_ids, const double *embeddings, int start, int n,
                                double *kv, double *resid, double *qbuf, double *hidden, void *stream) {
  TfDims m;
  if (int rc = tf_dims(m, d_model, n_heads, n_layers, vocab, max_len)) return rc;
  if (n < 1 || start < 0 || start + n > max_len || (!token_ids && !embeddings)) {
    set_error("transformer forward: rows [%d, %d) outside [0, %d)", start, start + n, max_len);
    return AURAS_E_ARG;
  }
  const size_t smem_qkv = sizeof(double) * 2 * TF_R * m.d;
  const size_t smem_blk = tf_block_smem(m);
  if (smem_blk > 200 * 1024) {
    set_error("transformer forward: %zu B of shared memory for d=%d h=%d max_len=%d", smem_blk, m.d, m.h,
              m.max_len);
    return AURAS_E_ARG;
  }
  static thread_local size_t configured = 0;
  if (smem_blk > 48 * 1024 && smem_blk > configured) {
    AURAS_CUDA(cudaFuncSetAttribute(tf_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_blk));
    configured = smem_blk;
  }
  cudaStream_t st = as_stream(stream);
  const int grid = (n + TF_R - 1) / TF_R;
  for (int l = 0; l < n_layers; ++l) {
    tf_qkv<<<grid, TF_THREADS, smem_qkv, st>>>(params, m, l, token_ids, embeddings, start, n, kv, resid, qbuf);
    tf_block<<<grid, TF_THREADS, smem_blk, st>>>(params, m, l, start, n, kv, resid, qbuf, hidden);
  }
  AURAS_LAUNCHED("tf_forward");
  return AURAS_OK;
}

extern "C" int auras_tf_logits(const double *params, int d_model, int vocab, const double *hidden, int n,
                               double *logits, int *argmax, void *stream) {
  if (n < 1 || d_model <= 0 || vocab <= 0) {
    set_error("transformer logits: bad sizes n=%d d=%d vocab=%d", n, d_model, vocab);
    return AURAS_E_ARG;
  }
  tf_logits<<<n, TF_THREADS, 0, as_stream(stream)>>>(params, d_model, vocab, hidden, logits, argmax);
  AURAS_LAUNCHED("tf_logits");
  return AURAS_OK;
}
