// Causal pre-norm transformer with a KV cache in HBM, fp64 (fp/transformer.py:69-211),
// the model behind the autoregressive merged prefill.
//
// One forward = rows [start, start + n) of a sequence whose rows [0, start)
// already sit in the KV cache: a prefill is start = 0, a decode is n = 1,
// start = cache length.  Row-parallel kernels, layers + 1 launches:
//
//   tf_embed_qkv : token / embedding + position -> LN1 -> q, k, v of layer 0;
//                  k, v go straight into the cache row, q into a scratch row
//   tf_block(l)  : causal attention of the row over cache rows 0..pos, out
//                  projection + residual, LN2, GELU MLP + residual, then LN1 +
//                  q, k, v of layer l + 1 (the final LN after the last layer)
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

#ifndef TF_ROWS
#define TF_ROWS 1
#endif
constexpr int TF_R = TF_ROWS;  // rows per CTA
#ifndef TF_NTHREADS
#define TF_NTHREADS 256
#endif
constexpr int TF_THREADS = TF_NTHREADS;
constexpr int TF_MAXDH = 32;
constexpr int TF_KPL = 8;      // keys per lane: max_len <= TF_KPL * 32 * warps per head
#ifdef TF_TIMING
__device__ unsigned long long tf_dbg[1024 * 16];
__device__ __forceinline__ void tf_mark(int i) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tf_dbg[blockIdx.x * 16 + i] = t;
  }
}
#define TF_MARK(i) tf_mark(i)
#else
#define TF_MARK(i)
#endif   // head width bound (attention partials live in registers)

struct TfDims {
  int d, h, dh, layers, vocab, max_len;
};

// warps sharing one (row, head) of attention
__host__ __device__ inline int tf_warps_per_head(int h) {
  const int w = (TF_THREADS / 32) / (TF_R * h);
  return w < 1 ? 1 : w;
}

// Start offset of a row's reduction loops.  It depends on the row's position
// only (one row per CTA), so a row computes the same bits in every launch,
// while the CTAs of one launch start on different weight / key lines instead
// of all hammering the same L2 lines at once.
__host__ __device__ inline int tf_rot(int pos) { return TF_R == 1 ? pos * 5 : 0; }

// gemv partials [KS][TF_R][cols] or attention partials [warps][32][dh]
__host__ __device__ inline size_t tf_red_elems(int dh) {
  const size_t a = (size_t)TF_R * TF_THREADS, b = (size_t)TF_THREADS * dh;
  return a > b ? a : b;
}

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
__device__ __forceinline__ void tf_layer_norm(const double *x, double *y, int rows, int d, const double *g,
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

// out[r][j] = sum_i a[r][i] * W(i, j) for TF_R rows and columns j < ncols, with
// W(i, j) = W[(j / seg) * seg_stride + i * ld + j % seg] (seg = ncols for a
// plain [k, ncols] matrix; q|k|v as one 3d-column matrix otherwise).
// Latency bound: with few columns the k range is split over KS thread slices
// (partials reduced in a fixed order through `red`).  Kept out of line and
// lightly unrolled: each warp runs the kernel's code only a few times, so
// instruction fetch, not arithmetic, is what a big unrolled body costs.
enum TfEmit { TF_STORE, TF_ADD, TF_GELU_BIAS, TF_ADD_BIAS, TF_QKV };

struct TfOut {
  double *out;        // [TF_R][out_ld] (TF_QKV: q rows)
  int out_ld;
  const double *bias;
  double *kc, *vc;    // TF_QKV: cache rows of this layer
  int d, row0, pos0;  // TF_QKV: width, first qbuf row, first cache row
};

__device__ __forceinline__ void tf_emit(int mode, const TfOut &o, int r, int j, double v) {
  switch (mode) {
    case TF_STORE: o.out[r * o.out_ld + j] = v; break;
    case TF_ADD: o.out[r * o.out_ld + j] = o.out[r * o.out_ld + j] + v; break;
    case TF_GELU_BIAS: o.out[r * o.out_ld + j] = tf_gelu(v + o.bias[j]); break;
    // x + gelu(..) @ w2 + b2 evaluates left to right in numpy
    case TF_ADD_BIAS: o.out[r * o.out_ld + j] = (o.out[r * o.out_ld + j] + v) + o.bias[j]; break;
    default: {
      const int which = j / o.d, c = j % o.d;
      if (which == 0) o.out[(int64_t)(o.row0 + r) * o.d + c] = v;
      else (which == 1 ? o.kc : o.vc)[(int64_t)(o.pos0 + r) * o.d + c] = v;
    }
  }
}

__device__ __noinline__ void tf_rows_gemv(const double *a, int lda, int rows, int k, const double *W, int ncols,
                                          int seg, int64_t seg_stride, int ld, double *red, int mode,
                                          TfOut o, int rot) {
  const int KS = ncols >= TF_THREADS ? 1 : TF_THREADS / ncols;   // k slices
  const int jw = TF_THREADS / KS;                                // columns per pass
  const int kc = (k + KS - 1) / KS;
  const int sl = threadIdx.x / jw;
  for (int j0 = 0; j0 < ncols; j0 += jw) {
    const int j = j0 + threadIdx.x % jw;
    double acc[TF_R];
#pragma unroll
    for (int r = 0; r < TF_R; ++r) acc[r] = 0.0;
    if (j < ncols && sl < KS) {
      const double *wc = W + (int64_t)(j / seg) * seg_stride + j % seg;
      const int i0 = sl * kc, len = min(k, i0 + kc) - i0;
      // rotated start (a function of the row only, see tf_rot): CTAs that
      // read the same weights at the same moment hit different L2 lines
      int i = i0 + (len > 0 ? rot % len : 0);
#pragma unroll 16
      for (int c = 0; c < len; ++c) {
        const double w = __ldg(wc + (int64_t)i * ld);
#pragma unroll
        for (int r = 0; r < TF_R; ++r) acc[r] = fma(a[r * lda + i], w, acc[r]);
        if (++i == i0 + len) i = i0;
      }
    }
    if (KS == 1) {
      for (int r = 0; r < rows; ++r)
        if (j < ncols) tf_emit(mode, o, r, j, acc[r]);
      continue;
    }
    if (sl < KS) {
#pragma unroll
      for (int r = 0; r < TF_R; ++r) red[(sl * TF_R + r) * jw + threadIdx.x % jw] = acc[r];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < TF_R * jw; idx += TF_THREADS) {
      const int r = idx / jw, jj = idx % jw;
      double v = 0.0;
      for (int q = 0; q < KS; ++q) v += red[(q * TF_R + r) * jw + jj];
      if (r < rows && j0 + jj < ncols) tf_emit(mode, o, r, j0 + jj, v);
    }
    __syncthreads();
  }
}

// Causal attention (fp/transformer.py:134-141) of one (row, head) over cache
// rows 0..pos, split over `wpp` warps: warp `sub` takes keys
// kb = (t * wpp + sub) * 32 + lane (rotated by tf_rot, a function of the row
// only), so a lane holds few keys and their loads are in flight together.
// Each warp leaves (max, sum of exp, unnormalised weighted values) in `st`;
// the caller rescales and merges them.
__device__ __forceinline__ void tf_attend_part(const double *q, const double *kc, const double *vc, double *part,
                                               double *st, int hh, int pos, int sub, int wpp, TfDims m) {
  const int d = m.d, dh = m.dh, lane = threadIdx.x & 31;
  const double scale = sqrt((double)dh);
  double sk[TF_KPL];
  double mx = -INFINITY;
  const int krot = tf_rot(pos) % (pos + 1);
#pragma unroll
  for (int t = 0; t < TF_KPL; ++t) {
    const int kb = (t * wpp + sub) * 32 + lane;
    const int k = kb + krot > pos ? kb + krot - pos - 1 : kb + krot;
    sk[t] = -INFINITY;
    if (kb <= pos) {
      const double *kr = kc + (int64_t)k * d + hh * dh;
      double kv_[TF_MAXDH];        // all loads of the key row first
#pragma unroll
      for (int e = 0; e < TF_MAXDH; ++e) kv_[e] = e < dh ? __ldg(kr + e) : 0.0;
      double s = 0.0;
#pragma unroll
      for (int e = 0; e < TF_MAXDH; ++e)
        if (e < dh) s = fma(q[e], kv_[e], s);
      sk[t] = s / scale;
      mx = fmax(mx, sk[t]);
    }
  }
  mx = warp_max_d(mx);
  double sum = 0.0;
  double acc[TF_MAXDH];
#pragma unroll
  for (int e = 0; e < TF_MAXDH; ++e) acc[e] = 0.0;
#pragma unroll
  for (int t = 0; t < TF_KPL; ++t) {
    const int kb = (t * wpp + sub) * 32 + lane;
    const int k = kb + krot > pos ? kb + krot - pos - 1 : kb + krot;
    if (kb <= pos) {
      const double p = exp(sk[t] - mx);
      sum += p;
      const double *vr = vc + (int64_t)k * d + hh * dh;
#pragma unroll
      for (int e = 0; e < TF_MAXDH; ++e)
        if (e < dh) acc[e] = fma(p, __ldg(vr + e), acc[e]);
    }
  }
  sum = warp_sum_d(sum);
#pragma unroll
  for (int e = 0; e < TF_MAXDH; ++e)
    if (e < dh) part[lane * dh + e] = acc[e];
  __syncwarp();
  for (int e = lane; e < dh; e += 32) {
    double v = 0.0;
    for (int l = 0; l < 32; ++l) v += part[l * dh + e];
    st[2 + e] = v;
  }
  if (lane == 0) {
    st[0] = mx;
    st[1] = sum;
  }
  __syncwarp();
}

// LN1 + q|k|v of layer `layer` for the CTA's rows: k, v into the cache rows,
// q into qbuf.  xs holds the residual rows; `as`, `red` are scratch.
__device__ void tf_qkv_rows(const double *prm, const TfDims &m, int layer, int start, int r0, int rows,
                            const double *xs, double *as, double *red, double *kv, double *qbuf) {
  const int d = m.d;
  const TfLayer L = tf_layer(prm, m, layer);
  tf_layer_norm(xs, as, rows, d, L.ln1_g, L.ln1_b);
  __syncthreads();
  double *kc = kv + (int64_t)layer * 2 * m.max_len * d;
  double *vc = kc + (int64_t)m.max_len * d;
  TfOut o{qbuf, 0, nullptr, kc, vc, d, r0, start + r0};
  tf_rows_gemv(as, d, rows, d, L.wq, 3 * d, d, (int64_t)d * d, d, red, TF_QKV, o, tf_rot(start + r0));
}

__global__ void __launch_bounds__(TF_THREADS) tf_embed_qkv(const double *__restrict__ prm, TfDims m,
                                                           const int *__restrict__ ids,
                                                           const double *__restrict__ emb, int start, int n,
                                                           double *__restrict__ kv, double *__restrict__ resid,
                                                           double *__restrict__ qbuf) {
  extern __shared__ double sm[];
  const int d = m.d;
  double *xs = sm;                 // [TF_R][d]
  double *as = xs + TF_R * d;      // [TF_R][d]
  double *red = as + TF_R * d;     // [TF_R][TF_THREADS] gemv partials
  const int r0 = blockIdx.x * TF_R;
  const int rows = min(TF_R, n - r0);
  // fp/transformer.py:104-109,126: token (or given) embedding + position
  for (int idx = threadIdx.x; idx < TF_R * d; idx += TF_THREADS) {
    const int r = idx / d, c = idx % d;
    double v = 0.0;
    if (r < rows) {
      const int row = r0 + r;
      const double e = ids ? prm[(int64_t)ids[row] * d + c] : emb[(int64_t)row * d + c];
      v = e + prm[(int64_t)m.vocab * d + (int64_t)(start + row) * d + c];
      resid[(int64_t)row * d + c] = v;
    }
    xs[idx] = v;
  }
  __syncthreads();
  tf_qkv_rows(prm, m, 0, start, r0, rows, xs, as, red, kv, qbuf);
}

// Attention + MLP of `layer`, then LN1 + q|k|v of layer + 1 (or the final LN).
__global__ void __launch_bounds__(TF_THREADS) tf_block(const double *__restrict__ prm, TfDims m, int layer,
                                                       int start, int n, double *__restrict__ kv,
                                                       double *__restrict__ resid, double *__restrict__ qbuf,
                                                       double *__restrict__ hidden) {
  extern __shared__ double sm[];
  const int d = m.d, H = m.h, P = m.max_len;
  double *xs = sm;                  // [TF_R][d]   residual rows
  double *at = xs + TF_R * d;       // [TF_R][d]   attention output / LN output
  double *qs = at + TF_R * d;       // [TF_R][d]   query rows
  double *hs = qs + TF_R * d;       // [TF_R][4d]  MLP hidden
  double *red = hs + TF_R * 4 * d;  // gemv / attention partials
  double *sc = red + tf_red_elems(m.dh);  // per-warp attention stats [TF_R*H*wpp][dh + 2]
  const int r0 = blockIdx.x * TF_R;
  const int rows = min(TF_R, n - r0);
  const int warp = threadIdx.x >> 5;
  const double *kc = kv + (int64_t)layer * 2 * P * d;
  TF_MARK(0);
  const double *vc = kc + (int64_t)P * d;
  for (int idx = threadIdx.x; idx < TF_R * d; idx += TF_THREADS) {
    const bool in = idx / d < rows;
    xs[idx] = in ? resid[(int64_t)(r0 + idx / d) * d + idx % d] : 0.0;
    qs[idx] = in ? qbuf[(int64_t)(r0 + idx / d) * d + idx % d] : 0.0;
  }
  __syncthreads();
  TF_MARK(1);

  // causal attention: wpp warps per (row, head), then the rescaled merge
  const int wpp = tf_warps_per_head(H);
  const int dh = m.dh;
  for (int pw = warp; pw < TF_R * H * wpp; pw += TF_THREADS / 32) {
    const int pair = pw / wpp, r = pair / H, hh = pair % H;
    if (r < rows)
      tf_attend_part(qs + r * d + hh * dh, kc, vc, red + (pw % (TF_THREADS / 32)) * 32 * dh,
                     sc + (int64_t)pw * (dh + 2), hh, start + r0 + r, pw % wpp, wpp, m);
  }
  __syncthreads();
  TF_MARK(2);
  for (int idx = threadIdx.x; idx < rows * H * dh; idx += TF_THREADS) {
    const int pair = idx / dh, e = idx % dh;
    const double *st = sc + (int64_t)pair * wpp * (dh + 2);
    double M = -INFINITY;
    for (int w = 0; w < wpp; ++w) M = fmax(M, st[w * (dh + 2)]);
    double tot = 0.0, o = 0.0;
    for (int w = 0; w < wpp; ++w) {
      const double mw = st[w * (dh + 2)];
      if (mw == -INFINITY) continue;          // a warp that saw no key
      const double f = exp(mw - M);
      tot += st[w * (dh + 2) + 1] * f;
      o += st[w * (dh + 2) + 2 + e] * f;
    }
    at[(pair / H) * d + (pair % H) * dh + e] = o / tot;
  }
  __syncthreads();
  TF_MARK(3);
  const TfLayer L = tf_layer(prm, m, layer);
  // x = x + attn @ wo
  tf_rows_gemv(at, d, rows, d, L.wo, d, d, 0, d, red, TF_ADD, TfOut{xs, d}, tf_rot(start + r0));
  __syncthreads();
  TF_MARK(4);
  tf_layer_norm(xs, at, rows, d, L.ln2_g, L.ln2_b);
  __syncthreads();
  TF_MARK(5);
  tf_rows_gemv(at, d, rows, d, L.w1, 4 * d, 4 * d, 0, 4 * d, red, TF_GELU_BIAS, TfOut{hs, 4 * d, L.b1}, tf_rot(start + r0));
  __syncthreads();
  TF_MARK(6);
  // x = x + gelu(..) @ w2 + b2   (left to right, as numpy evaluates it)
  tf_rows_gemv(hs, 4 * d, rows, 4 * d, L.w2, d, d, 0, d, red, TF_ADD_BIAS, TfOut{xs, d, L.b2}, tf_rot(start + r0));
  __syncthreads();
  TF_MARK(7);
  if (layer == m.layers - 1) {
    const double *lnf = prm + tf_layer_base(m, m.layers);
    tf_layer_norm(xs, at, rows, d, lnf, lnf + d);
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * d; idx += TF_THREADS)
      hidden[(int64_t)(r0 + idx / d) * d + idx % d] = at[idx];
  } else {
    for (int idx = threadIdx.x; idx < rows * d; idx += TF_THREADS)
      resid[(int64_t)(r0 + idx / d) * d + idx % d] = xs[idx];
    tf_qkv_rows(prm, m, layer + 1, start, r0, rows, xs, at, red, kv, qbuf);
  }
  __syncthreads();
  TF_MARK(8);
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
  return sizeof(double) * ((size_t)TF_R * 7 * m.d + tf_red_elems(m.dh) +
                           (size_t)TF_R * m.h * tf_warps_per_head(m.h) * (m.dh + 2));
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
  if (m.dh > TF_MAXDH) {
    set_error("transformer forward: head width %d > %d", m.dh, TF_MAXDH);
    return AURAS_E_ARG;
  }
  if (max_len > TF_KPL * 32 * tf_warps_per_head(m.h)) {
    set_error("transformer forward: max_len %d > %d for %d heads", max_len,
              TF_KPL * 32 * tf_warps_per_head(m.h), m.h);
    return AURAS_E_ARG;
  }
  if (n < 1 || start < 0 || start + n > max_len || (!token_ids && !embeddings)) {
    set_error("transformer forward: rows [%d, %d) outside [0, %d)", start, start + n, max_len);
    return AURAS_E_ARG;
  }
  const size_t smem_qkv = sizeof(double) * (2 * TF_R * m.d + TF_R * TF_THREADS);
  const size_t smem_blk = tf_block_smem(m);
  if (smem_blk > 200 * 1024) {
    set_error("transformer forward: %zu B of shared memory for d=%d h=%d max_len=%d", smem_blk, m.d, m.h,
              m.max_len);
    return AURAS_E_ARG;
  }
  if (smem_blk > 48 * 1024)
    if (int rc = ensure_smem_attr(tf_block, (int)smem_blk)) return rc;
  if (smem_qkv > 48 * 1024) {
    set_error("transformer forward: d=%d too wide", m.d);
    return AURAS_E_ARG;
  }
  cudaStream_t st = as_stream(stream);
  const int grid = (n + TF_R - 1) / TF_R;
  tf_embed_qkv<<<grid, TF_THREADS, smem_qkv, st>>>(params, m, token_ids, embeddings, start, n, kv, resid, qbuf);
  for (int l = 0; l < n_layers; ++l)
    tf_block<<<grid, TF_THREADS, smem_blk, st>>>(params, m, l, start, n, kv, resid, qbuf, hidden);
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

#ifdef TF_TIMING
extern "C" int auras_tf_debug_times(unsigned long long *out, int n) {
  return cudaMemcpyFromSymbol(out, auras::tf_dbg, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -1;
}
#endif
