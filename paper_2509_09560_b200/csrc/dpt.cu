// DP-T denoiser (Diffusion Policy's TransformerForDiffusion; BASELINE
// configs[3]) -- the pieces around the GEMMs.  Every linear layer runs on the
// tcgen05 conv path (auras_conv, 1-row convolutions over the token axis);
// these kernels stage a batch of in-flight samples, run the small attentions
// and apply the scheduler update:
//
//   dpt_prep   : per sample (agent, lane, inference step i): the noisy action
//                x_i from its request lane -> bf16 token rows (padded to 64
//                channels); the agent's observation tokens from the ring slot
//                the frame fetched (device-resolved slot) -> bf16 rows; the
//                time token temb[i] + cond_pos[0]
//   dpt_cond   : cond rows 1..n_obs = projected observation tokens + cond_pos
//   attention  : softmax(q k^T / sqrt(dh) + mask) v with key j visible to
//                query n iff j <= n + mask_off (causal self-attention: 0; the
//                memory mask t >= s - 1: 1), one warp per (sample, head, query)
//   dpt_update : DDPM / DDIM step of every sample from its eps, written back
//                to the request lane (the same arithmetic as the UNet path's
//                final step)
#include <cmath>

#include "common.cuh"

namespace auras {
namespace {

__global__ void dpt_prep_kernel(const int *__restrict__ agents, const int *__restrict__ lanes,
                                const int *__restrict__ steps, const float *__restrict__ x_lanes, int lanes_per_agent,
                                int horizon, int adim, __nv_bfloat16 *__restrict__ xin,
                                const float *__restrict__ ring, int64_t ring_agent_stride, int slot_floats,
                                const int64_t *__restrict__ fetched, int tok_w, int n_obs,
                                __nv_bfloat16 *__restrict__ gcbuf, int gpad, const float *__restrict__ temb, int E,
                                __nv_bfloat16 *__restrict__ c, const float *__restrict__ cond_pos) {
  const int s = blockIdx.x;
  const int agent = agents[s], lane = lanes[s], i = steps[s];
  const float *x = x_lanes + ((int64_t)agent * lanes_per_agent + lane) * horizon * adim;
  for (int e = threadIdx.x; e < horizon * 64; e += blockDim.x) {
    const int t = e >> 6, a = e & 63;
    xin[(int64_t)s * horizon * 64 + e] = __float2bfloat16_rn(a < adim ? x[t * adim + a] : 0.f);
  }
  const int slot = (int)fetched[0];
  const float *gc = ring + agent * ring_agent_stride + (int64_t)slot * slot_floats;
  for (int e = threadIdx.x; e < n_obs * gpad; e += blockDim.x) {
    const int j = e / gpad, k = e % gpad;
    gcbuf[(int64_t)s * n_obs * gpad + e] = __float2bfloat16_rn(k < tok_w ? gc[j * tok_w + k] : 0.f);
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    c[(int64_t)s * (1 + n_obs) * E + e] = __float2bfloat16_rn(temb[(int64_t)i * E + e] + cond_pos[e]);
}

// Per iteration: the cross-attention K|V rows of every sample from the time
// table (by inference step) and the frame's observation rows (by agent).
__global__ void dpt_kv_gather_kernel(__nv_bfloat16 *__restrict__ kv2, const __nv_bfloat16 *__restrict__ kvt,
                                     const __nv_bfloat16 *__restrict__ kvo, const int *__restrict__ agents,
                                     const int *__restrict__ steps, int tc, int lw) {
  const int s = blockIdx.x / tc, r = blockIdx.x % tc;
  const __nv_bfloat16 *src = r == 0 ? kvt + (int64_t)steps[s] * lw : kvo + ((int64_t)agents[s] * (tc - 1) + r - 1) * lw;
  __nv_bfloat16 *dst = kv2 + ((int64_t)s * tc + r) * lw;
  const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
  uint4 *d4 = reinterpret_cast<uint4 *>(dst);
  for (int i = threadIdx.x; i < lw / 8; i += blockDim.x) d4[i] = s4[i];
}

__global__ void dpt_cond_kernel(const __nv_bfloat16 *__restrict__ cobs, __nv_bfloat16 *__restrict__ c,
                                const float *__restrict__ cond_pos, int S, int n_obs, int E) {
  const int64_t total = (int64_t)S * n_obs * E;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(i % E);
    const int64_t r = i / E;
    const int j = (int)(r % n_obs);
    const int64_t s = r / n_obs;
    c[(s * (1 + n_obs) + 1 + j) * E + e] = __float2bfloat16_rn(__bfloat162float(cobs[i]) + cond_pos[(1 + j) * E + e]);
  }
}

__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int DA_MAXK = 32;   // keys per query (horizon / cond tokens)
constexpr int DA_MAXE = 4;    // head columns per lane (dh <= 128)

__global__ void dpt_attention_kernel(const __nv_bfloat16 *__restrict__ q, int ldq, const __nv_bfloat16 *__restrict__ k,
                                     int ldk, const __nv_bfloat16 *__restrict__ v, int ldv,
                                     __nv_bfloat16 *__restrict__ out, int ldo, int S, int Nq, int Nk, int H, int dh,
                                     int mask_off, float scale) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= S * H * Nq) return;
  const int n = w % Nq, h = (w / Nq) % H, s = w / (Nq * H);
  const __nv_bfloat16 *qr = q + ((int64_t)s * Nq + n) * ldq + h * dh;
  float qv[DA_MAXE];
#pragma unroll
  for (int u = 0; u < DA_MAXE; ++u) {
    const int e = lane + 32 * u;
    qv[u] = e < dh ? __bfloat162float(qr[e]) * scale : 0.f;
  }
  const int nk = min(Nk, n + mask_off + 1);
  float sc[DA_MAXK];
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < DA_MAXK; ++j) {
    sc[j] = -INFINITY;
    if (j < nk) {
      const __nv_bfloat16 *kr = k + ((int64_t)s * Nk + j) * ldk + h * dh;
      float a = 0.f;
#pragma unroll
      for (int u = 0; u < DA_MAXE; ++u) {
        const int e = lane + 32 * u;
        if (e < dh) a = fmaf(qv[u], __bfloat162float(kr[e]), a);
      }
      sc[j] = wsum(a);
      mx = fmaxf(mx, sc[j]);
    }
  }
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < DA_MAXK; ++j) {
    sc[j] = j < nk ? __expf(sc[j] - mx) : 0.f;
    sum += sc[j];
  }
  const float inv = 1.f / sum;
#pragma unroll
  for (int u = 0; u < DA_MAXE; ++u) {
    const int e = lane + 32 * u;
    if (e >= dh) continue;
    float a = 0.f;
#pragma unroll
    for (int j = 0; j < DA_MAXK; ++j)
      if (j < nk) a = fmaf(sc[j], __bfloat162float(v[((int64_t)s * Nk + j) * ldv + h * dh + e]), a);
    out[((int64_t)s * Nq + n) * ldo + h * dh + e] = __float2bfloat16_rn(a * inv);
  }
}

__global__ void dpt_update_kernel(const float *__restrict__ eps, int eps_pitch, const int *__restrict__ agents,
                                  const int *__restrict__ lanes, const int *__restrict__ steps, float *x_lanes,
                                  const float *__restrict__ noise_lanes, int lanes_per_agent, int horizon, int adim,
                                  auras_sched sch) {
  const int s = blockIdx.x;
  const int agent = agents[s], lane = lanes[s], i = steps[s];
  float *x = x_lanes + ((int64_t)agent * lanes_per_agent + lane) * horizon * adim;
  const float *z = noise_lanes
                       ? noise_lanes + (((int64_t)agent * lanes_per_agent + lane) * sch.n_steps + i) * horizon * adim
                       : nullptr;
  const float sab = sch.sqrt_ab[i], s1m = sch.sqrt_1mab[i];
  const float cx0 = sch.c_x0[i], cxt = sch.c_xt[i], ceps = sch.c_eps[i], sig = sch.sigma[i];
  for (int e = threadIdx.x; e < horizon * adim; e += blockDim.x) {
    const int t = e / adim, a = e % adim;
    const float xt = x[e], ep = eps[((int64_t)s * horizon + t) * eps_pitch + a];
    float x0 = (xt - s1m * ep) / sab;
    if (sch.clip_sample) x0 = fminf(fmaxf(x0, -1.f), 1.f);
    float nx = cx0 * x0 + cxt * xt + ceps * ep;
    if (sch.ddpm && z) nx += sig * z[e];
    x[e] = nx;
  }
}

}  // namespace
}  // namespace auras

using namespace auras;

extern "C" int auras_dpt_prep(const int *agents, const int *lanes, const int *steps, int S, const float *x_lanes,
                              int lanes_per_agent, int horizon, int adim, void *xin, const float *ring,
                              int64_t ring_agent_stride, int slot_floats, const int64_t *fetched, int tok_w, int n_obs,
                              void *gcbuf, int gpad, const float *temb, int E, void *c, const float *cond_pos,
                              void *stream) {
  if (S < 1 || adim > 64 || tok_w > gpad) {
    set_error("dpt_prep: bad sizes S=%d adim=%d tok_w=%d gpad=%d", S, adim, tok_w, gpad);
    return AURAS_E_ARG;
  }
  dpt_prep_kernel<<<S, 256, 0, as_stream(stream)>>>(agents, lanes, steps, x_lanes, lanes_per_agent, horizon, adim,
                                                    static_cast<__nv_bfloat16 *>(xin), ring, ring_agent_stride,
                                                    slot_floats, fetched, tok_w, n_obs,
                                                    static_cast<__nv_bfloat16 *>(gcbuf), gpad, temb, E,
                                                    static_cast<__nv_bfloat16 *>(c), cond_pos);
  AURAS_LAUNCHED("dpt_prep");
  return AURAS_OK;
}

extern "C" int auras_dpt_cond(const void *cobs, void *c, const float *cond_pos, int S, int n_obs, int E, void *stream) {
  const int64_t total = (int64_t)S * n_obs * E;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 1184);
  dpt_cond_kernel<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const __nv_bfloat16 *>(cobs),
                                                       static_cast<__nv_bfloat16 *>(c), cond_pos, S, n_obs, E);
  AURAS_LAUNCHED("dpt_cond");
  return AURAS_OK;
}

extern "C" int auras_attention(const void *q, int ldq, const void *k, int ldk, const void *v, int ldv, void *out,
                               int ldo, int S, int Nq, int Nk, int heads, int dh, int mask_off, void *stream) {
  if (S < 1 || Nq < 1 || Nk < 1 || Nk > DA_MAXK || dh < 1 || dh > 32 * DA_MAXE) {
    set_error("attention: bad sizes S=%d Nq=%d Nk=%d dh=%d", S, Nq, Nk, dh);
    return AURAS_E_ARG;
  }
  const int warps = S * heads * Nq;
  dpt_attention_kernel<<<(warps + 7) / 8, 256, 0, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16 *>(q), ldq, static_cast<const __nv_bfloat16 *>(k), ldk,
      static_cast<const __nv_bfloat16 *>(v), ldv, static_cast<__nv_bfloat16 *>(out), ldo, S, Nq, Nk, heads, dh,
      mask_off, 1.f / sqrtf((float)dh));
  AURAS_LAUNCHED("attention");
  return AURAS_OK;
}

extern "C" int auras_dpt_update(const float *eps, int eps_pitch, const int *agents, const int *lanes, const int *steps,
                                int S, float *x_lanes, const float *noise_lanes, int lanes_per_agent, int horizon,
                                int adim, const auras_sched *sched, void *stream) {
  if (S < 1 || !sched) {
    set_error("dpt_update: bad arguments");
    return AURAS_E_ARG;
  }
  dpt_update_kernel<<<S, 128, 0, as_stream(stream)>>>(eps, eps_pitch, agents, lanes, steps, x_lanes, noise_lanes,
                                                      lanes_per_agent, horizon, adim, *sched);
  AURAS_LAUNCHED("dpt_update");
  return AURAS_OK;
}

extern "C" int auras_dpt_kv_gather(void *kv2, const void *kvt, const void *kvo, const int *agents, const int *steps,
                                   int S, int tc, int lw, void *stream) {
  if (S < 1 || tc < 1 || lw % 8) {
    set_error("dpt_kv_gather: bad sizes S=%d tc=%d lw=%d", S, tc, lw);
    return AURAS_E_ARG;
  }
  dpt_kv_gather_kernel<<<S * tc, 256, 0, as_stream(stream)>>>(static_cast<__nv_bfloat16 *>(kv2),
                                                              static_cast<const __nv_bfloat16 *>(kvt),
                                                              static_cast<const __nv_bfloat16 *>(kvo), agents, steps,
                                                              tc, lw);
  AURAS_LAUNCHED("dpt_kv_gather");
  return AURAS_OK;
}
