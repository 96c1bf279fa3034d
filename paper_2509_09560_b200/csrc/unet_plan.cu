// The batched, staggered-timestep denoise chain (K3-K6 of SURVEY.md §2.4).
//
// One call runs every iteration of one frame for all in-flight samples:
//   for r in [0, iters):  prep(r) -> [conv GEMM -> fused epilogue] x ops -> final(r)
// prep(r) resolves each sample's diffusion timestep (start[s] + r) and the
// ring slot its agent fetched in-kernel, and loads x_t; the epilogues gather
// FiLM rows as film_tau[timestep] + ring_film[agent][slot]; final(r) applies
// the 1x1 output conv and the DDPM/DDIM update and writes x_{t-1} back to the
// request lane (GenerationModel.step, fp/policy.py:217-228, for a neural
// policy).  The chain can be captured once per (S, iters) into a CUDA graph.
#include <algorithm>
#include <cstring>
#include <map>
#include <utility>
#include <vector>

#include "common.cuh"
#include "conv.cuh"

namespace auras {

constexpr int kMaxS = 64;

struct UnetCtrl {             // per-frame control, uploaded by value
  int lanes[kMaxS], agents[kMaxS], start[kMaxS], count[kMaxS];
  float *x_lanes;
  const float *noise_lanes;
  const int64_t *fetched;
  int S, lanes_per_agent;
};

struct UnetDev {              // device-resident per-sample state
  UnetCtrl ctrl;
  int r;                      // iteration index within the frame, advanced in-graph
  int tau_row[kMaxS];
  int64_t film_b_off[kMaxS];
};

__global__ void unet_set_ctrl(UnetDev *dev, UnetCtrl c) {
  dev->ctrl = c;
  dev->r = 0;
}

__global__ void unet_advance(UnetDev *dev) { dev->r += 1; }

template <typename T>
__global__ void unet_prep(UnetDev *dev, auras_sched sch, int horizon, int adim, T *xin,
                          int x_pitch, int64_t ring_slot_stride, int64_t ring_agent_stride) {
  const int s = blockIdx.x;
  const UnetCtrl &c = dev->ctrl;
  const int r = dev->r;
  const int agent = c.agents[s], lane = c.lanes[s];
  int i = c.start[s] + r;
  i = i < sch.n_steps ? i : sch.n_steps - 1;
  if (threadIdx.x == 0) {
    dev->tau_row[s] = sch.timestep[i];
    const int64_t slot = c.fetched[0];   // one ring version schedule per lock-stepped agent group
    dev->film_b_off[s] = agent * ring_agent_stride + slot * ring_slot_stride;
  }
  const float *x = c.x_lanes + ((int64_t)agent * c.lanes_per_agent + lane) * horizon * adim;
  for (int e = threadIdx.x; e < horizon * x_pitch; e += blockDim.x) {
    const int t = e / x_pitch, ch = e - t * x_pitch;
    const float v = ch < adim ? x[t * adim + ch] : 0.f;
    Elem<T>::store(xin + ((int64_t)s * horizon + t) * x_pitch + ch, v);
  }
}

// eps = W_out . y + b (1x1 conv to action_dim) then the scheduler update.
template <typename T>
__global__ void unet_final(UnetDev *dev, auras_sched sch, int horizon, int adim, const T *y,
                           int y_pitch, int cin, const float *wf, const float *bf) {
  __shared__ float eps[512];
  const int s = blockIdx.x;
  const UnetCtrl &c = dev->ctrl;
  const int r = dev->r;
  const int lane_id = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = wid; o < horizon * adim; o += nw) {
    const int t = o / adim, a = o - t * adim;
    const T *yr = y + ((int64_t)s * horizon + t) * y_pitch;
    float acc = 0.f;
    for (int k = lane_id; k < cin; k += 32) acc = fmaf(wf[a * cin + k], Elem<T>::load(yr + k), acc);
    acc = warp_sum(acc);
    if (lane_id == 0) eps[o] = acc + bf[a];
  }
  __syncthreads();
  if (r >= c.count[s]) return;                        // sample finished its share this frame
  const int i = c.start[s] + r;
  const int agent = c.agents[s], lane = c.lanes[s];
  float *x = c.x_lanes + ((int64_t)agent * c.lanes_per_agent + lane) * horizon * adim;
  const float *z = c.noise_lanes
                       ? c.noise_lanes + (((int64_t)agent * c.lanes_per_agent + lane) * sch.n_steps + i) * horizon * adim
                       : nullptr;
  const float sab = sch.sqrt_ab[i], s1m = sch.sqrt_1mab[i];
  const float cx0 = sch.c_x0[i], cxt = sch.c_xt[i], ceps = sch.c_eps[i], sig = sch.sigma[i];
  for (int e = threadIdx.x; e < horizon * adim; e += blockDim.x) {
    const float xt = x[e], ep = eps[e];
    float x0 = (xt - s1m * ep) / sab;
    if (sch.clip_sample) x0 = fminf(fmaxf(x0, -1.f), 1.f);
    float nx = cx0 * x0 + cxt * xt + ceps * ep;
    if (sch.ddpm && z) nx += sig * z[e];
    x[e] = nx;
  }
}

}  // namespace auras

using namespace auras;

struct auras_unet_plan {
  std::vector<auras_conv_op> ops;
  int dtype, s_max, horizon, adim, film_width, final_cin;
  int64_t ring_slot_stride, ring_agent_stride;
  const float *film_tau, *ring_film, *final_b;
  const float *final_w;
  auras_sched sched;
  void *x_in;
  int x_pitch;
  float *partial = nullptr;
  int64_t partial_floats = 0;
  UnetDev *dev = nullptr;
  std::map<int, cudaGraphExec_t> graphs;     // one denoise step per batch size S
};

// One denoise step for S samples: prep -> (GEMM, epilogue) x ops -> final -> advance.
static int unet_launch_step(auras_unet_plan *p, int S, cudaStream_t st) {
  {
    if (p->dtype == AURAS_DT_BF16)
      unet_prep<__nv_bfloat16><<<S, 128, 0, st>>>(p->dev, p->sched, p->horizon, p->adim,
                                                  static_cast<__nv_bfloat16 *>(p->x_in), p->x_pitch,
                                                  p->ring_slot_stride, p->ring_agent_stride);
    else
      unet_prep<float><<<S, 128, 0, st>>>(p->dev, p->sched, p->horizon, p->adim,
                                          static_cast<float *>(p->x_in), p->x_pitch, p->ring_slot_stride,
                                          p->ring_agent_stride);
    AURAS_LAUNCHED("unet_prep");
    for (const auras_conv_op &op : p->ops) {
      ConvGemmArgs g;
      EpiArgs e;
      int rc = conv_op_to_args(op, S, p->dtype, p->partial, g, e);
      if (rc) return rc;
      if (op.film_off >= 0) {
        e.film_a = p->film_tau;
        e.film_a_row = p->dev->tau_row;
        e.film_a_stride = p->film_width;
        e.film_b = p->ring_film;
        e.film_b_off = p->dev->film_b_off;
      }
      if ((rc = run_gemm(g, p->dtype, st))) return rc;
      if ((rc = run_epilogue(e, S, p->dtype, st))) return rc;
    }
    const auras_conv_op &last = p->ops.back();
    if (p->dtype == AURAS_DT_BF16)
      unet_final<__nv_bfloat16><<<S, 256, 0, st>>>(p->dev, p->sched, p->horizon, p->adim,
                                                   static_cast<const __nv_bfloat16 *>(last.out), last.out_pitch,
                                                   p->final_cin, p->final_w, p->final_b);
    else
      unet_final<float><<<S, 256, 0, st>>>(p->dev, p->sched, p->horizon, p->adim,
                                           static_cast<const float *>(last.out), last.out_pitch, p->final_cin,
                                           p->final_w, p->final_b);
    AURAS_LAUNCHED("unet_final");
    unet_advance<<<1, 1, 0, st>>>(p->dev);
    AURAS_LAUNCHED("unet_advance");
  }
  return AURAS_OK;
}

extern "C" {

auras_unet_plan *auras_unet_plan_create(const auras_conv_op *ops, int n_ops, int dtype, int s_max,
                                        int horizon, int action_dim, const float *film_tau,
                                        const float *ring_film, int film_width, int64_t ring_slot_stride,
                                        int64_t ring_agent_stride, const void *final_w, const float *final_b,
                                        int final_cin, const auras_sched *sched, void *x_in_buffer,
                                        int x_in_pitch) {
  if (!ops || n_ops <= 0 || s_max <= 0 || s_max > kMaxS || !sched || horizon * action_dim > 512) {
    set_error("unet_plan_create: bad args (s_max <= %d)", kMaxS);
    return nullptr;
  }
  auto *p = new auras_unet_plan();
  p->ops.assign(ops, ops + n_ops);
  p->dtype = dtype;
  p->s_max = s_max;
  p->horizon = horizon;
  p->adim = action_dim;
  p->film_tau = film_tau;
  p->ring_film = ring_film;
  p->film_width = film_width;
  p->ring_slot_stride = ring_slot_stride;
  p->ring_agent_stride = ring_agent_stride;
  p->final_w = static_cast<const float *>(final_w);
  p->final_b = final_b;
  p->final_cin = final_cin;
  p->sched = *sched;
  p->x_in = x_in_buffer;
  p->x_pitch = x_in_pitch;
  for (const auto &op : p->ops) {
    int64_t f = 0;
    for (int s = 1; s <= s_max; ++s) f = std::max(f, conv_scratch_floats(op, s, dtype));
    if (f > p->partial_floats) p->partial_floats = f;
  }
  if (cudaMalloc(&p->partial, sizeof(float) * p->partial_floats) != cudaSuccess ||
      cudaMalloc(&p->dev, sizeof(UnetDev)) != cudaSuccess ||
      cudaMemset(p->dev, 0, sizeof(UnetDev)) != cudaSuccess) {
    set_error("unet_plan_create: cudaMalloc failed");
    auras_unet_plan_destroy(p);
    return nullptr;
  }
  return p;
}

void auras_unet_plan_destroy(auras_unet_plan *p) {
  if (!p) return;
  for (auto &kv : p->graphs) cudaGraphExecDestroy(kv.second);
  if (p->partial) cudaFree(p->partial);
  if (p->dev) cudaFree(p->dev);
  delete p;
}

int auras_unet_generate(auras_unet_plan *p, int S, const int *lanes, const int *agents, const int *start,
                        const int *count, int iters, int lanes_per_agent, float *x_lanes,
                        const float *noise_lanes, const int64_t *fetched, int use_graph, void *stream) {
  if (!p || S <= 0 || S > p->s_max || iters < 0 || !x_lanes || !fetched) {
    set_error("unet_generate: bad args (S=%d s_max=%d)", S, p ? p->s_max : -1);
    return AURAS_E_ARG;
  }
  if (iters == 0) return AURAS_OK;
  cudaStream_t st = as_stream(stream);
  UnetCtrl c;
  memset(&c, 0, sizeof(c));
  for (int s = 0; s < S; ++s) {
    c.lanes[s] = lanes[s];
    c.agents[s] = agents[s];
    c.start[s] = start[s];
    c.count[s] = count[s];
    if (start[s] < 0 || start[s] + count[s] > p->sched.n_steps) {
      set_error("unet_generate: sample %d steps [%d, %d) outside schedule of %d", s, start[s],
                start[s] + count[s], p->sched.n_steps);
      return AURAS_E_ARG;
    }
  }
  c.x_lanes = x_lanes;
  c.noise_lanes = noise_lanes;
  c.fetched = fetched;
  c.S = S;
  c.lanes_per_agent = lanes_per_agent;
  unet_set_ctrl<<<1, 1, 0, st>>>(p->dev, c);
  AURAS_LAUNCHED("unet_set_ctrl");
  if (!use_graph) {
    for (int r = 0; r < iters; ++r) {
      int rc = unet_launch_step(p, S, st);
      if (rc) return rc;
    }
    return AURAS_OK;
  }
  auto it = p->graphs.find(S);
  if (it == p->graphs.end()) {
    cudaGraph_t g;
    AURAS_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    int rc = unet_launch_step(p, S, st);
    cudaError_t ce = cudaStreamEndCapture(st, &g);
    if (rc) return rc;
    AURAS_CUDA(ce);
    cudaGraphExec_t ge;
    ce = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);
    AURAS_CUDA(ce);
    AURAS_CUDA(cudaGraphUpload(ge, st));
    it = p->graphs.emplace(S, ge).first;
  }
  for (int r = 0; r < iters; ++r) AURAS_CUDA(cudaGraphLaunch(it->second, st));
  return AURAS_OK;
}

}  // extern "C"
