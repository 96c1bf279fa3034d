// Per-frame control of the batched denoise chain, shared by the layer-by-layer
// launcher (unet_plan.cu) and the persistent megakernel (unet_mega.cu).
#pragma once
#include "common.cuh"

namespace auras {

constexpr int kMaxS = 64;

struct UnetCtrl {             // per-frame control, uploaded by value
  int lanes[kMaxS], agents[kMaxS], start[kMaxS], count[kMaxS];
  float *x_lanes;
  const float *noise_lanes;
  const int64_t *fetched;
  int S, lanes_per_agent;
  int iters;                  // denoise iterations this frame (run inside one launch by the cluster kernel)
};

struct UnetDev {              // device-resident per-sample state
  UnetCtrl ctrl;
  int r;                      // iteration index within the frame, advanced in-graph
  int tau_row[kMaxS];
  int64_t film_b_off[kMaxS];
};

// Sample s: resolve its diffusion timestep for iteration r and the ring slot
// its agent fetched in-kernel; load x_t into the conv input (channels padded).
template <typename T>
__device__ void prep_body(UnetDev *dev, int s, int tid, int nthr, const auras_sched &sch, int horizon, int adim,
                          T *xin, int x_pitch, int64_t ring_slot_stride, int64_t ring_agent_stride, int r_it = -1) {
  const UnetCtrl &c = dev->ctrl;
  const int r = r_it >= 0 ? r_it : dev->r;
  const int agent = c.agents[s], lane = c.lanes[s];
  int i = c.start[s] + r;
  i = i < sch.n_steps ? i : sch.n_steps - 1;
  if (tid == 0) {
    dev->tau_row[s] = sch.timestep[i];
    const int64_t slot = c.fetched[0];   // one ring version schedule per lock-stepped agent group
    dev->film_b_off[s] = agent * ring_agent_stride + slot * ring_slot_stride;
  }
  const float *x = c.x_lanes + ((int64_t)agent * c.lanes_per_agent + lane) * horizon * adim;
  for (int e = tid; e < horizon * x_pitch; e += nthr) {
    const int t = e / x_pitch, ch = e - t * x_pitch;
    const float v = ch < adim ? x[t * adim + ch] : 0.f;
    Elem<T>::store(xin + ((int64_t)s * horizon + t) * x_pitch + ch, v);
  }
}

// eps = W_out . y + b (1x1 conv to action_dim) then the DDPM/DDIM update of
// sample s, written back to its request lane.  `eps` is >= horizon*adim floats
// of block-shared scratch; `sync` synchronises the nthr participating threads.
template <typename T, typename Sync>
__device__ void final_body(UnetDev *dev, int s, int tid, int nthr, const auras_sched &sch, int horizon, int adim,
                           const T *y, int y_pitch, int cin, const float *wf, const float *bf, float *eps,
                           Sync sync, int r_it = -1) {
  const UnetCtrl &c = dev->ctrl;
  const int r = r_it >= 0 ? r_it : dev->r;
  const int lane_id = tid & 31, wid = tid >> 5, nw = nthr >> 5;
  for (int o = wid; o < horizon * adim; o += nw) {
    const int t = o / adim, a = o - t * adim;
    const T *yr = y + ((int64_t)s * horizon + t) * y_pitch;
    float acc = 0.f;
    for (int k = lane_id; k < cin; k += 32) acc = fmaf(wf[a * cin + k], Elem<T>::load(yr + k), acc);
    acc = warp_sum(acc);
    if (lane_id == 0) eps[o] = acc + bf[a];
  }
  sync();
  if (r >= c.count[s]) return;                        // sample finished its share this frame
  const int i = c.start[s] + r;
  const int agent = c.agents[s], lane = c.lanes[s];
  float *x = c.x_lanes + ((int64_t)agent * c.lanes_per_agent + lane) * horizon * adim;
  const float *z = c.noise_lanes
                       ? c.noise_lanes + (((int64_t)agent * c.lanes_per_agent + lane) * sch.n_steps + i) * horizon * adim
                       : nullptr;
  const float sab = sch.sqrt_ab[i], s1m = sch.sqrt_1mab[i];
  const float cx0 = sch.c_x0[i], cxt = sch.c_xt[i], ceps = sch.c_eps[i], sig = sch.sigma[i];
  for (int e = tid; e < horizon * adim; e += nthr) {
    const float xt = x[e], ep = eps[e];
    float x0 = (xt - s1m * ep) / sab;
    if (sch.clip_sample) x0 = fminf(fmaxf(x0, -1.f), 1.f);
    float nx = cx0 * x0 + cxt * xt + ceps * ep;
    if (sch.ddpm && z) nx += sig * z[e];
    x[e] = nx;
  }
}

}  // namespace auras
