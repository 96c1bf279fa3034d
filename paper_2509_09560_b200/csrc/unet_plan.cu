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
#include <cstdlib>
#include <cstring>
#include <map>
#include <utility>
#include <vector>

#include "common.cuh"
#include "conv.cuh"
#include <functional>

#include "unet.cuh"
#include "mega.cuh"
#include "cluster.cuh"

namespace auras {

__global__ void unet_set_ctrl(UnetDev *dev, UnetCtrl c) {
  dev->ctrl = c;
  dev->r = 0;
}

__global__ void unet_advance(UnetDev *dev) { dev->r += 1; }
// after a cluster-kernel launch that ran all of the frame's iterations
__global__ void unet_advance_iters(UnetDev *dev) { dev->r += max(1, dev->ctrl.iters); }

template <typename T>
__global__ void unet_prep(UnetDev *dev, auras_sched sch, int horizon, int adim, T *xin, int x_pitch,
                          int64_t ring_slot_stride, int64_t ring_agent_stride) {
  prep_body<T>(dev, blockIdx.x, threadIdx.x, blockDim.x, sch, horizon, adim, xin, x_pitch, ring_slot_stride,
               ring_agent_stride);
}

template <typename T>
__global__ void unet_final(UnetDev *dev, auras_sched sch, int horizon, int adim, const T *y, int y_pitch, int cin,
                           const float *wf, const float *bf) {
  __shared__ float eps[512];
  final_body<T>(dev, blockIdx.x, threadIdx.x, blockDim.x, sch, horizon, adim, y, y_pitch, cin, wf, bf, eps,
                [] __device__() { __syncthreads(); });
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
  bool use_mega = false;                     // persistent megakernel (bf16, tcgen05 engine)
  std::map<int, MegaConfig> mega;
  bool use_cluster = false;                  // cluster megakernel (DSMEM split-K + GroupNorm)
  std::map<int, ClConfig> clus;
  std::map<int, int> use_clus_for;           // per S: 1 cluster kernel, 0 L2 split-K megakernel
  float *dry_x = nullptr;                    // scratch request lanes for autotuning runs
  int64_t *dry_fetched = nullptr;
  TiledCache tiled;                          // tiled weight copies shared by all S
  TiledCache tiled_cl;                       // the cluster kernel's copies (m-tile pairs interleaved)
};

static int mega_kernel_launch(auras_unet_plan *p, int S, bool cluster, cudaStream_t st) {
  if (cluster) {
    auto it = p->clus.find(S);
    if (it == p->clus.end()) { set_error("cluster config for S=%d not built", S); return AURAS_E_ARG; }
    return clus_launch(it->second, st);
  }
  auto it = p->mega.find(S);
  if (it == p->mega.end()) { set_error("megakernel config for S=%d not built", S); return AURAS_E_ARG; }
  return mega_launch(it->second, st);
}

// One denoise step through the persistent megakernel picked for S.
// One step of the persistent kernels: the L2 split-K megakernel runs one denoise
// iteration per launch; the cluster kernel runs every iteration of the frame
// (UnetCtrl::iters) in one launch.
static int unet_mega_step(auras_unet_plan *p, int S, cudaStream_t st) {
  const bool cl = p->use_clus_for[S] == 1;
  int rc = mega_kernel_launch(p, S, cl, st);
  if (rc) return rc;
  if (cl) {
    unet_advance_iters<<<1, 1, 0, st>>>(p->dev);
    AURAS_LAUNCHED("unet_advance_iters");
  } else {
    unet_advance<<<1, 1, 0, st>>>(p->dev);
    AURAS_LAUNCHED("unet_advance");
  }
  return AURAS_OK;
}

static int build_cluster_config(auras_unet_plan *p, int S, const MegaParams &base, int bn_var, ClConfig &out) {
  ClParams cb;
  memset(&cb, 0, sizeof(cb));
  cb.dev = base.dev;
  cb.sched = base.sched;
  cb.horizon = base.horizon;
  cb.adim = base.adim;
  cb.xin = base.xin;
  cb.x_pitch = base.x_pitch;
  cb.ring_slot_stride = base.ring_slot_stride;
  cb.ring_agent_stride = base.ring_agent_stride;
  cb.y_final = base.y_final;
  cb.y_pitch = base.y_pitch;
  cb.final_cin = base.final_cin;
  cb.wf = base.wf;
  cb.bf = base.bf;
  ClConfig cc;
  cc.bn_var = bn_var;
  int rc = clus_build(cc, p->ops, S, p->x_in, cb, p->film_tau, p->film_width, p->ring_film, p->tiled_cl);
  if (rc) {
    clus_free(cc);
    return rc;
  }
  out = cc;
  return AURAS_OK;
}

static float time_launches(const std::function<int()> &launch, cudaStream_t st, int reps = 3) {
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) || cudaEventCreate(&e1)) return 1e30f;
  float best = 1e30f;
  for (int r = 0; r <= reps; ++r) {
    cudaEventRecord(e0, st);
    if (launch()) { best = 1e30f; break; }
    cudaEventRecord(e1, st);
    if (cudaEventSynchronize(e1) != cudaSuccess) { best = 1e30f; break; }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0) best = std::min(best, ms);                 // r = 0 warms up
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

// The cluster kernel for batch S: the 64-column variant, and for S >= 16 also
// the 128-column one, timed on a dry batch; the faster is kept (AURAS_CL_VARIANT
// = 64 | 128 forces one).
static int prepare_dry_batch(auras_unet_plan *p, int S, cudaStream_t st);
static int choose_cluster_config(auras_unet_plan *p, int S, const MegaParams &base, cudaStream_t st) {
  const char *fv = getenv("AURAS_CL_VARIANT");
  const int forced = fv ? atoi(fv) : 0;
  ClConfig c64, c128;
  int rc64 = forced == 128 ? AURAS_E_ARG : build_cluster_config(p, S, base, 64, c64);
  int rc128 = (forced == 64 || (S < 16 && forced != 128)) ? AURAS_E_ARG : build_cluster_config(p, S, base, 128, c128);
  if (rc64 && rc128) return rc64 ? rc64 : rc128;
  if (!rc64 && !rc128) {
    int rc = prepare_dry_batch(p, S, st);
    if (rc) { clus_free(c64); clus_free(c128); return rc; }
    const float t64 = time_launches([&] { return clus_launch(c64, st); }, st);
    const float t128 = time_launches([&] { return clus_launch(c128, st); }, st);
    if (t128 < t64) { clus_free(c64); rc64 = AURAS_E_ARG; }
    else { clus_free(c128); rc128 = AURAS_E_ARG; }
  }
  p->clus.emplace(S, rc64 ? c128 : c64);
  return AURAS_OK;
}

// Time both persistent kernels on a dry batch of S samples (scratch request
// lanes; every buffer they write is either scratch or rewritten by the next
// real step's prep) and keep the faster one for this S.
static int prepare_dry_batch(auras_unet_plan *p, int S, cudaStream_t st) {
  if (!p->dry_x) {
    AURAS_CUDA(cudaMalloc(&p->dry_x, sizeof(float) * kMaxS * p->horizon * p->adim));
    AURAS_CUDA(cudaMemset(p->dry_x, 0, sizeof(float) * kMaxS * p->horizon * p->adim));
    AURAS_CUDA(cudaMalloc(&p->dry_fetched, sizeof(int64_t) * 4));
    AURAS_CUDA(cudaMemset(p->dry_fetched, 0, sizeof(int64_t) * 4));
  }
  UnetCtrl c;
  memset(&c, 0, sizeof(c));
  for (int s = 0; s < S; ++s) {
    c.lanes[s] = s;
    c.count[s] = 1;
  }
  c.x_lanes = p->dry_x;
  c.fetched = p->dry_fetched;
  c.S = S;
  c.lanes_per_agent = S;
  unet_set_ctrl<<<1, 1, 0, st>>>(p->dev, c);
  AURAS_LAUNCHED("unet_set_ctrl");
  return AURAS_OK;
}

static int autotune_mega(auras_unet_plan *p, int S, cudaStream_t st, int *pick) {
  int rc0 = prepare_dry_batch(p, S, st);
  if (rc0) return rc0;
  float best[2] = {1e30f, 1e30f};
  cudaEvent_t e0, e1;
  AURAS_CUDA(cudaEventCreate(&e0));
  AURAS_CUDA(cudaEventCreate(&e1));
  int rc = AURAS_OK;
  for (int rep = 0; rep < 4 && !rc; ++rep)
    for (int k = 0; k < 2 && !rc; ++k) {
      cudaEventRecord(e0, st);
      rc = mega_kernel_launch(p, S, k == 1, st);
      cudaEventRecord(e1, st);
      if (!rc && cudaEventSynchronize(e1) == cudaSuccess) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0) best[k] = std::min(best[k], ms);        // rep 0 warms both
      }
    }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rc) return rc;
  AURAS_CUDA(cudaGetLastError());
  *pick = best[1] < best[0] ? 1 : 0;
  return AURAS_OK;
}

static int unet_ensure_mega(auras_unet_plan *p, int S, cudaStream_t st) {
  if (!p->use_mega || p->use_clus_for.count(S)) return AURAS_OK;
  const auras_conv_op &last = p->ops.back();
  MegaParams base = mega_base_params(p->dev, p->sched, p->horizon, p->adim, p->x_in, p->x_pitch, p->ring_slot_stride,
                                     p->ring_agent_stride, last.out, last.out_pitch, p->final_cin, p->final_w,
                                     p->final_b);
  // AURAS_MEGA_KERNEL = "cluster" | "l2" forces one kernel; default: autotune per S
  const char *force = getenv("AURAS_MEGA_KERNEL");
  bool want_cluster = p->use_cluster && !(force && !strcmp(force, "l2"));
  bool want_l2 = !(force && !strcmp(force, "cluster") && p->use_cluster);
  if (want_cluster && choose_cluster_config(p, S, base, st)) {
    if (force && !strcmp(force, "cluster")) return AURAS_E_ARG;
    want_cluster = false;                     // shapes the cluster kernel does not cover
    want_l2 = true;
  }
  if (want_l2) {
    MegaConfig mc;
    int rc = mega_build(mc, p->ops, S, p->x_in, p->x_pitch, base, p->film_tau, p->film_width, p->ring_film,
                        p->tiled);
    if (rc) {
      mega_free(mc);
      return rc;
    }
    p->mega.emplace(S, mc);
  }
  int pick = want_cluster ? 1 : 0;
  if (want_cluster && want_l2) {
    int rc = autotune_mega(p, S, st, &pick);
    if (rc) return rc;
  }
  p->use_clus_for[S] = pick;
  return AURAS_OK;
}

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
  p->use_mega = false;
  if (dtype == AURAS_DT_BF16 && !getenv("AURAS_NO_MEGA")) {
    p->use_mega = true;
    for (const auto &op : p->ops) {
      ConvGemmArgs g;
      EpiArgs e;
      if (conv_op_to_args(op, 1, dtype, nullptr, g, e) || g.engine != 1) p->use_mega = false;
    }
  }
  p->use_cluster = p->use_mega && !getenv("AURAS_NO_CLUSTER");
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
  for (auto &kv : p->mega) mega_free(kv.second);
  for (auto &kv : p->clus) clus_free(kv.second);
  if (p->dry_x) cudaFree(p->dry_x);
  if (p->dry_fetched) cudaFree(p->dry_fetched);
  mega_free_tiled(p->tiled);
  mega_free_tiled(p->tiled_cl);
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
  c.iters = iters;
  int rc0 = unet_ensure_mega(p, S, st);
  if (rc0) return rc0;
  // launches per frame: one for the cluster kernel (all iterations inside), else one per iteration
  const int launches = (p->use_mega && p->use_clus_for[S] == 1) ? 1 : iters;
  auto step = p->use_mega ? unet_mega_step : unet_launch_step;
  unet_set_ctrl<<<1, 1, 0, st>>>(p->dev, c);
  AURAS_LAUNCHED("unet_set_ctrl");
  if (!use_graph) {
    for (int r = 0; r < launches; ++r) {
      int rc = step(p, S, st);
      if (rc) return rc;
    }
    return AURAS_OK;
  }
  auto it = p->graphs.find(S);
  if (it == p->graphs.end()) {
    cudaGraph_t g;
    AURAS_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    int rc = step(p, S, st);
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
  for (int r = 0; r < launches; ++r) AURAS_CUDA(cudaGraphLaunch(it->second, st));
  return AURAS_OK;
}

}  // extern "C"

extern "C" {

int auras_unet_kernel_for(const auras_unet_plan *p, int S) {
  if (!p) return AURAS_E_ARG;
  if (!p->use_mega) return 0;
  auto it = p->use_clus_for.find(S);
  return it == p->use_clus_for.end() ? -1 : 1 + it->second;
}

// Health of the persistent kernels: 0, or 1 when a dependency wait in a
// cluster-kernel launch gave up after its timeout (the pipeline stalled; the
// launch's outputs are garbage).  Reads and clears the sticky error words;
// synchronous (call where the host already waits on the generation stream).
int auras_unet_check(auras_unet_plan *p) {
  if (!p) return AURAS_E_ARG;
  int bad = 0;
  for (auto &kv : p->clus) {
    const int v = clus_error(kv.second);
    if (v < 0) { set_error("reading the cluster kernel's error word failed"); return AURAS_E_CUDA; }
    bad |= v;
  }
  return bad;
}

int auras_unet_launches_per_iter(const auras_unet_plan *p) {
  if (!p) return AURAS_E_ARG;
  return p->use_mega ? 2 : 3 + 2 * (int)p->ops.size();
}

// Diagnostics: enable a per-task globaltimer trace for the megakernel of batch
// size S (buffer: int64[n_tasks][8] + int64[grid][1024][3]); returns n_tasks, copies the task table
// (int32[n_tasks][4]) to `tasks_out` when non-NULL.  Graphs captured before the
// call keep their old parameters, so call it before the first generate.
int auras_unet_mega_trace(auras_unet_plan *p, int S, long long *trace, int *tasks_out, int max_tasks) {
  if (!p || !p->use_mega) { set_error("megakernel not in use"); return AURAS_E_ARG; }
  int rc = unet_ensure_mega(p, S, nullptr);
  if (rc) return rc;
  const int4 *tasks;
  int n_tasks;
  if (p->use_clus_for[S] == 1) {
    ClConfig &cc = p->clus[S];
    tasks = cc.tasks;
    n_tasks = cc.n_tasks;
    clus_set_trace(cc, trace);
  } else {
    MegaConfig &mc = p->mega[S];
    tasks = mc.tasks;
    n_tasks = mc.n_tasks;
    mega_set_trace(mc, trace);
  }
  if (tasks_out) {
    if (n_tasks > max_tasks) { set_error("task buffer too small"); return AURAS_E_ARG; }
    AURAS_CUDA(cudaMemcpy(tasks_out, tasks, sizeof(int4) * n_tasks, cudaMemcpyDeviceToHost));
  }
  return n_tasks;
}

}  // extern "C"
