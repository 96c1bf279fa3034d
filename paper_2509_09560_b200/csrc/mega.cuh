// Host interface of the persistent denoise megakernel (unet_mega.cu).
#pragma once
#include <cuda.h>

#include <utility>
#include <vector>

#include "conv.cuh"
#include "unet.cuh"

namespace auras {

struct MegaOp;
struct MegaParams {
  const MegaOp *ops;
  const int4 *tasks;
  const int *cta_begin;
  int *ctr;
  int n_ops, S;
  UnetDev *dev;
  auras_sched sched;
  int horizon, adim;
  __nv_bfloat16 *xin;
  int x_pitch;
  int64_t ring_slot_stride, ring_agent_stride;
  const __nv_bfloat16 *y_final;
  int y_pitch, final_cin;
  const float *wf, *bf;
  long long *trace;         // optional [n_tasks][8] globaltimer stamps (NULL = off)
  int spin_ns;              // back-off between counter polls
  long long *kbtrace;       // optional [grid][1024][3]: per-k-block A ready, B ready, MMA issued
  int a_depth;              // weight-ring stages actually used (<= na)
  int na;                   // weight-ring stages (the rest of the ring smem is activations)
};

struct MegaConfig {
  MegaOp *ops = nullptr;
  int4 *tasks = nullptr;
  int *cta_begin = nullptr;
  int *ctr = nullptr;
  float *partials = nullptr;
  int n_ops = 0, n_tasks = 0, grid = 0, S = 0;
  MegaParams params;
};

MegaParams mega_base_params(UnetDev *dev, const auras_sched &sched, int horizon, int adim, void *xin, int x_pitch,
                            int64_t slot_stride, int64_t agent_stride, const void *y_final, int y_pitch, int cin,
                            const float *wf, const float *bf);
using TiledCache = std::vector<std::pair<const void *, void *>>;   // (row-major weights, tiled copy)
int mega_build(MegaConfig &mc, const std::vector<auras_conv_op> &ops, int S, const void *x_in, int x_pitch,
               const MegaParams &base, const float *film_tau, int film_width, const float *ring_film,
               TiledCache &cache);
void mega_free_tiled(TiledCache &cache);
// weights re-laid out as [m_tile][k_block][128][64] (cached per plan) and their tensor map
// nmt = 2: m-tiles interleaved in pairs per k-block ([pair][kb][2][128][64]);
// such copies go in their own cache
int tiled_weights(TiledCache &cache, const auras_conv_op &o, void **out, int nmt = 1);
int make_tiled_weight_map(CUtensorMap *tm, const void *wt, int rows_total, int box_rows = 128);
int mega_launch(const MegaConfig &mc, cudaStream_t st);
int mega_set_trace(MegaConfig &mc, long long *trace);
void mega_free(MegaConfig &mc);

}  // namespace auras
