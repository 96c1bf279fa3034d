// Cluster (DSMEM) helpers and the host interface of the cluster denoise
// megakernel (unet_cluster.cu).
#pragma once
#include <cuda.h>

#include <vector>

#include "conv.cuh"
#include "mega.cuh"
#include "tc_util.cuh"
#include "unet.cuh"

namespace auras {

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// Whole-cluster barrier; every thread of every CTA must execute it.
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Address of the same shared-memory offset in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

__device__ __forceinline__ void st_cluster_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

__device__ __forceinline__ void st_cluster_v4_b32(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

// DSMEM store that also signals `bytes` of completed transaction on an mbarrier
// of the destination CTA (the receiver waits on its own barrier; no separate
// release/arrive round trip).
__device__ __forceinline__ void st_async_v4_b32(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                                uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
               "r"(a), "r"(b), "r"(c), "r"(d), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void st_async_b32(uint32_t addr, uint32_t a, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(addr), "r"(a), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void st_async_v2_f32(uint32_t addr, float a, float b, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(addr), "f"(a),
               "f"(b), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void st_cluster_v2(uint32_t addr, float a, float b) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}

__device__ __forceinline__ void st_release_i32(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Release-ordered counter increment (prior writes ordered by a CTA barrier
// become visible before the increment), one instruction instead of
// __threadfence + atomicAdd.
__device__ __forceinline__ void red_release_add(int *p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAITC:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONEC;\n"
      "bra LAB_WAITC;\n"
      "DONEC:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_5d_warp(void *dst, const CUtensorMap *tm, uint64_t *bar, uint32_t bytes,
                                                 int c0, int c1, int c2, int c3, int c4) {
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "@px mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n"
      "@px cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%4, %5, %6, %7, "
      "%8}], [%2];\n"
      "}\n" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(bytes), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

// ---------------------------------------------------------------- host interface
struct ClOp;
struct ClParams {
  const ClOp *ops;
  const int4 *tasks;
  const int *cl_begin;      // per-cluster task ranges
  int *ctr;                 // [n_ops] tile completions x 8, [1] prep, then pair flags
  int *flags;
  float2 *gstats;           // per tile of a 256-channel GroupNorm: (mean, M2) per sample
  int *err;                 // sticky error word: 1 = a dependency wait timed out
  int n_ops, S, nc, n_tasks;
  int l2_prefetch;          // L2 prefetch mode for the ring overflow of a task's weights
  int hack;                 // timing experiments (AURAS_CL_HACK); 0 in production
  int fault;                // stall injection for the watchdog test (AURAS_FAULT_STALL); 0 in production
  long long spin_timeout_ns;
  int spin_mode;
  UnetDev *dev;
  auras_sched sched;
  int horizon, adim;
  __nv_bfloat16 *xin;
  int x_pitch;
  int64_t ring_slot_stride, ring_agent_stride;
  const __nv_bfloat16 *y_final;
  int y_pitch, final_cin;
  const float *wf, *bf;
  long long *trace;         // optional [n_tasks][8] globaltimer stamps
};

struct BlockedBuf {           // kernel-owned channel-blocked copy of a plan activation buffer
  const void *orig = nullptr;
  __nv_bfloat16 *ptr = nullptr;
  int T = 0;
  int64_t plane = 0;          // elements per 64-channel block: S * T * 64
};

struct ClConfig {
  std::vector<BlockedBuf> blocked;
  ClOp *ops = nullptr;
  int4 *tasks = nullptr;
  int *cl_begin = nullptr;
  int *ctr = nullptr;
  float2 *gstats = nullptr;
  int ctr_ints = 0, n_ops = 0, n_tasks = 0, nc = 0, S = 0;
  int bn_var = 64;            // kernel variant: 64 or 128 columns per tile task (set before clus_build)
  ClParams params;
};

int clus_build(ClConfig &cc, const std::vector<auras_conv_op> &ops, int S, const void *x_in,
               const ClParams &base, const float *film_tau, int film_width, const float *ring_film,
               TiledCache &cache);
int clus_launch(const ClConfig &cc, cudaStream_t st);
int clus_error(const ClConfig &cc);
int clus_set_trace(ClConfig &cc, long long *trace);
void clus_free(ClConfig &cc);

}  // namespace auras
