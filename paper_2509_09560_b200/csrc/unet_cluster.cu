// Cluster dataflow megakernel: one launch runs every denoise iteration of a
// frame of the ConditionalUnet1D for all S in-flight samples (SURVEY.md §2.4
// K3-K5), with split-K reduction and GroupNorm statistics kept on chip.
//
// Why a second design (unet_mega.cu is the first): there, split-K partials go
// through L2 and a separate epilogue unit reduces them, so every layer of the
// 34-deep dependency chain pays drain -> HBM/L2 round trip -> epilogue ->
// counter -> next layer, ~12-18 us per layer under a saturated weight stream.
// Here a thread-block CLUSTER of 8 CTAs owns an output tile (128 channels, or
// 256 for the 2048-channel layers, x up to 64 / 128 columns) of one conv; its
// 8 CTAs split K 8 ways, and
//
//   * each CTA's tcgen05 accumulator (TMEM) is pushed row-slice-wise as fp16
//     into the owning CTA's shared memory with st.async, which signals the
//     owner's transaction mbarrier (reduce-scatter: CTA r owns channels
//     16r..16r+15 of each 128-channel tile; no cluster barrier);
//   * the owner sums the 8 slices in a fixed order (deterministic), adds the
//     bias, and computes GroupNorm statistics of 8-channel atoms in registers
//     (warp shuffles); atom statistics (mean, M2) go to every CTA of the
//     cluster the same way and are merged per group (Chan's formula, fixed
//     order).  Groups of 256 channels split over two clusters exchange tile
//     statistics through global memory;
//   * GroupNorm affine, Mish/ReLU, FiLM (per-sample rows gathered from the
//     timestep table and the context ring slot the sample fetched), residual
//     and the (optionally zero-stuffed) bf16 / fp32 store run on the same
//     registers, then one release per CTA on the op's completion counter.
//
// Warp roles per CTA (512 threads): warps 0-3 weight TMA producers (never wait
// on data -- the HBM weight stream runs ahead across layers and iterations),
// warp 4 UMMA issuer, warps 5-7 activation (implicit im2col) TMA producers
// gated on the producing ops' counters, warps 8-15 epilogue (8-11 also drain
// TMEM).  Each cluster walks a static list of tile tasks in layer order, once
// per iteration; counters accumulate over the iterations.  The grid is as
// many clusters as fit co-resident.  Deadlock freedom: tasks only wait on
// strictly earlier ops (or, across iterations, on the previous iteration's
// final tasks), except a GroupNorm pair, which is scheduled on two clusters in
// the same round (see clus_build).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "epi.cuh"
#include "tc_util.cuh"
#include "unet.cuh"
#include "mega.cuh"
#include "cluster.cuh"

#include <cuda_fp16.h>

namespace auras {

constexpr int CL = 8;                     // CTAs per cluster (portable maximum)
constexpr int CK_THREADS = 512;
// Warp roles.  One TMA-issuing warp has ~one bulk tensor copy in flight at a
// time (~0.4 us each, whatever the box size or ring depth; measured,
// scratch/ubench/tma_w2.cu), so both operand streams are spread over warps.
constexpr int CK_NWW = 4;                 // weight producer warps 0..3: warp w fills ring stages ia % 4 == w
constexpr int CK_MMA_WARP = 4;
constexpr int CK_BW0 = 5, CK_NBW = 3;     // activation TMA warps 5..7: warp 5 + (stage % 3)
constexpr int CK_EW0 = 8;
                                          // epilogue warps 8..15 (8..11 also drain TMEM)
constexpr int CK_EPI = 256;
constexpr int CK_A_BYTES = 128 * 64 * 2;  // one 128 x 64 weight box
constexpr int CK_A_STAGE = 2 * CK_A_BYTES;
constexpr int CK_BRING = 44 * 1024;       // activation ring (1 k-block per stage)
constexpr int CK_NBMAX = 16;
constexpr int CK_SMAX = 16;               // max samples per tile

// Shared-memory layout of the two kernel variants: BN = 64 columns per tile
// task (4 weight stages) for small batches, BN = 128 (3 weight stages, wider
// receive buffers) for many samples per step, where a 64-column tile would
// re-stream each layer's weights over 4-5 rounds of tasks.
template <int BN>
struct ClLay {
#ifndef CK_NA128
#define CK_NA128 3
#endif
  static constexpr int NA = BN == 64 ? 4 : CK_NA128;          // weight stages (2 k-blocks each)
  static constexpr int OFF_B = NA * CK_A_STAGE;
  static constexpr int OFF_RECV = OFF_B + CK_BRING;
  // one receive buffer (two alternate): >= CL x rows x (bn + 8) halves for rows x bn <= 16 BN
  static constexpr int RECV_BYTES = BN == 64 ? CL * 32 * 40 * 2 : CL * 32 * 72 * 2;
  static constexpr int OFF_STATS = OFF_RECV + 2 * RECV_BYTES;
  static constexpr int OFF_EPS = OFF_STATS + CL * 64 * 8;   // stats: CL x (atoms x samples <= 64) float2
  // range-safe partials (rare path): per receive buffer a flag word and exponent bytes
  // [src][owned row <= 32][16-column chunk <= 8]
  static constexpr int EXP_BYTES = CL * 32 * 8;
  static constexpr int OFF_EXPF = OFF_EPS + 1024;           // final-task scratch above (horizon x adim floats)
  static constexpr int OFF_EXP = OFF_EXPF + 16;
  static constexpr int OFF_BAR = OFF_EXP + 2 * EXP_BYTES;
  static constexpr int NBARS = 2 * NA + 2 * CK_NBMAX + 2 + 2 + 4;
  static constexpr size_t SMEM = 1024 + OFF_BAR + NBARS * 8 + 16;
  static_assert(SMEM <= 232448, "cluster kernel shared memory");
  static_assert(CL * 16 * (BN + 8) * 2 <= RECV_BYTES, "receive buffer");
};

enum { K_GEMM = 0, K_PREP = 2, K_FINAL = 3 };

struct alignas(64) ClOp {
  CUtensorMap tmA;            // weights, 256-row boxes: one TMA op per 32 KB ring stage
  CUtensorMap tmA1;           // 128-row boxes (odd tail k-block of a K share)
  CUtensorMap tmB;
  EpiArgs epi;
  int M, Cin, Wo, stride, pad, s_box, rows, bn, kb_total, kps, m_tiles, tiles;
  int bstage, nbst;
  int gn, cg, pair, flag_base;
  int lwo, lbn, lsb, lcg;     // log2 of Wo, bn, s_box, cg (all powers of two)
  int nmt;                    // 128-row m-tiles per task (2: a 256-channel GroupNorm group stays in one cluster)
  int rsh;                    // receive-buffer row stride (halves)
  // activation addressing: element (s, t, c) at base + (c >> 6) * plane + (s * T + t) * row + (c & 63)
  // (channel-blocked [C/64][S][T][64] buffers owned by this kernel, or the plan's [S][T][pitch] layout)
  const uint8_t *wt;          // tiled weights (L2 prefetch addresses)
  __nv_bfloat16 *out_base;
  const __nv_bfloat16 *res_base;
  int64_t out_plane, res_plane;
  int out_row, out_T, res_row, res_T;
  int gemm_dep[3], gemm_tgt[3];
  int epi_dep[2], epi_tgt[2];
};

__device__ __forceinline__ long long ck_time() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Per-task, per-rank globaltimer stamps (diagnostics): trace[(t * CL + rank) * 16 + k]
#define CK_TR(k) (P.trace[((int64_t)t * CL + rank) * 16 + (k)] = ck_time())

// Dependency wait.  Polls with relaxed loads (an ld.acquire.gpu in the loop
// emits an L1 invalidation per probe), then one acquire load.  A wait longer
// than P.spin_timeout_ns (2 s; AURAS_SPIN_TIMEOUT_MS) flags P.err -- surfaced by
// the host as DeadlockDetected (auras_unet_check) -- and gives up instead of
// hanging the GPU.
__device__ __forceinline__ int ld_relaxed_i32(const int *p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __noinline__ void ck_spin_slow(int *err, long long timeout_ns, const int *ctr, int target) {
  const long long t0 = ck_time();
  for (int n = 1; ld_relaxed_i32(ctr) < target; ++n)
    if ((n & 1023) == 0 && ck_time() - t0 > timeout_ns) {
      atomicExch(err, 1);
      return;
    }
}

__device__ __noinline__ void ck_spin_slow_acq(int *err, long long timeout_ns, const int *ctr, int target) {
  const long long t0 = ck_time();
  for (int n = 1; ld_acquire_i32(ctr) < target; ++n)
    if ((n & 1023) == 0 && ck_time() - t0 > timeout_ns) {
      atomicExch(err, 1);
      return;
    }
}

__device__ __forceinline__ void ck_spin(const ClParams &P, const int *ctr, int target) {
  if (P.spin_mode == 2) {
    if (ld_acquire_i32(ctr) < target) ck_spin_slow_acq(P.err, P.spin_timeout_ns, ctr, target);
    return;
  }
  if (ld_relaxed_i32(ctr) < target) ck_spin_slow(P.err, P.spin_timeout_ns, ctr, target);
  if (P.spin_mode == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  else (void)ld_acquire_i32(ctr);
}

// Counters accumulate over the frame's iterations: iteration `it` needs
// (it + 1) x the per-iteration count.
__device__ __forceinline__ void ck_wait_dep(const ClParams &P, const int *prep_done, int d, int tgt, int it) {
  if (d == -2) ck_spin(P, prep_done, P.S * (it + 1));
  else if (d >= 0) ck_spin(P, &P.ctr[d], P.fault ? 0x7fffffff : tgt * (it + 1));   // fault: stall injection (tests)
}

// Equal-count merge of k (mean, M2) pairs of n0 values each (fixed order).
__device__ __forceinline__ float2 merge_equal(const float2 *st, int stride, int k, float n0) {
  float m = 0.f;
  for (int i = 0; i < k; ++i) m += st[i * stride].x;
  m /= (float)k;
  float q = 0.f, d2 = 0.f;
  for (int i = 0; i < k; ++i) {
    q += st[i * stride].y;
    const float d = st[i * stride].x - m;
    d2 += d * d;
  }
  return make_float2(m, q + n0 * d2);
}

// Rare path of the slice sum: 8 fp16 slices, each scaled back by 2^e (its
// exponent byte; sources 32 x 8 bytes apart).  Out of line so the common path
// keeps its registers.
__device__ __noinline__ float ck_sum_scaled(const __half *rp, int stride, const uint8_t *eb) {
  float acc = 0.f;
  for (int src = 0; src < CL; ++src)
    acc += __half2float(rp[src * stride]) * __int_as_float((127 + (int)eb[src * 32 * 8]) << 23);
  return acc;
}

template <int BN>
__global__ void __launch_bounds__(CK_THREADS, 1) unet_cluster(const __grid_constant__ ClParams P) {
  using Lay = ClLay<BN>;
  constexpr int CK_BN = BN;
  constexpr int CK_NA = Lay::NA;
  constexpr int RECV_BYTES = Lay::RECV_BYTES;
  constexpr int VMAX = BN == 64 ? 4 : 8;
#ifdef CK_TMEM_ALL
  constexpr int CK_TMEM_COLS = 512;
#else
  constexpr int CK_TMEM_COLS = 4 * BN;
#endif   // values per epilogue thread (8: 128-column tiles)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KB alignment by an offset from the __shared__ array itself, so every
  // derived pointer stays in the shared window (LDS/STS, not generic LD/ST)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sA = smem;
  uint8_t *sB = smem + Lay::OFF_B;
  __half *recv = reinterpret_cast<__half *>(smem + Lay::OFF_RECV);
  float2 *stats = reinterpret_cast<float2 *>(smem + Lay::OFF_STATS);
  float *eps = reinterpret_cast<float *>(smem + Lay::OFF_EPS);
  uint32_t *expf = reinterpret_cast<uint32_t *>(smem + Lay::OFF_EXPF);
  uint8_t *exps = smem + Lay::OFF_EXP;
  uint64_t *fullA = reinterpret_cast<uint64_t *>(smem + Lay::OFF_BAR);
  uint64_t *emptyA = fullA + CK_NA;
  uint64_t *fullB = emptyA + CK_NA;
  uint64_t *emptyB = fullB + CK_NBMAX;
  uint64_t *tfull = emptyB + CK_NBMAX;
  uint64_t *tempty = tfull + 2;
  uint64_t *rbar = tempty + 2;             // transaction barriers: [buf] partials received, [2 + i] statistics received
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rbar + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_ctarank();
  const int cid = blockIdx.x / CL;
  const int t0 = P.cl_begin[cid], t1 = P.cl_begin[cid + 1];
  int *done = P.ctr;
  int *prep_done = P.ctr + P.n_ops;

  if (threadIdx.x == 0) {
    for (int i = 0; i < CK_NA; ++i) { mbar_init(&fullA[i], 1); mbar_init(&emptyA[i], 1); }
    for (int i = 0; i < CK_NBMAX; ++i) { mbar_init(&fullB[i], 1); mbar_init(&emptyB[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 8); }
    for (int i = 0; i < 4; ++i) mbar_init(&rbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == CK_MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(CK_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < (16 + 2 * Lay::EXP_BYTES) / 16; i += CK_THREADS)
    reinterpret_cast<uint4 *>(smem + Lay::OFF_EXPF)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();                       // peers' barriers initialised before any remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // the frame's denoise iterations all run in this launch (control word set per frame)
  const int iters = max(1, P.dev->ctrl.iters), r0 = P.dev->r;
  if (P.trace && threadIdx.x == 0) P.trace[16 * CL * (int64_t)P.n_tasks + 2 * blockIdx.x] = ck_time();

  if (warp < CK_NWW) {
    // ------------------------------------------------ weights: this CTA's K share of every task
    // L2 prefetch of the part of a task's K share that does not fit in the
    // ring (P.l2_prefetch: 1 = per-line prefetch.global.L2 from the LSU path,
    // 2 = one bulk prefetch per warp through the copy engine).  Issued when the
    // producers enter the task, i.e. while the previous task drains and the
    // layer's dependency is still unresolved, so the HBM stream keeps flowing
    // through the epilogue chain and the ring refills from L2.
    const int pf = P.l2_prefetch;
    int ia = 0;
    for (int it = 0; it < iters; ++it)
    for (int t = t0; t < t1; ++t) {
      const int4 tk = P.tasks[t];
      if ((tk.x & 0xff) != K_GEMM) continue;
      if (pf) {
        const ClOp *op = &P.ops[tk.x >> 8];
        const int kps = op->kps, kbt = op->kb_total, nmt = op->nmt;
        const int kb0 = rank * kps, kb1 = min(kbt, kb0 + kps);
        const int64_t row0 = (int64_t)tk.y * nmt * kbt * 128;
        const int64_t lo = (row0 + (int64_t)kb0 * 128 * nmt) * 128 + (int64_t)CK_NA * CK_A_STAGE;
        const int64_t hi = (row0 + (int64_t)kb1 * 128 * nmt) * 128;
        if (hi > lo) {
          const uint8_t *base = op->wt;
          if (pf == 1) {
            for (int64_t b = lo + (int64_t)(warp * 32 + lane) * 128; b < hi; b += CK_NWW * 32 * 128)
              asm volatile("prefetch.global.L2 [%0];" ::"l"(base + b));
          } else if (pf == 3) {
            for (int64_t b = lo + (int64_t)(warp * 32 + lane) * 128; b < hi; b += CK_NWW * 32 * 128)
              asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(base + b));
          } else if (lane == 0) {
            const int64_t chunk = ((hi - lo + CK_NWW - 1) / CK_NWW + 15) & ~15ll;
            const int64_t a = lo + warp * chunk, e = min(hi, a + chunk);
            if (e > a)
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + a), "r"((uint32_t)(e - a))
                           : "memory");
          }
        }
      }
      const ClOp *op = &P.ops[tk.x >> 8];
      const int kps = op->kps, kbt = op->kb_total;
      const int kb0 = rank * kps, kb1 = min(kbt, kb0 + kps);
      const int nmt = op->nmt;
      // tiled layouts: [m_tile][k_block][128][64] (nmt = 1), [pair][k_block][2][128][64] (nmt = 2);
      // a ring stage (32 KB) is one 256-row box either way
      const int row0 = tk.y * nmt * kbt * 128;
      if (nmt == 1) {                               // stage = 2 k-blocks of one m-tile
        for (int kb = kb0; kb < kb1; kb += 2, ++ia) {
          const int st = ia % CK_NA;
          if (st % CK_NWW != warp) continue;         // a stage always has the same issuing warp
          const bool two = kb + 1 < kb1;
          mbar_wait(&emptyA[st], ((ia / CK_NA) & 1) ^ 1);
          if (P.hack & 2) { if (lane == 0) mbar_arrive(&fullA[st]); __syncwarp(); continue; }
          tma_load_2d_warp(sA + st * CK_A_STAGE, two ? &op->tmA : &op->tmA1, &fullA[st],
                           two ? CK_A_STAGE : CK_A_BYTES, 0, row0 + kb * 128);
        }
      } else {                                      // stage = 1 k-block of both m-tiles
        for (int kb = kb0; kb < kb1; ++kb, ++ia) {
          const int st = ia % CK_NA;
          if (st % CK_NWW != warp) continue;         // a stage always has the same issuing warp
          mbar_wait(&emptyA[st], ((ia / CK_NA) & 1) ^ 1);
          if (P.hack & 2) { if (lane == 0) mbar_arrive(&fullA[st]); __syncwarp(); continue; }
          tma_load_2d_warp(sA + st * CK_A_STAGE, &op->tmA, &fullA[st], CK_A_STAGE, 0, row0 + kb * 256);
        }
      }
    }
  } else if (warp >= CK_BW0 && warp < CK_BW0 + CK_NBW) {
    // ------------------------------------------------ activations: after the producing ops
    // k-block j of a task goes to ring stage j % nbst, issued by warp 5 + stage % 3
    const int bw = warp - CK_BW0;
    uint32_t par = 0;
    for (int it = 0; it < iters; ++it)
    for (int t = t0; t < t1; ++t) {
      const int4 tk = P.tasks[t];
      if ((tk.x & 0xff) != K_GEMM) continue;
      const ClOp *op = &P.ops[tk.x >> 8];
      const int bstage = op->bstage, nbst = op->nbst;
      const int kps = op->kps, kbt = op->kb_total, Cin = op->Cin, pad = op->pad, stride = op->stride;
      const int sbox = op->s_box;
      const uint32_t bbytes = op->rows * 128;
      const CUtensorMap *tmB = &op->tmB;
      if (lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(tmB) : "memory");   // descriptor fetch off the critical path
        if (!(P.hack & 32768))
          for (int d = 0; d < 3; ++d) ck_wait_dep(P, prep_done, op->gemm_dep[d], op->gemm_tgt[d], it);
        fence_proxy_async();
        if (P.trace && bw == 0) CK_TR(0);
      }
      __syncwarp();
      const int kb0 = rank * kps, kb1 = min(kbt, kb0 + kps);
      for (int kb = kb0, j = 0; kb < kb1; ++kb, ++j) {
        const int sb = j % nbst;
        if (sb % CK_NBW != bw) continue;
        mbar_wait(&emptyB[sb], ((par >> sb) & 1) ^ 1);
        par ^= 1u << sb;
        const int k = kb * 64;
        const int tap = k / Cin, c0 = k - tap * Cin;
        const int off = tap - pad;
        const int q = off >= 0 ? off / stride : -((-off + stride - 1) / stride);
        const int h = off - q * stride;
        if ((P.hack & 1) && (j > 0 || (P.hack & 16384))) { if (lane == 0) mbar_arrive(&fullB[sb]); __syncwarp(); continue; }
        if (P.hack & 8) {
          if (lane == ((j / CK_NBW) & 31)) {
            mbar_expect_tx(&fullB[sb], bbytes);
            asm volatile(
                "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
                "%6, %7}], [%2];" ::"r"(smem_u32(sB + sb * bstage)),
                "l"(tmB), "r"(smem_u32(&fullB[sb])), "r"(0), "r"(h), "r"(q), "r"(tk.z * sbox), "r"(c0 >> 6)
                : "memory");
          }
          __syncwarp();
          continue;
        }
        tma_load_5d_warp(sB + sb * bstage, tmB, &fullB[sb], bbytes, 0, h, q, tk.z * sbox, c0 >> 6);
      }
    }
  } else if (warp == CK_MMA_WARP) {
    // ------------------------------------------------ MMA issuer
    // One warp issues every UMMA of the CTA; with N = 32..64 its instruction
    // stream, not the tensor pipe, bounds a k-block, so the loop is kept lean:
    // ring slots advance incrementally, descriptors come from precomputed
    // shared-memory addresses, one elected lane issues a whole K = 64 block.
    int ia = 0, gi = 0, sa = 0;
    uint32_t par = 0, pa_bits = 0;
    const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB);
    for (int it = 0; it < iters; ++it)
    for (int t = t0; t < t1; ++t) {
      const int4 tk = P.tasks[t];
      if ((tk.x & 0xff) != K_GEMM) continue;
      const ClOp *op = &P.ops[tk.x >> 8];
      const int kps = op->kps, kbt = op->kb_total, bn = op->bn, bstage = op->bstage, nbst = op->nbst;
      const int buf = gi & 1;
      mbar_wait(&tempty[buf], ((gi >> 1) & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t idesc = umma_idesc(bn);
      const uint32_t dt = tmem + buf * 2 * CK_BN;
      const int kb0 = rank * kps, kb1 = min(kbt, kb0 + kps);
      int sb = 0;
      if (op->nmt == 2) {                           // two accumulators: m-tile u at column u * CK_BN
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&fullA[sa], (pa_bits >> sa) & 1);
          mbar_wait(&fullB[sb], (par >> sb) & 1);
          if (P.trace && lane == 0 && kb == kb0) CK_TR(1);
          par ^= 1u << sb;
          pa_bits ^= 1u << sa;
          if (!(P.hack & 1024))
            umma_kblock2_warp(dt, dt + CK_BN, umma_desc(sA0 + sa * CK_A_STAGE), umma_desc(sB0 + sb * bstage), idesc,
                              kb > kb0 ? 1u : 0u);
          umma_commit_warp(&emptyB[sb]);
          umma_commit_warp(&emptyA[sa]);
          sb = sb + 1 == nbst ? 0 : sb + 1;
          sa = sa + 1 == CK_NA ? 0 : sa + 1;
          ++ia;
        }
      } else {
        for (int kb = kb0; kb < kb1; kb += 2) {
          mbar_wait(&fullA[sa], (pa_bits >> sa) & 1);
          pa_bits ^= 1u << sa;
          const uint32_t a0 = sA0 + sa * CK_A_STAGE;
          const int nk = min(2, kb1 - kb);
          for (int i = 0; i < nk; ++i) {
            mbar_wait(&fullB[sb], (par >> sb) & 1);
            if (P.trace && lane == 0 && kb == kb0 && i == 0) CK_TR(1);
            par ^= 1u << sb;
            if (!(P.hack & 1024))
              umma_kblock_warp(dt, umma_desc(a0 + i * CK_A_BYTES), umma_desc(sB0 + sb * bstage), idesc,
                               (kb > kb0 || i > 0) ? 1u : 0u);
            umma_commit_warp(&emptyB[sb]);
            sb = sb + 1 == nbst ? 0 : sb + 1;
          }
          umma_commit_warp(&emptyA[sa]);
          sa = sa + 1 == CK_NA ? 0 : sa + 1;
          ++ia;
        }
      }
      if (P.trace && lane == 0) CK_TR(2);
      if (kb1 > kb0) umma_commit_warp(&tfull[buf]);
      else if (lane == 0) mbar_arrive(&tfull[buf]);      // empty K share: the drain pushes zeros
      __syncwarp();
      ++gi;
    }
  } else if (warp >= CK_EW0) {
    // ------------------------------------------------ epilogue warps
    const int et = threadIdx.x - 32 * CK_EW0;
    const int ew = warp - CK_EW0;
    auto esync = [] __device__() { named_sync(1, CK_EPI); };
    int gi = 0, gn_i = 0;
    for (int it = 0; it < iters; ++it)
    for (int t = t0; t < t1; ++t) {
      const int4 tk = P.tasks[t];
      const int type = tk.x & 0xff, opi = tk.x >> 8;
      if (type == K_GEMM) {
        const ClOp *op = &P.ops[opi];
        const EpiArgs e = op->epi;
        const int M = op->M, Wo = op->Wo, sbox = op->s_box, rows = op->rows, bn = op->bn;
        const int kps = op->kps, kbt = op->kb_total, gn = op->gn, cg = op->cg, pair = op->pair;
        // timing ablations (AURAS_CL_HACK, scratch/r2_ab.sh; 0 in production): 256 no statistics
        // exchange, 512 no partials exchange, 1024 no UMMA, 2048 no apply / store, 16384 (with 1)
        // no activation boxes, 32768 no dependency waits
        const int gnx = gn && !(P.hack & 256);
        const int nmt = op->nmt, mt0 = tk.y * nmt, nt = tk.z, S = P.S;
        const int lwo = op->lwo, lsb = op->lsb, lcg = op->lcg;
        const int RPC = 16 * nmt;                        // rows (channels) owned by this CTA
        const int RSH = op->rsh;                         // receive row stride (halves)
        const int A = 2 * nmt;                           // 8-channel GroupNorm atoms owned
        const int nkb = max(0, min(kbt, (rank + 1) * kps) - rank * kps);
        const bool film = e.film_off >= 0;
        const int buf = gi & 1;
        // receive buffers alternate by task: a peer pushing task t+1 has passed
        // barrier A of task t, so every CTA is done reading task t-1's buffer
        __half *recvb = recv + buf * (RECV_BYTES / 2);
        // channel of owned row r (0..RPC-1): tile r >> 4, row 16 * rank + (r & 15) of that tile
        auto chan = [&](int r) { return (mt0 + (r >> 4)) * 128 + 16 * rank + (r & 15); };
        // ---- residual producers and the per-sample FiLM rows (prep) first
        if (et == 0) {
          // bytes this CTA will receive: 16 * nmt rows x bn fp16 partials from each of the 8
          // CTAs; with GroupNorm, (mean, M2) of 2 * nmt atoms x s_box samples from each
          if (!(P.hack & 512)) mbar_expect_tx(&rbar[buf], (uint32_t)(CL * 16 * nmt * bn * 2));
          if (gnx) mbar_expect_tx(&rbar[2 + (gn_i & 1)], (uint32_t)(CL * 2 * nmt * sbox * 8));
          if (film) ck_spin(P, prep_done, S * (it + 1));
          if (!(P.hack & 32768))
            for (int d = 0; d < 2; ++d) ck_wait_dep(P, prep_done, op->epi_dep[d], op->epi_tgt[d], it);
          if (P.trace) CK_TR(12);
        }
        esync();
        // ---- element ownership.  Thread et belongs to (atom pa, sample pj) pair pi = et / L
        //      (L lanes per pair, L | 32, L >= Wo).  With L >= 2 Wo (NH = 1) lane li < 2 Wo owns
        //      channels 4 hh .. 4 hh + 3 (hh = li / Wo) of the atom's 8 rows; with L = Wo (NH = 2,
        //      128-column tiles) lane li owns all 8 -- at time tq = li % Wo, tile column
        //      col = pj * Wo + tq.  The slice sums, the atom statistics (warp shuffles), the
        //      group merge and the store all run on these registers: no staging, no CTA barrier.
        const int lL = min(5, 8 - lsb - nmt), L = 1 << lL;         // L = min(32, 256 / (A * sbox))
        const int NH = (VMAX == 4 || L >= 2 * Wo) ? 1 : 2;
        const int pi = et >> lL, li = et & (L - 1);
        const int pa = pi >> lsb, pj = pi & (sbox - 1);
        const bool in_pair = pi < A * sbox;
        const int hh = NH == 1 ? li >> lwo : 0, tq = li & (Wo - 1);
        const int col = pj * Wo + tq;
        const int s = nt * sbox + pj;
        const int row0 = 8 * pa + 4 * hh;                  // first owned row (0..RPC-1)
        const int ch0 = chan(row0);                        // its channel (4 or 8 consecutive channels)
        const bool mine = in_pair && li < (2 * Wo) / NH && col < rows && s < S && ch0 < M;
        float bias[VMAX], gam[VMAX], bet[VMAX], sc[VMAX], bi[VMAX], v[VMAX], r[VMAX];
#pragma unroll
        for (int k = 0; k < VMAX; ++k) {
          bias[k] = 0.f; gam[k] = 1.f; bet[k] = 0.f; sc[k] = 1.f; bi[k] = 0.f; r[k] = 0.f;
        }
        if (mine) {
          const float *fa = film ? e.film_a + (int64_t)e.film_a_row[s] * e.film_a_stride + e.film_off : nullptr;
          const float *fb = (film && e.film_b) ? e.film_b + e.film_b_off[s] + e.film_off : nullptr;
#pragma unroll
          for (int k = 0; k < VMAX; ++k) {
            if (k >= 4 * NH) break;
            const int ch = ch0 + k;
            if (e.bias) bias[k] = e.bias[ch];
            if (gn) { gam[k] = e.gn_gamma[ch]; bet[k] = e.gn_beta[ch]; }
            if (fa) {
              sc[k] = fa[ch] + (fb ? fb[ch] : 0.f);
              bi[k] = fa[M + ch] + (fb ? fb[M + ch] : 0.f);
            }
          }
#pragma unroll
          for (int h = 0; h < VMAX / 4; ++h) {
            if (h >= NH) break;
            const int c4 = ch0 + 4 * h;
            if (e.res) {                                 // 4 bf16 channels of the residual
              const uint2 u = __ldcg(reinterpret_cast<const uint2 *>(
                  op->res_base + (c4 >> 6) * op->res_plane + ((int64_t)s * op->res_T + tq) * op->res_row + (c4 & 63)));
              const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.x));
              const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.y));
              r[4 * h] = f0.x; r[4 * h + 1] = f0.y; r[4 * h + 2] = f1.x; r[4 * h + 3] = f1.y;
            } else if (e.res_f32) {
              const float4 f = __ldcg(reinterpret_cast<const float4 *>(e.res_f32 + ((int64_t)s * Wo + tq) * M + c4));
              r[4 * h] = f.x; r[4 * h + 1] = f.y; r[4 * h + 2] = f.z; r[4 * h + 3] = f.w;
            }
          }
        }
        // ---- drain TMEM and push row slices to their owners (reduce-scatter over DSMEM):
        //      all 8 epilogue warps, warps ew and ew + 4 (same TMEM lane quadrant) taking
        //      alternate 16-column chunks
        {
          mbar_wait(&tfull[buf], (gi >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (P.trace && et == 0) CK_TR(3);
          const int quad = ew & 3, half = ew >> 2;
          const int m = quad * 32 + lane;
          const int cpu = bn >> 4, nch = nmt * cpu;
          for (int q = half; q < nch; q += 2) {
            const int u = q / cpu, c = (q - u * cpu) * 16;
            // fp16 partial sums (K/8 terms each, fp32-accumulated in TMEM): half the
            // DSMEM traffic; the owner sums the 8 slices in fp32
            const uint32_t dst = mapa_shared(smem_u32(recvb + (rank * RPC + u * 16 + (m & 15)) * RSH), m >> 4);
            const uint32_t rbar_dst = mapa_shared(smem_u32(&rbar[buf]), m >> 4);
            {
              float x[16];
              if (nkb > 0) {
                tmem_ld16(tmem + buf * 2 * CK_BN + u * CK_BN + c + ((uint32_t)(quad * 32) << 16), x);
              } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) x[i] = 0.f;
              }
              // range safety: a row whose 16 partials reach 2^15 goes as fp16(x 2^-e), its
              // exponent e written to the owner's exponent bytes (and flag) before the data; the
              // data's complete_tx (release, cluster scope) publishes them.  Rare path only:
              // otherwise e = 0 and nothing extra is sent.
              // (columns past the tile's `rows` hold products of stale operand rows: excluded)
              float mx = 0.f;
              if (c + 16 <= rows) {
#pragma unroll
                for (int i = 0; i < 16; ++i) mx = fmaxf(mx, fabsf(x[i]));
              } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) mx = fmaxf(mx, c + i < rows ? fabsf(x[i]) : 0.f);
              }
#ifndef CK_NO_RANGE
              if (__any_sync(0xffffffffu, mx >= 32768.f) && !(P.hack & 128)) {
                const int ex = min(126, max(0, ((__float_as_int(mx) >> 23) & 0xff) - 127 - 14));
                if (ex > 0) {
                  const float down = __int_as_float((127 - ex) << 23);
#pragma unroll
                  for (int i = 0; i < 16; ++i) x[i] *= down;
                  const uint32_t ea = mapa_shared(
                      smem_u32(exps + buf * Lay::EXP_BYTES + (rank * 32 + u * 16 + (m & 15)) * 8 + (c >> 4)), m >> 4);
                  asm volatile("st.shared::cluster.u8 [%0], %1;" ::"r"(ea), "h"((unsigned short)ex) : "memory");
                  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(mapa_shared(smem_u32(expf + buf), m >> 4)),
                               "r"(1u)
                               : "memory");
                }
                asm volatile("fence.acq_rel.cluster;" ::: "memory");
              }
#endif
              uint32_t hw[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const __half2 h2 = __floats2half2_rn(x[2 * i], x[2 * i + 1]);
                hw[i] = *reinterpret_cast<const uint32_t *>(&h2);
              }
              if (!(P.hack & 512)) {
                st_async_v4_b32(dst + c * 2, hw[0], hw[1], hw[2], hw[3], rbar_dst);
                st_async_v4_b32(dst + c * 2 + 16, hw[4], hw[5], hw[6], hw[7], rbar_dst);
              }
            }
          }
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[buf]);
          if (P.trace && et == 0) CK_TR(4);
        }
        if (!(P.hack & 512)) mbar_wait_cluster(&rbar[buf], (gi >> 1) & 1);   // all 8 CTAs' partials have landed
        if (P.trace && et == 0) CK_TR(5);
        // ---- fixed-order sum of the 8 K slices + bias (fp32); slices a source scaled
        //      (exponent bytes, flagged per buffer: rare) are scaled back out of line
#ifndef CK_NO_RANGE
        const uint32_t scaled = expf[buf];
#else
        const uint32_t scaled = 0;
#endif
        if (!scaled) {
#pragma unroll
          for (int k = 0; k < VMAX; ++k) {
            float acc = bias[k];
            if (mine && k < 4 * NH) {
              const __half *rp = recvb + (row0 + k) * RSH + col;
#pragma unroll
              for (int src = 0; src < CL; ++src) acc += __half2float(rp[src * RPC * RSH]);
            }
            v[k] = acc;
          }
        } else {
#pragma unroll
          for (int k = 0; k < VMAX; ++k) {
            float acc = bias[k];
            if (mine && k < 4 * NH)
              acc += ck_sum_scaled(recvb + (row0 + k) * RSH + col, RPC * RSH,
                                   exps + buf * Lay::EXP_BYTES + (row0 + k) * 8 + (col >> 4));
            v[k] = acc;
          }
        }
        const float n0 = 8.f * Wo;
        const int fi = pair ? op->flag_base + nt * op->m_tiles + mt0 : 0;
        float mean_g = 0.f, rstd_g = 1.f;
        if (gnx) {
          // ---- atom statistics: 8 rows x Wo columns of (pa, pj), butterfly over the pair's L lanes
          if (in_pair) {
            float sum = 0.f, sq = 0.f;
#pragma unroll
            for (int k = 0; k < VMAX; ++k)
              if (mine && k < 4 * NH) { sum += v[k]; sq += v[k] * v[k]; }
            for (int o = 1; o < L; o <<= 1) {
              sum += __shfl_xor_sync(0xffffffffu, sum, o);
              sq += __shfl_xor_sync(0xffffffffu, sq, o);
            }
            const float mean = sum / n0;
            const float m2a = fmaxf(sq - sum * mean, 0.f);
            for (int dst = li; dst < CL; dst += L) {      // lane li -> CTAs li, li + L, ...
              st_async_v2_f32(mapa_shared(smem_u32(stats + (rank * A + pa) * sbox + pj), dst), mean, m2a,
                              mapa_shared(smem_u32(&rbar[2 + (gn_i & 1)]), dst));
            }
            if (pair && li == (CL & (L - 1)))            // the partner tile reads its atoms from L2
              __stcg(&P.gstats[((int64_t)fi * 16 + rank * 2 + pa) * CK_SMAX + pj], make_float2(mean, m2a));
          }
          if (pair) {                                     // published before the exchange
            esync();
            if (et == 0) red_release_add(&P.flags[fi], 1);
          }
        }
        if (P.trace && et == 0) CK_TR(6);
        if (gnx) mbar_wait_cluster(&rbar[2 + (gn_i & 1)], (gn_i >> 1) & 1);   // every peer's statistics
        if (P.trace && et == 0) CK_TR(7);
        if (gnx) {
          // ---- merge the atoms of each group (butterfly, fixed lane order); task atoms are
          //      numbered in channel order q = tile * 16 + within-tile atom; 256-channel groups
          //      split over two tasks also merge the partner tile's statistics from L2.  Every
          //      lane of the pair ends with the group's (mean, rstd).
          float2 gs = make_float2(0.f, 0.f);
          float ncount = 1.f;
          if (pair) {                                     // partner tile's 8 CTAs have published
            if (et == 0) ck_spin(P, &P.flags[fi ^ 1], CL);
            esync();
          }
          if (in_pair && !(P.hack & 4096)) {           // (4096: timing probe -- skip the merge arithmetic)
            const int cha = chan(8 * pa);
            const int gf = (cha >> lcg) << lcg;
            const int tlo = mt0 * 128, thi = min((mt0 + nmt) * 128, M);
            const int lo = max(gf, tlo), hi = min(gf + cg, thi);
            const int q0 = (lo - tlo) >> 3, kq = (hi - lo) >> 3;
            auto atom = [&](const float2 *base, int q) {  // task atom q -> stats entry
              const int w = q & 15, u = q >> 4;
              return base[((w >> 1) * A + 2 * u + (w & 1)) * sbox + pj];
            };
            // butterfly merge of kq equal-count atoms (lane li takes atoms li, li + L, ...)
            auto merge = [&](const float2 *base, bool global) {
              auto get = [&](int q) {
                return global ? __ldcg(base + (int64_t)(q0 + q) * CK_SMAX + pj) : atom(base, q0 + q);
              };
              float m = 0.f;
              for (int q = li; q < kq; q += L) m += get(q).x;
              for (int o = 1; o < L; o <<= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
              m /= (float)kq;
              float qs = 0.f;
              for (int q = li; q < kq; q += L) {
                const float2 at = get(q);
                const float d = at.x - m;
                qs += at.y + n0 * d * d;
              }
              for (int o = 1; o < L; o <<= 1) qs += __shfl_xor_sync(0xffffffffu, qs, o);
              return make_float2(m, qs);
            };
            gs = merge(stats, false);
            ncount = n0 * kq;
            if (pair) {                                   // partner tile (16 atoms), lower tile first
              const float2 other = merge(P.gstats + (int64_t)(fi ^ 1) * 16 * CK_SMAX, true);
              const float2 lo2 = (mt0 & 1) ? other : gs, hi2 = (mt0 & 1) ? gs : other;
              const float m = 0.5f * (lo2.x + hi2.x);
              const float d0 = lo2.x - m, d1 = hi2.x - m;
              gs = make_float2(m, (lo2.y + hi2.y) + ncount * (d0 * d0 + d1 * d1));
              ncount *= 2.f;
            }
          }
          mean_g = gs.x;
          rstd_g = rsqrtf(gs.y / ncount + 1e-5f);
        }
        if (P.trace && et == 0) CK_TR(8);
        // ---- normalise, activate, FiLM, residual (registers) and store 4 channels per half
        if (mine && !(P.hack & 2048)) {
          const float rba = e.res_before_act ? 1.f : 0.f;
          const float is_mish = e.act == AURAS_ACT_MISH ? 1.f : 0.f;
          const float is_relu = e.act == AURAS_ACT_RELU ? 1.f : 0.f;
          const float is_none = 1.f - is_mish - is_relu;
          float y[VMAX];
#pragma unroll
          for (int k = 0; k < VMAX; ++k) {
            float x = gn ? (v[k] - mean_g) * rstd_g * gam[k] + bet[k] : v[k];
            x += rba * r[k];
            const float ex = __expf(fminf(x, 20.f));
            const float nn = ex * (ex + 2.f);
            const float ratio = __fdividef(nn, nn + 2.f);
            const float xm = x * (x > 20.f ? 1.f : ratio);
            x = is_mish * xm + is_relu * fmaxf(x, 0.f) + is_none * x;
            x = x * sc[k] + bi[k];
            y[k] = x + (1.f - rba) * r[k];
          }
#pragma unroll
          for (int h = 0; h < VMAX / 4; ++h) {
            if (h >= NH) break;
            const int c4 = ch0 + 4 * h;
            if (e.out) {
              const __nv_bfloat162 b0 = __floats2bfloat162_rn(y[4 * h], y[4 * h + 1]);
              const __nv_bfloat162 b1 = __floats2bfloat162_rn(y[4 * h + 2], y[4 * h + 3]);
              const int ox2 = e.out_stuff ? 2 * tq : tq;
              __nv_bfloat16 *dst = op->out_base + (c4 >> 6) * op->out_plane +
                                   ((int64_t)s * op->out_T + ox2) * op->out_row + (c4 & 63);
              *reinterpret_cast<uint2 *>(dst) =
                  make_uint2(*reinterpret_cast<const uint32_t *>(&b0), *reinterpret_cast<const uint32_t *>(&b1));
              if (e.out_stuff) *reinterpret_cast<uint2 *>(dst + op->out_row) = make_uint2(0, 0);
            }
            if (e.out_f32)
              *reinterpret_cast<float4 *>(e.out_f32 + ((int64_t)s * Wo + tq) * M + c4) =
                  make_float4(y[4 * h], y[4 * h + 1], y[4 * h + 2], y[4 * h + 3]);
          }
        }
        if (P.trace && et == 0) CK_TR(9);
        fence_proxy_async();
        esync();
        if (scaled) {                                            // every reader is past the sum: reset for task gi + 2
          for (int i = et; i < Lay::EXP_BYTES / 16; i += CK_EPI)
            reinterpret_cast<uint4 *>(exps + buf * Lay::EXP_BYTES)[i] = make_uint4(0, 0, 0, 0);
          if (et == 0) expf[buf] = 0;
        }
        if (et == 0) {
          if (P.trace) CK_TR(10);
          red_release_add(&done[opi], 1);
          if (P.trace) CK_TR(11);
        }
        ++gi;
        gn_i += gnx;
      } else if (type == K_PREP) {
        if (tk.w != rank || it > 0) continue;            // later iterations: prepared by the final task
        if (P.trace && et == 0) CK_TR(0);
        prep_body<__nv_bfloat16>(P.dev, tk.y, et, CK_EPI, P.sched, P.horizon, P.adim, P.xin, P.x_pitch,
                                 P.ring_slot_stride, P.ring_agent_stride, r0);
        fence_proxy_async();
        esync();
        if (et == 0) {
          __threadfence();
          atomicAdd(prep_done, 1);
          if (P.trace) CK_TR(11);
        }
      } else if (type == K_FINAL) {
        if (tk.w != rank) continue;
        if (et == 0) ck_spin(P, &done[P.n_ops - 1], P.ops[P.n_ops - 1].tiles * CL * (it + 1));
        if (P.trace && et == 0) CK_TR(0);
        esync();
        final_body<__nv_bfloat16>(P.dev, tk.y, et, CK_EPI, P.sched, P.horizon, P.adim, P.y_final, P.y_pitch,
                                  P.final_cin, P.wf, P.bf, eps, esync, r0 + it);
        if (it + 1 < iters) {
          // the sample's next iteration input, from the x this task just wrote (every op of
          // this iteration has finished: nothing still reads the conv input buffer)
          esync();
          prep_body<__nv_bfloat16>(P.dev, tk.y, et, CK_EPI, P.sched, P.horizon, P.adim, P.xin, P.x_pitch,
                                   P.ring_slot_stride, P.ring_agent_stride, r0 + it + 1);
          fence_proxy_async();
          esync();
          if (et == 0) {
            __threadfence();
            atomicAdd(prep_done, 1);
          }
        }
        if (P.trace && et == 0) CK_TR(11);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();                       // no CTA leaves while peers may still touch its smem
  if (P.trace && threadIdx.x == 0) P.trace[16 * CL * (int64_t)P.n_tasks + 2 * blockIdx.x + 1] = ck_time();
  if (warp == CK_MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CK_TMEM_COLS));
}

// ---------------------------------------------------------------- host side

static int pow2_ceil(int x) {
  int p = 1;
  while (p < x) p *= 2;
  return p;
}

static bool same_buf(const void *a, const void *b) { return a != nullptr && a == b; }

template <int BN>
static int cluster_capacity_t() {
  // per device: the smem attribute is set on, and the occupancy queried for, the current device
  static int cached[64];
  static bool init = false;
  if (!init) { for (int &c : cached) c = -1; init = true; }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) { cudaGetLastError(); return 0; }
  if (cached[dev] >= 0) return cached[dev];
  if (ensure_smem_attr(unet_cluster<BN>, (int)ClLay<BN>::SMEM) != AURAS_OK) {
    cudaGetLastError();
    return cached[dev] = 0;
  }
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(CL * 16);
  cfg.blockDim = dim3(CK_THREADS);
  cfg.dynamicSmemBytes = ClLay<BN>::SMEM;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = CL;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, unet_cluster<BN>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  return cached[dev] = n;
}

static int cluster_capacity(int bn_var) { return bn_var == 128 ? cluster_capacity_t<128>() : cluster_capacity_t<64>(); }

static BlockedBuf *find_blocked(ClConfig &cc, const void *orig) {
  for (auto &b : cc.blocked)
    if (b.orig == orig) return &b;
  return nullptr;
}

// 5-D view of a channel-blocked activation buffer: {64 channels, phase (the
// conv stride), time / stride, sample, channel block}; box {64, 1, Wo, s_box, 1}.
static int make_act_map_blocked(CUtensorMap *tm, const void *base, int Cin, int T, int stride, int S, int64_t plane,
                                int Wo, int s_box) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return AURAS_E_CUDA; }
  cuuint64_t dims[5] = {64, (cuuint64_t)stride, (cuuint64_t)(T / stride), (cuuint64_t)S, (cuuint64_t)(Cin / 64)};
  cuuint64_t strides[4] = {128, (cuuint64_t)128 * stride, (cuuint64_t)128 * T, (cuuint64_t)plane * 2};
  cuuint32_t box[5] = {64, 1, (cuuint32_t)Wo, (cuuint32_t)s_box, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("blocked activation map: CUresult %d", (int)r); return AURAS_E_CUDA; }
  return AURAS_OK;
}

int clus_build(ClConfig &cc, const std::vector<auras_conv_op> &ops, int S, const void *x_in,
               const ClParams &base, const float *film_tau, int film_width, const float *ring_film,
               TiledCache &cache) {
  const int n = (int)ops.size();
  const int bn_var = cc.bn_var == 128 ? 128 : 64;
  cc.bn_var = bn_var;
  int nc = std::min(cluster_capacity(bn_var), 16);
  if (const char *e = getenv("AURAS_CLUSTERS")) nc = std::min(nc, atoi(e));
  nc &= ~1;                                   // GroupNorm pairs need an even cluster count
  if (nc < 2) { set_error("cluster kernel: only %d co-resident 8-CTA clusters", nc); return AURAS_E_ARG; }
  // columns per tile task: narrower tiles mean less DSMEM traffic per CTA and
  // more clusters per layer, at the cost of re-streaming weights per n-tile
  int bn_cap = bn_var;
  if (const char *e = getenv("AURAS_CL_BN")) bn_cap = std::max(16, std::min(bn_var, atoi(e)));
  const char *de = getenv("AURAS_CL_DUAL");
  const bool dual = de ? atoi(de) != 0 : true;
  std::vector<ClOp> hops(n);
  int n_flags = 0;
  for (int i = 0; i < n; ++i) {
    const auras_conv_op &o = ops[i];
    ClOp &m = hops[i];
    memset(&m, 0, sizeof(m));
    ConvGemmArgs g;
    EpiArgs e;
    int rc = conv_op_to_args(o, S, AURAS_DT_BF16, nullptr, g, e);
    if (rc) return rc;
    if (!gemm_sm100_supported(g) || o.Ho != 1 || o.pool_out) {
      set_error("cluster kernel: op %d not a 1-D tcgen05 conv", i);
      return AURAS_E_ARG;
    }
    if (o.Wo > 32 || o.Wo < 2 || (o.Wo & (o.Wo - 1)) || o.M % 8) {
      set_error("cluster kernel: op %d shape", i);
      return AURAS_E_ARG;
    }
    if (o.out && (o.out_pitch % 8 || o.out_coff % 8)) { set_error("cluster kernel: op %d out align", i); return AURAS_E_ARG; }
    if (o.res && (o.res_pitch % 8 || o.res_coff % 8)) { set_error("cluster kernel: op %d res align", i); return AURAS_E_ARG; }
    m.gn = o.gn_gamma != nullptr;
    m.cg = m.gn ? o.M / o.groups : 0;
    if (m.gn && (o.M % o.groups || m.cg % 8 || (m.cg <= 128 ? 128 % m.cg : m.cg != 256))) {
      set_error("cluster kernel: op %d GroupNorm of %d channels", i, m.cg);
      return AURAS_E_ARG;
    }
    m.M = o.M; m.Cin = o.Cin; m.Wo = o.Wo; m.stride = o.stride; m.pad = o.pad_w;
    m.m_tiles = (o.M + 127) / 128;
    // two m-tiles per task when the layer has more tiles than there are clusters
    // (16 tiles of a 2048-channel layer on 14 clusters would take two rounds) or
    // a GroupNorm group spans two tiles (its statistics then stay in-cluster)
    m.nmt = (dual && m.m_tiles % 2 == 0 && (m.m_tiles > nc || m.cg == 256)) ? 2 : 1;
    m.pair = m.gn && m.cg == 256 && m.nmt == 1;
    const int cap = m.nmt == 2 ? bn_cap / 2 : bn_cap;
    {
      // samples per column tile: as few tiles as the width allows, each padded up to a
      // power of two (the TMA box zero-fills samples past S; the epilogue skips them),
      // so e.g. S = 5..7 stream each layer's weights once, like S = 8
      const int smax = std::min(CK_SMAX, std::max(1, cap / o.Wo));
      const int ntl = (S + smax - 1) / smax;
      m.s_box = std::min(smax, pow2_ceil((S + ntl - 1) / ntl));
    }
    m.rows = m.s_box * o.Wo;
    m.bn = std::max(16, m.rows);
    if (m.nmt == 2 && (m.bn > bn_var / 2 || 4 * m.s_box > 64)) {
      set_error("cluster kernel: op %d dual tile", i);
      return AURAS_E_ARG;
    }
    {
      const int lLh = std::min(5, 8 - (int)std::log2((double)m.s_box) - m.nmt);
      if ((1 << lLh) < o.Wo || (bn_var == 64 && (1 << lLh) < 2 * o.Wo)) {
        set_error("cluster kernel: op %d epilogue lanes", i);
        return AURAS_E_ARG;
      }
    }
    m.rsh = m.bn + 8;
    m.kb_total = o.Kp / 64;
    m.kps = (m.kb_total + CL - 1) / CL;
    const int n_tiles = (S + m.s_box - 1) / m.s_box;
    m.tiles = (m.m_tiles / m.nmt) * n_tiles;
    if (m.pair && (m.m_tiles & 1)) { set_error("cluster kernel: op %d odd tile pair", i); return AURAS_E_ARG; }
    auto lg = [](int x) { int l = 0; while ((1 << l) < x) ++l; return l; };
    m.lwo = lg(m.Wo);
    m.lbn = lg(m.bn);
    m.lsb = lg(m.s_box);
    m.lcg = m.gn ? lg(m.cg) : 0;
    if (m.gn && (1 << m.lcg) != m.cg) { set_error("cluster kernel: op %d group size", i); return AURAS_E_ARG; }
    m.bstage = m.bn * 128;
    m.nbst = std::min(CK_NBMAX, CK_BRING / m.bstage);
    m.epi = e;
    if (o.film_off >= 0) {
      m.epi.film_a = film_tau;
      m.epi.film_a_row = base.dev->tau_row;
      m.epi.film_a_stride = film_width;
      m.epi.film_b = ring_film;
      m.epi.film_b_off = base.dev->film_b_off;
    }
    if (m.pair) {
      m.flag_base = n_flags;
      n_flags += m.tiles;
    }
    void *wt = nullptr;
    if ((rc = tiled_weights(cache, o, &wt, m.nmt))) return rc;
    m.wt = static_cast<const uint8_t *>(wt);
    if ((rc = make_tiled_weight_map(&m.tmA, wt, m.m_tiles * m.kb_total * 128, 256))) return rc;
    if ((rc = make_tiled_weight_map(&m.tmA1, wt, m.m_tiles * m.kb_total * 128, 128))) return rc;
    // ---- activation buffers: every tensor a later op reads through TMA is re-laid
    //      out channel-blocked, [C/64][S][T][64], so an im2col box row run is
    //      contiguous (TMA serves strided 128-byte rows at ~17 GB/s per SM)
    if (o.in_coff % 64 || o.out_coff % 64 || o.res_coff % 64 || o.Cin % 64) {
      set_error("cluster kernel: op %d channel offsets not 64-aligned", i);
      return AURAS_E_ARG;
    }
    const __nv_bfloat16 *in_base;
    int64_t in_plane;
    int in_T;
    if (o.in == x_in) {                         // the prep's [S][T][64] input is already blocked (C = 64)
      if (o.in_pitch != 64 || o.in_coff) { set_error("cluster kernel: x buffer pitch"); return AURAS_E_ARG; }
      in_base = static_cast<const __nv_bfloat16 *>(o.in);
      in_T = o.W;
      in_plane = (int64_t)S * in_T * 64;
    } else {
      const BlockedBuf *b = find_blocked(cc, o.in);
      if (!b || b->T != o.W) { set_error("cluster kernel: op %d input not produced in-kernel", i); return AURAS_E_ARG; }
      in_base = b->ptr + (o.in_coff >> 6) * b->plane;
      in_plane = b->plane;
      in_T = b->T;
    }
    if ((rc = make_act_map_blocked(&m.tmB, in_base, o.Cin, in_T, o.stride, S, in_plane, o.Wo, m.s_box))) return rc;
    if (o.out) {
      if (i == n - 1) {                         // read by the final 1x1 conv: keep the plan's layout
        m.out_base = static_cast<__nv_bfloat16 *>(o.out) + o.out_coff;
        m.out_plane = 64;
        m.out_row = o.out_pitch;
        m.out_T = o.out_stuff ? 2 * o.Wo : o.Wo;
      } else {
        const int T = o.out_stuff ? 2 * o.Wo : o.Wo;
        BlockedBuf *b = find_blocked(cc, o.out);
        if (!b) {
          BlockedBuf nb;
          nb.orig = o.out;
          nb.T = T;
          nb.plane = (int64_t)S * T * 64;
          const size_t bytes = (size_t)(o.out_pitch / 64) * nb.plane * 2;
          AURAS_CUDA(cudaMalloc(&nb.ptr, bytes));
          AURAS_CUDA(cudaMemset(nb.ptr, 0, bytes));
          cc.blocked.push_back(nb);
          b = &cc.blocked.back();
        }
        if (b->T != T) { set_error("cluster kernel: op %d output length", i); return AURAS_E_ARG; }
        m.out_base = b->ptr + (o.out_coff >> 6) * b->plane;
        m.out_plane = b->plane;
        m.out_row = 64;
        m.out_T = T;
      }
    }
    if (o.res) {
      const BlockedBuf *b = find_blocked(cc, o.res);
      if (!b) { set_error("cluster kernel: op %d residual not produced in-kernel", i); return AURAS_E_ARG; }
      m.res_base = b->ptr + (o.res_coff >> 6) * b->plane;
      m.res_plane = b->plane;
      m.res_row = 64;
      m.res_T = b->T;
    }
    for (int d = 0; d < 3; ++d) m.gemm_dep[d] = -1;
    for (int d = 0; d < 2; ++d) m.epi_dep[d] = -1;
    int nd = 0;
    if (o.in == x_in) m.gemm_dep[nd++] = -2;
    for (int j = i - 1; j >= 0 && nd < 3; --j)
      if (same_buf(ops[j].out, o.in)) m.gemm_dep[nd++] = j;
    int ne = 0;
    for (int j = i - 1; j >= 0 && ne < 2; --j)
      if (same_buf(ops[j].out, o.res) || same_buf(ops[j].out_f32, o.res_f32)) m.epi_dep[ne++] = j;
    if (o.res && o.res == x_in) { set_error("cluster kernel: residual from the x buffer"); return AURAS_E_ARG; }
    for (int d = 0; d < 3; ++d) m.gemm_tgt[d] = m.gemm_dep[d] >= 0 ? hops[m.gemm_dep[d]].tiles * CL : 0;
    for (int d = 0; d < 2; ++d) m.epi_tgt[d] = m.epi_dep[d] >= 0 ? hops[m.epi_dep[d]].tiles * CL : 0;
  }
  // per-cluster task lists, layer order
  std::vector<std::vector<int4>> per(nc);
  for (int s = 0; s < S; ++s) per[s % nc].push_back(make_int4(K_PREP, s, 0, (s / nc) % CL));
  int rot = 0;
  for (int i = 0; i < n; ++i) {
    const ClOp &m = hops[i];
    if (m.pair && (rot & 1)) rot = (rot + 1) % nc;     // pairs land on clusters (2c, 2c+1) in one round
    const int groups = m.m_tiles / m.nmt, n_tiles = m.tiles / groups;
    int q = 0;
    for (int nt = 0; nt < n_tiles; ++nt)
      for (int mg = 0; mg < groups; ++mg, ++q) per[(rot + q) % nc].push_back(make_int4(K_GEMM | (i << 8), mg, nt, 0));
    rot = (rot + q) % nc;
  }
  for (int s = 0; s < S; ++s) per[(rot + s) % nc].push_back(make_int4(K_FINAL, s, 0, (s / nc) % CL));
  // The activation ring is re-cut per op (stage = bn x 128 B).  A task whose op
  // does not depend on the cluster's previous task could load its activations
  // while that task's UMMAs still read overlapping stages of the old cut, so a
  // cut change is only allowed across a dependency (always true for the UNets
  // built here; other shapes fall back to the L2 megakernel).
  {
    std::vector<std::vector<char>> dep(n, std::vector<char>(n, 0));   // dep[i][j]: op i waits (transitively) on op j
    for (int i = 0; i < n; ++i) {
      for (int d = 0; d < 3; ++d)
        if (hops[i].gemm_dep[d] >= 0) dep[i][hops[i].gemm_dep[d]] = 1;
      for (int d = 0; d < 2; ++d)
        if (hops[i].epi_dep[d] >= 0) dep[i][hops[i].epi_dep[d]] = 1;
      for (int j = 0; j < i; ++j)
        if (dep[i][j])
          for (int k = 0; k < j; ++k)
            if (dep[j][k]) dep[i][k] = 1;
    }
    for (int c = 0; c < nc; ++c) {
      int prev = -1;
      for (const int4 &tk : per[c]) {
        if ((tk.x & 0xff) != K_GEMM) continue;
        const int cur = tk.x >> 8;
        if (prev >= 0 && cur != prev && hops[cur].bstage != hops[prev].bstage && !(cur > prev && dep[cur][prev])) {
          set_error("cluster kernel: ops %d -> %d change the activation ring cut without a dependency", prev, cur);
          return AURAS_E_ARG;
        }
        prev = cur;
      }
    }
  }
  std::vector<int4> flat;
  std::vector<int> begin(nc + 1, 0);
  for (int c = 0; c < nc; ++c) {
    begin[c] = (int)flat.size();
    flat.insert(flat.end(), per[c].begin(), per[c].end());
  }
  begin[nc] = (int)flat.size();

  AURAS_CUDA(cudaMalloc(&cc.ops, sizeof(ClOp) * n));
  AURAS_CUDA(cudaMalloc(&cc.tasks, sizeof(int4) * flat.size()));
  AURAS_CUDA(cudaMalloc(&cc.cl_begin, sizeof(int) * (nc + 1)));
  cc.ctr_ints = n + 1 + std::max(1, n_flags) + 1;   // ... + the sticky error word (last)
  AURAS_CUDA(cudaMalloc(&cc.ctr, sizeof(int) * cc.ctr_ints));
  AURAS_CUDA(cudaMemset(cc.ctr, 0, sizeof(int) * cc.ctr_ints));
  AURAS_CUDA(cudaMalloc(&cc.gstats, sizeof(float2) * 16 * CK_SMAX * std::max(1, n_flags)));
  AURAS_CUDA(cudaMemcpy(cc.ops, hops.data(), sizeof(ClOp) * n, cudaMemcpyHostToDevice));
  AURAS_CUDA(cudaMemcpy(cc.tasks, flat.data(), sizeof(int4) * flat.size(), cudaMemcpyHostToDevice));
  AURAS_CUDA(cudaMemcpy(cc.cl_begin, begin.data(), sizeof(int) * (nc + 1), cudaMemcpyHostToDevice));
  cc.n_ops = n;
  cc.n_tasks = (int)flat.size();
  cc.nc = nc;
  cc.S = S;
  cc.params = base;
  cc.params.ops = cc.ops;
  cc.params.tasks = cc.tasks;
  cc.params.cl_begin = cc.cl_begin;
  cc.params.ctr = cc.ctr;
  cc.params.flags = cc.ctr + n + 1;
  cc.params.err = cc.ctr + cc.ctr_ints - 1;
  cc.params.gstats = cc.gstats;
  cc.params.n_ops = n;
  cc.params.S = S;
  cc.params.nc = nc;
  cc.params.n_tasks = cc.n_tasks;
  {
    const char *e = getenv("AURAS_CL_L2PF");
    cc.params.l2_prefetch = e ? atoi(e) : 0;
    e = getenv("AURAS_CL_HACK");        // timing experiments only: 1 = skip activation boxes, 2 = skip weights
    cc.params.hack = e ? atoi(e) : 0;
    e = getenv("AURAS_SPIN_TIMEOUT_MS");
    cc.params.spin_timeout_ns = (long long)((e ? atof(e) : 2000.0) * 1e6);
    e = getenv("AURAS_SPIN_MODE");
    cc.params.spin_mode = e ? atoi(e) : 0;
    e = getenv("AURAS_FAULT_STALL");    // tests: every layer dependency becomes unreachable
    cc.params.fault = e ? atoi(e) : 0;
  }
  return AURAS_OK;
}

int clus_launch(const ClConfig &cc, cudaStream_t st) {
  // counters and pair flags restart every launch; the error word (last int) is
  // sticky until the host reads it (clus_error)
  AURAS_CUDA(cudaMemsetAsync(cc.ctr, 0, sizeof(int) * (cc.ctr_ints - 1), st));
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(CL * cc.nc);
  cfg.blockDim = dim3(CK_THREADS);
  cfg.dynamicSmemBytes = cc.bn_var == 128 ? ClLay<128>::SMEM : ClLay<64>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = CL;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  if (cc.bn_var == 128) {
    if (int rc = ensure_smem_attr(unet_cluster<128>, (int)ClLay<128>::SMEM)) return rc;
    AURAS_CUDA(cudaLaunchKernelEx(&cfg, unet_cluster<128>, cc.params));
  } else {
    if (int rc = ensure_smem_attr(unet_cluster<64>, (int)ClLay<64>::SMEM)) return rc;
    AURAS_CUDA(cudaLaunchKernelEx(&cfg, unet_cluster<64>, cc.params));
  }
  return AURAS_OK;
}

// Reads and clears the kernel's error word (1: a dependency wait timed out).
// Synchronous: call where the host already waits on the generation stream.
int clus_error(const ClConfig &cc) {
  if (!cc.ctr) return 0;
  int v = 0;
  if (cudaMemcpy(&v, cc.ctr + cc.ctr_ints - 1, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  if (v) cudaMemset(cc.ctr + cc.ctr_ints - 1, 0, sizeof(int));
  return v;
}

int clus_set_trace(ClConfig &cc, long long *trace) {
  cc.params.trace = trace;
  return AURAS_OK;
}

void clus_free(ClConfig &cc) {
  for (auto &b : cc.blocked) cudaFree(b.ptr);
  cudaFree(cc.ops);
  cudaFree(cc.tasks);
  cudaFree(cc.cl_begin);
  cudaFree(cc.ctr);
  cudaFree(cc.gstats);
  cc = ClConfig();
}

}  // namespace auras
