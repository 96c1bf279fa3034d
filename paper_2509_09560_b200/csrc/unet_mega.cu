// Persistent dataflow megakernel: ONE launch runs a whole denoise step of the
// ConditionalUnet1D for all S in-flight samples.
//
// Why: layer by layer, every conv costs a GEMM launch plus an epilogue launch
// of 5-14 us each, dominated by prologue / pipeline fill, while its weights need
// 0.4-6.5 us of HBM time.  Here every CTA (one per SM) walks a static task list
// (built on the host, ordered by layer) with warp-specialised roles:
//
//   warp 0  A producer : TMA-streams weight tiles of ALL its upcoming GEMM tasks
//                        into an 8-stage ring, never waiting on activations --
//                        weights do not depend on the previous layer, so the
//                        HBM stream runs ahead across layer boundaries;
//   warp 2  B producer : per GEMM task, waits (acquire) on the completion
//                        counters of the layers producing its input, then TMAs
//                        the implicit-im2col activation tiles;
//   warp 1  MMA        : one elected lane issues tcgen05.mma (M=128, N<=128,
//                        K=16) into a double-buffered TMEM accumulator;
//   warps 4-7          : drain TMEM into fp32 split-K partials and signal the
//                        layer's GEMM counter; run the fused epilogue units
//                        (split reduce + bias + GroupNorm + Mish + FiLM +
//                        residual, deterministic order) once a layer's GEMMs
//                        are all done; run the per-sample prep (x_t, timestep,
//                        ring slot) and final (1x1 conv + DDPM/DDIM update).
//
// Dependencies are global int counters (release: fence + atomicAdd; acquire:
// ld.acquire spin), with fence.proxy.async between generic epilogue stores and
// the TMA reads of the next layer.  Deadlock freedom: each CTA processes its
// list in layer order and a task only waits on tasks of strictly earlier
// layers; the grid is one CTA per SM so all CTAs are co-resident.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "epi.cuh"
#include "tc_util.cuh"
#include "unet.cuh"
#include "mega.cuh"

namespace auras {

constexpr int MK_THREADS = 384;              // 4 role warps + 8 epilogue warps
constexpr int MK_EPI = 256;                  // epilogue-unit threads (warps 4-11)
constexpr int MK_KS = 2;                 // k-blocks (64 wide) per pipeline stage
constexpr int MK_NA = 5;                 // max weight stages (2 x 16 KB each); runtime P.na <= MK_NA
constexpr int MK_BN = 256;               // max N per GEMM task (TMEM: 2 buffers x 256 columns)
constexpr int MK_A_BYTES = 128 * 64 * 2;         // one 128 x 64 weight box
constexpr int MK_A_STAGE = MK_KS * MK_A_BYTES;
// smem holds the weight ring (P.na stages) followed by the activation ring
// (P.bring bytes, carved per task into stages of KS * round_up(bn*128, 1KB)):
// 160 KB / 48 KB for batches of <= 128 columns, 128 KB / 96 KB beyond.
constexpr int MK_RINGS = 208 * 1024;
constexpr int MK_NBMAX = 12;
constexpr size_t MK_SMEM = 1024 + (size_t)MK_RINGS + 1024 + 4 * 600;

enum { T_GEMM = 0, T_EPI = 1, T_PREP = 2, T_FINAL = 3 };

struct alignas(64) MegaOp {
  CUtensorMap tmA;
  CUtensorMap tmB;
  EpiArgs epi;
  int M, N, Cin, Wo, stride, pad, S, s_box, rows, bn, kb_total, kb_per_split, splits, gemm_tasks, epi_units;
  int bstage, nbst;         // activation-ring stage bytes and stage count for this op
  int gemm_dep[3];          // -1 none, -2 prep
  int epi_dep[2];
};

__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void spin_ns(const int *ctr, int target, int ns) {
  while (ld_acquire_i32(ctr) < target) {
    if (ns) __nanosleep(ns);
  }
}

__device__ __forceinline__ void wait_dep(const MegaParams &P, int *epi_done, int *prep_done, int d) {
  if (d == -2) spin_ns(prep_done, P.S, P.spin_ns);
  else if (d >= 0) spin_ns(&epi_done[d], P.ops[d].epi_units, P.spin_ns);
}

__global__ void __launch_bounds__(MK_THREADS, 1) unet_mega(const __grid_constant__ MegaParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;
  const int NA = P.na;
  uint8_t *sB = sA + NA * MK_A_STAGE;
  uint64_t *fullA = reinterpret_cast<uint64_t *>(sA + MK_RINGS);
  uint64_t *emptyA = fullA + MK_NA;
  uint64_t *fullB = emptyA + MK_NA;
  uint64_t *emptyB = fullB + MK_NBMAX;
  uint64_t *tfull = emptyB + MK_NBMAX;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
  float *red = reinterpret_cast<float *>(tmem_slot + 8);
  float *eps = red + 32;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = P.cta_begin[blockIdx.x], t1 = P.cta_begin[blockIdx.x + 1];
  int *gemm_done = P.ctr;
  int *epi_done = P.ctr + P.n_ops;
  int *prep_done = P.ctr + 2 * P.n_ops;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NA; ++i) { mbar_init(&fullA[i], 1); mbar_init(&emptyA[i], 1); }
    for (int i = 0; i < MK_NBMAX; ++i) { mbar_init(&fullB[i], 1); mbar_init(&emptyB[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * MK_BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ A producer: weights, never blocked on data
    // (warp-uniform loop; one lane elected inside the PTX)
    int ia = 0;
    for (int t = t0; t < t1; ++t) {
      const int4 tk = P.tasks[t];
      if ((tk.x & 0xff) != T_GEMM) continue;
      const MegaOp *op = &P.ops[tk.x >> 8];
      const int kps = op->kb_per_split, kbt = op->kb_total;     // snapshot: no reloads in the loop
      const CUtensorMap *tmA = &op->tmA;
      const int kb0 = tk.w * kps, kb1 = min(kbt, kb0 + kps);
      const int row0 = tk.y * kbt * 128;          // tiled layout [m_tile][k_block][128][64]
      for (int kb = kb0; kb < kb1; kb += MK_KS, ++ia) {
        const int st = ia % NA;
        const int two = kb + 1 < kb1;
        mbar_wait(&emptyA[st], ((ia / NA) & 1) ^ 1);
        if (P.a_depth < NA && ia >= P.a_depth)           // optional cap on weights in flight
          mbar_wait(&emptyA[(ia - P.a_depth) % NA], (((ia - P.a_depth) / NA) & 1));
        tma_load_2d_pair_warp(sA + st * MK_A_STAGE, tmA, &fullA[st], (1 + two) * MK_A_BYTES, 0, row0 + kb * 128,
                              row0 + (kb + 1) * 128, two);
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------ B producer: activations, after dependencies
    uint32_t par = 0;                 // per-slot use parity of the activation ring
    for (int t = t0; t < t1; ++t) {
      const int4 tk = P.tasks[t];
      if ((tk.x & 0xff) != T_GEMM) continue;
      const MegaOp *op = &P.ops[tk.x >> 8];
      const int bstage = op->bstage, nbst = op->nbst;
      const int dep0 = op->gemm_dep[0], dep1 = op->gemm_dep[1], dep2 = op->gemm_dep[2];
      const int kps = op->kb_per_split, kbt = op->kb_total, Cin = op->Cin, pad = op->pad;
      const int stride = op->stride, sbox = op->s_box;
      const uint32_t bbytes = op->rows * 128;
      const CUtensorMap *tmB = &op->tmB;
      if (lane == 0) {
        wait_dep(P, epi_done, prep_done, dep0);
        wait_dep(P, epi_done, prep_done, dep1);
        wait_dep(P, epi_done, prep_done, dep2);
        fence_proxy_async();
        if (P.trace) P.trace[8 * t + 0] = gtime();
      }
      __syncwarp();
      const int kb0 = tk.w * kps, kb1 = min(kbt, kb0 + kps);
      for (int kb = kb0; kb < kb1; kb += MK_KS) {
        const int st = ((kb - kb0) / MK_KS) % nbst;
        const int nk = min(MK_KS, kb1 - kb);
        mbar_wait(&emptyB[st], ((par >> st) & 1) ^ 1);
        par ^= 1u << st;
        mbar_expect_tx_warp(&fullB[st], nk * bbytes);
        for (int i = 0; i < nk; ++i) {
          const int k = (kb + i) * 64;
          const int tap = k / Cin, c0 = k - tap * Cin;
          const int off = tap - pad;
          const int q = off >= 0 ? off / stride : -((-off + stride - 1) / stride);
          const int h = off - q * stride;
          tma_4d_warp(sB + st * MK_KS * bstage + i * bstage, tmB, &fullB[st], c0, h, q, tk.z * sbox);
        }
      }
      if (lane == 0 && P.trace) P.trace[8 * t + 1] = gtime();
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    int ia = 0, gi = 0;
    uint32_t par = 0;
    for (int t = t0; t < t1; ++t) {
      const int4 tk = P.tasks[t];
      if ((tk.x & 0xff) != T_GEMM) continue;
      const MegaOp *op = &P.ops[tk.x >> 8];
      const int kps = op->kb_per_split, kbt = op->kb_total, bn = op->bn;
      const int bstage = op->bstage, nbst = op->nbst;
      const int buf = gi & 1;
      mbar_wait(&tempty[buf], ((gi >> 1) & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t idesc = umma_idesc(bn);
      const uint32_t dt = tmem + buf * MK_BN;
      const int kb0 = tk.w * kps, kb1 = min(kbt, kb0 + kps);
      if (P.trace && lane == 0) P.trace[8 * t + 4] = gtime();
      for (int kb = kb0; kb < kb1; kb += MK_KS, ++ia) {
        const int sa = ia % NA, sb = ((kb - kb0) / MK_KS) % nbst;
        const int nk = min(MK_KS, kb1 - kb);
        mbar_wait(&fullA[sa], (ia / NA) & 1);
        if (P.trace && lane == 0 && kb == kb0) P.trace[8 * t + 5] = gtime();
        long long *kt = (P.kbtrace && ia < 1024) ? P.kbtrace + ((int64_t)blockIdx.x * 1024 + ia) * 3 : nullptr;
        if (kt && lane == 0) kt[0] = gtime();
        mbar_wait(&fullB[sb], (par >> sb) & 1);
        if (kt && lane == 0) kt[1] = gtime();
        par ^= 1u << sb;
        if (P.trace && lane == 0 && kb == kb0) P.trace[8 * t + 6] = gtime();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int i = 0; i < nk; ++i) {
          const uint32_t a0 = smem_u32(sA + sa * MK_A_STAGE + i * MK_A_BYTES);
          const uint32_t b0 = smem_u32(sB + sb * MK_KS * bstage + i * bstage);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16_warp(dt, umma_desc(a0 + kk * 32), umma_desc(b0 + kk * 32), idesc,
                           (kb > kb0 || i > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit_warp(&emptyA[sa]);
        umma_commit_warp(&emptyB[sb]);
        if (kt && lane == 0) kt[2] = gtime();
        __syncwarp();
      }
      umma_commit_warp(&tfull[buf]);
      if (lane == 0 && P.trace) P.trace[8 * t + 7] = gtime();
      __syncwarp();
      ++gi;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue warps: 4-7 drain TMEM, 4-11 run units
    const int et = threadIdx.x - 128;
    const int ew = warp - 4;
    const bool drainer = ew < 4;
    auto dsync = [] __device__() { named_sync(1, 128); };
    auto sync = [] __device__() { named_sync(2, MK_EPI); };
    int gi = 0;
    for (int t = t0; t < t1; ++t) {
      const int4 tk = P.tasks[t];
      const int type = tk.x & 0xff, opi = tk.x >> 8;
      if (type == T_GEMM) {
        if (!drainer) continue;
        const MegaOp *op = &P.ops[opi];
        const int oM = op->M, oN = op->N, oWo = op->Wo, orows = op->rows, oS = op->S, osbox = op->s_box;
        const int obn = op->bn;
        float *opart = op->epi.partial;
        const int buf = gi & 1;
        mbar_wait(&tfull[buf], (gi >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (P.trace && et == 0) P.trace[8 * t + 2] = gtime();
        const int m = tk.y * 128 + ew * 32 + lane;
        const int s0 = tk.z * osbox;
        const int nvalid = min(orows, (oS - s0) * oWo);
        float *out = opart + (int64_t)tk.w * oN * oM + (int64_t)m * oN + (int64_t)s0 * oWo;   // [split][m][n]
        for (int c = 0; c < obn; c += 16) {
          float v[16];
          tmem_ld16(tmem + buf * MK_BN + c + ((uint32_t)(ew * 32) << 16), v);
          if (m < oM) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              if (c + j < nvalid)
                *reinterpret_cast<float4 *>(out + c + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        dsync();
        if (et == 0) {                              // one fence after the barrier releases the CTA's stores
          __threadfence();
          atomicAdd(&gemm_done[opi], 1);
          if (P.trace) P.trace[8 * t + 3] = gtime();
        }
        ++gi;
      } else if (type == T_EPI) {
        const MegaOp *op = &P.ops[opi];
        const EpiArgs e = op->epi;                  // by value: registers, no reloads after fences
        const int need = op->gemm_tasks, d0 = op->epi_dep[0], d1 = op->epi_dep[1];
        if (et == 0) {                              // residual producers + per-sample FiLM rows
          spin_ns(prep_done, P.S, P.spin_ns);
          wait_dep(P, epi_done, prep_done, d0);
          wait_dep(P, epi_done, prep_done, d1);
        }
        sync();
        auto gate = [&] __device__() {              // this layer's GEMM partials
          if (et == 0) spin_ns(&gemm_done[opi], need, P.spin_ns);
          sync();
          if (P.trace && et == 0) P.trace[8 * t + 0] = gtime();
        };
        if (epi_fits_regs(e, tk.z, MK_EPI)) {
          long long st3[3] = {0, 0, 0};
          epi_unit_regs<__nv_bfloat16>(e, tk.y, tk.z, et, MK_EPI, red, sync, gate, P.trace ? st3 : nullptr);
          if (P.trace && et == 0) {
            P.trace[8 * t + 2] = st3[0];
            P.trace[8 * t + 3] = st3[1];
            P.trace[8 * t + 4] = st3[2];
          }
        } else {
          gate();
          epi_unit<__nv_bfloat16>(e, tk.y, tk.z, et, MK_EPI, red, sync);
        }
        fence_proxy_async();
        sync();
        if (et == 0) {
          __threadfence();
          atomicAdd(&epi_done[opi], 1);
          if (P.trace) P.trace[8 * t + 1] = gtime();
        }
      } else if (type == T_PREP) {
        prep_body<__nv_bfloat16>(P.dev, tk.y, et, MK_EPI, P.sched, P.horizon, P.adim, P.xin, P.x_pitch,
                                 P.ring_slot_stride, P.ring_agent_stride);
        fence_proxy_async();
        sync();
        if (et == 0) {
          __threadfence();
          atomicAdd(prep_done, 1);
        }
      } else if (type == T_FINAL) {
        if (et == 0) spin_ns(&epi_done[P.n_ops - 1], P.ops[P.n_ops - 1].epi_units, P.spin_ns);
        sync();
        final_body<__nv_bfloat16>(P.dev, tk.y, et, MK_EPI, P.sched, P.horizon, P.adim, P.y_final, P.y_pitch,
                                  P.final_cin, P.wf, P.bf, eps, sync);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * MK_BN));
}

// ---------------------------------------------------------------- host side

// Weights re-laid out as [m_tile][k_block][128 rows][64] so that every 16 KB
// TMA box -- and a task's whole run of k-blocks -- is contiguous in HBM.
__global__ void tile_weights_kernel(const __nv_bfloat16 *__restrict__ src, __nv_bfloat16 *__restrict__ dst, int M,
                                    int Kp, int m_tiles, int nmt) {
  const int KB = Kp / 64;
  const int64_t total = (int64_t)m_tiles * KB * 128 * 8;     // 16-byte chunks
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int chunk = i & 7;
    const int64_t rowi = i >> 3;
    const int r = rowi & 127;
    int64_t tile = rowi >> 7;
    if (nmt == 2) {                     // pairs of m-tiles interleaved per k-block: [pair][kb][2][128][64]
      const int u = tile & 1;
      const int64_t q = tile >> 1;
      tile = ((q / KB) * 2 + u) * KB + q % KB;
    }
    const int kb = tile % KB, mt = tile / KB;
    const int m = mt * 128 + r;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (m < M) v = *reinterpret_cast<const uint4 *>(src + (int64_t)m * Kp + kb * 64 + chunk * 8);
    *reinterpret_cast<uint4 *>(dst + rowi * 64 + chunk * 8) = v;
  }
}

int make_tiled_weight_map(CUtensorMap *tm, const void *wt, int rows_total, int box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return AURAS_E_CUDA; }
  cuuint64_t dims[2] = {64, (cuuint64_t)rows_total};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(wt), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("tiled weight map: CUresult %d", (int)r); return AURAS_E_CUDA; }
  return AURAS_OK;
}

int tiled_weights(TiledCache &cache, const auras_conv_op &o, void **out, int nmt) {
  // the pair-interleaved copy of the same weights is a different entry (odd key)
  const void *key = nmt == 2 ? static_cast<const void *>(static_cast<const char *>(o.w) + 1) : o.w;
  for (auto &kv : cache)
    if (kv.first == key) { *out = kv.second; return AURAS_OK; }
  const int m_tiles = (o.M + 127) / 128;
  const size_t bytes = (size_t)m_tiles * o.Kp * 128 * 2;
  void *d = nullptr;
  AURAS_CUDA(cudaMalloc(&d, bytes));
  tile_weights_kernel<<<1184, 256>>>(static_cast<const __nv_bfloat16 *>(o.w), static_cast<__nv_bfloat16 *>(d), o.M,
                                     o.Kp, m_tiles, nmt);
  AURAS_LAUNCHED("tile_weights_kernel");
  AURAS_CUDA(cudaDeviceSynchronize());
  cache.emplace_back(key, d);
  *out = d;
  return AURAS_OK;
}

static bool same_buffer(const void *a, const void *b) { return a != nullptr && a == b; }

// Build the per-S task table.  `ops` are the plan's conv ops in execution order.
int mega_build(MegaConfig &mc, const std::vector<auras_conv_op> &ops, int S, const void *x_in, int x_pitch,
               const MegaParams &base, const float *film_tau, int film_width, const float *ring_film,
               TiledCache &cache) {
  const int n = (int)ops.size();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // leave a few SMs to the perception stream, which runs concurrently
  const char *rs = getenv("AURAS_MEGA_RESERVE");
  const int reserve = rs ? atoi(rs) : 8;
  sms = std::max(16, sms - std::max(0, reserve));
  // ring split: wide batches (> 128 columns per task) trade weight prefetch for activation stages
  int rows_max = 0;
  for (const auto &o : ops) rows_max = std::max(rows_max, std::min(S, MK_BN / o.Wo) * o.Wo);
  const int bn_max = rows_max > 128 ? MK_BN : 128;
  const int na = bn_max > 128 ? 4 : MK_NA;
  const int bring = MK_RINGS - na * MK_A_STAGE;
  std::vector<MegaOp> hops(n);
  std::vector<int64_t> part_off(n);
  int64_t part_total = 0;
  for (int i = 0; i < n; ++i) {
    const auras_conv_op &o = ops[i];
    MegaOp &m = hops[i];
    memset(&m, 0, sizeof(m));
    ConvGemmArgs g;
    EpiArgs e;
    int rc = conv_op_to_args(o, S, AURAS_DT_BF16, nullptr, g, e);
    if (rc) return rc;
    if (!gemm_sm100_supported(g)) { set_error("megakernel: op %d not supported by the tcgen05 engine", i); return AURAS_E_ARG; }
    m.M = o.M; m.N = S * o.Wo; m.Cin = o.Cin; m.Wo = o.Wo; m.stride = o.stride; m.pad = o.pad_w; m.S = S;
    m.s_box = std::min(S, bn_max / o.Wo);
    m.rows = m.s_box * o.Wo;
    m.bn = (m.rows + 15) / 16 * 16;
    m.kb_total = o.Kp / 64;
    m.bstage = (m.bn * 128 + 1023) / 1024 * 1024;
    m.nbst = std::min(MK_NBMAX, bring / (MK_KS * m.bstage));
    if (m.nbst < 1) { set_error("megakernel: B stage too large"); return AURAS_E_ARG; }
    const int m_tiles = (o.M + 127) / 128, n_tiles = (S + m.s_box - 1) / m.s_box;
    // split-K: enough CTAs to stream big layers at full HBM rate, but at least
    // ~128 KB of weights per task so small layers do not drown in partials
    const int64_t wbytes = (int64_t)o.M * o.Kp * 2;
    int want = (int)std::max<int64_t>(1, wbytes / ((int64_t)m_tiles * n_tiles * 128 * 1024));
    want = std::min(want, std::max(1, sms / (m_tiles * n_tiles)));
    want = std::min(want, m.kb_total);
    m.kb_per_split = (m.kb_total + want - 1) / want;
    m.splits = (m.kb_total + m.kb_per_split - 1) / m.kb_per_split;
    m.gemm_tasks = m_tiles * n_tiles * m.splits;
    const bool gn = o.gn_gamma != nullptr;
    m.epi_units = S * (gn ? o.groups : (o.M + 63) / 64);
    m.epi = e;
    m.epi.splits = m.splits;
    if (o.film_off >= 0) {
      m.epi.film_a = film_tau;
      m.epi.film_a_row = base.dev->tau_row;          // device address arithmetic only
      m.epi.film_a_stride = film_width;
      m.epi.film_b = ring_film;
      m.epi.film_b_off = base.dev->film_b_off;
    }
    part_off[i] = part_total;
    part_total += (int64_t)m.splits * m.N * m.M;
    void *wt = nullptr;
    if ((rc = tiled_weights(cache, o, &wt))) return rc;
    if ((rc = make_tiled_weight_map(&m.tmA, wt, m_tiles * m.kb_total * 128))) return rc;
    if ((rc = make_act_map(&m.tmB, o.in, o.in_coff, o.Cin, o.in_pitch, o.W, o.stride, S, o.Wo, m.s_box))) return rc;
    // dependencies: producers of the input buffer (or the prep), of the residuals
    int nd = 0;
    for (int d = 0; d < 3; ++d) m.gemm_dep[d] = -1;
    for (int d = 0; d < 2; ++d) m.epi_dep[d] = -1;
    if (o.in == x_in) m.gemm_dep[nd++] = -2;
    for (int j = i - 1; j >= 0 && nd < 3; --j)
      if (same_buffer(ops[j].out, o.in)) m.gemm_dep[nd++] = j;
    int ne = 0;
    for (int j = i - 1; j >= 0 && ne < 2; --j) {
      if (same_buffer(ops[j].out, o.res) || same_buffer(ops[j].out_f32, o.res_f32)) m.epi_dep[ne++] = j;
    }
    if (o.res && o.res == x_in) { set_error("megakernel: residual from the x buffer"); return AURAS_E_ARG; }
  }
  // tasks, layer by layer, round-robin over CTAs
  std::vector<std::vector<int4>> per(sms);
  for (int s = 0; s < S; ++s) per[s % sms].push_back(make_int4(T_PREP, s, 0, 0));
  int rot = 0;
  for (int i = 0; i < n; ++i) {
    const MegaOp &m = hops[i];
    const int m_tiles = (m.M + 127) / 128, n_tiles = (S + m.s_box - 1) / m.s_box;
    int k = 0;
    for (int sp = 0; sp < m.splits; ++sp)
      for (int nt = 0; nt < n_tiles; ++nt)
        for (int mt = 0; mt < m_tiles; ++mt, ++k)
          per[(rot + k) % sms].push_back(make_int4(T_GEMM | (i << 8), mt, nt, sp));
    rot = (rot + k) % sms;
    const bool gn = ops[i].gn_gamma != nullptr;
    const int gy = gn ? ops[i].groups : (m.M + 63) / 64;
    int u = 0;
    const int units = S * gy;
    for (int s = 0; s < S; ++s)        // spread the units evenly over the grid (one per CTA when possible)
      for (int g = 0; g < gy; ++g, ++u)
        per[(rot + (int)((int64_t)u * sms / units)) % sms].push_back(make_int4(T_EPI | (i << 8), s, g, 0));
    rot = (rot + 1) % sms;
  }
  for (int s = 0; s < S; ++s) per[(rot + s) % sms].push_back(make_int4(T_FINAL, s, 0, 0));
  std::vector<int4> flat;
  std::vector<int> begin(sms + 1, 0);
  for (int c = 0; c < sms; ++c) {
    begin[c] = (int)flat.size();
    flat.insert(flat.end(), per[c].begin(), per[c].end());
  }
  begin[sms] = (int)flat.size();

  AURAS_CUDA(cudaMalloc(&mc.partials, sizeof(float) * std::max<int64_t>(1, part_total)));
  for (int i = 0; i < n; ++i) hops[i].epi.partial = mc.partials + part_off[i];
  AURAS_CUDA(cudaMalloc(&mc.ops, sizeof(MegaOp) * n));
  AURAS_CUDA(cudaMalloc(&mc.tasks, sizeof(int4) * flat.size()));
  AURAS_CUDA(cudaMalloc(&mc.cta_begin, sizeof(int) * (sms + 1)));
  AURAS_CUDA(cudaMalloc(&mc.ctr, sizeof(int) * (2 * n + 1)));
  AURAS_CUDA(cudaMemcpy(mc.ops, hops.data(), sizeof(MegaOp) * n, cudaMemcpyHostToDevice));
  AURAS_CUDA(cudaMemcpy(mc.tasks, flat.data(), sizeof(int4) * flat.size(), cudaMemcpyHostToDevice));
  AURAS_CUDA(cudaMemcpy(mc.cta_begin, begin.data(), sizeof(int) * (sms + 1), cudaMemcpyHostToDevice));
  mc.n_ops = n;
  mc.n_tasks = (int)flat.size();
  mc.grid = sms;
  mc.S = S;
  mc.params = base;
  mc.params.ops = mc.ops;
  mc.params.tasks = mc.tasks;
  mc.params.cta_begin = mc.cta_begin;
  mc.params.ctr = mc.ctr;
  mc.params.n_ops = n;
  mc.params.S = S;
  const char *sn = getenv("AURAS_MEGA_SPIN_NS");
  mc.params.spin_ns = sn ? atoi(sn) : 0;
  const char *ad = getenv("AURAS_MEGA_A_DEPTH");
  mc.params.na = na;
  mc.params.a_depth = ad ? std::max(1, std::min(na, atoi(ad))) : na;
  return ensure_smem_attr(unet_mega, (int)MK_SMEM);
}

int mega_launch(const MegaConfig &mc, cudaStream_t st) {
  AURAS_CUDA(cudaMemsetAsync(mc.ctr, 0, sizeof(int) * (2 * mc.n_ops + 1), st));
  unet_mega<<<mc.grid, MK_THREADS, MK_SMEM, st>>>(mc.params);
  AURAS_LAUNCHED("unet_mega");
  return AURAS_OK;
}

int mega_set_trace(MegaConfig &mc, long long *trace) {
  mc.params.trace = trace;
  mc.params.kbtrace = trace ? trace + (int64_t)mc.n_tasks * 8 : nullptr;
  return AURAS_OK;
}

void mega_free_tiled(TiledCache &cache) {
  for (auto &kv : cache) cudaFree(kv.second);
  cache.clear();
}

void mega_free(MegaConfig &mc) {
  cudaFree(mc.ops);
  cudaFree(mc.tasks);
  cudaFree(mc.cta_begin);
  cudaFree(mc.ctr);
  cudaFree(mc.partials);
  mc = MegaConfig();
}

MegaParams mega_base_params(UnetDev *dev, const auras_sched &sched, int horizon, int adim, void *xin, int x_pitch,
                            int64_t slot_stride, int64_t agent_stride, const void *y_final, int y_pitch, int cin,
                            const float *wf, const float *bf) {
  MegaParams p;
  memset(&p, 0, sizeof(p));
  p.dev = dev;
  p.sched = sched;
  p.horizon = horizon;
  p.adim = adim;
  p.xin = static_cast<__nv_bfloat16 *>(xin);
  p.x_pitch = x_pitch;
  p.ring_slot_stride = slot_stride;
  p.ring_agent_stride = agent_stride;
  p.y_final = static_cast<const __nv_bfloat16 *>(y_final);
  p.y_pitch = y_pitch;
  p.final_cin = cin;
  p.wf = wf;
  p.bf = bf;
  return p;
}

}  // namespace auras
