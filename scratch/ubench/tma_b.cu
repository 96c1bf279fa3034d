// Throughput of the denoise kernel's activation TMA loads (4-D im2col view,
// box {64 ch, 1, Wo, s_box}, 128-byte rows strided by the channel pitch)
// versus contiguous 2-D weight boxes, one CTA per SM, L2-resident source.
#include <cstdio>
#include <vector>
#include "../../paper_2509_09560_b200/csrc/tc_util.cuh"
using namespace auras;
namespace auras {
void set_error(const char *fmt, ...) {}
int cuda_check(cudaError_t e, const char *what) { if (e) { printf("%s: %s\n", what, cudaGetErrorString(e)); return -1; } return 0; }
}
constexpr int STAGES = 12;
__global__ void bench(const __grid_constant__ CUtensorMap tm, int mode, int iters, int stage_bytes, int cin, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *buf = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  uint64_t *full = reinterpret_cast<uint64_t *>(buf + STAGES * stage_bytes);
  if (threadIdx.x == 0) { for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  long long t0 = clock64();
  for (int i = 0; i < iters + STAGES; ++i) {
    const int st = i % STAGES;
    if (i >= STAGES) mbar_wait(&full[st], ((i / STAGES) - 1) & 1);
    if (i < iters) {
      if (mode == 0) {
        const int kb = (i + blockIdx.x) % (5 * cin / 64);
        const int k = kb * 64, tap = k / cin, c0 = k - tap * cin;
        tma_load_4d_warp(buf + st * stage_bytes, &tm, &full[st], stage_bytes, c0, 0, tap, 0);
      } else if (mode == 2) {       // 3-D {C, T, S}
        const int kb = (i + blockIdx.x) % (5 * cin / 64);
        const int k = kb * 64, tap = k / cin, c0 = k - tap * cin;
        asm volatile("{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, 0xffffffff;\n"
                     "@px mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n"
                     "@px cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%4, %5, %6}], [%2];\n}\n"
                     :: "r"(smem_u32(buf + st * stage_bytes)), "l"(&tm), "r"(smem_u32(&full[st])), "r"(stage_bytes), "r"(c0), "r"(tap - 2), "r"(0) : "memory");
      } else if (mode == 3) {       // 2-D {C, S*T}: strided rows, one box of Wo*sbox rows
        const int kb = (i + blockIdx.x) % (5 * cin / 64);
        const int k = kb * 64, tap = k / cin, c0 = k - tap * cin;
        tma_load_2d_warp(buf + st * stage_bytes, &tm, &full[st], stage_bytes, c0, tap);
      } else {
        tma_load_2d_warp(buf + st * stage_bytes, &tm, &full[st], stage_bytes, 0, ((i + blockIdx.x * 7) % 1024) * 128);
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
  const int S = 8, T = 8, C = 2048, Wo = 4, sbox = 8;
  void *act, *w;
  cudaMalloc(&act, (size_t)S * T * (C + 64) * 2);
  cudaMemset(act, 0, (size_t)S * T * (C + 64) * 2);
  cudaMalloc(&w, (size_t)1024 * 128 * 128);
  cudaMemset(w, 0, (size_t)1024 * 128 * 128);
  long long *out; cudaMalloc(&out, 148 * 8);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int pitch_extra : {0}) {
  const int P = C + pitch_extra;
  for (int mode : {1}) {
    CUtensorMap tm;
    int stage;
    if (mode == 0) {
      // the kernel's view: {C, stride=1, T, S}, pitch C, box {64, 1, Wo, sbox}
      make_act_map(&tm, act, 0, C, C, T, 1, S, Wo, sbox);
      stage = Wo * sbox * 128;
    } else if (mode == 2) {
      EncodeTiledFn enc = encode_fn();
      cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)T, (cuuint64_t)S};
      cuuint64_t str[2] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * T};
      cuuint32_t box[3] = {64, (cuuint32_t)Wo, (cuuint32_t)sbox}; cuuint32_t es[3] = {1, 1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, act, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      stage = Wo * sbox * 128;
    } else if (mode == 3) {
      EncodeTiledFn enc = encode_fn();
      cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)(T * S)};
      cuuint64_t str[1] = {(cuuint64_t)P * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)(Wo * sbox)}; cuuint32_t es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, act, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      stage = Wo * sbox * 128;
    } else {
      EncodeTiledFn enc = encode_fn();
      cuuint64_t dims[2] = {64, 1024 * 128}; cuuint64_t str[1] = {128}; cuuint32_t box[2] = {64, 128}; cuuint32_t es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      stage = 16384;
    }
    const size_t smem = 1024 + STAGES * stage + 256;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int grid : {1, 16, 64, 112, 148}) {
      const int iters = 2000;
      bench<<<grid, 64, smem>>>(tm, mode, iters, stage, C, out);
      cudaDeviceSynchronize();
      bench<<<grid, 64, smem>>>(tm, mode, iters, stage, C, out);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<long long> h(grid);
      cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost);
      long long mx = 0; for (auto v : h) mx = v > mx ? v : mx;
      const double us = mx / (clk * 1e-3);
      printf("pitch %d: %s grid %3d: %.3f us per box (%d B), %.1f GB/s per SM, %.0f GB/s total %s\n",
             P, mode == 0 ? "act 4-D box" : mode == 2 ? "act 3-D box" : mode == 3 ? "act 2-D strided" : "weight 2-D box", grid, us / iters, stage, (double)stage * iters / us * 1e-3,
             (double)stage * iters * grid / us * 1e-3, cudaGetErrorString(e));
    }
  }
  }
}
