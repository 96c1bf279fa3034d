// Internal kernel-argument structs shared by the conv engines and the UNet plan.
#pragma once
#include "common.cuh"

namespace auras {

struct ConvGemmArgs {
  const void *w;      // [M][Kp]
  const void *in;     // NHWC view
  float *partial;     // [splits][N][M]
  int M, N, Kp, Kreal, Cin;
  int H, W, in_pitch, in_coff;
  int kh, kw, stride, pad_h, pad_w;
  int Ho, Wo;
  int splits, kchunk;
  int engine;         // 0 SIMT, 1 tcgen05 + TMA im2col (1-D), 2 tcgen05 + gathered im2col
  int cta_target;     // engine 2: CTAs to aim for (0: a 32-CTA slice of the GPU)
};

struct EpiArgs {
  float *partial;             // [splits][N][M]; split 0 receives the reduced sum
  const float *bias, *gn_gamma, *gn_beta;
  const void *res;
  const float *res_f32;
  void *out;
  float *out_f32;
  const float *film_a;        // FiLM rows: film_a[row_a(s) * film_a_stride + off ...]
  const int *film_a_row;      // per-sample row (NULL: row = s)
  int64_t film_a_stride;
  const float *film_b;        // optional second FiLM source, per-sample float offset
  const int64_t *film_b_off;
  int M, N, Ho, Wo, splits, groups, act, res_before_act, film_off;
  int out_pitch, out_coff, res_pitch, res_coff, out_stuff, pool_out;
};

struct LinArgs {
  const void *w;
  const float *bias;
  const float *x;
  float *y;
  int M, K, ldw, mish_in, N, ldx, ldy;
};

int conv_op_to_args(const auras_conv_op &op, int S, int dtype, float *partial, ConvGemmArgs &g, EpiArgs &e);
int run_gemm(const ConvGemmArgs &g, int dtype, cudaStream_t st);
int run_epilogue(const EpiArgs &e, int S, int dtype, cudaStream_t st);
int64_t conv_scratch_floats(const auras_conv_op &op, int S, int dtype);

// tcgen05 / TMA engine (gemm_sm100.cu)
bool gemm_sm100_supported(const ConvGemmArgs &g);
int gemm_sm100_splits(const ConvGemmArgs &g);
// tcgen05 engine with a thread-gathered im2col operand (gemm_gather_sm100.cu)
bool gemm_gather_supported(const ConvGemmArgs &g);
int gemm_gather_splits(const ConvGemmArgs &g);
int launch_gemm_gather(const ConvGemmArgs &g, cudaStream_t st);
int launch_gemm_sm100(const ConvGemmArgs &g, cudaStream_t st);

}  // namespace auras
