// tcgen05 / TMA implicit-GEMM engine (placeholder until the sm_100a kernel lands).
#include "conv.cuh"

namespace auras {
bool gemm_sm100_supported(const ConvGemmArgs &) { return false; }
int launch_gemm_sm100(const ConvGemmArgs &, cudaStream_t) {
  set_error("tcgen05 engine not built");
  return AURAS_E_ARG;
}
}  // namespace auras
