// Shared device helpers for the Auras B200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "auras_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "auras_b200 targets sm_100a (B200) only"
#endif

namespace auras {

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...);
int cuda_check(cudaError_t e, const char *what);
#define AURAS_CUDA(call) do { int _rc = ::auras::cuda_check((call), #call); if (_rc) return _rc; } while (0)
#define AURAS_LAUNCHED(what) do { int _rc = ::auras::cuda_check(cudaGetLastError(), what); if (_rc) return _rc; } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute is per device, so a process-wide flag would miss the second
// GPU of the disaggregated variant.
template <typename F>
inline int ensure_smem_attr(F *func, int bytes) {
  struct Entry {
    const void *f;
    int dev, bytes;
  };
  static thread_local Entry cache[64];
  static thread_local int n = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = -1;
  for (int i = 0; i < n; ++i)
    if (cache[i].f == reinterpret_cast<const void *>(func) && cache[i].dev == dev && cache[i].bytes >= bytes)
      return AURAS_OK;
  const int rc = cuda_check(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
                            "cudaFuncSetAttribute");
  if (rc) return rc;
  if (n < 64) cache[n++] = Entry{reinterpret_cast<const void *>(func), dev, bytes};
  return AURAS_OK;
}

// ---------------------------------------------------------------- numerics
template <typename T> struct Elem;
template <> struct Elem<float> {
  static __device__ __forceinline__ float load(const float *p) { return *p; }
  static __device__ __forceinline__ void store(float *p, float v) { *p = v; }
};
template <> struct Elem<__nv_bfloat16> {
  static __device__ __forceinline__ float load(const __nv_bfloat16 *p) { return __bfloat162float(*p); }
  static __device__ __forceinline__ void store(__nv_bfloat16 *p, float v) { *p = __float2bfloat16_rn(v); }
};

// Mish(x) = x * tanh(softplus(x)).  With e = exp(x):
// tanh(log(1 + e)) = (e^2 + 2e) / (e^2 + 2e + 2)  -- one exp, one division.
__device__ __forceinline__ float mish(float x) {
  if (x > 20.f) return x;                     // torch's softplus threshold
  const float e = __expf(x);
  const float n = e * (e + 2.f);
  return x * __fdividef(n, n + 2.f);
}

__device__ __forceinline__ float activate(float v, int act) {
  if (act == AURAS_ACT_RELU) return v > 0.f ? v : 0.f;
  if (act == AURAS_ACT_MISH) return mish(v);
  if (act == AURAS_ACT_GELU) return 0.5f * v * (1.f + erff(v * 0.70710678118654752f));   // exact (erf) GELU
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum for blockDim.x a multiple of 32 (<= 1024); `red` has >= 32 slots.
__device__ __forceinline__ float block_sum(float v, float *red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  float t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.f;
  if (wid == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  float r = red[0];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------- memory ordering
__device__ __forceinline__ void st_release_gpu(int64_t *p, int64_t v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_gpu(const int64_t *p) {
  int64_t v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

}  // namespace auras
