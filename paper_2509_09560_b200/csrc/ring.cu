// Public-context ring (ContextStore, fp/context.py:98-175) and the reference's
// fp64 refinement policy (fp/policy.py:217-246) on the device.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace auras {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_check(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return AURAS_OK;
  set_error("%s: %s", what, cudaGetErrorString(e));
  return AURAS_E_CUDA;
}

__device__ __forceinline__ int ring_slot(int64_t frame, int capacity) {
  int64_t r = frame % capacity;
  return static_cast<int>(r < 0 ? r + capacity : r);
}

// Version word written last with release semantics: a consumer that
// acquire-loads the version observes every payload store that preceded it.
__device__ void commit_slot(int64_t *meta, int64_t *state, int capacity, int64_t frame,
                            int64_t expected_version) {
  const int slot = ring_slot(frame, capacity);
  const int64_t v = state[0] + 1;
  if (v != expected_version) state[3] = 1;     // host/device version drift
  if (state[1] >= 0 && frame < state[1]) state[3] = 2;  // StaleWrite seen on device
  meta[2 * slot + 0] = frame;
  __threadfence();
  st_release_gpu(&meta[2 * slot + 1], v);
  state[0] = v;
  state[1] = frame;
  state[2] += 1;
}

__global__ void ring_commit_kernel(int64_t *meta, int64_t *state, int capacity, int64_t frame,
                                   int64_t expected_version) {
  commit_slot(meta, state, capacity, frame, expected_version);
}

// System-scope variant for a ring that lives on another GPU.
__global__ void ring_commit_sys_kernel(int64_t *meta, int64_t *state, int capacity, int64_t frame,
                                       int64_t expected_version) {
  const int slot = ring_slot(frame, capacity);
  const int64_t v = state[0] + 1;
  if (v != expected_version) state[3] = 1;
  if (state[1] >= 0 && frame < state[1]) state[3] = 2;
  meta[2 * slot + 0] = frame;
  __threadfence_system();
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(&meta[2 * slot + 1]), "l"(v) : "memory");
  state[0] = v;
  state[1] = frame;
  state[2] += 1;
}

__global__ void ring_fetch_kernel(const int64_t *meta, const int64_t *state, int capacity,
                                  int64_t target, int64_t *out, int64_t *log, int64_t log_index) {
  int slot = ring_slot(target, capacity);
  int64_t v = ld_acquire_gpu(&meta[2 * slot + 1]);
  int64_t f = meta[2 * slot + 0];
  if (v <= 0 || f != target) {                  // publisher skipped: newest context
    const int64_t last = state[1];
    slot = ring_slot(last, capacity);
    v = ld_acquire_gpu(&meta[2 * slot + 1]);
    f = meta[2 * slot + 0];
  }
  out[0] = slot;
  out[1] = v;
  out[2] = f;
  if (log) log[log_index] = v;
}

// ---------------------------------------------------------------- ring stress (test)
// t/test_context_store.py:148-183 on the device: block 0 publishes versions
// 1..n into a `capacity`-slot ring with the product's order (version word
// invalidated with a release store, payload written by the whole block, then
// commit_slot: frame, fence, version with release); blocks 1..readers fetch the
// newest entry concurrently, seqlock style: acquire the version, read the
// payload, fence, re-read the version.  A read whose two versions agree must
// carry the writer's words for that version (fp/context.py:28-36 checks a
// checksum; here every word is checked) and versions must never go backwards.
// counts[r] = {consistent reads, retries, torn reads, version regressions}.
__device__ __forceinline__ double stress_word(int64_t v, int j) { return (double)v * 4096.0 + (double)j; }

__global__ void ring_stress_kernel(int64_t *meta, int64_t *state, double *payload, int capacity, int words,
                                   int n, int *done, unsigned long long *counts) {
  if (blockIdx.x == 0) {
    for (int64_t v = 1; v <= n; ++v) {
      const int64_t frame = v - 1;
      const int slot = ring_slot(frame, capacity);
      if (threadIdx.x == 0) st_release_gpu(&meta[2 * slot + 1], -1);
      __syncthreads();
      for (int j = threadIdx.x; j < words; j += blockDim.x) payload[(int64_t)slot * words + j] = stress_word(v, j);
      __syncthreads();
      if (threadIdx.x == 0) commit_slot(meta, state, capacity, frame, v);
      __syncthreads();
      __nanosleep(1000);                            // give readers a window between publishes
    }
    if (threadIdx.x == 0) {
      __threadfence();
      atomicExch(done, 1);
    }
    return;
  }
  __shared__ int64_t s_v;
  __shared__ int s_bad, s_stop;
  unsigned long long ok = 0, retry = 0, torn = 0, regress = 0;
  int64_t last = 0;
  for (;;) {
    if (threadIdx.x == 0) {
      s_stop = atomicAdd(done, 0);
      int64_t vc;
      asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(vc) : "l"(&state[0]) : "memory");
      int64_t v1 = -1;
      if (vc > 0) v1 = ld_acquire_gpu(&meta[2 * ring_slot(vc - 1, capacity) + 1]);
      s_v = (vc > 0 && v1 == vc) ? vc : 0;
      s_bad = 0;
    }
    __syncthreads();
    const int64_t v = s_v;
    const int stop = s_stop;
    if (v > 0) {
      const int slot = ring_slot(v - 1, capacity);
      int bad = 0;
      for (int j = threadIdx.x; j < words; j += blockDim.x) {
        double x;
        asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(x) : "l"(&payload[(int64_t)slot * words + j]) : "memory");
        bad |= x != stress_word(v, j);
      }
      __threadfence();                              // payload reads before the re-check
      if (bad) atomicOr(&s_bad, 1);
      __syncthreads();
      if (threadIdx.x == 0) {
        int64_t v2;
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v2) : "l"(&meta[2 * slot + 1]) : "memory");
        if (v2 != v) ++retry;                       // overwritten while reading: discard
        else if (s_bad) ++torn;
        else {
          ++ok;
          if (v < last) ++regress;
          last = v;
        }
      }
    } else if (threadIdx.x == 0) {
      ++retry;
    }
    __syncthreads();
    if (stop) break;
  }
  if (threadIdx.x == 0) {
    unsigned long long *c = counts + 4 * (blockIdx.x - 1);
    c[0] = ok;
    c[1] = retry;
    c[2] = torn;
    c[3] = regress;
  }
}

// ---------------------------------------------------------------- toy policy

__global__ void toy_ingest_kernel(double *latent, int lane, double o0, double o1, double o2,
                                  double o3, double *x, double x0, double x1) {
  latent[4 * lane + 0] = o0;
  latent[4 * lane + 1] = o1;
  latent[4 * lane + 2] = o2;
  latent[4 * lane + 3] = o3;
  x[2 * lane + 0] = x0;
  x[2 * lane + 1] = x1;
}

__global__ void toy_publish_kernel(const double *latent, int lane, double *payload,
                                   int64_t *meta, int64_t *state, int capacity, int64_t frame,
                                   int64_t version) {
  const int slot = ring_slot(frame, capacity);
  // invalidate, write the payload, then release the version (seqlock order)
  st_release_gpu(&meta[2 * slot + 1], -1);
  // fp/policy.py:286  conditioning = latent[:2] - latent[2:4]
  payload[2 * slot + 0] = __dsub_rn(latent[4 * lane + 0], latent[4 * lane + 2]);
  payload[2 * slot + 1] = __dsub_rn(latent[4 * lane + 1], latent[4 * lane + 3]);
  commit_slot(meta, state, capacity, frame, version);
}

struct ToyBatch {
  int lanes[64];
  int iters[64];
};

__global__ void toy_generate_kernel(double *x, ToyBatch batch, int n, double eta,
                                    const double *payload, const int64_t *fetched) {
  const int i = threadIdx.x;
  if (i >= n) return;
  const int slot = static_cast<int>(fetched[0]);   // slot resolved in-kernel by ring_fetch
  const double h0 = payload[2 * slot + 0], h1 = payload[2 * slot + 1];
  const int lane = batch.lanes[i];
  double a = x[2 * lane + 0], b = x[2 * lane + 1];
  for (int k = 0; k < batch.iters[i]; ++k) {
    // fp/policy.py:224  new = x + eta * (target - x), evaluated as numpy does
    a = __dadd_rn(a, __dmul_rn(eta, __dsub_rn(h0, a)));
    b = __dadd_rn(b, __dmul_rn(eta, __dsub_rn(h1, b)));
  }
  x[2 * lane + 0] = a;
  x[2 * lane + 1] = b;
}

__global__ void toy_finish_kernel(const double *x, int lane, double max_action, double *out) {
  double a = x[2 * lane + 0], b = x[2 * lane + 1];
  // np.linalg.norm of a 2-vector on this stack is sqrt(fma(b, b, a*a)) (OpenBLAS ddot)
  const double norm = __dsqrt_rn(__fma_rn(b, b, __dmul_rn(a, a)));
  if (norm > max_action) {
    const double s = __ddiv_rn(max_action, norm);
    a = __dmul_rn(a, s);
    b = __dmul_rn(b, s);
  }
  out[0] = a;
  out[1] = b;
}

__global__ void copy_bytes_kernel(uint4 *dst, const uint4 *src, int64_t n16, uint8_t *dtail,
                                  const uint8_t *stail, int ntail) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  if (blockIdx.x == 0 && threadIdx.x < ntail) dtail[threadIdx.x] = stail[threadIdx.x];
}

}  // namespace auras

using namespace auras;

extern "C" {

const char *auras_last_error(void) { return g_err; }

int auras_abi_version(void) { return 4; }

int auras_device_ok(int device) {
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return 0;
  return p.major == 10 && p.minor == 0;
}

int auras_ring_commit(int64_t *meta, int64_t *state, int capacity, int64_t frame,
                      int64_t expected_version, void *stream) {
  if (!meta || !state || capacity < 2) { set_error("ring_commit: bad args"); return AURAS_E_ARG; }
  ring_commit_kernel<<<1, 1, 0, as_stream(stream)>>>(meta, state, capacity, frame, expected_version);
  AURAS_LAUNCHED("ring_commit_kernel");
  return AURAS_OK;
}

// Action emission buffer: pinned host memory mapped into the device address
// space, so the finish kernel writes the emitted action straight to host memory and a reader only
// waits for that kernel's completion event (no device-to-host copy on the action path).
int auras_host_mapped_alloc(size_t bytes, void **host, void **dev) {
  if (!host || !dev || bytes == 0) {
    set_error("host_mapped_alloc: bad args");
    return AURAS_E_ARG;
  }
  *host = nullptr;
  *dev = nullptr;
  AURAS_CUDA(cudaHostAlloc(host, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(*host, 0, bytes);
  const cudaError_t e = cudaHostGetDevicePointer(dev, *host, 0);
  if (e != cudaSuccess) {
    cudaFreeHost(*host);
    *host = nullptr;
    return cuda_check(e, "host_mapped_alloc");
  }
  return AURAS_OK;
}

int auras_host_mapped_free(void *host) {
  if (host) AURAS_CUDA(cudaFreeHost(host));
  return AURAS_OK;
}

int auras_ring_stress(int capacity, int words, int n_versions, int readers, unsigned long long *counts_host) {
  if (capacity < 2 || words < 1 || n_versions < 1 || readers < 1 || readers > 64 || !counts_host) {
    set_error("ring_stress: bad args");
    return AURAS_E_ARG;
  }
  int64_t *meta = nullptr, *state = nullptr;
  double *payload = nullptr;
  int *done = nullptr;
  unsigned long long *counts = nullptr;
  int rc = AURAS_OK;
  if ((rc = cuda_check(cudaMalloc(&meta, sizeof(int64_t) * 2 * capacity), "malloc")) ||
      (rc = cuda_check(cudaMalloc(&state, sizeof(int64_t) * 4), "malloc")) ||
      (rc = cuda_check(cudaMalloc(&payload, sizeof(double) * (size_t)capacity * words), "malloc")) ||
      (rc = cuda_check(cudaMalloc(&done, sizeof(int)), "malloc")) ||
      (rc = cuda_check(cudaMalloc(&counts, sizeof(unsigned long long) * 4 * readers), "malloc")))
    goto out;
  cudaMemset(meta, 0, sizeof(int64_t) * 2 * capacity);
  cudaMemset(payload, 0, sizeof(double) * (size_t)capacity * words);
  cudaMemset(done, 0, sizeof(int));
  {
    const int64_t st0[4] = {0, -1, 0, 0};
    cudaMemcpy(state, st0, sizeof(st0), cudaMemcpyHostToDevice);
  }
  ring_stress_kernel<<<1 + readers, 256>>>(meta, state, payload, capacity, words, n_versions, done, counts);
  if ((rc = cuda_check(cudaGetLastError(), "ring_stress_kernel"))) goto out;
  if ((rc = cuda_check(cudaDeviceSynchronize(), "ring_stress_kernel"))) goto out;
  rc = cuda_check(cudaMemcpy(counts_host, counts, sizeof(unsigned long long) * 4 * readers,
                             cudaMemcpyDeviceToHost), "copy counts");
out:
  cudaFree(meta);
  cudaFree(state);
  cudaFree(payload);
  cudaFree(done);
  cudaFree(counts);
  return rc;
}

int auras_ring_commit_sys(int64_t *meta, int64_t *state, int capacity, int64_t frame,
                          int64_t expected_version, void *stream) {
  if (!meta || !state || capacity < 2) { set_error("ring_commit_sys: bad args"); return AURAS_E_ARG; }
  ring_commit_sys_kernel<<<1, 1, 0, as_stream(stream)>>>(meta, state, capacity, frame, expected_version);
  AURAS_LAUNCHED("ring_commit_sys_kernel");
  return AURAS_OK;
}

int auras_enable_peer(int device, int peer) {
  if (device == peer) return AURAS_OK;
  int prev = 0;
  AURAS_CUDA(cudaGetDevice(&prev));
  AURAS_CUDA(cudaSetDevice(device));
  int can = 0;
  cudaDeviceCanAccessPeer(&can, device, peer);
  cudaError_t e = can ? cudaDeviceEnablePeerAccess(peer, 0) : cudaErrorPeerAccessUnsupported;
  if (e == cudaErrorPeerAccessAlreadyEnabled) e = cudaSuccess;
  cudaGetLastError();
  cudaSetDevice(prev);
  return cuda_check(e, "cudaDeviceEnablePeerAccess");
}

int auras_peer_copy(void *dst, int64_t dst_pitch, const void *src, int64_t src_pitch, int64_t width,
                    int64_t rows, void *stream) {
  if (!dst || !src || width < 0 || rows < 0 || dst_pitch < width || src_pitch < width) {
    set_error("peer_copy: bad args");
    return AURAS_E_ARG;
  }
  if (width == 0 || rows == 0) return AURAS_OK;
  AURAS_CUDA(cudaMemcpy2DAsync(dst, (size_t)dst_pitch, src, (size_t)src_pitch, (size_t)width, (size_t)rows,
                               cudaMemcpyDefault, as_stream(stream)));
  return AURAS_OK;
}

int auras_ring_fetch(const int64_t *meta, const int64_t *state, int capacity, int64_t target,
                     int64_t *out, int64_t *version_log, int64_t log_index, void *stream) {
  if (!meta || !state || !out || capacity < 2) { set_error("ring_fetch: bad args"); return AURAS_E_ARG; }
  ring_fetch_kernel<<<1, 1, 0, as_stream(stream)>>>(meta, state, capacity, target, out, version_log,
                                                    log_index);
  AURAS_LAUNCHED("ring_fetch_kernel");
  return AURAS_OK;
}

int auras_ring_write(void *payload, int64_t slot_bytes, int slot, const void *src, int64_t bytes,
                     void *stream) {
  if (!payload || !src || bytes > slot_bytes || slot < 0) { set_error("ring_write: bad args"); return AURAS_E_ARG; }
  uint8_t *dst = static_cast<uint8_t *>(payload) + slot_bytes * slot;
  const bool aligned = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  if (!aligned) {
    AURAS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, as_stream(stream)));
    return AURAS_OK;
  }
  const int64_t n16 = bytes / 16;
  const int ntail = static_cast<int>(bytes - n16 * 16);
  int blocks = static_cast<int>((n16 + 255) / 256);
  blocks = blocks < 1 ? 1 : (blocks > 592 ? 592 : blocks);
  copy_bytes_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
      reinterpret_cast<uint4 *>(dst), reinterpret_cast<const uint4 *>(src), n16, dst + n16 * 16,
      static_cast<const uint8_t *>(src) + n16 * 16, ntail);
  AURAS_LAUNCHED("copy_bytes_kernel");
  return AURAS_OK;
}

int auras_toy_ingest(double *latent, int lane, const double obs[4], double *x_state,
                     const double x0[2], void *stream) {
  if (!latent || !x_state || !obs || !x0 || lane < 0) { set_error("toy_ingest: bad args"); return AURAS_E_ARG; }
  toy_ingest_kernel<<<1, 1, 0, as_stream(stream)>>>(latent, lane, obs[0], obs[1], obs[2], obs[3],
                                                    x_state, x0[0], x0[1]);
  AURAS_LAUNCHED("toy_ingest_kernel");
  return AURAS_OK;
}

int auras_toy_publish(const double *latent, int lane, double *ring_payload, int64_t *meta,
                      int64_t *state, int capacity, int64_t frame, int64_t version, void *stream) {
  if (!latent || !ring_payload || !meta || !state || capacity < 2) { set_error("toy_publish: bad args"); return AURAS_E_ARG; }
  toy_publish_kernel<<<1, 1, 0, as_stream(stream)>>>(latent, lane, ring_payload, meta, state,
                                                     capacity, frame, version);
  AURAS_LAUNCHED("toy_publish_kernel");
  return AURAS_OK;
}

int auras_toy_generate(double *x_state, const int *lanes, const int *iters, int n, double eta,
                       const double *ring_payload, const int64_t *fetched, void *stream) {
  if (n < 0 || n > 64 || !x_state || !ring_payload || !fetched) { set_error("toy_generate: bad args (n=%d)", n); return AURAS_E_ARG; }
  if (n == 0) return AURAS_OK;
  ToyBatch b;
  memset(&b, 0, sizeof(b));
  for (int i = 0; i < n; ++i) { b.lanes[i] = lanes[i]; b.iters[i] = iters[i]; }
  toy_generate_kernel<<<1, 64, 0, as_stream(stream)>>>(x_state, b, n, eta, ring_payload, fetched);
  AURAS_LAUNCHED("toy_generate_kernel");
  return AURAS_OK;
}

int auras_toy_finish(const double *x_state, int lane, double max_action, double *out, void *stream) {
  if (!x_state || !out) { set_error("toy_finish: bad args"); return AURAS_E_ARG; }
  toy_finish_kernel<<<1, 1, 0, as_stream(stream)>>>(x_state, lane, max_action, out);
  AURAS_LAUNCHED("toy_finish_kernel");
  return AURAS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- scripted token policy
// fp/policy.py:110-161: the displacement in the fetched context (vision row 0,
// the toy ring payload {x, y}) quantised into the 7-token schema
// (sign, mag / 8, mag % 8) per axis + STOP, repeated cyclically for l_a > 7.
// Token p of a request depends only on the context it reads and p.

namespace {
__device__ int ar_token(double dx, double dy, double max_action, int p) {
  const int k = p % 7;
  if (k == 6) return 0;                                  // STOP_TOKEN
  const double raw = k < 3 ? dx : dy;
  const double width = max_action / 63.0;
  const double v = fmin(fmax(raw, -max_action), max_action);
  int mag = (int)floor(fabs(v) / width + 0.5);
  mag = mag < 63 ? mag : 63;
  const int sign = mag == 0 ? 0 : (v > 0.0 ? 1 : 2);
  const int j = k % 3;
  return j == 0 ? sign : (j == 1 ? mag / 8 : mag % 8);
}

struct ArBatch {
  int lanes[64], starts[64], counts[64];
};

__global__ void ar_generate_kernel(int *tokens, int l_a, ArBatch b, int n, const double *ring_payload,
                                   const int64_t *fetched, double max_action) {
  const int64_t slot = fetched[0];
  const double dx = ring_payload[slot * 2], dy = ring_payload[slot * 2 + 1];
  for (int r = 0; r < n; ++r)
    for (int i = threadIdx.x; i < b.counts[r]; i += blockDim.x) {
      const int p = b.starts[r] + i;
      if (p < l_a) tokens[b.lanes[r] * l_a + p] = ar_token(dx, dy, max_action, p);
    }
}

__global__ void ar_finish_kernel(const int *tokens, int lane, int l_a, double *out) {
  for (int i = threadIdx.x; i < l_a; i += blockDim.x) out[i] = (double)tokens[lane * l_a + i];
}

__global__ void ring_copy_slot_kernel(double *payload, int elems, int src, int dst) {
  for (int i = threadIdx.x; i < elems; i += blockDim.x) payload[dst * elems + i] = payload[src * elems + i];
}
}  // namespace

extern "C" {

int auras_ar_generate(int *tokens, int l_a, const int *lanes, const int *starts, const int *counts, int n,
                      const double *ring_payload, const int64_t *fetched, double max_action, void *stream) {
  if (n < 0 || n > 64 || l_a < 1 || !tokens || !ring_payload || !fetched) {
    set_error("ar_generate: bad args (n=%d, l_a=%d)", n, l_a);
    return AURAS_E_ARG;
  }
  if (n == 0) return AURAS_OK;
  ArBatch b;
  memset(&b, 0, sizeof(b));
  for (int i = 0; i < n; ++i) { b.lanes[i] = lanes[i]; b.starts[i] = starts[i]; b.counts[i] = counts[i]; }
  ar_generate_kernel<<<1, 64, 0, as_stream(stream)>>>(tokens, l_a, b, n, ring_payload, fetched, max_action);
  AURAS_LAUNCHED("ar_generate_kernel");
  return AURAS_OK;
}

int auras_ar_finish(const int *tokens, int lane, int l_a, double *out, void *stream) {
  if (!tokens || !out || lane < 0 || l_a < 1) { set_error("ar_finish: bad args"); return AURAS_E_ARG; }
  ar_finish_kernel<<<1, 64, 0, as_stream(stream)>>>(tokens, lane, l_a, out);
  AURAS_LAUNCHED("ar_finish_kernel");
  return AURAS_OK;
}

int auras_ring_copy_slot(double *payload, int elems, int src, int dst, void *stream) {
  if (!payload || elems < 1 || src < 0 || dst < 0) { set_error("ring_copy_slot: bad args"); return AURAS_E_ARG; }
  if (src == dst) return AURAS_OK;
  ring_copy_slot_kernel<<<1, 128, 0, as_stream(stream)>>>(payload, elems, src, dst);
  AURAS_LAUNCHED("ring_copy_slot_kernel");
  return AURAS_OK;
}

}  // extern "C"
