// Fused conv epilogue body, shared by the standalone epilogue kernel and the
// persistent denoise megakernel (unet_mega.cu).
#pragma once
#include "conv.cuh"

namespace auras {

// Sum over `nthr` threads that synchronise with `sync()`; every thread gets
// the same value, accumulated in a fixed order (deterministic).
template <typename Sync>
__device__ __forceinline__ float unit_sum(float v, float *red, int tid, int nthr, Sync sync) {
  v = warp_sum(v);
  sync();
  if ((tid & 31) == 0) red[tid >> 5] = v;
  sync();
  float t = 0.f;
  for (int i = 0; i < (nthr >> 5); ++i) t += red[i];
  return t;
}

// One epilogue unit: sample s, GroupNorm group gy (or 64-channel block without
// GroupNorm).  Three passes over the L2-resident partials:
//   1) v = bias + sum_split partial  (written back in place), group sum
//   2) group variance around the mean
//   3) normalise, affine, activation, FiLM, residual, store (stuffed/pooled)
// Register-resident variant (P % 4 == 0 and <= 16 values per thread): every
// load the unit needs -- partials of all splits (float4), bias, GroupNorm
// affine, FiLM rows, residual -- is issued in one round, statistics come from
// registers, then one store pass.  Partials are [split][m][n], n = s*P + p.
template <typename T, typename Sync, typename Gate>
__device__ __forceinline__ void epi_unit_regs(const EpiArgs &a, int s, int gy, int tid, int nthr, float *red,
                                              Sync sync, Gate gate, long long *stamp = nullptr) {
  constexpr int U = 4;
  const bool gn = a.gn_gamma != nullptr;
  const int cg = gn ? a.M / a.groups : min(64, a.M - gy * 64);
  const int c0 = gn ? gy * cg : gy * 64;
  const int P = a.Ho * a.Wo, P4 = P >> 2;
  const int cnt4 = cg * P4;
  // R lanes share one float4 vector when there are fewer vectors than threads;
  // each lane sums every R-th split, a butterfly combines them (fixed order).
  int R = 1;
  while (R < 8 && cnt4 * R * 2 <= nthr) R <<= 1;
  const int lane_r = tid & (R - 1);
  const int vt = tid / R, vstride = nthr / R;
  const float *base = a.partial;
  const int64_t NM = (int64_t)a.N * a.M;
  const float *fa = nullptr, *fb = nullptr;
  if (a.film_off >= 0) {
    const int ra = a.film_a_row ? a.film_a_row[s] : s;
    fa = a.film_a + (int64_t)ra * a.film_a_stride + a.film_off;
    if (a.film_b) fb = a.film_b + a.film_b_off[s] + a.film_off;
  }
  const T *res = static_cast<const T *>(a.res);
  float v[U][4], rv[U][4];
  float gam[U], bet[U], sc[U], bi[U];
  int cc_[U], p0_[U];
  bool ok_[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int vi = vt + u * vstride;
    const bool ok = vi < cnt4;
    ok_[u] = ok;
    const int cc = ok ? vi / P4 : 0;
    const int p0 = ok ? (vi - cc * P4) * 4 : 0;
    const int c = c0 + cc;
    cc_[u] = cc;
    p0_[u] = p0;
    const float b0 = (ok && a.bias && lane_r == 0) ? a.bias[c] : 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) v[u][q] = b0;
    gam[u] = (ok && gn) ? a.gn_gamma[c] : 1.f;
    bet[u] = (ok && gn) ? a.gn_beta[c] : 0.f;
    sc[u] = 1.f;
    bi[u] = 0.f;
    if (ok && fa) {
      sc[u] = fa[c];
      bi[u] = fa[a.M + c];
      if (fb) { sc[u] += fb[c]; bi[u] += fb[a.M + c]; }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float r = 0.f;
      if (ok) {
        const int p = p0 + q;
        if (res) r = Elem<T>::load(res + ((int64_t)s * P + p) * a.res_pitch + a.res_coff + c);
        else if (a.res_f32) r = a.res_f32[((int64_t)s * P + p) * a.M + c];
      }
      rv[u][q] = r;
    }
  }
  gate();          // everything above is independent of this layer's GEMMs; partials are not
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (!ok_[u]) continue;
    const float *col = base + (int64_t)(c0 + cc_[u]) * a.N + (int64_t)s * P + p0_[u];
    int z = lane_r;
    for (; z + 7 * R < a.splits; z += 8 * R) {          // 8 independent float4 loads in flight
      float4 t[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) t[j] = *reinterpret_cast<const float4 *>(col + (z + j * R) * NM);
      v[u][0] += ((t[0].x + t[1].x) + (t[2].x + t[3].x)) + ((t[4].x + t[5].x) + (t[6].x + t[7].x));
      v[u][1] += ((t[0].y + t[1].y) + (t[2].y + t[3].y)) + ((t[4].y + t[5].y) + (t[6].y + t[7].y));
      v[u][2] += ((t[0].z + t[1].z) + (t[2].z + t[3].z)) + ((t[4].z + t[5].z) + (t[6].z + t[7].z));
      v[u][3] += ((t[0].w + t[1].w) + (t[2].w + t[3].w)) + ((t[4].w + t[5].w) + (t[6].w + t[7].w));
    }
    for (; z + 3 * R < a.splits; z += 4 * R) {
      const float4 t0 = *reinterpret_cast<const float4 *>(col + z * NM);
      const float4 t1 = *reinterpret_cast<const float4 *>(col + (z + R) * NM);
      const float4 t2 = *reinterpret_cast<const float4 *>(col + (z + 2 * R) * NM);
      const float4 t3 = *reinterpret_cast<const float4 *>(col + (z + 3 * R) * NM);
      v[u][0] += (t0.x + t1.x) + (t2.x + t3.x);
      v[u][1] += (t0.y + t1.y) + (t2.y + t3.y);
      v[u][2] += (t0.z + t1.z) + (t2.z + t3.z);
      v[u][3] += (t0.w + t1.w) + (t2.w + t3.w);
    }
    for (; z < a.splits; z += R) {
      const float4 t = *reinterpret_cast<const float4 *>(col + z * NM);
      v[u][0] += t.x; v[u][1] += t.y; v[u][2] += t.z; v[u][3] += t.w;
    }
  }
  for (int o = 1; o < R; o <<= 1) {
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) v[u][q] += __shfl_xor_sync(0xffffffffu, v[u][q], o);
  }
  const bool owner = lane_r == 0;
  float mean = 0.f, rstd = 1.f;
  if (gn) {
    float ls = 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ok_[u] && owner) ls += (v[u][0] + v[u][1]) + (v[u][2] + v[u][3]);
    const int cnt = cnt4 * 4;
    mean = unit_sum(ls, red, tid, nthr, sync) / cnt;
    if (stamp && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(stamp[0]));
    float lq = 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ok_[u] && owner)
#pragma unroll
        for (int q = 0; q < 4; ++q) { const float d = v[u][q] - mean; lq += d * d; }
    rstd = rsqrtf(unit_sum(lq, red, tid, nthr, sync) / cnt + 1e-5f);
    if (stamp && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(stamp[1]));
  }
  T *out = static_cast<T *>(a.out);
  const int wout = a.out_stuff ? 2 * a.Wo : a.Wo;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (!ok_[u]) continue;
    const int c = c0 + cc_[u];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if ((q & (R - 1)) != lane_r && R <= 4) continue;       // lanes of a vector split the stores
      if (R > 4 && !(lane_r < 4 && q == lane_r)) continue;
      const int p = p0_[u] + q;
      float y = v[u][q];
      if (gn) y = (y - mean) * rstd * gam[u] + bet[u];
      if (a.res_before_act) y += rv[u][q];
      y = activate(y, a.act);
      if (fa) y = y * sc[u] + bi[u];
      if (!a.res_before_act) y += rv[u][q];
      if (a.out_f32) a.out_f32[((int64_t)s * P + p) * a.M + c] = y;
      if (out) {
        const int oy = p / a.Wo, ox = p - oy * a.Wo;
        const int ox2 = a.out_stuff ? 2 * ox : ox;
        T *dst = out + ((int64_t)(s * a.Ho + oy) * wout + ox2) * a.out_pitch + a.out_coff + c;
        Elem<T>::store(dst, y);
        if (a.out_stuff) Elem<T>::store(dst + a.out_pitch, 0.f);
      }
    }
  }
  if (stamp && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(stamp[2]));
}

// True when the unit takes the register-resident path (epi_unit_regs).
__device__ __forceinline__ bool epi_fits_regs(const EpiArgs &a, int gy, int nthr) {
  const bool gn = a.gn_gamma != nullptr;
  const int cg0 = gn ? a.M / a.groups : min(64, a.M - gy * 64);
  const int P0 = a.Ho * a.Wo;
  return !a.pool_out && (P0 & 3) == 0 && cg0 * P0 <= 16 * nthr;
}

template <typename T, typename Sync>
__device__ void epi_unit(const EpiArgs &a, int s, int gy, int tid, int nthr, float *red, Sync sync) {
  const bool gn = a.gn_gamma != nullptr;
  if (epi_fits_regs(a, gy, nthr)) {
    epi_unit_regs<T>(a, s, gy, tid, nthr, red, sync, [] __device__() {});
    return;
  }
  const int cg = gn ? a.M / a.groups : min(64, a.M - gy * 64);
  const int c0 = gn ? gy * cg : gy * 64;
  const int P = a.Ho * a.Wo;
  const int cnt = cg * P;
  float *base = a.partial;
  const int64_t NM = (int64_t)a.N * a.M;

  // pass 1: split-K reduction with 4 elements x 4 splits of loads in flight per thread
  float lsum = 0.f;
  for (int i0 = tid; i0 < cnt; i0 += 4 * nthr) {
    int64_t off[4];
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * nthr;
      const int ii = i < cnt ? i : i0;
      const int cc = ii / P, p = ii - cc * P, c = c0 + cc;
      off[u] = (int64_t)c * a.N + s * P + p;          // partial[split][m][n]
      v[u] = a.bias ? a.bias[c] : 0.f;
    }
    int z = 0;
    for (; z + 4 <= a.splits; z += 4) {
      float t[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int u = 0; u < 4; ++u) t[q][u] = base[(z + q) * NM + off[u]];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] += (t[0][u] + t[1][u]) + (t[2][u] + t[3][u]);
    }
    for (; z < a.splits; ++z)
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] += base[z * NM + off[u]];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i0 + u * nthr < cnt) {
        base[off[u]] = v[u];
        lsum += v[u];
      }
    }
  }
  float mean = 0.f, rstd = 1.f;
  if (gn) {
    mean = unit_sum(lsum, red, tid, nthr, sync) / cnt;
    float lsq = 0.f;
    for (int i = tid; i < cnt; i += nthr) {
      const int cc = i / P, p = i - cc * P, c = c0 + cc;
      const float d = base[(int64_t)c * a.N + s * P + p] - mean;
      lsq += d * d;
    }
    const float var = unit_sum(lsq, red, tid, nthr, sync) / cnt;
    rstd = rsqrtf(var + 1e-5f);
  } else {
    sync();
  }

  T *out = static_cast<T *>(a.out);
  const T *res = static_cast<const T *>(a.res);
  const float *fa = nullptr, *fb = nullptr;
  if (a.film_off >= 0) {
    const int ra = a.film_a_row ? a.film_a_row[s] : s;
    fa = a.film_a + (int64_t)ra * a.film_a_stride + a.film_off;
    if (a.film_b) fb = a.film_b + a.film_b_off[s] + a.film_off;
  }
  const int wout = a.out_stuff ? 2 * a.Wo : a.Wo;
  for (int i = tid; i < cnt; i += nthr) {
    const int cc = i / P, p = i - cc * P, c = c0 + cc;
    const int64_t row = (int64_t)(s * P + p);
    const int64_t pidx = (int64_t)c * a.N + s * P + p;
    float y = base[pidx];
    if (gn) y = (y - mean) * rstd * a.gn_gamma[c] + a.gn_beta[c];
    const int oy = p / a.Wo, ox = p - oy * a.Wo;
    float r = 0.f;
    if (res) {
      r = Elem<T>::load(res + ((int64_t)(s * a.Ho + oy) * a.Wo + ox) * a.res_pitch + a.res_coff + c);
    } else if (a.res_f32) {
      r = a.res_f32[row * a.M + c];
    }
    if (a.res_before_act) y += r;
    y = activate(y, a.act);
    if (fa) {
      float sc = fa[c], bi = fa[a.M + c];
      if (fb) { sc += fb[c]; bi += fb[a.M + c]; }
      y = y * sc + bi;
    }
    if (!a.res_before_act) y += r;
    if (a.out_f32 && !a.pool_out) a.out_f32[row * a.M + c] = y;
    if (a.pool_out) {
      base[pidx] = y;                   // staged for the fixed-order pooling below
    } else if (out) {
      const int ox2 = a.out_stuff ? 2 * ox : ox;
      T *dst = out + ((int64_t)(s * a.Ho + oy) * wout + ox2) * a.out_pitch + a.out_coff + c;
      Elem<T>::store(dst, y);
      if (a.out_stuff) Elem<T>::store(dst + a.out_pitch, 0.f);
    }
  }
  if (a.pool_out) {                    // deterministic global average pool
    sync();
    for (int i = tid; i < cg; i += nthr) {
      float acc = 0.f;
      for (int p = 0; p < P; ++p) acc += base[(int64_t)(c0 + i) * a.N + s * P + p];
      a.out_f32[(int64_t)s * a.M + c0 + i] = acc / P;
    }
  }
}

}  // namespace auras
