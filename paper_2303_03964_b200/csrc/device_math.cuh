// Small device helpers shared by the sm_100a kernels (product path only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tfdp_internal.h"

namespace tfdp {

// PDL (tfdp_internal.h launch_chained): let the next chain kernel be scheduled now / wait
// until the predecessor grid has completed with its writes visible.  No-ops for kernels
// launched without the attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// MUFU.RCP: one SFU op, ~1 ulp.  s = 1 + d^2 >= 1 so no denormal inputs.
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// s^-gamma for s >= 1.  G = 1..8: integer gamma (1 MUFU + G-1.. FMULs); G = 0: general
// gamma via exp2(-gamma log2 s) (2 MUFU).  The t-kernel K = (1 + d^2)^-gamma.
template <int G>
__device__ __forceinline__ float pow_neg(float s, float neg_gamma) {
  if constexpr (G == 0) {
    return ex2_approx(neg_gamma * lg2_approx(s));
  } else {
    const float r = rcp_approx(s);
    if constexpr (G == 1) return r;
    if constexpr (G == 2) return r * r;
    if constexpr (G == 3) return r * r * r;
    if constexpr (G == 4) { const float r2 = r * r; return r2 * r2; }
    float q = r;
#pragma unroll
    for (int i = 1; i < G; ++i) q *= r;
    return q;
  }
}

// Order-preserving float <-> uint mapping for exact atomic min/max of fp32 values.
__device__ __forceinline__ unsigned int f2key(float f) {
  const unsigned int u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(unsigned int k) {
  const unsigned int u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// Attraction of one CSR row (P:286-288 Eq. newforce, phi = 1 t-force term R17), without
// the -alpha factor: sum_j (1 + beta / (1 + d^2)) (x_i - x_j).  Four edges per round: all
// column indices, then all neighbour positions are loaded before any arithmetic, so a
// thread keeps up to 8 independent loads in flight (the row walk is latency-bound).
__device__ __forceinline__ float2 attraction_edges(const float2* __restrict__ xy, float2 xi,
                                                   const int32_t* __restrict__ col, int64_t e,
                                                   int64_t e1, float beta) {
  float sx = 0.f, sy = 0.f;
  auto term = [&](float2 xj) {
    const float dx = xi.x - xj.x, dy = xi.y - xj.y;
    const float s = fmaf(dx, dx, fmaf(dy, dy, 1.0f));
    const float c = fmaf(beta, rcp_approx(s), 1.0f);
    sx = fmaf(c, dx, sx);
    sy = fmaf(c, dy, sy);
  };
  for (; e + 4 <= e1; e += 4) {
    const int j0 = __ldg(col + e), j1 = __ldg(col + e + 1), j2 = __ldg(col + e + 2),
              j3 = __ldg(col + e + 3);
    const float2 x0 = __ldg(xy + j0), x1 = __ldg(xy + j1), x2 = __ldg(xy + j2), x3 = __ldg(xy + j3);
    term(x0);
    term(x1);
    term(x2);
    term(x3);
  }
  for (; e < e1; ++e) term(__ldg(xy + __ldg(col + e)));
  return make_float2(sx, sy);
}

__device__ __forceinline__ float2 attraction_sum(const float2* __restrict__ xy, float2 xi,
                                                 const int64_t* __restrict__ row_ptr,
                                                 const int32_t* __restrict__ col, int64_t i,
                                                 float beta) {
  return attraction_edges(xy, xi, col, row_ptr[i], row_ptr[i + 1], beta);
}

// Row sum with the heavy-row split: rows above kHeavyDeg edges add their precomputed chunk
// sums in chunk order (kernels_heavy.cu); the others walk their edges.
__device__ __forceinline__ float2 attraction_sum_hv(const float2* __restrict__ xy, float2 xi,
                                                    const int64_t* __restrict__ row_ptr,
                                                    const int32_t* __restrict__ col, int64_t i,
                                                    const ForceArgs& fa) {
  const int64_t e0 = row_ptr[i], e1 = row_ptr[i + 1];
  if (fa.hv_part && e1 - e0 > kHeavyDeg) {
    const long long f = fa.hv_first[i];
    const int nc = (int)((e1 - e0 + kHeavyChunk - 1) / kHeavyChunk);
    float sx = 0.f, sy = 0.f;
    for (int c = 0; c < nc; ++c) {
      const float2 q = fa.hv_part[f + c];
      sx += q.x;
      sy += q.y;
    }
    return make_float2(sx, sy);
  }
  return attraction_edges(xy, xi, col, e0, e1, fa.beta);
}

// Attraction row sum with the refinement mask's edge weight (la on edges whose both ends are
// in the focal region): rows outside the region take the unmasked path (weight 1).
__device__ __forceinline__ float2 attraction_sum_masked(const float2* __restrict__ xy, float2 xi,
                                                        const int64_t* __restrict__ row_ptr,
                                                        const int32_t* __restrict__ col,
                                                        int64_t i, float beta,
                                                        const unsigned char* __restrict__ label,
                                                        float la) {
  if (!label || !label[i]) return attraction_sum(xy, xi, row_ptr, col, i, beta);
  float sx = 0.f, sy = 0.f;
  for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
    const int j = __ldg(col + e);
    const float2 xj = __ldg(xy + j);
    const float dx = xi.x - xj.x, dy = xi.y - xj.y;
    const float s = fmaf(dx, dx, fmaf(dy, dy, 1.0f));
    float c = fmaf(beta, rcp_approx(s), 1.0f);
    if (label[j]) c *= la;
    sx = fmaf(c, dx, sx);
    sy = fmaf(c, dy, sy);
  }
  return make_float2(sx, sy);
}

// Masked repulsion from the unmasked R (already x rho) and the region sum S1 (R23):
// rho [w0 (S - S1) + w1 S1] = w0 R + rho (w1 - w0) S1.
__device__ __forceinline__ float2 focus_repulsion(float2 R, int64_t i, int64_t t, float rho,
                                                  const FocusArgs& fo) {
  const bool in = fo.label[i] != 0;
  const float w0 = in ? 1.0f : fo.ls, w1 = in ? fo.lf : 1.0f;
  const float c = rho * (w1 - w0);
  const float2 s1 = fo.s1[t];
  return make_float2(fmaf(c, s1.x, w0 * R.x), fmaf(c, s1.y, w0 * R.y));
}

// Lagrange basis on K equispaced nodes t_c = (c + 1/2)/K of [0, 1] (R8):
// l_c(u) = prod_{c' != c} (u - t_c') / (t_c - t_c').  Constants fold at compile time.
template <int K>
__device__ __forceinline__ void lagrange(float u, float (&l)[K]) {
#pragma unroll
  for (int c = 0; c < K; ++c) {
    float v = 1.0f;
#pragma unroll
    for (int cp = 0; cp < K; ++cp) {
      if (cp != c) {
        const float tc = (c + 0.5f) / K, tcp = (cp + 0.5f) / K;
        v *= (u - tcp) * (1.0f / (tc - tcp));
      }
    }
    l[c] = v;
  }
}

}  // namespace tfdp
