// Exact all-pairs t-force repulsion (P:454, P:463-465 Eq. repfK) + CSR attraction
// + position update — sm_100a.
//
// exact_partial: unit of work = (block of 1024 targets, source chunk c).  Each thread
// holds kExactTPT targets in registers; sources are staged through shared memory as two
// float arrays (x, y) and read back in pairs (j, j+1) as warp-wide LDS.64 broadcasts.  The
// pair arithmetic runs on packed fp32x2 instructions (sm_100a FADD2 / FFMA2 / FMUL2) with
// lanes = the two sources: per two pairs (gamma = 2) 2 FADD2 (dx, dy), 2 FFMA2 (s = 1 + d^2),
// 2 MUFU.RCP, 1 FMUL2 (w^2), 2 FFMA2 (accumulate) = 4.5 issue slots per pair: bound by the
// SFU (one MUFU.RCP per pair) with the FMA pipe at ~88 % of it (moving one reciprocal in
// 8..64 to an FMA-pipe Newton iteration measured slower: tools/mbench_exact.cu v3) —
// DESIGN.md §Kernels.  Sums: fp32 within a
// tile (<= 1024 terms, even and odd sources in separate lanes), fp64 across tiles and
// chunks.  Source chunks depend on n only, and every target sums its chunks in index order,
// so the forces are bitwise identical for any number of target shards (R15).
#include "device_math.cuh"
#include "tfdp_internal.h"

namespace tfdp {

namespace {
using u64 = unsigned long long;
__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(u64 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// (1 + d^2)^-gamma for the two lanes of s
template <int G>
__device__ __forceinline__ u64 weight2(u64 s, float neg_gamma) {
  float s1, s2;
  upk(s, s1, s2);
  if constexpr (G == 2) {
    const u64 w = pk(rcp_approx(s1), rcp_approx(s2));
    return mul2(w, w);
  } else {
    return pk(pow_neg<G>(s1, neg_gamma), pow_neg<G>(s2, neg_gamma));
  }
}
}  // namespace

template <int G>
__global__ void __launch_bounds__(kExactThreads)
exact_partial_kernel(const float2* __restrict__ xy, int64_t n, int64_t lo, int64_t n_local,
                     int64_t chunk, float neg_gamma, double2* __restrict__ part) {
  __shared__ __align__(16) float xs[kExactTile];
  __shared__ __align__(16) float ys[kExactTile];
  const int c = blockIdx.y;
  const int64_t src_begin = (int64_t)c * chunk;
  const int64_t src_end = min(n, src_begin + chunk);
  const int64_t tbase = (int64_t)blockIdx.x * kExactTargetsPerBlock + threadIdx.x;

  u64 tx[kExactTPT], ty[kExactTPT];  // (x_i, x_i), (y_i, y_i)
  double ax[kExactTPT], ay[kExactTPT];
#pragma unroll
  for (int r = 0; r < kExactTPT; ++r) {
    const int64_t t = tbase + (int64_t)r * kExactThreads;
    const float2 p = (t < n_local) ? xy[lo + t] : make_float2(0.f, 0.f);
    tx[r] = pk(p.x, p.x);
    ty[r] = pk(p.y, p.y);
    ax[r] = 0.0;
    ay[r] = 0.0;
  }
  const u64 one = pk(1.0f, 1.0f);

  for (int64_t base = src_begin; base < src_end; base += kExactTile) {
    const int cnt = (int)min((int64_t)kExactTile, src_end - base);
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += kExactThreads) {
      const float2 p = xy[base + j];
      xs[j] = p.x;
      ys[j] = p.y;
    }
    __syncthreads();
    u64 fx[kExactTPT], fy[kExactTPT];  // lanes: even / odd sources of the tile
#pragma unroll
    for (int r = 0; r < kExactTPT; ++r) fx[r] = fy[r] = pk(0.f, 0.f);
    const int cnt2 = cnt & ~1;
    int j = 0;
    // 32 source pairs per round, fully unrolled (C5: 4.17 -> 4.35e12 pairs/s against the
    // 2-pair unroll), then the remainder of a partial tile
    constexpr int kPairsPerRound = 32;
    for (; j + 2 * kPairsPerRound <= cnt2; j += 2 * kPairsPerRound) {
#pragma unroll
      for (int jj = 0; jj < kPairsPerRound; ++jj) {
        const u64 qx = *reinterpret_cast<const u64*>(xs + j + 2 * jj);  // (x_j, x_j+1)
        const u64 qy = *reinterpret_cast<const u64*>(ys + j + 2 * jj);
#pragma unroll
        for (int r = 0; r < kExactTPT; ++r) {
          const u64 dx = sub2(tx[r], qx);  // r_ij = x_i - x_j
          const u64 dy = sub2(ty[r], qy);
          const u64 sq = fma2(dy, dy, fma2(dx, dx, one));  // 1 + |r_ij|^2
          const u64 w = weight2<G>(sq, neg_gamma);         // (1 + d^2)^-gamma
          fx[r] = fma2(w, dx, fx[r]);
          fy[r] = fma2(w, dy, fy[r]);
        }
      }
    }
#pragma unroll 2
    for (; j < cnt2; j += 2) {
      const u64 qx = *reinterpret_cast<const u64*>(xs + j);  // (x_j, x_j+1)
      const u64 qy = *reinterpret_cast<const u64*>(ys + j);
#pragma unroll
      for (int r = 0; r < kExactTPT; ++r) {
        const u64 dx = sub2(tx[r], qx);  // r_ij = x_i - x_j
        const u64 dy = sub2(ty[r], qy);
        const u64 s = fma2(dy, dy, fma2(dx, dx, one));  // 1 + |r_ij|^2
        const u64 w = weight2<G>(s, neg_gamma);         // (1 + d^2)^-gamma
        fx[r] = fma2(w, dx, fx[r]);
        fy[r] = fma2(w, dy, fy[r]);
      }
    }
    if (cnt2 < cnt) {  // odd tail: one source in lane 0, lane 1 contributes 0
      const u64 qx = pk(xs[cnt2], 0.f), qy = pk(ys[cnt2], 0.f);
      const u64 lane0 = pk(1.0f, 0.0f);
#pragma unroll
      for (int r = 0; r < kExactTPT; ++r) {
        const u64 dx = mul2(sub2(tx[r], qx), lane0);
        const u64 dy = mul2(sub2(ty[r], qy), lane0);
        const u64 s = fma2(dy, dy, fma2(dx, dx, one));
        const u64 w = weight2<G>(s, neg_gamma);
        fx[r] = fma2(w, dx, fx[r]);
        fy[r] = fma2(w, dy, fy[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < kExactTPT; ++r) {
      float a0, a1, b0, b1;
      upk(fx[r], a0, a1);
      upk(fy[r], b0, b1);
      ax[r] += (double)a0 + (double)a1;
      ay[r] += (double)b0 + (double)b1;
    }
  }
#pragma unroll
  for (int r = 0; r < kExactTPT; ++r) {
    const int64_t t = tbase + (int64_t)r * kExactThreads;
    if (t < n_local) part[(int64_t)c * n_local + t] = make_double2(ax[r], ay[r]);
  }
}

void launch_exact_partial(const float2* xy, int64_t n, int64_t lo, int64_t n_local,
                          int64_t chunk, int n_chunks, ForceArgs fa, double2* part,
                          cudaStream_t s) {
  if (n_local <= 0) return;
  dim3 grid((unsigned)((n_local + kExactTargetsPerBlock - 1) / kExactTargetsPerBlock),
            (unsigned)n_chunks);
  const float ng = -fa.gamma;
  switch (fa.gamma_int) {
    case 1: exact_partial_kernel<1><<<grid, kExactThreads, 0, s>>>(xy, n, lo, n_local, chunk, ng, part); break;
    case 2: exact_partial_kernel<2><<<grid, kExactThreads, 0, s>>>(xy, n, lo, n_local, chunk, ng, part); break;
    case 3: exact_partial_kernel<3><<<grid, kExactThreads, 0, s>>>(xy, n, lo, n_local, chunk, ng, part); break;
    case 4: exact_partial_kernel<4><<<grid, kExactThreads, 0, s>>>(xy, n, lo, n_local, chunk, ng, part); break;
    case 8: exact_partial_kernel<8><<<grid, kExactThreads, 0, s>>>(xy, n, lo, n_local, chunk, ng, part); break;
    default: exact_partial_kernel<0><<<grid, kExactThreads, 0, s>>>(xy, n, lo, n_local, chunk, ng, part); break;
  }
}

// Attraction over one CSR row: -alpha sum_j (1 + beta / (1 + d^2)) (x_i - x_j).
__device__ __forceinline__ float2 attraction_row(const float2* __restrict__ xy, float2 xi,
                                                 const int64_t* __restrict__ row_ptr,
                                                 const int32_t* __restrict__ col, int64_t i,
                                                 const ForceArgs& fa) {
  const float2 s = attraction_sum_hv(xy, xi, row_ptr, col, i, fa);
  return make_float2(-fa.alpha * s.x, -fa.alpha * s.y);
}

__global__ void __launch_bounds__(kNodeThreads)
exact_finish_kernel(const float2* __restrict__ xy, float2* __restrict__ xy_next, int64_t lo,
                    int64_t n_local, int n_chunks, const double2* __restrict__ part,
                    const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                    ForceArgs fa, FocusArgs fo, float eta, int iter, int update,
                    float2* __restrict__ rep_out, float2* __restrict__ att_out,
                    unsigned long long* diverge, const PeerRoute* __restrict__ rt, int next_buf) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_local) return;
  const int64_t i = lo + t;
  double sx = 0.0, sy = 0.0;
  for (int c = 0; c < n_chunks; ++c) {  // fixed chunk order -> deterministic (R15)
    const double2 d = part[(int64_t)c * n_local + t];
    sx += d.x;
    sy += d.y;
  }
  float Rx = (float)(fa.rho * sx), Ry = (float)(fa.rho * sy);
  const float2 xi = xy[i];
  float2 A;
  if (fo.label) {  // local refinement mask (R23)
    const float2 Rm = focus_repulsion(make_float2(Rx, Ry), i, t, fa.rho, fo);
    Rx = Rm.x;
    Ry = Rm.y;
    const float2 as = attraction_sum_masked(xy, xi, row_ptr, col, i, fa.beta, fo.label, fo.la);
    A = make_float2(-fa.alpha * as.x, -fa.alpha * as.y);
  } else {
    A = attraction_row(xy, xi, row_ptr, col, i, fa);
  }
  if (update) {
    const float nx = fmaf(eta, Rx + A.x, xi.x);
    const float ny = fmaf(eta, Ry + A.y, xi.y);
    xy_next[i] = make_float2(nx, ny);
    if (rt)  // p > 1, fused position all-gather: into every other rank's copy
      for (int j = 0; j < rt->world; ++j)
        if (j != rt->rank) rt->xy[next_buf][j][i] = make_float2(nx, ny);
    if (!isfinite(nx) || !isfinite(ny))
      atomicMin(diverge, ((unsigned long long)(unsigned)iter << 32) | (unsigned long long)i);
  } else {
    if (rep_out) rep_out[t] = make_float2(Rx, Ry);
    if (att_out) att_out[t] = A;
  }
}

void launch_exact_finish(const float2* xy, float2* xy_next, int64_t lo, int64_t n_local,
                         int n_chunks, const double2* part, const int64_t* row_ptr,
                         const int32_t* col, ForceArgs fa, FocusArgs fo, float eta, int iter,
                         int update, float2* rep_out, float2* att_out,
                         unsigned long long* diverge, cudaStream_t s, const PeerRoute* route,
                         int next_buf) {
  if (n_local <= 0) return;
  const unsigned blocks = (unsigned)((n_local + kNodeThreads - 1) / kNodeThreads);
  exact_finish_kernel<<<blocks, kNodeThreads, 0, s>>>(xy, xy_next, lo, n_local, n_chunks, part,
                                                      row_ptr, col, fa, fo, eta, iter, update,
                                                      rep_out, att_out, diverge, route,
                                                      next_buf);
}

}  // namespace tfdp
