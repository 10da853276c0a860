// Exact all-pairs t-force repulsion (P:454, P:463-465 Eq. repfK) + CSR attraction
// + position update — sm_100a.
//
// exact_partial: unit of work = (block of 1024 targets, source chunk c).  Each thread
// holds kExactTPT targets in registers; sources are staged through shared memory in
// tiles of kExactTile float2 and read back as warp-wide broadcasts, so one LDS.64 feeds
// kExactTPT pair evaluations.  Per pair (gamma = 2): 2 FADD, 2 FFMA (s = 1 + d^2),
// 1 MUFU.RCP, 1 FMUL, 2 FFMA (accumulate) — the FP32/SFU-pipe bound of DESIGN.md §Kernels.
// Sums: fp32 within a tile (<= 1024 terms), fp64 across tiles and chunks.  Source chunks
// depend on n only, and every target sums its chunks in index order, so the forces are
// bitwise identical for any number of target shards (R15).
#include "device_math.cuh"
#include "tfdp_internal.h"

namespace tfdp {

template <int G>
__global__ void __launch_bounds__(kExactThreads)
exact_partial_kernel(const float2* __restrict__ xy, int64_t n, int64_t lo, int64_t n_local,
                     int64_t chunk, float neg_gamma, double2* __restrict__ part) {
  __shared__ float2 tile[kExactTile];
  const int c = blockIdx.y;
  const int64_t src_begin = (int64_t)c * chunk;
  const int64_t src_end = min(n, src_begin + chunk);
  const int64_t tbase = (int64_t)blockIdx.x * kExactTargetsPerBlock + threadIdx.x;

  float tx[kExactTPT], ty[kExactTPT];
  double ax[kExactTPT], ay[kExactTPT];
#pragma unroll
  for (int r = 0; r < kExactTPT; ++r) {
    const int64_t t = tbase + (int64_t)r * kExactThreads;
    const float2 p = (t < n_local) ? xy[lo + t] : make_float2(0.f, 0.f);
    tx[r] = p.x;
    ty[r] = p.y;
    ax[r] = 0.0;
    ay[r] = 0.0;
  }

  for (int64_t base = src_begin; base < src_end; base += kExactTile) {
    const int cnt = (int)min((int64_t)kExactTile, src_end - base);
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += kExactThreads) tile[j] = xy[base + j];
    __syncthreads();
    float fx[kExactTPT], fy[kExactTPT];
#pragma unroll
    for (int r = 0; r < kExactTPT; ++r) fx[r] = fy[r] = 0.f;
#pragma unroll 4
    for (int j = 0; j < cnt; ++j) {
      const float2 q = tile[j];
#pragma unroll
      for (int r = 0; r < kExactTPT; ++r) {
        const float dx = tx[r] - q.x;  // r_ij = x_i - x_j
        const float dy = ty[r] - q.y;
        const float s = fmaf(dx, dx, fmaf(dy, dy, 1.0f));  // 1 + |r_ij|^2
        const float wgt = pow_neg<G>(s, neg_gamma);        // (1 + d^2)^-gamma
        fx[r] = fmaf(wgt, dx, fx[r]);
        fy[r] = fmaf(wgt, dy, fy[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < kExactTPT; ++r) {
      ax[r] += (double)fx[r];
      ay[r] += (double)fy[r];
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
                                                 float alpha, float beta) {
  const float2 s = attraction_sum(xy, xi, row_ptr, col, i, beta);
  return make_float2(-alpha * s.x, -alpha * s.y);
}

__global__ void __launch_bounds__(kNodeThreads)
exact_finish_kernel(const float2* __restrict__ xy, float2* __restrict__ xy_next, int64_t lo,
                    int64_t n_local, int n_chunks, const double2* __restrict__ part,
                    const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                    ForceArgs fa, float eta, int iter, int update, float2* __restrict__ rep_out,
                    float2* __restrict__ att_out, unsigned long long* diverge) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_local) return;
  const int64_t i = lo + t;
  double sx = 0.0, sy = 0.0;
  for (int c = 0; c < n_chunks; ++c) {  // fixed chunk order -> deterministic (R15)
    const double2 d = part[(int64_t)c * n_local + t];
    sx += d.x;
    sy += d.y;
  }
  const float Rx = (float)(fa.rho * sx), Ry = (float)(fa.rho * sy);
  const float2 xi = xy[i];
  const float2 A = attraction_row(xy, xi, row_ptr, col, i, fa.alpha, fa.beta);
  if (update) {
    const float nx = fmaf(eta, Rx + A.x, xi.x);
    const float ny = fmaf(eta, Ry + A.y, xi.y);
    xy_next[i] = make_float2(nx, ny);
    if (!isfinite(nx) || !isfinite(ny))
      atomicMin(diverge, ((unsigned long long)(unsigned)iter << 32) | (unsigned long long)i);
  } else {
    if (rep_out) rep_out[t] = make_float2(Rx, Ry);
    if (att_out) att_out[t] = A;
  }
}

void launch_exact_finish(const float2* xy, float2* xy_next, int64_t lo, int64_t n_local,
                         int n_chunks, const double2* part, const int64_t* row_ptr,
                         const int32_t* col, ForceArgs fa, float eta, int iter, int update,
                         float2* rep_out, float2* att_out, unsigned long long* diverge,
                         cudaStream_t s) {
  if (n_local <= 0) return;
  const unsigned blocks = (unsigned)((n_local + kNodeThreads - 1) / kNodeThreads);
  exact_finish_kernel<<<blocks, kNodeThreads, 0, s>>>(xy, xy_next, lo, n_local, n_chunks, part,
                                                      row_ptr, col, fa, eta, iter, update,
                                                      rep_out, att_out, diverge);
}

}  // namespace tfdp
