// PivotMDS initialisation on the device (NEXT-2, SPEC init_pivot_mds S:110-118,
// Brandes & Pich 2006).  Steps:
//   1. p pivots by max-min farthest-point selection: one cooperative BFS kernel per pivot
//      (level-synchronous frontier queues, grid.sync between levels), then a column kernel
//      that writes D[:, j] (unreachable -> eccentricity + 1, R24), updates the min-distance
//      to the pivot set and selects the next pivot with one 64-bit atomicMax of
//      (min distance, ~index) — ties go to the lowest index;
//   2. double centring of the squared distances (row means, column means, grand mean) and
//      the p x p Gram matrix C^T C of C = -1/2 (D2 - r - c + g), accumulated per block in
//      fp64 over fixed row ranges and summed in a fixed order (deterministic);
//   3. top-2 eigenvectors of C^T C by power iteration with deflation (one block, fp64),
//      sign rule: largest-|.| component positive;
//   4. positions C v_k, centred, scaled to mean edge length 1 (fixed-order reductions).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "device_math.cuh"
#include "tfdp_internal.h"

namespace cg = cooperative_groups;

namespace tfdp {

namespace {

constexpr int kBfsThreads = 256;
constexpr int kRed = 256;

__global__ void __launch_bounds__(kBfsThreads)
bfs_coop_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int src,
                int* __restrict__ dist, int* __restrict__ q0, int* __restrict__ q1,
                int* __restrict__ cnt /*[4]: 3 rotating sizes + ecc*/) {
  cg::grid_group grid = cg::this_grid();
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int nt = gridDim.x * blockDim.x;
  if (gt == 0) {
    dist[src] = 0;
    q0[0] = src;
    cnt[0] = 1;
    cnt[1] = 0;
    cnt[2] = 0;
  }
  grid.sync();
  int* cur = q0;
  int* nxt = q1;
  int level = 0;
  for (;;) {
    const int size = __ldcg(cnt + level % 3);
    if (size == 0) break;
    int* next_cnt = cnt + (level + 1) % 3;
    for (int idx = gt; idx < size; idx += nt) {
      const int u = __ldcg(cur + idx);
      for (int64_t e = rp[u]; e < rp[u + 1]; ++e) {
        const int v = col[e];
        if (__ldcg(dist + v) < 0 && atomicCAS(dist + v, -1, level + 1) == -1) {
          cg::coalesced_group g = cg::coalesced_threads();
          int base = 0;
          if (g.thread_rank() == 0) base = atomicAdd(next_cnt, (int)g.size());
          base = g.shfl(base, 0);
          nxt[base + g.thread_rank()] = v;
        }
      }
    }
    if (gt == 0) cnt[(level + 2) % 3] = 0;
    grid.sync();
    int* t = cur;
    cur = nxt;
    nxt = t;
    ++level;
  }
  if (gt == 0) cnt[3] = level - 1;  // eccentricity of src within its component
}

// D[:, j] (column-major, int32), min distance to the pivot set, next-pivot key.
__global__ void __launch_bounds__(256)
pmds_column_kernel(const int* __restrict__ dist, int n, const int* __restrict__ cnt,
                   int* __restrict__ Dj, int* __restrict__ mind, int first,
                   unsigned long long* __restrict__ best) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long key = 0ull;
  if (i < n) {
    const int d = dist[i] >= 0 ? dist[i] : cnt[3] + 1;
    Dj[i] = d;
    const int m = first ? d : min(mind[i], d);
    mind[i] = m;
    key = ((unsigned long long)(unsigned)m << 32) | (unsigned long long)(0xffffffffu - (unsigned)i);
  }
  // warp max of the key (distance, then lowest index)
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, key, o);
    key = y > key ? y : key;
  }
  if ((threadIdx.x & 31) == 0 && key) atomicMax(best, key);
}

// fixed-order block sums: part[b] = sum of v over [b * per, (b + 1) * per)
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double s[kRed];
  s[threadIdx.x] = v;
  __syncthreads();
  for (int w = kRed / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  const double r = s[0];
  __syncthreads();
  return r;
}

// row means r_i = mean_j D_ij^2
__global__ void __launch_bounds__(256)
pmds_rowmean_kernel(const int* __restrict__ D, int n, int p, double* __restrict__ r) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int j = 0; j < p; ++j) {
    const double d = (double)D[(int64_t)j * n + i];
    s += d * d;
  }
  r[i] = s / p;
}

// column means c_j = mean_i D_ij^2: one block per column, fixed strides and tree
__global__ void __launch_bounds__(kRed)
pmds_colmean_kernel(const int* __restrict__ D, int n, double* __restrict__ c) {
  const int j = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += kRed) {
    const double d = (double)D[(int64_t)j * n + i];
    s += d * d;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) c[j] = s / n;
}

// Gram partials: block b accumulates C^T C over rows [b * rows_per, ...) (upper triangle)
constexpr int kMaxPivots = 64;
constexpr int kGramRows = 32;

__global__ void __launch_bounds__(256)
pmds_gram_kernel(const int* __restrict__ D, int n, int p, const double* __restrict__ r,
                 const double* __restrict__ c, int rows_per, double* __restrict__ part) {
  __shared__ double tile[kGramRows][kMaxPivots];
  __shared__ double cs[kMaxPivots];
  __shared__ double gsh;
  if (threadIdx.x == 0) {
    double g = 0.0;
    for (int j = 0; j < p; ++j) g += c[j];
    gsh = g / p;
  }
  for (int j = threadIdx.x; j < p; j += blockDim.x) cs[j] = c[j];
  __syncthreads();
  const double g = gsh;
  const int npairs = p * (p + 1) / 2;
  double acc[9];  // <= ceil(2080 / 256) = 9 pairs per thread
  int pa[9], pb[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    acc[q] = 0.0;
    // pair index -> (a, b), a <= b, row-major upper triangle
    int a = 0, rem = threadIdx.x + q * blockDim.x;
    while (a < p && rem >= p - a) {
      rem -= p - a;
      ++a;
    }
    pa[q] = a;
    pb[q] = a + rem;
  }
  const int r0 = blockIdx.x * rows_per, r1 = min(n, r0 + rows_per);
  for (int base = r0; base < r1; base += kGramRows) {
    const int rows = min(kGramRows, r1 - base);
    __syncthreads();
    for (int t = threadIdx.x; t < rows * p; t += blockDim.x) {
      const int rr = t / p, j = t - rr * p;
      const int i = base + rr;
      const double d = (double)D[(int64_t)j * n + i];
      tile[rr][j] = -0.5 * (d * d - r[i] - cs[j] + g);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const int pr = threadIdx.x + q * blockDim.x;
      if (pr < npairs) {
        const int a = pa[q], b = pb[q];
        double s = acc[q];
        for (int rr = 0; rr < rows; ++rr) s = fma(tile[rr][a], tile[rr][b], s);
        acc[q] = s;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const int pr = threadIdx.x + q * blockDim.x;
    if (pr < npairs) part[(int64_t)blockIdx.x * npairs + pr] = acc[q];
  }
}

// fixed-order sum of the Gram partials -> full symmetric M[p][p]
__global__ void pmds_gram_reduce_kernel(const double* __restrict__ part, int nb, int p,
                                        double* __restrict__ M) {
  const int npairs = p * (p + 1) / 2;
  for (int pr = blockIdx.x * blockDim.x + threadIdx.x; pr < npairs; pr += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[(int64_t)b * npairs + pr];
    int a = 0, rem = pr;
    while (rem >= p - a) {
      rem -= p - a;
      ++a;
    }
    const int bb = a + rem;
    M[a * p + bb] = s;
    M[bb * p + a] = s;
  }
}

// Power iteration with deflation for the top-2 eigenvectors of M (one block, p <= 64).
__global__ void __launch_bounds__(64)
pmds_eig_kernel(const double* __restrict__ M, int p, double* __restrict__ V /*[2][p]*/,
                double* __restrict__ lam /*[2]*/) {
  __shared__ double v[kMaxPivots], w[kMaxPivots], u1[kMaxPivots];
  __shared__ double red[2];
  const int j = threadIdx.x;
  for (int a = 0; a < 2; ++a) {
    if (j < p) v[j] = 1.0 + (double)j / (double)(p + 1) + 0.5 * a * ((j & 1) ? -1.0 : 1.0);
    __syncthreads();
    double lambda = 0.0;
    for (int it = 0; it < 200000; ++it) {
      if (j < p) {
        double s = 0.0;
        for (int k = 0; k < p; ++k) s = fma(M[j * p + k], v[k], s);
        w[j] = s;
      }
      __syncthreads();
      if (a == 1) {  // deflate: w -= (u1 . w) u1
        if (j == 0) {
          double d = 0.0;
          for (int k = 0; k < p; ++k) d = fma(u1[k], w[k], d);
          red[0] = d;
        }
        __syncthreads();
        if (j < p) w[j] -= red[0] * u1[j];
        __syncthreads();
      }
      if (j == 0) {
        double nn = 0.0;
        for (int k = 0; k < p; ++k) nn = fma(w[k], w[k], nn);
        red[1] = sqrt(nn);
      }
      __syncthreads();
      lambda = red[1];
      double diff = 0.0;
      if (lambda > 0.0 && j < p) {
        const double nv = w[j] / lambda;
        diff = fabs(nv - v[j]);
        v[j] = nv;
      }
      // block-wide max of diff (p <= 64: two warps)
      __shared__ double dmax[2];
      double dm = diff;
      for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
      if ((j & 31) == 0) dmax[j >> 5] = dm;
      __syncthreads();
      const double dd = fmax(dmax[0], blockDim.x > 32 ? dmax[1] : 0.0);
      __syncthreads();
      if (lambda == 0.0 || dd < 1e-15) break;
    }
    // sign rule: largest |component| positive (lowest index on ties)
    if (j == 0) {
      int arg = 0;
      for (int k = 1; k < p; ++k)
        if (fabs(v[k]) > fabs(v[arg])) arg = k;
      red[0] = v[arg] < 0 ? -1.0 : 1.0;
      lam[a] = lambda;
    }
    __syncthreads();
    if (j < p) {
      v[j] *= red[0];
      V[a * p + j] = v[j];
      if (a == 0) u1[j] = v[j];
    }
    __syncthreads();
  }
}

// positions C v_k (fp64) -> tmp[i]; block partial sums of the coordinates
__global__ void __launch_bounds__(kRed)
pmds_project_kernel(const int* __restrict__ D, int n, int p, const double* __restrict__ r,
                    const double* __restrict__ c, const double* __restrict__ V,
                    const double* __restrict__ lam, double2* __restrict__ X,
                    double* __restrict__ part /*[2][nb]*/) {
  __shared__ double cs[kMaxPivots], v0[kMaxPivots], v1[kMaxPivots];
  __shared__ double gsh;
  if (threadIdx.x == 0) {
    double g = 0.0;
    for (int j = 0; j < p; ++j) g += c[j];
    gsh = g / p;
  }
  const bool use1 = lam[1] > 1e-12 * lam[0];  // rank < 2: the second axis stays 0 (R24)
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    cs[j] = c[j];
    v0[j] = lam[0] > 0.0 ? V[j] : 0.0;
    v1[j] = use1 ? V[p + j] : 0.0;
  }
  __syncthreads();
  const int i = blockIdx.x * kRed + threadIdx.x;
  double x = 0.0, y = 0.0;
  if (i < n) {
    const double g = gsh;
    for (int j = 0; j < p; ++j) {
      const double d = (double)D[(int64_t)j * n + i];
      const double cij = -0.5 * (d * d - r[i] - cs[j] + g);
      x = fma(cij, v0[j], x);
      y = fma(cij, v1[j], y);
    }
    X[i] = make_double2(x, y);
  }
  const double sx = block_sum(x);
  const double sy = block_sum(y);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = sx;
    part[gridDim.x + blockIdx.x] = sy;
  }
}

// mean edge length partials of the centred positions (caller-order CSR, one row per thread)
__global__ void __launch_bounds__(kRed)
pmds_edge_kernel(const double2* __restrict__ X, int n, const int64_t* __restrict__ rp,
                 const int32_t* __restrict__ col, double* __restrict__ part) {
  const int i = blockIdx.x * kRed + threadIdx.x;
  double s = 0.0;
  if (i < n) {
    const double2 a = X[i];
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const double2 b = X[col[e]];
      s += sqrt((a.x - b.x) * (a.x - b.x) + (a.y - b.y) * (a.y - b.y));
    }
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// sums the nb partials in a fixed order into out[k] for k < nk (part layout [nk][nb])
__global__ void __launch_bounds__(kRed)
pmds_sum_kernel(const double* __restrict__ part, int nb, int nk, double* __restrict__ out) {
  for (int k = 0; k < nk; ++k) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nb; b += kRed) s += part[(int64_t)k * nb + b];
    s = block_sum(s);
    if (threadIdx.x == 0) out[k] = s;
  }
}

__global__ void __launch_bounds__(kRed)
pmds_finish_kernel(const double2* __restrict__ X, int n, const double* __restrict__ sums,
                   double nnz, float2* __restrict__ xy) {
  const int i = blockIdx.x * kRed + threadIdx.x;
  if (i >= n) return;
  const double mx = sums[0] / n, my = sums[1] / n;
  const double L = nnz > 0 ? sums[2] / nnz : 0.0;
  const double s = L > 0 ? 1.0 / L : 1.0;
  const double2 a = X[i];
  xy[i] = make_float2((float)((a.x - mx) * s), (float)((a.y - my) * s));
}

unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace

int pmds_max_pivots() { return kMaxPivots; }

size_t pmds_scratch_bytes(int64_t n, int p) {
  const int64_t nb = nblk(n, kRed);
  const int npairs = p * (p + 1) / 2;
  const int64_t gb = std::min<int64_t>(1184, nb);
  return (size_t)n * 4 * 4            // dist, q0, q1, mind
         + (size_t)n * p * 4          // D
         + (size_t)n * 8 + 64 * 8     // r, c
         + (size_t)n * 16             // X
         + (size_t)gb * npairs * 8    // gram partials
         + (size_t)p * p * 8 + 4 * p * 8 + (size_t)3 * nb * 8 + 1024 + 20 * 256;  // + take() rounding
}

// Returns the number of kernel launches; pivots_out (host, p entries) receives the pivots.
cudaError_t launch_pmds(const int64_t* rp, const int32_t* col, int64_t n64, int64_t nnz, int p,
                        unsigned long long seed_pivot, void* scratch, float2* xy,
                        int* pivots_out, int64_t* launches, const char** stage,
                        cudaStream_t s) {
  const int n = (int)n64;
  *stage = "";
  char* q = static_cast<char*>(scratch);
  auto take = [&](size_t b) {
    char* r = q;
    q += (b + 255) / 256 * 256;
    return r;
  };
  int* dist = (int*)take((size_t)n * 4);
  int* q0 = (int*)take((size_t)n * 4);
  int* q1 = (int*)take((size_t)n * 4);
  int* mind = (int*)take((size_t)n * 4);
  int* D = (int*)take((size_t)n * p * 4);
  double* r = (double*)take((size_t)n * 8);
  double* c = (double*)take(64 * 8);
  double2* X = (double2*)take((size_t)n * 16);
  const int nb = (int)nblk(n, kRed);
  const int gram_blocks = std::min(1184, nb);
  const int npairs = p * (p + 1) / 2;
  double* gpart = (double*)take((size_t)gram_blocks * npairs * 8);
  double* M = (double*)take((size_t)p * p * 8);
  double* V = (double*)take((size_t)2 * p * 8);
  double* lam = (double*)take(2 * 8);
  double* part = (double*)take((size_t)3 * nb * 8);
  double* sums = (double*)take(4 * 8);
  int* cnt = (int*)take(4 * 4);
  unsigned long long* best = (unsigned long long*)take(8);

  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_coop_kernel, kBfsThreads, 0);
  if (e != cudaSuccess) {
    *stage = "occupancy";
    return e;
  }
  const int bfs_blocks = std::max(1, std::min(nsm * per_sm, (int)nblk(n, kBfsThreads)));
  int64_t L = 0;
  int piv = (int)(seed_pivot % (unsigned long long)n);
  for (int j = 0; j < p; ++j) {
    pivots_out[j] = piv;
    cudaMemsetAsync(dist, 0xff, (size_t)n * 4, s);
    void* args[] = {(void*)&rp, (void*)&col, (void*)&piv, (void*)&dist, (void*)&q0, (void*)&q1, (void*)&cnt};
    e = cudaLaunchCooperativeKernel((void*)bfs_coop_kernel, bfs_blocks, kBfsThreads, args, 0, s);
    if (e != cudaSuccess) {
      *stage = "cooperative BFS launch";
      return e;
    }
    e = cudaMemsetAsync(best, 0, 8, s);
    if (e != cudaSuccess) {
      *stage = "memset best";
      return e;
    }
    pmds_column_kernel<<<nblk(n, 256), 256, 0, s>>>(dist, n, cnt, D + (int64_t)j * n, mind,
                                                     j == 0 ? 1 : 0, best);
    e = cudaGetLastError();
    if (e != cudaSuccess) {
      *stage = "column kernel launch";
      return e;
    }
    L += 2;
    if (j + 1 < p) {
      unsigned long long key = 0;
      e = cudaMemcpyAsync(&key, best, 8, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) {
        *stage = "pivot selection";
        return e;
      }
      piv = (int)(0xffffffffu - (unsigned)(key & 0xffffffffull));
    }
  }
  pmds_rowmean_kernel<<<nblk(n, 256), 256, 0, s>>>(D, n, p, r);
  pmds_colmean_kernel<<<p, kRed, 0, s>>>(D, n, c);
  const int rows_per = (n + gram_blocks - 1) / gram_blocks;
  pmds_gram_kernel<<<gram_blocks, 256, 0, s>>>(D, n, p, r, c, rows_per, gpart);
  pmds_gram_reduce_kernel<<<nblk(npairs, 256), 256, 0, s>>>(gpart, gram_blocks, p, M);
  pmds_eig_kernel<<<1, 64, 0, s>>>(M, p, V, lam);
  pmds_project_kernel<<<nb, kRed, 0, s>>>(D, n, p, r, c, V, lam, X, part);
  pmds_sum_kernel<<<1, kRed, 0, s>>>(part, nb, 2, sums);
  // centre in place before the edge lengths (they are translation invariant, but the
  // finish kernel reuses the same sums)
  pmds_edge_kernel<<<nb, kRed, 0, s>>>(X, n, rp, col, part + 2 * nb);
  pmds_sum_kernel<<<1, kRed, 0, s>>>(part + 2 * nb, nb, 1, sums + 2);
  pmds_finish_kernel<<<nb, kRed, 0, s>>>(X, n, sums, (double)nnz, xy);
  L += 11;
  *launches += L;
  *stage = "centring / Gram / eigen / projection";
  return cudaGetLastError();
}

}  // namespace tfdp
