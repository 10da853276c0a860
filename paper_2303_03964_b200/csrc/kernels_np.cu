// Neighbourhood preservation NP1 of the current layout on the device (NEXT-3; P:599-606,
// S:421-429): NP1 = (1/n) sum_i |N_G(i) ∩ N_L(i, k_i)| / |N_G(i) ∪ N_L(i, k_i)|, k_i =
// deg(i), N_L = the k_i nearest other nodes in the layout, ties by lower node id, degree-0
// nodes contribute 1.  Both sets have k_i elements, so |∪| = 2 k_i - |∩|: only the
// intersection ("hits") is computed.
//
// Exact kNN membership without materialising neighbour lists:
//   1. uniform G x G cell grid over the bounding square (G = ceil(sqrt(n/2)), ~2 nodes per
//      cell), nodes counting-sorted by cell (histogram, exclusive scan, scatter);
//   2. one warp per target i: expand Chebyshev rings of cells around i's cell until they
//      hold >= k_i + 1 nodes (ring r) — the k-th nearest other node is then within
//      D = sqrt2 (r + 2) cs (one ring of slack for the fp32 cell assignment) — and take the
//      candidates within D from the cells within ceil(D / cs) + 1 rings (each row of cells
//      is one contiguous range of the sorted arrays);
//   3. radix select (4 x 8 bits) of the k-th smallest d^2 among the candidates;
//   4. a graph neighbour j is in N_L iff d_ij^2 < t*, or d_ij^2 == t* and fewer than
//      `want` tied candidates have a lower id (tie rule).
// d^2 = (dx dx) + (dy dy) with every operation rounded in IEEE fp32 (no contraction): the
// oracle's np1_hits(dist="fp32") takes the same integer decisions (R22).
#include <algorithm>
#include <cmath>

#include "device_math.cuh"
#include "tfdp_internal.h"

namespace tfdp {

namespace {

constexpr int kNpWarps = 8;  // warps (targets) per block of the query kernel

struct NpGrid {
  float lo_x, lo_y;
  float cs, inv_cs;  // cell side and its inverse
  int G;
};

__device__ __forceinline__ float d2_rn(float2 a, float2 b) {
  const float dx = __fsub_rn(b.x, a.x), dy = __fsub_rn(b.y, a.y);
  return __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
}

__device__ __forceinline__ int cell_coord(float v, float lo, float inv_cs, int G) {
  const float t = (v - lo) * inv_cs;
  int c = (int)t;  // t >= 0 up to rounding; clamped below
  return min(max(c, 0), G - 1);
}

__global__ void np_grid_kernel(const BoxKeys* __restrict__ keys, int G, NpGrid* __restrict__ out) {
  const BoxKeys b = *keys;
  const float x0 = key2f(b.minx), y0 = key2f(b.miny);
  float L = fmaxf(key2f(b.maxx) - x0, key2f(b.maxy) - y0);
  if (!(L > 0.f)) L = 1.f;  // all points coincident: any cell size works
  NpGrid g;
  g.lo_x = x0;
  g.lo_y = y0;
  g.cs = L / (float)G;
  g.inv_cs = (float)G / L;
  g.G = G;
  *out = g;
}

__global__ void __launch_bounds__(256)
np_count_kernel(const float2* __restrict__ xy, int64_t n, const NpGrid* __restrict__ grid,
                int* __restrict__ cell, long long* __restrict__ hist) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const NpGrid g = *grid;
  const float2 p = xy[i];
  const int c = cell_coord(p.y, g.lo_y, g.inv_cs, g.G) * g.G + cell_coord(p.x, g.lo_x, g.inv_cs, g.G);
  cell[i] = c;
  atomicAdd(reinterpret_cast<unsigned long long*>(hist + c), 1ull);
}

__global__ void __launch_bounds__(256)
np_scatter_kernel(const float2* __restrict__ xy, int64_t n, const int* __restrict__ cell,
                  const int* __restrict__ ids, long long* __restrict__ cursor,
                  float2* __restrict__ sxy, int* __restrict__ sid) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long s =
      (long long)atomicAdd(reinterpret_cast<unsigned long long*>(cursor + cell[i]), 1ull);
  sxy[s] = xy[i];
  sid[s] = ids ? ids[i] : (int)i;
}

// Calls f(a, b) for the contiguous sorted range of each row of cells in the Chebyshev box
// of radius R around (cx, cy), clamped to the grid.
template <typename F>
__device__ __forceinline__ void for_box_rows(const long long* __restrict__ start, int G, int cx,
                                             int cy, int R, F&& f) {
  const int x0 = max(cx - R, 0), x1 = min(cx + R, G - 1);
  const int y0 = max(cy - R, 0), y1 = min(cy + R, G - 1);
  for (int y = y0; y <= y1; ++y) f(start[(int64_t)y * G + x0], start[(int64_t)y * G + x1 + 1]);
}

__global__ void __launch_bounds__(32 * kNpWarps)
np_query_kernel(const float2* __restrict__ xy, int64_t n, int64_t lo, int64_t n_local,
                const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                const int* __restrict__ ids, const NpGrid* __restrict__ grid,
                const long long* __restrict__ start, const float2* __restrict__ sxy,
                const int* __restrict__ sid, int* __restrict__ hits) {
  __shared__ unsigned hist_s[kNpWarps][256];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * kNpWarps + wib;
  if (q >= n_local) return;
  const int64_t t = lo + q;
  const int64_t e0 = row_ptr[t], e1 = row_ptr[t + 1];
  const int k = (int)(e1 - e0);
  if (k == 0) {
    if (lane == 0) hits[q] = 0;
    return;
  }
  if ((int64_t)k >= n - 1) {  // every other node is a layout neighbour
    if (lane == 0) hits[q] = k;
    return;
  }
  const NpGrid g = *grid;
  const int G = g.G;
  const float2 xi = xy[t];
  const int my_id = ids ? ids[t] : (int)t;
  const int cx = cell_coord(xi.x, g.lo_x, g.inv_cs, G), cy = cell_coord(xi.y, g.lo_y, g.inv_cs, G);

  // 1. rings until >= k + 1 nodes (self included)
  long long cnt = 0;
  int r = 0;
  for (;; ++r) {
    long long c = 0;
    if (r == 0) {
      if (lane == 0) c = start[(int64_t)cy * G + cx + 1] - start[(int64_t)cy * G + cx];
    } else {
      for (int qq = lane; qq < 8 * r; qq += 32) {
        const int side = qq / (2 * r), pos = qq % (2 * r);
        int x, y;
        if (side == 0) { x = cx - r + pos; y = cy - r; }
        else if (side == 1) { x = cx + r; y = cy - r + pos; }
        else if (side == 2) { x = cx + r - pos; y = cy + r; }
        else { x = cx - r; y = cy + r - pos; }
        if (x >= 0 && x < G && y >= 0 && y < G) {
          const int64_t cc = (int64_t)y * G + x;
          c += start[cc + 1] - start[cc];
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    cnt += c;
    if (cnt >= (long long)k + 1) break;
    if (r >= G) break;  // the box covers the grid (cnt == n >= k + 1 already)
  }
  // 2. candidate disc
  const float D = 1.41421356f * (float)(r + 2) * g.cs * 1.0001f;
  const float D2 = D * D;
  const int R = (int)ceilf((float)(r + 2) * 1.41421356f) + 1;

  // 3. radix select of the k-th smallest candidate d^2 (self excluded)
  unsigned prefix = 0u, mask = 0u;
  int want = k;  // 1-based rank still to be located inside the current prefix class
  unsigned* h = hist_s[wib];
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = lane; b < 256; b += 32) h[b] = 0u;
    __syncwarp();
    for_box_rows(start, G, cx, cy, R, [&](long long a, long long b) {
      for (long long s = a + lane; s < b; s += 32) {
        const float d2 = d2_rn(xi, sxy[s]);
        const unsigned bits = __float_as_uint(d2);
        if (d2 <= D2 && (bits & mask) == prefix && sid[s] != my_id)
          atomicAdd(&h[(bits >> shift) & 255u], 1u);
      }
    });
    __syncwarp();
    // bucket holding rank `want`: lane l owns bins 8l .. 8l+7
    unsigned loc[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      loc[j] = h[8 * lane + j];
      sum += loc[j];
    }
    unsigned incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const unsigned excl = incl - sum;
    const bool mine = excl < (unsigned)want && (unsigned)want <= incl;
    const unsigned ballot = __ballot_sync(0xffffffffu, mine);
    const int owner = __ffs(ballot) - 1;
    int bucket = 0, below = 0;
    if (lane == owner) {
      unsigned acc = excl;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (acc + loc[j] >= (unsigned)want) {
          bucket = 8 * lane + j;
          below = (int)acc;
          break;
        }
        acc += loc[j];
      }
    }
    bucket = __shfl_sync(0xffffffffu, bucket, owner);
    below = __shfl_sync(0xffffffffu, below, owner);
    want -= below;
    prefix |= (unsigned)bucket << shift;
    mask |= 255u << shift;
    __syncwarp();
  }
  const unsigned tstar = prefix;  // bits of the k-th smallest d^2; `want` of its ties are in

  // 4. intersection with the graph neighbourhood
  int hit = 0;
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    const int j = col[e];
    const unsigned bits = __float_as_uint(d2_rn(xi, xy[j]));
    if (bits < tstar) {
      ++hit;
    } else if (bits == tstar) {
      const int jid = ids ? ids[j] : j;
      int lower = 0;  // tied candidates with a lower id (this lane alone; ties are rare)
      for_box_rows(start, G, cx, cy, R, [&](long long a, long long b) {
        for (long long s = a; s < b; ++s) {
          const int id = sid[s];
          if (id < jid && id != my_id && __float_as_uint(d2_rn(xi, sxy[s])) == tstar) ++lower;
        }
      });
      if (lower < want) ++hit;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hit += __shfl_xor_sync(0xffffffffu, hit, o);
  if (lane == 0) hits[q] = hit;
}

// Fixed-order reduction of sum_i (k_i == 0 ? 1 : h_i / (2 k_i - h_i)): block partials over
// fixed ranges, then one block in fixed order (deterministic).
constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum_fixed(double v) {
  __shared__ double s[kRedThreads];
  s[threadIdx.x] = v;
  __syncthreads();
  for (int w = kRedThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  return s[0];
}

__global__ void __launch_bounds__(kRedThreads)
np_partial_kernel(const int* __restrict__ hits, const int64_t* __restrict__ row_ptr, int64_t lo,
                  int64_t n_local, double* __restrict__ part) {
  const int64_t per = (int64_t)kRedThreads * 8;
  const int64_t b0 = (int64_t)blockIdx.x * per;
  double v = 0.0;
#pragma unroll 1
  for (int j = 0; j < 8; ++j) {
    const int64_t q = b0 + (int64_t)j * kRedThreads + threadIdx.x;
    if (q < n_local) {
      const int64_t t = lo + q;
      const int k = (int)(row_ptr[t + 1] - row_ptr[t]);
      const int h = hits[q];
      v += k == 0 ? 1.0 : (double)h / (double)(2 * k - h);
    }
  }
  const double s = block_sum_fixed(v);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kRedThreads)
np_final_kernel(const double* __restrict__ part, int nb, double inv_n, double* __restrict__ out) {
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += kRedThreads) v += part[b];
  const double s = block_sum_fixed(v);
  if (threadIdx.x == 0) *out = s * inv_n;
}

__global__ void __launch_bounds__(256)
unpermute_int_kernel(const int* __restrict__ in, const int* __restrict__ perm, int64_t n,
                     int* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[perm[i]] = in[i];
}

unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace

int np_grid_side(int64_t n) {
  const double g = std::ceil(std::sqrt((double)n / 2.0));
  return (int)std::min(4096.0, std::max(1.0, g));
}

size_t np_scratch_bytes(int64_t n, int64_t n_local) {
  auto rnd = [](size_t b) { return (b + 255) / 256 * 256; };
  const int64_t G = np_grid_side(n);
  const int64_t cells = G * G;
  const int64_t per = (int64_t)kRedThreads * 8;
  const int64_t nb = (n_local + per - 1) / per;
  return rnd(sizeof(NpGrid)) + 2 * rnd((size_t)(cells + 1) * 8) +
         rnd(((size_t)(cells + 1) / 1024 + 2) * 8) + 2 * rnd((size_t)n * 4) + rnd((size_t)n * 8) +
         rnd((size_t)(nb + 1) * 8);
}

int launch_np1(const float2* xy, int64_t n, int64_t lo, int64_t n_local, const int64_t* row_ptr,
               const int32_t* col, const int* ids, const BoxKeys* box_keys, void* scratch,
               int* hits_out, double* np_part_out, cudaStream_t s) {
  const int G = np_grid_side(n);
  const int64_t cells = (int64_t)G * G;
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) / 256 * 256;
    return r;
  };
  NpGrid* grid = reinterpret_cast<NpGrid*>(take(sizeof(NpGrid)));
  long long* hist = reinterpret_cast<long long*>(take((size_t)(cells + 1) * 8));
  long long* start = reinterpret_cast<long long*>(take((size_t)(cells + 1) * 8));
  long long* sums = reinterpret_cast<long long*>(take(((size_t)(cells + 1) / 1024 + 2) * 8));
  int* cell = reinterpret_cast<int*>(take((size_t)n * 4));
  int* sid = reinterpret_cast<int*>(take((size_t)n * 4));
  float2* sxy = reinterpret_cast<float2*>(take((size_t)n * 8));
  int* hits = hits_out;
  const int64_t per = (int64_t)kRedThreads * 8;
  const int nb = (int)((n_local + per - 1) / per);
  double* part = reinterpret_cast<double*>(take((size_t)(nb + 1) * 8));
  np_grid_kernel<<<1, 1, 0, s>>>(box_keys, G, grid);
  cudaMemsetAsync(hist, 0, (size_t)(cells + 1) * 8, s);
  np_count_kernel<<<nblk(n, 256), 256, 0, s>>>(xy, n, grid, cell, hist);
  exclusive_scan_ll(hist, start, cells + 1, sums, s);  // start[cells] = n
  cudaMemcpyAsync(hist, start, (size_t)(cells + 1) * 8, cudaMemcpyDeviceToDevice, s);  // cursors
  np_scatter_kernel<<<nblk(n, 256), 256, 0, s>>>(xy, n, cell, ids, hist, sxy, sid);
  if (n_local > 0)
    np_query_kernel<<<nblk(n_local, kNpWarps), 32 * kNpWarps, 0, s>>>(
        xy, n, lo, n_local, row_ptr, col, ids, grid, start, sxy, sid, hits);
  if (nb > 0) {
    np_partial_kernel<<<nb, kRedThreads, 0, s>>>(hits, row_ptr, lo, n_local, part);
    np_final_kernel<<<1, kRedThreads, 0, s>>>(part, nb, 1.0 / (double)n, np_part_out);
  } else {
    cudaMemsetAsync(np_part_out, 0, sizeof(double), s);
  }
  return 6 + (nb > 0 ? 2 : 0) + (n_local > 0 ? 1 : 0);  // kernels (incl. the 3 scan kernels)
}

void launch_unpermute_int(const int* in, const int* perm, int64_t n, int* out, cudaStream_t s) {
  unpermute_int_kernel<<<nblk(n, 256), 256, 0, s>>>(in, perm, n, out);
}

}  // namespace tfdp
