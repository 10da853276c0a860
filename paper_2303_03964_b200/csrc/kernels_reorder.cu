// Spatial reordering of the nodes (a locality optimisation of the ibFFT path; no paper
// arithmetic).  Nodes are renumbered internally in Morton (Z) order of a 1024 x 1024 grid
// over the bounding box, so that consecutive threads of spread / gather touch neighbouring
// grid cells and neighbouring positions.  Counting sort: key histogram (atomics), exclusive
// scan, scatter; then positions, the permutation and the CSR are rebuilt in the new order.
// The public API keeps the caller's node order (api.cpp permutes on input, un-permutes on
// output).  Within one cell the order is whatever the atomics produce (results are
// permutation-equivariant; only fp summation order changes, R15).
#include <algorithm>

#include "device_math.cuh"
#include "tfdp_internal.h"

namespace tfdp {

namespace {

constexpr int kMortonBits = 8;  // 256 x 256 cells -> 65536 bins (~15 nodes per bin at C4)
constexpr int kBins = 1 << (2 * kMortonBits);

__device__ __forceinline__ unsigned spread_bits(unsigned v) {  // 8 bits -> even positions
  v &= (1u << kMortonBits) - 1u;
  v = (v | (v << 8)) & 0x00ff00ffu;
  v = (v | (v << 4)) & 0x0f0f0f0fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}

__global__ void __launch_bounds__(256)
morton_keys_kernel(const float2* __restrict__ xy, int64_t n, const BoxKeys* __restrict__ box,
                   int* __restrict__ keys, long long* __restrict__ hist) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const BoxKeys b = *box;
  const float x0 = key2f(b.minx), y0 = key2f(b.miny);
  const float L = fmaxf(fmaxf(key2f(b.maxx) - x0, key2f(b.maxy) - y0), 1e-30f);
  constexpr float top = (float)((1 << kMortonBits) - 1);
  const float s = (top + 0.999f) / L;
  const float2 p = xy[i];
  const unsigned cx = (unsigned)fminf(top, fmaxf(0.f, (p.x - x0) * s));
  const unsigned cy = (unsigned)fminf(top, fmaxf(0.f, (p.y - y0) * s));
  const int k = (int)(spread_bits(cx) | (spread_bits(cy) << 1));
  keys[i] = k;
  // warp-aggregated: an almost sorted layout puts whole warps on one bin
  const unsigned act = __activemask();
  const unsigned grp = __match_any_sync(act, k);
  if ((threadIdx.x & 31) == __ffs(grp) - 1)
    atomicAdd(reinterpret_cast<unsigned long long*>(hist + k), (unsigned long long)__popc(grp));
}

// Exclusive scan, three passes: per-block scan + block totals, scan of totals, add.
constexpr int kScanBlock = 1024;

__device__ __forceinline__ long long block_exclusive_scan(long long v, long long* total) {
  __shared__ long long warp_sums[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    long long w = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) warp_sums[lane] = w;
  }
  __syncthreads();
  const long long incl = x + (warp > 0 ? warp_sums[warp - 1] : 0);
  if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
  return incl - v;
}

__global__ void __launch_bounds__(kScanBlock)
scan_blocks_kernel(const long long* __restrict__ in, long long* __restrict__ out, int64_t n,
                   long long* __restrict__ block_sums) {
  const int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  const long long v = i < n ? in[i] : 0;
  long long tot;
  const long long ex = block_exclusive_scan(v, &tot);
  if (i < n) out[i] = ex;
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanBlock)
scan_sums_kernel(long long* __restrict__ sums, int nb) {
  // one block, sequential chunks of kScanBlock
  long long carry = 0;
  for (int base = 0; base < nb; base += kScanBlock) {
    const int i = base + threadIdx.x;
    const long long v = i < nb ? sums[i] : 0;
    long long tot;
    const long long ex = block_exclusive_scan(v, &tot);
    __syncthreads();
    if (i < nb) sums[i] = ex + carry;
    carry += tot;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kScanBlock)
scan_add_kernel(long long* __restrict__ out, int64_t n, const long long* __restrict__ sums) {
  const int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  if (i < n) out[i] += sums[blockIdx.x];
}

// slot i (old internal order) -> new position of its caller id in the new permutation
__global__ void __launch_bounds__(256)
scatter_kernel(const int* __restrict__ keys, long long* __restrict__ offs, int64_t n,
               const int* __restrict__ perm_old, int* __restrict__ perm_new) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int key = keys[i];
  // warp-aggregated slot allocation: one atomic per (warp, bin)
  const unsigned act = __activemask();
  const unsigned grp = __match_any_sync(act, key);
  const int lane = threadIdx.x & 31, leader = __ffs(grp) - 1;
  unsigned long long base = 0;
  if (lane == leader)
    base = atomicAdd(reinterpret_cast<unsigned long long*>(offs + key), (unsigned long long)__popc(grp));
  base = __shfl_sync(grp, base, leader);
  const long long pos = (long long)base + __popc(grp & ((1u << lane) - 1u));
  perm_new[pos] = perm_old[i];
}

// Applies a new permutation (computed here, or by rank 0 and broadcast so that every rank
// holds the same internal order): positions, inverse and degrees in the new order.
__global__ void __launch_bounds__(256)
apply_perm_kernel(const int* __restrict__ perm_new, const int* __restrict__ inv_old, int64_t n,
                  const float2* __restrict__ xy_old, float2* __restrict__ xy_new,
                  int* __restrict__ inv_new, const int64_t* __restrict__ row_ptr_o,
                  long long* __restrict__ deg_new) {
  const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= n) return;
  const int o = perm_new[pos];
  xy_new[pos] = xy_old[inv_old[o]];
  inv_new[o] = (int)pos;
  deg_new[pos] = row_ptr_o[o + 1] - row_ptr_o[o];
}

__global__ void __launch_bounds__(256)
remap_cols_kernel(const int* __restrict__ perm, const int* __restrict__ inv,
                  const int64_t* __restrict__ row_ptr_o, const int32_t* __restrict__ col_o,
                  const int64_t* __restrict__ row_ptr_p, int32_t* __restrict__ col_p, int64_t n) {
  // eight lanes per row (mean degrees are ~8-20): coalesced over each row's edges
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int lane = threadIdx.x & 7;
  if (w >= n) return;
  const int o = perm[w];
  const int64_t s = row_ptr_o[o], e = row_ptr_o[o + 1], d = row_ptr_p[w];
  for (int64_t k = s + lane; k < e; k += 8) col_p[d + (k - s)] = inv[col_o[k]];
}

__global__ void __launch_bounds__(256)
unpermute_kernel(const float2* __restrict__ in, const int* __restrict__ perm, int64_t n,
                 float2* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[perm[i]] = in[i];
}

__global__ void __launch_bounds__(256)
permute_kernel(const float2* __restrict__ in, const int* __restrict__ perm, int64_t n,
               float2* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[perm[i]];
}

__global__ void iota_kernel(int* __restrict__ perm, int* __restrict__ inv, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    perm[i] = (int)i;
    inv[i] = (int)i;
  }
}

unsigned blocks_for(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

void exclusive_scan(const long long* in, long long* out, int64_t n, long long* sums, cudaStream_t s) {
  const int nb = (int)blocks_for(n, kScanBlock);
  scan_blocks_kernel<<<nb, kScanBlock, 0, s>>>(in, out, n, sums);
  scan_sums_kernel<<<1, kScanBlock, 0, s>>>(sums, nb);
  scan_add_kernel<<<nb, kScanBlock, 0, s>>>(out, n, sums);
}

}  // namespace

void exclusive_scan_ll(const long long* in, long long* out, int64_t n, long long* sums,
                       cudaStream_t s) {
  exclusive_scan(in, out, n, sums, s);
}

size_t reorder_scratch_bytes(int64_t n) {
  // keys int[n], hist/offs ll[kBins], deg ll[n+1], sums ll[blocks]
  const int64_t nbins = kBins;
  const int64_t mx = std::max<int64_t>(nbins, n + 1);
  return (size_t)n * 4 + (size_t)nbins * 8 * 2 + (size_t)(n + 1) * 8 * 2 +
         (size_t)((mx + kScanBlock - 1) / kScanBlock + 1) * 8 + 1024;
}

void launch_iota(int* perm, int* inv, int64_t n, cudaStream_t s) {
  iota_kernel<<<blocks_for(n, 256), 256, 0, s>>>(perm, inv, n);
}

namespace {
struct Scratch {
  int* keys;
  long long *hist, *offs, *deg, *sums;
};
Scratch carve(void* scratch, int64_t n) {
  char* p = static_cast<char*>(scratch);
  Scratch q;
  q.keys = reinterpret_cast<int*>(p);
  p += ((size_t)n * 4 + 255) / 256 * 256;
  q.hist = reinterpret_cast<long long*>(p);
  p += (size_t)kBins * 8;
  q.offs = reinterpret_cast<long long*>(p);
  p += (size_t)kBins * 8;
  q.deg = reinterpret_cast<long long*>(p);
  p += (size_t)(n + 1) * 8;
  q.sums = reinterpret_cast<long long*>(p);
  return q;
}
}  // namespace

int launch_reorder_perm(const float2* xy_old, const BoxKeys* box, const int* perm_old,
                        int* perm_new, int64_t n, void* scratch, cudaStream_t s) {
  const Scratch q = carve(scratch, n);
  cudaMemsetAsync(q.hist, 0, (size_t)kBins * 8, s);
  morton_keys_kernel<<<blocks_for(n, 256), 256, 0, s>>>(xy_old, n, box, q.keys, q.hist);
  exclusive_scan(q.hist, q.offs, kBins, q.sums, s);
  scatter_kernel<<<blocks_for(n, 256), 256, 0, s>>>(q.keys, q.offs, n, perm_old, perm_new);
  return 5;
}

int launch_reorder_apply(const float2* xy_old, float2* xy_new, const int* inv_old,
                         const int* perm_new, int* inv_new, const int64_t* row_ptr_o,
                         const int32_t* col_o, int64_t* row_ptr_p, int32_t* col_p, int64_t n,
                         void* scratch, cudaStream_t s) {
  const Scratch q = carve(scratch, n);
  cudaMemsetAsync(q.deg + n, 0, sizeof(long long), s);
  apply_perm_kernel<<<blocks_for(n, 256), 256, 0, s>>>(perm_new, inv_old, n, xy_old, xy_new,
                                                       inv_new, row_ptr_o, q.deg);
  exclusive_scan(q.deg, reinterpret_cast<long long*>(row_ptr_p), n + 1, q.sums, s);
  remap_cols_kernel<<<blocks_for(n * 8, 256), 256, 0, s>>>(perm_new, inv_new, row_ptr_o, col_o,
                                                             row_ptr_p, col_p, n);
  return 5;
}

void launch_unpermute(const float2* in, const int* perm, int64_t n, float2* out, cudaStream_t s) {
  unpermute_kernel<<<blocks_for(n, 256), 256, 0, s>>>(in, perm, n, out);
}

void launch_permute(const float2* in, const int* perm, int64_t n, float2* out, cudaStream_t s) {
  permute_kernel<<<blocks_for(n, 256), 256, 0, s>>>(in, perm, n, out);
}

}  // namespace tfdp
