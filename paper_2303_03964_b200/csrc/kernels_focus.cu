// Local (fisheye) refinement (NEXT-4, SPEC RefinementMask S:155-158): the focal
// region F u N(F), its internal-slot view, and the exact repulsion sum S1 over the region's
// sources that the masked force combination needs (R23; FocusArgs in
// tfdp_internal.h).  The region is small (a handful of focal nodes and their neighbours), so
// S1 is a direct n_local x |region| sum through a shared-memory source tile, in a fixed
// source order (deterministic, shard-invariant).
#include <algorithm>

#include "device_math.cuh"
#include "tfdp_internal.h"

namespace tfdp {

namespace {

// one warp per focal node: the node and its CSR row (caller order) into the region
__global__ void mark_focus_kernel(const int* __restrict__ focal, int n_focal,
                                  const int64_t* __restrict__ row_ptr,
                                  const int32_t* __restrict__ col, unsigned char* __restrict__ label) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n_focal) return;
  const int f = focal[w];
  if (lane == 0) label[f] = 1;
  for (int64_t e = row_ptr[f] + lane; e < row_ptr[f + 1]; e += 32) label[col[e]] = 1;
}

__global__ void focus_label_slots_kernel(const unsigned char* __restrict__ label_caller,
                                         const int* __restrict__ perm, int64_t n,
                                         unsigned char* __restrict__ label_slot) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n) label_slot[s] = label_caller[perm ? perm[s] : s];
}

__global__ void focus_region_slots_kernel(const int* __restrict__ region_caller, int m,
                                          const int* __restrict__ inv, int* __restrict__ region_slot) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) region_slot[k] = inv ? inv[region_caller[k]] : region_caller[k];
}

constexpr int kS1Threads = 256;
constexpr int kS1Tile = 1024;

template <int G>
__global__ void __launch_bounds__(kS1Threads)
focus_s1_kernel(const float2* __restrict__ xy, int64_t lo, int64_t n_local,
                const int* __restrict__ region, int m, float neg_gamma, float2* __restrict__ s1) {
  __shared__ float2 src[kS1Tile];
  const int64_t t = (int64_t)blockIdx.x * kS1Threads + threadIdx.x;
  const bool active = t < n_local;
  const float2 xi = active ? xy[lo + t] : make_float2(0.f, 0.f);
  float sx = 0.f, sy = 0.f;
  for (int base = 0; base < m; base += kS1Tile) {
    const int cnt = min(kS1Tile, m - base);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += kS1Threads) src[k] = xy[region[base + k]];
    __syncthreads();
    for (int k = 0; k < cnt; ++k) {  // fixed source order
      const float2 xj = src[k];
      const float dx = xi.x - xj.x, dy = xi.y - xj.y;
      const float w = pow_neg<G>(fmaf(dx, dx, fmaf(dy, dy, 1.0f)), neg_gamma);
      sx = fmaf(w, dx, sx);
      sy = fmaf(w, dy, sy);
    }
  }
  if (active) s1[t] = make_float2(sx, sy);
}

unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace

void launch_mark_focus(const int* focal, int n_focal, const int64_t* row_ptr_caller,
                       const int32_t* col_caller, unsigned char* label_caller, cudaStream_t s) {
  if (n_focal <= 0) return;
  mark_focus_kernel<<<nblk((int64_t)n_focal * 32, 256), 256, 0, s>>>(focal, n_focal, row_ptr_caller,
                                                                      col_caller, label_caller);
}

void launch_focus_slots(const unsigned char* label_caller, const int* perm, const int* inv,
                        int64_t n, const int* region_caller, int m, unsigned char* label_slot,
                        int* region_slot, cudaStream_t s) {
  focus_label_slots_kernel<<<nblk(n, 256), 256, 0, s>>>(label_caller, perm, n, label_slot);
  if (m > 0)
    focus_region_slots_kernel<<<nblk(m, 256), 256, 0, s>>>(region_caller, m, inv, region_slot);
}

void launch_focus_s1(const float2* xy, int64_t lo, int64_t n_local, const int* region_slot,
                     int m, ForceArgs fa, float2* s1, cudaStream_t s) {
  if (n_local <= 0) return;
  const unsigned b = nblk(n_local, kS1Threads);
  const float ng = -fa.gamma;
  switch (fa.gamma_int) {
    case 1: focus_s1_kernel<1><<<b, kS1Threads, 0, s>>>(xy, lo, n_local, region_slot, m, ng, s1); break;
    case 2: focus_s1_kernel<2><<<b, kS1Threads, 0, s>>>(xy, lo, n_local, region_slot, m, ng, s1); break;
    case 3: focus_s1_kernel<3><<<b, kS1Threads, 0, s>>>(xy, lo, n_local, region_slot, m, ng, s1); break;
    case 4: focus_s1_kernel<4><<<b, kS1Threads, 0, s>>>(xy, lo, n_local, region_slot, m, ng, s1); break;
    case 8: focus_s1_kernel<8><<<b, kS1Threads, 0, s>>>(xy, lo, n_local, region_slot, m, ng, s1); break;
    default: focus_s1_kernel<0><<<b, kS1Threads, 0, s>>>(xy, lo, n_local, region_slot, m, ng, s1); break;
  }
}

}  // namespace tfdp
