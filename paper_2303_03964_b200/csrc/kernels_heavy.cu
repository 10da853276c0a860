// Degree-skew handling of the attraction row walk (VERDICT r1 missing
// 8) — sm_100a.  The finishing kernels walk one CSR row per thread, which is right for the
// mesh / RGG graphs (degrees ~4-20) but leaves a warp waiting on one thread for a power-law
// hub (Chung-Lu / LiveJournal-like graphs: degrees of 10^4 and more).  Rows with more
// than kHeavyDeg edges are cut into chunks of kHeavyChunk edges; one warp sums a chunk
// (lanes stride the chunk, fixed xor-shuffle reduction) into part[chunk], and the row's
// thread in the finishing kernel adds its chunk sums in chunk order — deterministic and
// independent of the target shards (R15).  The chunk index (first[i] = first chunk of row
// i) is rebuilt whenever the CSR is (init, renumbering).
#include <algorithm>

#include "device_math.cuh"
#include "tfdp_internal.h"

namespace tfdp {

namespace {

__global__ void __launch_bounds__(256)
heavy_count_kernel(const int64_t* __restrict__ row_ptr, int64_t n, long long* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) {
    cnt[n] = 0;
    return;
  }
  const int64_t d = row_ptr[i + 1] - row_ptr[i];
  cnt[i] = d > kHeavyDeg ? (d + kHeavyChunk - 1) / kHeavyChunk : 0;
}

// one warp per chunk of the rows [lo, hi): chunks [first[lo], first[hi]), grid-stride
__global__ void __launch_bounds__(256)
heavy_attr_kernel(const float2* __restrict__ xy, const int64_t* __restrict__ row_ptr,
                  const int32_t* __restrict__ col, const long long* __restrict__ first,
                  int64_t lo, int64_t hi, float beta, float2* __restrict__ part) {
  const long long c0 = first[lo], c1 = first[hi];
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (long long c = c0 + warp; c < c1; c += nw) {
    // row of chunk c: the last row r in [lo, hi) with first[r] <= c (binary search)
    int64_t a = lo, b = hi - 1;
    while (a < b) {
      const int64_t m = (a + b + 1) >> 1;
      if (first[m] <= c) a = m;
      else b = m - 1;
    }
    const int64_t r = a;
    const int64_t e0 = row_ptr[r] + (c - first[r]) * kHeavyChunk;
    const int64_t e1 = min(row_ptr[r + 1], e0 + kHeavyChunk);
    const float2 xi = xy[r];
    float sx = 0.f, sy = 0.f;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const float2 xj = __ldg(xy + __ldg(col + e));
      const float dx = xi.x - xj.x, dy = xi.y - xj.y;
      const float s = fmaf(dx, dx, fmaf(dy, dy, 1.0f));
      const float w = fmaf(beta, rcp_approx(s), 1.0f);
      sx = fmaf(w, dx, sx);
      sy = fmaf(w, dy, sy);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sx += __shfl_xor_sync(0xffffffffu, sx, o);
      sy += __shfl_xor_sync(0xffffffffu, sy, o);
    }
    if (lane == 0) part[c] = make_float2(sx, sy);
  }
}

}  // namespace

size_t heavy_scratch_bytes(int64_t n) {
  return (size_t)(n + 1) * 8 + (size_t)((n + 1 + 1023) / 1024 + 1) * 8 + 256;
}

void launch_heavy_build(const int64_t* row_ptr, int64_t n, long long* first, void* scratch,
                        cudaStream_t s) {
  long long* cnt = static_cast<long long*>(scratch);
  long long* sums = cnt + (n + 1);
  heavy_count_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, s>>>(row_ptr, n, cnt);
  exclusive_scan_ll(cnt, first, n + 1, sums, s);
}

void launch_heavy_attr(const float2* xy, const int64_t* row_ptr, const int32_t* col,
                       const long long* first, int64_t lo, int64_t hi, int64_t n_items_max,
                       float beta, float2* part, cudaStream_t s) {
  if (hi <= lo || n_items_max <= 0) return;
  const int64_t warps = std::min<int64_t>(n_items_max, 148 * 32);
  heavy_attr_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(xy, row_ptr, col, first,
                                                                        lo, hi, beta, part);
}

}  // namespace tfdp
