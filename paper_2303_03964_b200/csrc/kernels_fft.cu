// ibFFT path kernels — sm_100a.
//   bbox          exact fp32 min/max of the positions (ordered-uint keys, block partials)
//   setup         box -> (lo, L, N_int, w, h, centre) on the device, no host sync
//                 (R5/R5'/R6/R19); decides whether the kernel spectrum is stale
//   spread        step 1: Lagrange charges {1, x~, y~} onto the k x k nodes of each
//                 node's own interval; fp32 v4 reductions into L2
//   gather_update step 3 + assemble + attraction + update,
//                 fused bbox of the new positions for the next iteration
// The grid convolution (step 2) is kernels_fftconv.cu.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "device_math.cuh"
#include "tfdp_internal.h"

namespace tfdp {

namespace {
thread_local bool g_pdl_active = true;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TFDP_PDL");
    return !(e && e[0] == '0');
  }();
  return on && g_pdl_active;
}

void set_pdl_active(bool on) { g_pdl_active = on; }

// ------------------------------------------------------------------ bbox
// Two-level exact min/max: every block reduces its keys (warp __reduce + smem) and merges
// them with atomicMin/Max into one of kBoxSlots slots (block % kBoxSlots: ~60 blocks per
// slot, so no single-address hot spot); the consumer (setup / box_reduce, one block) reduces
// the slots and resets them to the identity for the next producer.
__device__ __forceinline__ void block_box_commit(unsigned kx0, unsigned ky0, unsigned kx1,
                                                 unsigned ky1, BoxKeys* slots) {
  __shared__ unsigned s[4][32];
  kx0 = __reduce_min_sync(0xffffffffu, kx0);
  ky0 = __reduce_min_sync(0xffffffffu, ky0);
  kx1 = __reduce_max_sync(0xffffffffu, kx1);
  ky1 = __reduce_max_sync(0xffffffffu, ky1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s[0][warp] = kx0;
    s[1][warp] = ky0;
    s[2][warp] = kx1;
    s[3][warp] = ky1;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    const bool v = lane < nw;
    kx0 = __reduce_min_sync(0xffffffffu, v ? s[0][lane] : 0xffffffffu);
    ky0 = __reduce_min_sync(0xffffffffu, v ? s[1][lane] : 0xffffffffu);
    kx1 = __reduce_max_sync(0xffffffffu, v ? s[2][lane] : 0u);
    ky1 = __reduce_max_sync(0xffffffffu, v ? s[3][lane] : 0u);
    if (lane == 0) {
      BoxKeys* sl = slots + (blockIdx.x % kBoxSlots);
      atomicMin(&sl->minx, kx0);
      atomicMin(&sl->miny, ky0);
      atomicMax(&sl->maxx, kx1);
      atomicMax(&sl->maxy, ky1);
    }
  }
}

__device__ __forceinline__ void reset_slots(BoxKeys* slots) {
  for (int i = threadIdx.x; i < kBoxSlots; i += blockDim.x)
    slots[i] = BoxKeys{0xffffffffu, 0xffffffffu, 0u, 0u};
}

// One block reduces the n_part slots, then (reset) resets them; all threads return the result.
__device__ BoxKeys block_reduce_partials(BoxKeys* part, int n_part, bool reset = true) {
  unsigned kx0 = 0xffffffffu, ky0 = 0xffffffffu, kx1 = 0u, ky1 = 0u;
  for (int i = threadIdx.x; i < n_part; i += blockDim.x) {
    const BoxKeys b = part[i];
    kx0 = min(kx0, b.minx);
    ky0 = min(ky0, b.miny);
    kx1 = max(kx1, b.maxx);
    ky1 = max(ky1, b.maxy);
  }
  __shared__ BoxKeys r[1];
  __shared__ unsigned s[4][32];
  kx0 = __reduce_min_sync(0xffffffffu, kx0);
  ky0 = __reduce_min_sync(0xffffffffu, ky0);
  kx1 = __reduce_max_sync(0xffffffffu, kx1);
  ky1 = __reduce_max_sync(0xffffffffu, ky1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s[0][warp] = kx0;
    s[1][warp] = ky0;
    s[2][warp] = kx1;
    s[3][warp] = ky1;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    const bool v = lane < nw;
    kx0 = __reduce_min_sync(0xffffffffu, v ? s[0][lane] : 0xffffffffu);
    ky0 = __reduce_min_sync(0xffffffffu, v ? s[1][lane] : 0xffffffffu);
    kx1 = __reduce_max_sync(0xffffffffu, v ? s[2][lane] : 0u);
    ky1 = __reduce_max_sync(0xffffffffu, v ? s[3][lane] : 0u);
    if (lane == 0) r[0] = BoxKeys{kx0, ky0, kx1, ky1};
  }
  __syncthreads();  // all slot reads are done
  if (reset) reset_slots(part);
  return r[0];
}

__global__ void __launch_bounds__(kNodeThreads)
bbox_kernel(const float2* __restrict__ xy, int64_t n, BoxKeys* part) {
  unsigned kx0 = 0xffffffffu, ky0 = 0xffffffffu, kx1 = 0u, ky1 = 0u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float2 p = xy[i];
    const unsigned a = f2key(p.x), b = f2key(p.y);
    kx0 = min(kx0, a);
    ky0 = min(ky0, b);
    kx1 = max(kx1, a);
    ky1 = max(ky1, b);
  }
  block_box_commit(kx0, ky0, kx1, ky1, part);
}

__global__ void __launch_bounds__(64)
box_reduce_kernel(BoxKeys* part, int n_part, BoxKeys* keys, int reset) {
  const BoxKeys b = block_reduce_partials(part, n_part, reset != 0);
  if (threadIdx.x == 0) *keys = b;
}

__global__ void __launch_bounds__(64) reset_slots_kernel(BoxKeys* slots) { reset_slots(slots); }

int bbox_blocks(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + kNodeThreads - 1) / kNodeThreads, 148 * 8));
}

void launch_reset_slots(BoxKeys* slots, cudaStream_t s) { reset_slots_kernel<<<1, 64, 0, s>>>(slots); }

int launch_bbox(const float2* xy, int64_t n, BoxKeys* part, cudaStream_t s) {
  bbox_kernel<<<bbox_blocks(n), kNodeThreads, 0, s>>>(xy, n, part);
  return kBoxSlots;
}

void launch_box_reduce(BoxKeys* part, int n_part, BoxKeys* keys, cudaStream_t s, bool reset) {
  box_reduce_kernel<<<1, 64, 0, s>>>(part, n_part, keys, reset ? 1 : 0);
}

// ------------------------------------------------------------------ setup
__global__ void __launch_bounds__(64)
setup_kernel(BoxKeys* part, int n_part, BoxKeys* keys, GridGeom* geom, int k,
             int n_int_min, int n_int_fixed, int n_int_cap, int P, int pitch, int* capped_flag,
             int rule, float gamma, KspecKey* kkey) {
  pdl_wait();
  pdl_trigger();
  const BoxKeys kb = block_reduce_partials(part, n_part);
  if (threadIdx.x != 0) return;
  *keys = kb;
  const float mnx = key2f(kb.minx), mny = key2f(kb.miny);
  const float mxx = key2f(kb.maxx), mxy = key2f(kb.maxy);
  // R6: bounding square anchored at (min x, min y), L = max(span_x, span_y) (fp32, R19)
  float L = fmaxf(__fsub_rn(mxx, mnx), __fsub_rn(mxy, mny));
  float lox = mnx, loy = mny;
  if (L == 0.0f) {  // all points coincident: unit square centred on them
    lox = __fsub_rn(mnx, 0.5f);
    loy = __fsub_rn(mny, 0.5f);
    L = 1.0f;
  }
  int nint;
  int capped = 0;
  bool unit = false;
  if (n_int_fixed > 0) {
    nint = n_int_fixed;
  } else {
    const float cl = ceilf(L);  // R5: N_int = max(n_int_min, ceil L)
    if (!(cl <= (float)n_int_cap)) {
      nint = n_int_cap;
      capped = 1;
    } else {
      nint = max(n_int_min, (int)cl);
      // R5': the span sets the count -> unit-width intervals, square of side N_int
      unit = rule == 0 && (int)cl >= n_int_min;
    }
  }
  if (nint > n_int_cap) {
    nint = n_int_cap;
    capped = 1;
    unit = false;
  }
  GridGeom g;
  g.lo_x = lox;
  g.lo_y = loy;
  g.L = L;
  g.w = unit ? 1.0f : __fdiv_rn(L, (float)nint);
  g.h = __fdiv_rn(g.w, (float)k);
  const float side = unit ? (float)nint : L;
  g.cx = __fmaf_rn(0.5f, side, lox);
  g.cy = __fmaf_rn(0.5f, side, loy);
  g.n_int = nint;
  g.k = k;
  g.M = nint * k;
  g.P = P;
  g.capped = capped;
  g.pitch = pitch;
  // K^ = FFT of the periodic kernel samples K(h d): a function of (P, h, gamma) only
  const KspecKey kk = *kkey;
  const unsigned hb = __float_as_uint(g.h), gb = __float_as_uint(gamma);
  g.kspec = !(kk.valid == 1 && kk.P == P && kk.h_bits == hb && kk.gamma_bits == gb);
  if (g.kspec) *kkey = KspecKey{P, hb, gb, 1};
  *geom = g;
  if (capped) atomicOr(capped_flag, 1);
}

void launch_setup(BoxKeys* part, int n_part, BoxKeys* keys, GridGeom* geom, int k,
                  int n_int_min, int n_int_fixed, int n_int_cap, int P, int pitch,
                  int* capped_flag, int rule, float gamma, KspecKey* kkey, cudaStream_t s) {
  launch_chained(setup_kernel, 1, 64, 0, s, part, n_part, keys, geom, k, n_int_min, n_int_fixed,
                 n_int_cap, P, pitch, capped_flag, rule, gamma, kkey);
}

// ------------------------------------------------------------------ interval coords
struct Cell {
  int bx, by;
  float ux, uy;
};

// b = min(floor((x - lo)/w), N_int - 1), u = (x - lo)/w - b, all in IEEE fp32 (R7, R19):
// the same operations as the oracle's interval_coords, so the integer decision matches.
__device__ __forceinline__ Cell cell_of(float2 p, const GridGeom& g) {
  Cell c;
  float tx = __fsub_rn(p.x, g.lo_x), ty = __fsub_rn(p.y, g.lo_y);
  if (g.w != 1.0f) {  // unit-width intervals (R5'): the division by 1 is exact, skip it
    tx = __fdiv_rn(tx, g.w);
    ty = __fdiv_rn(ty, g.w);
  }
  c.bx = max(0, min((int)floorf(tx), g.n_int - 1));
  c.by = max(0, min((int)floorf(ty), g.n_int - 1));
  c.ux = __fsub_rn(tx, (float)c.bx);
  c.uy = __fsub_rn(ty, (float)c.by);
  return c;
}

// ------------------------------------------------------------------ spread (step 1)
// The charges live channel-interleaved, float4 {C_1, C_x~, C_y~, 0} per grid node, so one
// node-to-grid-node contribution is ONE vector reduction (red.global.add.v4.f32) instead of
// three scalar ones into three planes: the L2 reduction units process a v4 RED at the
// instruction rate of a scalar one (tools/mbench_red.cu), and the spread is bound by that
// rate (3 k^2 -> k^2 REDs per node).
// Warp pre-aggregation for k >= 2: lanes whose nodes fall in the same interval have the
// same k x k target nodes, so the group's lowest lane sums the members' charges (their
// positions and Lagrange factors arrive by shuffles, in lane order) and issues the group's
// k^2 REDs alone.  Morton-ordered nodes put ~60 % of a warp's nodes in an interval shared
// with another lane at unit density.  Measured at C4 (us, plain / aggregated): k = 1
// 12.7 / 14.8 (one RED per node: the shuffles cost more than they save), k = 2 37.4 / 34.3,
// k = 3 83.9 / 71.9.
template <int K>
__global__ void __launch_bounds__(kNodeThreads)
spread_kernel(const float2* __restrict__ xy, int64_t lo, int64_t cnt,
              const GridGeom* __restrict__ geom, float4* __restrict__ grid, int by_lo,
              int by_hi) {
  constexpr bool kAgg = K >= 2;
  pdl_wait();
  pdl_trigger();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = t < cnt;
  if (kAgg ? __all_sync(0xffffffffu, !in) : !in) return;
  const GridGeom g = *geom;
  const float2 p = in ? xy[lo + t] : make_float2(g.cx, g.cy);
  const Cell c = cell_of(p, g);
  // interval-row filter: the multi-GPU slab mode spreads, from all positions, exactly the
  // nodes whose interval row lies in this rank's grid-row slab (by_lo = 0, by_hi = INT_MAX
  // on one GPU)
  const bool active = in && c.by >= by_lo && c.by < by_hi;
  if (!kAgg && !active) return;
  float lx[K], ly[K];
  lagrange<K>(c.ux, lx);
  lagrange<K>(c.uy, ly);
  const float xt = p.x - g.cx, yt = p.y - g.cy;  // box-centred channels (R11)
  float4 acc[K][K];
#pragma unroll
  for (int b = 0; b < K; ++b)
#pragma unroll
    for (int a = 0; a < K; ++a) {
      const float wgt = lx[a] * ly[b];
      acc[b][a] = make_float4(wgt, wgt * xt, wgt * yt, 0.0f);
    }
  if constexpr (kAgg) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned key = active ? (unsigned)c.by * (unsigned)g.n_int + (unsigned)c.bx : ~(unsigned)lane;
    const unsigned grp = __match_any_sync(full, key);
    const bool leader = (grp & ((1u << lane) - 1u)) == 0u;
    const int gmax = (int)__reduce_max_sync(full, (unsigned)__popc(grp));
    unsigned rest = grp & (grp - 1u);  // members after the leader
    for (int r = 1; r < gmax; ++r) {
      const int src = rest ? __ffs(rest) - 1 : lane;
      const float mxt = __shfl_sync(full, xt, src), myt = __shfl_sync(full, yt, src);
      float mlx[K], mly[K];
#pragma unroll
      for (int a = 0; a < K; ++a) {
        mlx[a] = __shfl_sync(full, lx[a], src);
        mly[a] = __shfl_sync(full, ly[a], src);
      }
      if (leader && rest) {
#pragma unroll
        for (int b = 0; b < K; ++b)
#pragma unroll
          for (int a = 0; a < K; ++a) {
            const float wgt = mlx[a] * mly[b];
            acc[b][a].x += wgt;
            acc[b][a].y = fmaf(wgt, mxt, acc[b][a].y);
            acc[b][a].z = fmaf(wgt, myt, acc[b][a].z);
          }
      }
      rest &= rest - 1u;
    }
    if (!active || !leader) return;
  }
#pragma unroll
  for (int b = 0; b < K; ++b) {
    const int64_t row = (int64_t)(c.by * K + b) * g.pitch;
#pragma unroll
    for (int a = 0; a < K; ++a) atomicAdd(grid + row + c.bx * K + a, acc[b][a]);
  }
}

// ------------------------------------------------------------------ spread, privatised
// Shared-memory privatised, tile-binned variant (north star step 1): a
// block takes kNodeThreads * NPT consecutive nodes (in the internal Morton order they cover
// a compact patch of intervals), reduces the patch's interval box, accumulates its charges
// into a private shared-memory tile of that box and flushes the tile with ONE v4 RED per
// touched grid node.  sm_100a has no native fp32 add in the shared-memory atomic unit (an
// fp32 atomicAdd on shared memory is a CAS loop, ATOMS.CAST.SPIN), so the tile holds 64-bit
// fixed-point sums (2^32 scale; integer ATOMS.ADD.64, exact and order-independent; the
// quantum 2^-32 is far below the fp32 rounding of the values).  A patch whose box exceeds
// the tile capacity (random node order, outliers) falls back to per-node REDs.
template <int K>
__host__ __device__ constexpr int spread_tile_npt() { return K == 1 ? 4 : K == 2 ? 2 : 1; }
template <int K>
__host__ __device__ constexpr int spread_tile_cap() { return K == 1 ? 2048 : K == 2 ? 2048 : 2304; }

__device__ __forceinline__ void fx_add(unsigned long long* a, float v) {
  atomicAdd(a, (unsigned long long)__float2ll_rn(v * 4294967296.0f));
}
__device__ __forceinline__ float fx_get(unsigned long long a) {
  return (float)((double)(long long)a * (1.0 / 4294967296.0));
}

template <int K>
__global__ void __launch_bounds__(kNodeThreads)
spread_tile_kernel(const float2* __restrict__ xy, int64_t lo, int64_t cnt,
                   const GridGeom* __restrict__ geom, float4* __restrict__ grid) {
  constexpr int NPT = spread_tile_npt<K>();
  constexpr int CAP = spread_tile_cap<K>();
  extern __shared__ unsigned long long tile[];  // [3][CAP] fixed point
  __shared__ int sbox[4][kNodeThreads / 32];
  pdl_wait();
  pdl_trigger();
  const GridGeom g = *geom;
  const int64_t base = (int64_t)blockIdx.x * kNodeThreads * NPT;
  float2 p[NPT];
  Cell c[NPT];
  bool act[NPT];
  int bx0 = INT32_MAX, by0 = INT32_MAX, bx1 = -1, by1 = -1;
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    const int64_t t = base + j * kNodeThreads + threadIdx.x;
    act[j] = t < cnt;
    p[j] = act[j] ? xy[lo + t] : make_float2(g.cx, g.cy);
    c[j] = cell_of(p[j], g);
    if (act[j]) {
      bx0 = min(bx0, c[j].bx);
      bx1 = max(bx1, c[j].bx);
      by0 = min(by0, c[j].by);
      by1 = max(by1, c[j].by);
    }
  }
  // block interval box (uniform decision below)
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    bx0 = __reduce_min_sync(0xffffffffu, bx0);
    by0 = __reduce_min_sync(0xffffffffu, by0);
    bx1 = __reduce_max_sync(0xffffffffu, bx1);
    by1 = __reduce_max_sync(0xffffffffu, by1);
    if (lane == 0) {
      sbox[0][warp] = bx0;
      sbox[1][warp] = by0;
      sbox[2][warp] = bx1;
      sbox[3][warp] = by1;
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kNodeThreads / 32; ++w) {
      bx0 = min(bx0, sbox[0][w]);
      by0 = min(by0, sbox[1][w]);
      bx1 = max(bx1, sbox[2][w]);
      by1 = max(by1, sbox[3][w]);
    }
  }
  if (bx1 < 0) return;  // no active node in the block
  const int W = (bx1 - bx0 + 1) * K, H = (by1 - by0 + 1) * K;
  const bool priv = W * H <= CAP;
  if (priv) {
    const int WH = W * H;
    for (int i = threadIdx.x; i < WH; i += kNodeThreads) {
      tile[i] = 0ull;
      tile[CAP + i] = 0ull;
      tile[2 * CAP + i] = 0ull;
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    if (!act[j]) continue;
    float lx[K], ly[K];
    lagrange<K>(c[j].ux, lx);
    lagrange<K>(c[j].uy, ly);
    const float xt = p[j].x - g.cx, yt = p[j].y - g.cy;  // box-centred channels (R11)
#pragma unroll
    for (int b = 0; b < K; ++b) {
#pragma unroll
      for (int a = 0; a < K; ++a) {
        const float wgt = lx[a] * ly[b];
        if (priv) {
          const int o = ((c[j].by - by0) * K + b) * W + (c[j].bx - bx0) * K + a;
          fx_add(tile + o, wgt);
          fx_add(tile + CAP + o, wgt * xt);
          fx_add(tile + 2 * CAP + o, wgt * yt);
        } else {
          atomicAdd(grid + (int64_t)(c[j].by * K + b) * g.pitch + c[j].bx * K + a,
                    make_float4(wgt, wgt * xt, wgt * yt, 0.0f));
        }
      }
    }
  }
  if (!priv) return;
  __syncthreads();
  for (int i = threadIdx.x; i < W * H; i += kNodeThreads) {
    const unsigned long long a0 = tile[i], a1 = tile[CAP + i], a2 = tile[2 * CAP + i];
    if ((a0 | a1 | a2) != 0ull) {
      const int r = i / W, q = i - r * W;
      atomicAdd(grid + (int64_t)(by0 * K + r) * g.pitch + bx0 * K + q,
                make_float4(fx_get(a0), fx_get(a1), fx_get(a2), 0.0f));
    }
  }
}

// Spread variant.  Measured at C4 (tools/spread_ab.sh, profiles/r2_spread_ab.txt; us per
// launch, REDs / privatised tile): input layout k = 1 10.8 / 20.6, k = 2 25.3 / 35.6,
// k = 3 59.9 / 73.6; clustered layout (1000 Gaussian clusters) k = 1 10.9 / 20.7, k = 3
// 50.7 / 70.5.  The shared-memory atomics (CAS loops) cost more than the L2 reductions they
// save, so the per-node v4 REDs are the default; TFDP_SPREAD=tile selects the privatised
// kernel (A/B runs; it is parity-tested like the default).
bool spread_tiles() {
  static const bool t = [] {
    const char* e = std::getenv("TFDP_SPREAD");
    return e && e[0] == 't';
  }();
  return t;
}

void launch_spread(const float2* xy, int64_t lo, int64_t cnt, const GridGeom* geom, int k,
                   float4* grid, cudaStream_t s, int by_lo, int by_hi) {
  if (cnt <= 0) return;
  if (spread_tiles() && by_lo == 0 && by_hi == INT32_MAX) {
#define TFDP_ST(KK)                                                                          \
  {                                                                                          \
    constexpr int per = kNodeThreads * spread_tile_npt<KK>();                                \
    const size_t smb = 3 * sizeof(unsigned long long) * spread_tile_cap<KK>();              \
    static bool attr = [] {                                                                  \
      cudaFuncSetAttribute(spread_tile_kernel<KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)(3 * sizeof(unsigned long long) * spread_tile_cap<KK>()));   \
      return true;                                                                           \
    }();                                                                                     \
    (void)attr;                                                                              \
    launch_chained(spread_tile_kernel<KK>, (unsigned)((cnt + per - 1) / per), kNodeThreads, smb, \
                   s, xy, lo, cnt, geom, grid);                                              \
  }
    if (k == 1) TFDP_ST(1)
    else if (k == 2) TFDP_ST(2)
    else TFDP_ST(3)
#undef TFDP_ST
    return;
  }
  const unsigned blocks = (unsigned)((cnt + kNodeThreads - 1) / kNodeThreads);
  if (k == 1)
    launch_chained(spread_kernel<1>, blocks, kNodeThreads, 0, s, xy, lo, cnt, geom, grid, by_lo, by_hi);
  else if (k == 2)
    launch_chained(spread_kernel<2>, blocks, kNodeThreads, 0, s, xy, lo, cnt, geom, grid, by_lo, by_hi);
  else
    launch_chained(spread_kernel<3>, blocks, kNodeThreads, 0, s, xy, lo, cnt, geom, grid, by_lo, by_hi);
}

// ------------------------------------------------------------------ gather + update
template <int K>
__global__ void __launch_bounds__(kNodeThreads)
gather_update_kernel(const float2* __restrict__ xy, float2* __restrict__ xy_next, int64_t lo,
                     int64_t n_local, const GridGeom* __restrict__ geom,
                     const float* __restrict__ phi, const int64_t* __restrict__ row_ptr,
                     const int32_t* __restrict__ col, ForceArgs fa, FocusArgs fo, float eta,
                     int iter, int update, float2* __restrict__ rep_out,
                     float2* __restrict__ att_out, unsigned long long* diverge,
                     BoxKeys* next_part, const PeerRoute* __restrict__ rt, int next_buf,
                     const float2* __restrict__ A_pre) {
  pdl_wait();
  pdl_trigger();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = t < n_local;
  unsigned kx0 = 0xffffffffu, ky0 = 0xffffffffu, kx1 = 0u, ky1 = 0u;
  if (active) {
    const int64_t i = lo + t;
    const GridGeom g = *geom;
    const float2 p = xy[i];
    const Cell c = cell_of(p, g);
    float lx[K], ly[K];
    lagrange<K>(c.ux, lx);
    lagrange<K>(c.uy, ly);
    const int64_t plane = (int64_t)g.pitch * g.pitch;
    float psi0 = 0.f, psi1 = 0.f, psi2 = 0.f;
#pragma unroll
    for (int b = 0; b < K; ++b) {
      const int64_t row = (int64_t)(c.by * K + b) * g.pitch;
#pragma unroll
      for (int a = 0; a < K; ++a) {
        const int64_t idx = row + c.bx * K + a;
        const float wgt = lx[a] * ly[b];
        psi0 = fmaf(wgt, __ldg(phi + idx), psi0);
        psi1 = fmaf(wgt, __ldg(phi + plane + idx), psi1);
        psi2 = fmaf(wgt, __ldg(phi + 2 * plane + idx), psi2);
      }
    }
    const float xt = p.x - g.cx, yt = p.y - g.cy;
    // F^r = x~ psi_1 - psi_x~  (Eqs. Fr1/Fr2); fused to limit cancellation (R11)
    float Rx = fa.rho * fmaf(xt, psi0, -psi1);
    float Ry = fa.rho * fmaf(yt, psi0, -psi2);
    float2 as;
    if (fo.label) {  // local refinement mask (R23)
      const float2 Rm = focus_repulsion(make_float2(Rx, Ry), i, t, fa.rho, fo);
      Rx = Rm.x;
      Ry = Rm.y;
      as = attraction_sum_masked(xy, p, row_ptr, col, i, fa.beta, fo.label, fo.la);
    } else if (!A_pre) {
      as = attraction_sum_hv(xy, p, row_ptr, col, i, fa);
    }
    // A_pre: the attraction, computed from the same positions by attraction_kernel on the
    // side stream while the FFT passes ran (it does not depend on the grid)
    const float ax = A_pre && !fo.label ? A_pre[t].x : -fa.alpha * as.x;
    const float ay = A_pre && !fo.label ? A_pre[t].y : -fa.alpha * as.y;
    if (update) {
      const float nx = fmaf(eta, Rx + ax, p.x);
      const float ny = fmaf(eta, Ry + ay, p.y);
      xy_next[i] = make_float2(nx, ny);
      if (rt)  // slab mode, fused position all-gather: into every other rank's copy
        for (int j = 0; j < rt->world; ++j)
          if (j != rt->rank) rt->xy[next_buf][j][i] = make_float2(nx, ny);
      if (!isfinite(nx) || !isfinite(ny)) {
        atomicMin(diverge, ((unsigned long long)(unsigned)iter << 32) | (unsigned long long)i);
      } else {
        kx0 = kx1 = f2key(nx);
        ky0 = ky1 = f2key(ny);
      }
    } else {
      if (rep_out) rep_out[t] = make_float2(Rx, Ry);
      if (att_out) att_out[t] = make_float2(ax, ay);
    }
  }
  if (update && next_part) block_box_commit(kx0, ky0, kx1, ky1, next_part);
}

// Attraction of the shard's nodes, A_t = -alpha sum_j (1 + beta/s)(x_i - x_j) (P:286-288,
// P:301-303), written for gather_update: it depends only on the positions, so it runs on the
// side stream concurrently with spread and the FFT passes instead of on the critical path.
__global__ void __launch_bounds__(kNodeThreads)
attraction_kernel(const float2* __restrict__ xy, int64_t lo, int64_t n_local,
                  const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                  ForceArgs fa, float2* __restrict__ A) {
  // grid-stride: the default grid is one thread per node; a small grid (blocks > 0 in
  // launch_attraction) trickles beside the FFT passes instead of flooding the SMs
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_local;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = lo + t;
    const float2 s = attraction_sum_hv(xy, xy[i], row_ptr, col, i, fa);
    A[t] = make_float2(-fa.alpha * s.x, -fa.alpha * s.y);
  }
}

void launch_attraction(const float2* xy, int64_t lo, int64_t n_local, const int64_t* row_ptr,
                       const int32_t* col, ForceArgs fa, float2* A, cudaStream_t s, int blocks) {
  if (n_local <= 0) return;
  const int64_t full = (n_local + kNodeThreads - 1) / kNodeThreads;
  const unsigned g = (unsigned)(blocks > 0 ? std::min<int64_t>(blocks, full) : full);
  attraction_kernel<<<g, kNodeThreads, 0, s>>>(xy, lo, n_local, row_ptr, col, fa, A);
}

void launch_gather_update(const float2* xy, float2* xy_next, int64_t lo, int64_t n_local,
                          const GridGeom* geom, int k, const float* phi,
                          const int64_t* row_ptr, const int32_t* col, ForceArgs fa,
                          FocusArgs fo, float eta, int iter, int update, float2* rep_out,
                          float2* att_out, unsigned long long* diverge, BoxKeys* next_part,
                          cudaStream_t s, const PeerRoute* route, int next_buf,
                          const float2* A_pre) {
  if (n_local <= 0) return;
  const unsigned blocks = (unsigned)((n_local + kNodeThreads - 1) / kNodeThreads);
#define TFDP_GU(KK)                                                                         \
  launch_chained(gather_update_kernel<KK>, blocks, kNodeThreads, 0, s, xy, xy_next, lo,      \
                 n_local, geom, phi, row_ptr, col, fa, fo, eta, iter, update, rep_out, att_out, \
                 diverge, next_part, route, next_buf, A_pre)
  if (k == 1) TFDP_GU(1);
  else if (k == 2) TFDP_GU(2);
  else TFDP_GU(3);
#undef TFDP_GU
}

}  // namespace tfdp
