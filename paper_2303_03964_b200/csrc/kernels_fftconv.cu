// Hand-written FFT convolution of the ibFFT grid step (R9) — sm_100a.
//
// Replaces a zero-padded P x P 2-D R2C -> x K^ -> C2R (cuFFT) by four passes that never
// touch the zero padding and never write outputs that are discarded:
//   kspec_rows  K rows dy = 0..M-1, generated on the fly (K even in x and y, so each row
//               FFT is real): KA[q][dy], q = 0..P/2                        (1 x M FFTs)
//   rows_fwd    each pair of charge rows (a + i b) -> one complex FFT, untangled into
//               the half spectra of rows a and b: CA[c][q][row]            (3M/2 FFTs)
//   cols        per pair of columns q: K^ columns (one packed real-even FFT), then for
//               each channel FFT -> x K^ -> inverse FFT, keeping rows 0..M-1 (13 FFTs)
//   rows_inv    Hermitian rows -> one complex inverse FFT per row pair, keep 0..M-1
// Rows beyond M are zero and never loaded; outputs beyond M are never stored.  All FFTs
// are power-of-two Stockham radix-8/4/2 in shared memory with an fp64-generated twiddle
// table.  The 1/P^2 of the inverse is folded into the kernel samples.
#include <algorithm>

#include "device_math.cuh"
#include "tfdp_internal.h"

namespace tfdp {

namespace {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }
// multiply by -i
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }

template <int R>
__device__ __forceinline__ void dft(float2 (&v)[R]);

template <>
__device__ __forceinline__ void dft<2>(float2 (&v)[2]) {
  const float2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

template <>
__device__ __forceinline__ void dft<3>(float2 (&v)[3]) {
  // w = exp(-2 pi i / 3) = (-1/2, -sqrt3/2)
  const float c = -0.5f, sn = -0.86602540378443865f;
  const float2 s12 = cadd(v[1], v[2]), d12 = csub(v[1], v[2]);
  const float2 m = make_float2(fmaf(c, s12.x, v[0].x), fmaf(c, s12.y, v[0].y));
  const float2 t = make_float2(-sn * d12.y, sn * d12.x);  // i * sn * d12
  v[0] = cadd(v[0], s12);
  v[1] = cadd(m, t);
  v[2] = csub(m, t);
}

template <>
__device__ __forceinline__ void dft<5>(float2 (&v)[5]) {
  // direct 5-point DFT with the standard real/imag split
  const float c1 = 0.30901699437494742f, c2 = -0.80901699437494742f;
  const float s1 = -0.95105651629515357f, s2 = -0.58778525229247313f;
  const float2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
  const float2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
  const float2 x0 = v[0];
  const float2 m1 = make_float2(x0.x + c1 * a1.x + c2 * a2.x, x0.y + c1 * a1.y + c2 * a2.y);
  const float2 m2 = make_float2(x0.x + c2 * a1.x + c1 * a2.x, x0.y + c2 * a1.y + c1 * a2.y);
  // i*(s1 b1 + s2 b2), i*(s2 b1 - s1 b2)
  const float2 n1 = make_float2(-(s1 * b1.y + s2 * b2.y), s1 * b1.x + s2 * b2.x);
  const float2 n2 = make_float2(-(s2 * b1.y - s1 * b2.y), s2 * b1.x - s1 * b2.x);
  v[0] = cadd(x0, cadd(a1, a2));
  v[1] = cadd(m1, n1);
  v[4] = csub(m1, n1);
  v[2] = cadd(m2, n2);
  v[3] = csub(m2, n2);
}

template <>
__device__ __forceinline__ void dft<4>(float2 (&v)[4]) {
  // forward DFT-4: X_s = sum_r v_r (-i)^{rs}
  const float2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
  const float2 s13 = cadd(v[1], v[3]), d13 = mul_mi(csub(v[1], v[3]));
  v[0] = cadd(s02, s13);
  v[2] = csub(s02, s13);
  v[1] = cadd(d02, d13);
  v[3] = csub(d02, d13);
}

template <>
__device__ __forceinline__ void dft<8>(float2 (&v)[8]) {
  // radix-2 x radix-4: even/odd DFT-4s combined with W8^s
  float2 e[4] = {v[0], v[2], v[4], v[6]};
  float2 o[4] = {v[1], v[3], v[5], v[7]};
  dft<4>(e);
  dft<4>(o);
  const float h = 0.70710678118654752f;
  // W8^1 = (1 - i)/sqrt2, W8^2 = -i, W8^3 = (-1 - i)/sqrt2
  const float2 o1 = make_float2(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));
  const float2 o2 = mul_mi(o[2]);
  const float2 o3 = make_float2(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));
  v[0] = cadd(e[0], o[0]);
  v[4] = csub(e[0], o[0]);
  v[1] = cadd(e[1], o1);
  v[5] = csub(e[1], o1);
  v[2] = cadd(e[2], o2);
  v[6] = csub(e[2], o2);
  v[3] = cadd(e[3], o3);
  v[7] = csub(e[3], o3);
}

// Shared-memory layout of one FFT buffer: one float2 of padding per 8, which makes the
// strided Stockham stores of the first stages conflict-free.
__device__ __forceinline__ int pad(int i) { return i + (i >> 3); }
__host__ __device__ constexpr int padded_len(int N) { return N + (N >> 3) + 1; }

// Twiddle table (fp64-generated, fp32 stored), two-level so it fits in shared memory:
// tw[0..64) = exp(-2 pi i t / N), tw[64 + u] = exp(-2 pi i 64 u / N), u = 0..N/64; then
// exp(-2 pi i t / N) = tw[64 + (t >> 6)] * tw[t & 63]  (one complex product, ~1.5 ulp).
__host__ __device__ constexpr int tw_len(int N) { return 64 + N / 64 + 1; }

__device__ __forceinline__ float2 tw_at(const float2* __restrict__ tw, int t) {
  return cmul(tw[64 + (t >> 6)], tw[t & 63]);
}

// Twiddles w^r, r = 1..R-1, of one butterfly: at most three table lookups (w, w^2, w^4),
// the rest by at most two complex products.
template <int R>
__device__ __forceinline__ void twiddles(const float2* __restrict__ tw, int base, float2 (&w)[R]) {
  w[1] = tw_at(tw, base);
  if constexpr (R >= 3) w[2] = tw_at(tw, 2 * base);
  if constexpr (R >= 4) w[3] = cmul(w[1], w[2]);
  if constexpr (R == 5) w[4] = cmul(w[2], w[2]);
  if constexpr (R == 8) {
    w[4] = tw_at(tw, 4 * base);
    w[5] = cmul(w[4], w[1]);
    w[6] = cmul(w[4], w[2]);
    w[7] = cmul(w[4], w[3]);
  }
}

// In-place Stockham autosort stage (Govindaraju et al. 2008 formulation), radix R, size N,
// current sub-transform size Ns.  Every thread first loads + transforms its butterflies
// (registers), the block synchronises, then all results are stored: one buffer instead
// of ping-pong, so twice the FFTs fit in shared memory.  Requires blockDim.x >= N / 8.
template <int R>
struct PerThread { static constexpr int value = 1; };
template <> struct PerThread<4> { static constexpr int value = 2; };
template <> struct PerThread<2> { static constexpr int value = 4; };
template <> struct PerThread<3> { static constexpr int value = 3; };
template <> struct PerThread<5> { static constexpr int value = 2; };

template <int R>
__device__ __forceinline__ void stage(float2* buf, int N, int Ns, const float2* __restrict__ tw) {
  constexpr int MB = PerThread<R>::value;  // butterflies per thread (N/R <= MB * blockDim)
  const int nb = N / R;
  const int step = nb / Ns;  // N / (Ns R)
  const bool p2 = (Ns & (Ns - 1)) == 0;
  float2 v[MB][R];
#pragma unroll
  for (int b = 0; b < MB; ++b) {
    const int j = threadIdx.x + b * blockDim.x;
    if (j < nb) {
      const int k = p2 ? (j & (Ns - 1)) : (j % Ns);
#pragma unroll
      for (int r = 0; r < R; ++r) v[b][r] = buf[pad(j + r * nb)];
      if (Ns > 1) {
        float2 w[R];
        twiddles<R>(tw, k * step, w);
#pragma unroll
        for (int r = 1; r < R; ++r) v[b][r] = cmul(v[b][r], w[r]);
      }
      dft<R>(v[b]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < MB; ++b) {
    const int j = threadIdx.x + b * blockDim.x;
    if (j < nb) {
      const int k = p2 ? (j & (Ns - 1)) : (j % Ns);
      const int d = (j - k) * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) buf[pad(d + r * Ns)] = v[b][r];
    }
  }
  __syncthreads();
}

// Forward complex FFT of buf[0..N) (N = 2^a 3^b 5^c, padded layout) in shared memory, in
// place.  Power-of-two stages first (radix 8, then 4 / 2), odd radices last, so Ns is a
// power of two wherever possible.  Called by the whole block (blockDim.x >= N/8); the
// input must be visible (barrier) before the call; ends with a barrier.
__device__ void fft_smem(float2* buf, int N, const float2* __restrict__ tw) {
  int Ns = 1, rem = N;
  while (rem % 8 == 0) {
    stage<8>(buf, N, Ns, tw);
    Ns *= 8;
    rem /= 8;
  }
  if (rem % 4 == 0) {
    stage<4>(buf, N, Ns, tw);
    Ns *= 4;
    rem /= 4;
  }
  if (rem % 2 == 0) {
    stage<2>(buf, N, Ns, tw);
    Ns *= 2;
    rem /= 2;
  }
  while (rem % 3 == 0) {
    stage<3>(buf, N, Ns, tw);
    Ns *= 3;
    rem /= 3;
  }
  while (rem % 5 == 0) {
    stage<5>(buf, N, Ns, tw);
    Ns *= 5;
    rem /= 5;
  }
}

__global__ void twiddle_kernel(float2* tw, int N) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= tw_len(N)) return;
  const int t = i < 64 ? i : 64 * (i - 64);
  double s, c;
  sincospi(2.0 * (double)t / (double)N, &s, &c);
  tw[i] = make_float2((float)c, (float)-s);
}

// Copies the twiddle table to shared memory (caller synchronises before use).
__device__ __forceinline__ void load_tw(float2* dst, const float2* __restrict__ src, int N) {
  for (int i = threadIdx.x; i < tw_len(N); i += blockDim.x) dst[i] = src[i];
}

// ---------------------------------------------------------------- K spectrum rows
template <int G>
__global__ void __launch_bounds__(1024)
kspec_rows_kernel(const GridGeom* __restrict__ geom, int P, float neg_gamma,
                  const float2* __restrict__ tw, float* __restrict__ KA, int ka_pitch) {
  extern __shared__ float2 sm[];
  float2* a = sm;
  float2* tws = sm + padded_len(P);
  load_tw(tws, tw, P);
  const GridGeom g = *geom;
  const int M = g.M;
  const int dya = 2 * blockIdx.x, dyb = dya + 1;
  if (dya >= M) return;
  const float h2 = g.h * g.h;
  const float scale = 1.0f / ((float)P * (float)P);
  for (int x = threadIdx.x; x < P; x += blockDim.x) {
    const int dx = (x <= M - 1) ? x : ((x >= P - (M - 1)) ? x - P : INT32_MAX);
    float va = 0.f, vb = 0.f;
    if (dx != INT32_MAX) {
      const float dx2 = (float)(dx * dx);
      va = pow_neg<G>(fmaf(h2, dx2 + (float)(dya * dya), 1.0f), neg_gamma) * scale;
      if (dyb < M) vb = pow_neg<G>(fmaf(h2, dx2 + (float)(dyb * dyb), 1.0f), neg_gamma) * scale;
    }
    a[pad(x)] = make_float2(va, vb);
  }
  __syncthreads();
  fft_smem(a, P, tws);
  const float2* r = a;
  // real-even rows -> real spectra: row a in Re, row b in Im
  for (int q = threadIdx.x; q <= P / 2; q += blockDim.x) {
    const float2 z = r[pad(q)];
    KA[(int64_t)q * ka_pitch + dya] = z.x;
    if (dyb < M) KA[(int64_t)q * ka_pitch + dyb] = z.y;
  }
}

// ---------------------------------------------------------------- forward rows
__global__ void __launch_bounds__(1024)
rows_fwd_kernel(const GridGeom* __restrict__ geom, const float* __restrict__ C, int cpitch,
                int P, const float2* __restrict__ tw, float2* __restrict__ CA, int ca_pitch) {
  extern __shared__ float2 sm[];
  float2* a = sm;
  float2* tws = sm + padded_len(P);
  load_tw(tws, tw, P);
  const int M = geom->M;
  const int ra = 2 * blockIdx.x, rb = ra + 1;
  if (ra >= M) return;
  const int ch = blockIdx.y;
  const float* rowa = C + ((int64_t)ch * cpitch + ra) * cpitch;
  const float* rowb = rowa + cpitch;
  const bool hb = rb < M;
  for (int x = threadIdx.x; x < P; x += blockDim.x) {
    float va = 0.f, vb = 0.f;
    if (x < M) {
      va = rowa[x];
      if (hb) vb = rowb[x];
    }
    a[pad(x)] = make_float2(va, vb);
  }
  __syncthreads();
  fft_smem(a, P, tws);
  const float2* r = a;
  const int half = P / 2;
  float2* out = CA + (int64_t)ch * (half + 1) * ca_pitch;
  for (int q = threadIdx.x; q <= half; q += blockDim.x) {
    const float2 z = r[pad(q)];
    const float2 zc = conjf2(r[pad(q == 0 ? 0 : P - q)]);
    const float2 xa = make_float2(0.5f * (z.x + zc.x), 0.5f * (z.y + zc.y));
    const float2 xb = mul_mi(make_float2(0.5f * (z.x - zc.x), 0.5f * (z.y - zc.y)));
    float2* o = out + (int64_t)q * ca_pitch + ra;
    if (hb) {
      *reinterpret_cast<float4*>(o) = make_float4(xa.x, xa.y, xb.x, xb.y);
    } else {
      *o = xa;
    }
  }
}

// ---------------------------------------------------------------- columns
__global__ void __launch_bounds__(1024)
cols_kernel(const GridGeom* __restrict__ geom, float2* __restrict__ CA, int ca_pitch,
            const float* __restrict__ KA, int ka_pitch, int P, const float2* __restrict__ tw) {
  extern __shared__ float2 sm[];
  float2* a = sm;
  float2* tws = sm + padded_len(P);
  float* kh = reinterpret_cast<float*>(tws + tw_len(P));  // [2][P]
  load_tw(tws, tw, P);
  const int M = geom->M;
  const int half = P / 2;
  const int q0 = 2 * blockIdx.x, q1 = q0 + 1;
  const bool h1 = q1 <= half;
  // K^ columns q0, q1: real-even columns (mirror of dy = 0..M-1) packed as re/im
  for (int u = threadIdx.x; u < P; u += blockDim.x) {
    const int dy = (u <= M - 1) ? u : ((u >= P - (M - 1)) ? P - u : -1);
    float va = 0.f, vb = 0.f;
    if (dy >= 0) {
      va = KA[(int64_t)q0 * ka_pitch + dy];
      if (h1) vb = KA[(int64_t)q1 * ka_pitch + dy];
    }
    a[pad(u)] = make_float2(va, vb);
  }
  __syncthreads();
  {
    fft_smem(a, P, tws);
  const float2* r = a;
    for (int u = threadIdx.x; u < P; u += blockDim.x) {
      const float2 z = r[pad(u)];
      kh[u] = z.x;
      kh[P + u] = z.y;
    }
    __syncthreads();
  }
  for (int ch = 0; ch < 3; ++ch) {
    for (int s = 0; s < 2; ++s) {
      const int q = s ? q1 : q0;
      if (q > half) break;
      float2* col = CA + ((int64_t)ch * (half + 1) + q) * ca_pitch;
      for (int u = threadIdx.x; u < P; u += blockDim.x) a[pad(u)] = (u < M) ? col[u] : make_float2(0.f, 0.f);
      __syncthreads();
      fft_smem(a, P, tws);
      float2* r = a;
      // multiply by K^ (real) and conjugate for the inverse transform
      const float* k = kh + s * P;
      for (int u = threadIdx.x; u < P; u += blockDim.x) {
        const float2 z = r[pad(u)];
        const float kk = k[u];
        r[pad(u)] = make_float2(z.x * kk, -z.y * kk);
      }
      __syncthreads();
      fft_smem(r, P, tws);
      const float2* ri = r;
      for (int u = threadIdx.x; u < M; u += blockDim.x) {
        const float2 z = ri[pad(u)];
        col[u] = make_float2(z.x, -z.y);
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- inverse rows
__global__ void __launch_bounds__(1024)
rows_inv_kernel(const GridGeom* __restrict__ geom, const float2* __restrict__ CA, int ca_pitch,
                int P, const float2* __restrict__ tw, float* __restrict__ Phi, int cpitch) {
  extern __shared__ float2 sm[];
  float2* a = sm;
  float2* tws = sm + padded_len(P);
  load_tw(tws, tw, P);
  const int M = geom->M;
  const int ra = 2 * blockIdx.x, rb = ra + 1;
  if (ra >= M) return;
  const int ch = blockIdx.y;
  const bool hb = rb < M;
  const int half = P / 2;
  const float2* in = CA + (int64_t)ch * (half + 1) * ca_pitch;
  // Z[q] = Xa[q] + i Xb[q] over the full circle (Hermitian extension); stored conjugated
  // so that a forward FFT computes the inverse transform.
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    const int qq = (q <= half) ? q : P - q;
    float2 xa, xb = make_float2(0.f, 0.f);
    const float2* p = in + (int64_t)qq * ca_pitch + ra;
    if (hb) {
      const float4 v = *reinterpret_cast<const float4*>(p);
      xa = make_float2(v.x, v.y);
      xb = make_float2(v.z, v.w);
    } else {
      xa = *p;
    }
    if (q > half) {
      xa = conjf2(xa);
      xb = conjf2(xb);
    }
    const float2 z = make_float2(xa.x - xb.y, xa.y + xb.x);  // xa + i xb
    a[pad(q)] = conjf2(z);
  }
  __syncthreads();
  fft_smem(a, P, tws);
  const float2* r = a;
  float* pa = Phi + ((int64_t)ch * cpitch + ra) * cpitch;
  float* pb = pa + cpitch;
  for (int x = threadIdx.x; x < M; x += blockDim.x) {
    const float2 z = r[pad(x)];  // conj(result) = xa + i xb: xa = z.x, xb = -z.y
    pa[x] = z.x;
    if (hb) pb[x] = -z.y;
  }
}

__global__ void zero_planes_kernel(const GridGeom* __restrict__ geom, float* __restrict__ C, int cpitch) {
  const int M = geom->M;
  const int row = blockIdx.x;
  if (row >= M) return;
  float* p = C + ((int64_t)blockIdx.y * cpitch + row) * cpitch;
  for (int x = threadIdx.x; x < M; x += blockDim.x) p[x] = 0.f;
}

}  // namespace

void launch_twiddles(float2* tw, int P, cudaStream_t s) {
  twiddle_kernel<<<(tw_len(P) + 255) / 256, 256, 0, s>>>(tw, P);
}

void launch_zero_planes(const GridGeom* geom, float* C, int cpitch, int Mcap, cudaStream_t s) {
  zero_planes_kernel<<<dim3((unsigned)Mcap, 3), 256, 0, s>>>(geom, C, cpitch);
}

// Threads per FFT block: >= P/8 (one radix-8 butterfly each), multiple of 32, >= 128.
int fft_threads(int P) { return std::min(1024, std::max(128, ((P / 8) + 31) / 32 * 32)); }

size_t fftconv_smem_bytes(int P, int which) {
  // which: 0 rows (2 P float2), 1 cols (2 P float2 + 2 P float)
  const size_t base = (size_t)(padded_len(P) + tw_len(P)) * sizeof(float2);
  return which == 0 ? base : base + (size_t)2 * P * sizeof(float);
}

cudaError_t fftconv_prepare(int P) {
  const int r = (int)fftconv_smem_bytes(P, 0), c = (int)fftconv_smem_bytes(P, 1);
  cudaError_t e;
#define TFDP_ATTR(fn, bytes)                                                              \
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (bytes));     \
  if (e != cudaSuccess) return e;
  TFDP_ATTR(kspec_rows_kernel<0>, r);
  TFDP_ATTR(kspec_rows_kernel<1>, r);
  TFDP_ATTR(kspec_rows_kernel<2>, r);
  TFDP_ATTR(kspec_rows_kernel<3>, r);
  TFDP_ATTR(kspec_rows_kernel<4>, r);
  TFDP_ATTR(kspec_rows_kernel<8>, r);
  TFDP_ATTR(rows_fwd_kernel, r);
  TFDP_ATTR(rows_inv_kernel, r);
  TFDP_ATTR(cols_kernel, c);
#undef TFDP_ATTR
  return cudaSuccess;
}

void launch_kspec_rows(const GridGeom* geom, int P, int Mcap, ForceArgs fa, const float2* tw,
                       float* KA, int ka_pitch, cudaStream_t s) {
  const unsigned blocks = (unsigned)((Mcap + 1) / 2);
  const size_t sm = fftconv_smem_bytes(P, 0);
  const float ng = -fa.gamma;
  switch (fa.gamma_int) {
    case 1: kspec_rows_kernel<1><<<blocks, fft_threads(P), sm, s>>>(geom, P, ng, tw, KA, ka_pitch); break;
    case 2: kspec_rows_kernel<2><<<blocks, fft_threads(P), sm, s>>>(geom, P, ng, tw, KA, ka_pitch); break;
    case 3: kspec_rows_kernel<3><<<blocks, fft_threads(P), sm, s>>>(geom, P, ng, tw, KA, ka_pitch); break;
    case 4: kspec_rows_kernel<4><<<blocks, fft_threads(P), sm, s>>>(geom, P, ng, tw, KA, ka_pitch); break;
    case 8: kspec_rows_kernel<8><<<blocks, fft_threads(P), sm, s>>>(geom, P, ng, tw, KA, ka_pitch); break;
    default: kspec_rows_kernel<0><<<blocks, fft_threads(P), sm, s>>>(geom, P, ng, tw, KA, ka_pitch); break;
  }
}

void launch_rows_fwd(const GridGeom* geom, const float* C, int cpitch, int P, int Mcap,
                     const float2* tw, float2* CA, int ca_pitch, cudaStream_t s) {
  rows_fwd_kernel<<<dim3((unsigned)((Mcap + 1) / 2), 3), fft_threads(P), fftconv_smem_bytes(P, 0), s>>>(
      geom, C, cpitch, P, tw, CA, ca_pitch);
}

void launch_cols(const GridGeom* geom, float2* CA, int ca_pitch, const float* KA, int ka_pitch,
                 int P, const float2* tw, cudaStream_t s) {
  const unsigned blocks = (unsigned)((P / 2 + 1 + 1) / 2);
  cols_kernel<<<blocks, fft_threads(P), fftconv_smem_bytes(P, 1), s>>>(geom, CA, ca_pitch, KA, ka_pitch, P, tw);
}

void launch_rows_inv(const GridGeom* geom, const float2* CA, int ca_pitch, int P, int Mcap,
                     const float2* tw, float* Phi, int cpitch, cudaStream_t s) {
  rows_inv_kernel<<<dim3((unsigned)((Mcap + 1) / 2), 3), fft_threads(P), fftconv_smem_bytes(P, 0), s>>>(
      geom, CA, ca_pitch, P, tw, Phi, cpitch);
}

}  // namespace tfdp
