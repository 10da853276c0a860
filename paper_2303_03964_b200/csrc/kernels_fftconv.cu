// Hand-written FFT convolution of the ibFFT grid step (R9) — sm_100a.
//
// Replaces a zero-padded P x P 2-D R2C -> x K^ -> C2R by five passes that never transform
// the zero padding and never store outputs that are discarded:
//   kspec_rows  K rows dy = 0..P/2 of the periodic kernel generated on the fly (K is even
//               in x and y, so each row spectrum is real), four rows per block: KA[q][dy]
//   kspec_cols  four K^ columns per block (real-even): KH[q][u] (real), u = 0..P-1
//               (both skip unless setup found the held spectrum stale: K^ depends on
//               (P, h, gamma) only, and h = 1/k is constant under reading R5')
//   rows_fwd    four charge rows per block, two per complex FFT (a + i b), of one channel of
//               the interleaved charges, untangled into the half spectra CA[c][q][row] (32
//               contiguous bytes per q)
//   cols        two (channel, column) items per block: FFT -> x K^ -> inverse FFT, rows
//               0..M-1 kept
//   rows_inv    four Hermitian rows per block, two per complex inverse FFT, columns 0..M-1;
//               re-zeroes the same rows of the (consumed) charges, a third per channel block
// The inputs of every forward FFT are zero beyond P/2 (M <= P/2), so the first stage skips
// those loads; every inverse FFT keeps only outputs below P/2, so its last stage stores half.
//
// Every block runs TWO independent complex FFTs (lanes A, B) in SoA form: shared element e
// is the float4 {re_A, re_B, im_A, im_B} and a thread holds each value as two fp32x2 packs
// (re pair, im pair).  Then one LDS.128 / STS.128 moves a value of both FFTs; a complex add
// is 2 FADD2 for both lanes; a product with a twiddle (shared by the lanes: same position)
// is 4 instructions for both lanes with scalar-broadcast FMUL2/FFMA2 operands; a product
// by -i is a register renaming whose sign folds into the next FADD2; the twiddle chains are
// computed once for both FFTs.
//
// FFTs are in-place Stockham autosort stages (radix 16, then 16/8/4/2, then 3, 5) in shared
// memory, fully specialised at compile time for each supported P (P % 256 == 0,
// 2^a 3^b 5^c): every index, stride and loop bound is a constant.  One element of padding
// per 16 makes the strided stores conflict-free.  Twiddles come from a two-level
// fp64-generated table in shared memory and short product chains.  1/P^2 is folded into the
// kernel samples.
#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "device_math.cuh"
#include "tfdp_internal.h"

namespace tfdp {

namespace {

// ---------------------------------------------------------------- scalar complex (twiddles)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return __ffma2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x),
                    __fmul2_rn(make_float2(a.x, a.x), b));
}

// ---------------------------------------------------------------- SoA pair arithmetic
struct C2 {
  float2 re, im;  // (lane A, lane B)
};

__device__ __forceinline__ float2 bc(float s) { return make_float2(s, s); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ C2 add(C2 a, C2 b) {
  return {__fadd2_rn(a.re, b.re), __fadd2_rn(a.im, b.im)};
}
__device__ __forceinline__ C2 sub(C2 a, C2 b) {
  return {__fadd2_rn(a.re, neg2(b.re)), __fadd2_rn(a.im, neg2(b.im))};
}
__device__ __forceinline__ C2 mul_mi(C2 a) { return {a.im, neg2(a.re)}; }  // * (-i)
// a * (c + i s) for both lanes
__device__ __forceinline__ C2 mulw(C2 a, float c, float s) {
  return {__ffma2_rn(a.im, bc(-s), __fmul2_rn(a.re, bc(c))),
          __ffma2_rn(a.im, bc(c), __fmul2_rn(a.re, bc(s)))};
}
__device__ __forceinline__ C2 zero2() { return {make_float2(0.f, 0.f), make_float2(0.f, 0.f)}; }
__device__ __forceinline__ C2 ld(const float4* p) {
  const float4 q = *p;
  return {make_float2(q.x, q.y), make_float2(q.z, q.w)};
}
__device__ __forceinline__ void st(float4* p, C2 v) { *p = make_float4(v.re.x, v.re.y, v.im.x, v.im.y); }

template <int R>
__device__ __forceinline__ void dft(C2 (&v)[R]);

template <>
__device__ __forceinline__ void dft<2>(C2 (&v)[2]) {
  const C2 a = v[0], b = v[1];
  v[0] = add(a, b);
  v[1] = sub(a, b);
}

template <>
__device__ __forceinline__ void dft<3>(C2 (&v)[3]) {
  // w = exp(-2 pi i / 3) = (-1/2, -sqrt3/2)
  const float sn = -0.86602540378443865f;
  const C2 s12 = add(v[1], v[2]), d12 = sub(v[1], v[2]);
  const C2 m = {__ffma2_rn(s12.re, bc(-0.5f), v[0].re), __ffma2_rn(s12.im, bc(-0.5f), v[0].im)};
  const C2 t = {__fmul2_rn(d12.im, bc(-sn)), __fmul2_rn(d12.re, bc(sn))};  // i * sn * d12
  v[0] = add(v[0], s12);
  v[1] = add(m, t);
  v[2] = sub(m, t);
}

template <>
__device__ __forceinline__ void dft<5>(C2 (&v)[5]) {
  const float c1 = 0.30901699437494742f, c2 = -0.80901699437494742f;
  const float s1 = -0.95105651629515357f, s2 = -0.58778525229247313f;
  const C2 a1 = add(v[1], v[4]), b1 = sub(v[1], v[4]);
  const C2 a2 = add(v[2], v[3]), b2 = sub(v[2], v[3]);
  const C2 x0 = v[0];
  const C2 m1 = {__ffma2_rn(a2.re, bc(c2), __ffma2_rn(a1.re, bc(c1), x0.re)),
                 __ffma2_rn(a2.im, bc(c2), __ffma2_rn(a1.im, bc(c1), x0.im))};
  const C2 m2 = {__ffma2_rn(a2.re, bc(c1), __ffma2_rn(a1.re, bc(c2), x0.re)),
                 __ffma2_rn(a2.im, bc(c1), __ffma2_rn(a1.im, bc(c2), x0.im))};
  // n1 = i (s1 b1 + s2 b2), n2 = i (s2 b1 - s1 b2)
  const float2 u1r = __ffma2_rn(b2.re, bc(s2), __fmul2_rn(b1.re, bc(s1)));
  const float2 u1i = __ffma2_rn(b2.im, bc(s2), __fmul2_rn(b1.im, bc(s1)));
  const float2 u2r = __ffma2_rn(b2.re, bc(-s1), __fmul2_rn(b1.re, bc(s2)));
  const float2 u2i = __ffma2_rn(b2.im, bc(-s1), __fmul2_rn(b1.im, bc(s2)));
  const C2 n1 = {neg2(u1i), u1r}, n2 = {neg2(u2i), u2r};
  v[0] = add(x0, add(a1, a2));
  v[1] = add(m1, n1);
  v[4] = sub(m1, n1);
  v[2] = add(m2, n2);
  v[3] = sub(m2, n2);
}

template <>
__device__ __forceinline__ void dft<4>(C2 (&v)[4]) {
  const C2 s02 = add(v[0], v[2]), d02 = sub(v[0], v[2]);
  const C2 s13 = add(v[1], v[3]), d13 = mul_mi(sub(v[1], v[3]));
  v[0] = add(s02, s13);
  v[2] = sub(s02, s13);
  v[1] = add(d02, d13);
  v[3] = sub(d02, d13);
}

// o * W8 = o (h - i h) = (h (re + im), h (im - re));  o * W8^3 = o (-h - i h) =
// (h (im - re), -h (re + im))
__device__ __forceinline__ C2 mul_w8(C2 o, float h) {
  return {__fmul2_rn(__fadd2_rn(o.re, o.im), bc(h)), __fmul2_rn(__fadd2_rn(o.im, neg2(o.re)), bc(h))};
}
__device__ __forceinline__ C2 mul_w8_3(C2 o, float h) {
  return {__fmul2_rn(__fadd2_rn(o.im, neg2(o.re)), bc(h)), __fmul2_rn(__fadd2_rn(o.re, o.im), bc(-h))};
}

template <>
__device__ __forceinline__ void dft<8>(C2 (&v)[8]) {
  C2 e[4] = {v[0], v[2], v[4], v[6]};
  C2 o[4] = {v[1], v[3], v[5], v[7]};
  dft<4>(e);
  dft<4>(o);
  const float h = 0.70710678118654752f;
  const C2 o1 = mul_w8(o[1], h);
  const C2 o2 = mul_mi(o[2]);
  const C2 o3 = mul_w8_3(o[3], h);
  v[0] = add(e[0], o[0]);
  v[4] = sub(e[0], o[0]);
  v[1] = add(e[1], o1);
  v[5] = sub(e[1], o1);
  v[2] = add(e[2], o2);
  v[6] = sub(e[2], o2);
  v[3] = add(e[3], o3);
  v[7] = sub(e[3], o3);
}

// DFT-16 as 4 x 4 (Cooley-Tukey, r = 4 r1 + r2, s = s1 + 4 s2): DFT-4 over r1, twiddle
// W16^(r2 s1), DFT-4 over r2; outputs written back in natural order.
// ZU: inputs v[8..15] are zero (first stage of a zero-padded forward FFT): the first-level
// DFT-4s of (a, b, 0, 0) reduce to (a + b, a - i b, a - b, a + i b).
template <bool ZU = false>
__device__ __forceinline__ void dft16(C2 (&v)[16]) {
  C2 y[4][4];  // y[r2][s1]
#pragma unroll
  for (int r2 = 0; r2 < 4; ++r2) {
    if constexpr (ZU) {
      const C2 a = v[r2], b = v[r2 + 4], ib = mul_mi(b);  // -i b
      y[r2][0] = add(a, b);
      y[r2][1] = add(a, ib);
      y[r2][2] = sub(a, b);
      y[r2][3] = sub(a, ib);
    } else {
      C2 t[4] = {v[r2], v[r2 + 4], v[r2 + 8], v[r2 + 12]};
      dft<4>(t);
#pragma unroll
      for (int s1 = 0; s1 < 4; ++s1) y[r2][s1] = t[s1];
    }
  }
  const float h = 0.70710678118654752f;
  const float c1 = 0.92387953251128674f, s1_ = 0.38268343236508978f;  // cos, sin(pi/8)
  // W16^e = exp(-2 pi i e / 16) for the products e = r2 * s1
  y[1][1] = mulw(y[1][1], c1, -s1_);  // W1
  y[1][2] = mul_w8(y[1][2], h);       // W2
  y[1][3] = mulw(y[1][3], s1_, -c1);  // W3
  y[2][1] = mul_w8(y[2][1], h);       // W2
  y[2][2] = mul_mi(y[2][2]);          // W4 = -i
  y[2][3] = mul_w8_3(y[2][3], h);     // W6
  y[3][1] = mulw(y[3][1], s1_, -c1);  // W3
  y[3][2] = mul_w8_3(y[3][2], h);     // W6
  y[3][3] = mulw(y[3][3], -c1, s1_);  // W9
#pragma unroll
  for (int s1 = 0; s1 < 4; ++s1) {
    C2 t[4] = {y[0][s1], y[1][s1], y[2][s1], y[3][s1]};
    dft<4>(t);
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) v[s1 + 4 * s2] = t[s2];
  }
}

template <>
__device__ __forceinline__ void dft<16>(C2 (&v)[16]) {
  dft16<false>(v);
}

// Shared-memory layout: one element of padding per 16 (pad(i) = i + i/16): the strided
// Stockham stores of the first stages become conflict-free and, since every stride is a
// multiple of 16 (P % 256 == 0), address(r) = base + r * padded_stride.
__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded_len(int N) { return N + (N >> 4) + 1; }

// Half-spectrum layout CA (element (channel ch, frequency q, grid row r), H = P/2 + 1
// frequencies, ca_pitch rows, a multiple of kCaTile): row tiles of kCaTile rows,
// CA[ch][r / kCaTile][q][r % kCaTile].  A row pass over 4 rows writes / reads 32 B per q at a
// stride of 8 kCaTile bytes (a sequential sweep instead of the column-major stride of
// 8 ca_pitch bytes), the column pass reads a column as kCaTile * 8-byte runs.  Measured at
// C4 (rows_fwd + cols + rows_inv, us; column-major / tile 4 / 8 / 16 / 32): k = 1
// 76.9 / 75.2 / 75.4 / 78.0 / 78.0, k = 2 276 / 289 / 277 / 277 / 278, k = 3
// 692 / 674 / 649 / 675 / 670.
#ifndef TFDP_CA_TILE
#define TFDP_CA_TILE 8
#endif
constexpr int kCaTile = TFDP_CA_TILE;
static_assert(kCaTile >= 4 && (kCaTile & (kCaTile - 1)) == 0, "CA tile: power of 2 >= 4");
__device__ __forceinline__ int64_t ca_col_base(int ch, int q, int H, int ca_pitch) {
  return ((int64_t)ch * (ca_pitch / kCaTile) * H + q) * kCaTile;
}
// offset of row r from its column base
__device__ __forceinline__ int64_t ca_row_off(int r, int H) {
  return (int64_t)(r / kCaTile) * kCaTile * H + (r % kCaTile);
}

// Two-level twiddle table: tw[0..64) = exp(-2 pi i t / N), tw[64 + u] = exp(-2 pi i 64u / N),
// exp(-2 pi i t / N) = tw[64 + t/64] * tw[t % 64].
__host__ __device__ constexpr int tw_len(int N) { return 64 + N / 64 + 1; }
__device__ __forceinline__ float2 tw_at(const float2* __restrict__ tw, int t) {
  return cmul(tw[64 + (t >> 6)], tw[t & 63]);
}

// w^r for r = 1..R-1 from one table lookup and a product chain of depth <= 3.
template <int R>
__device__ __forceinline__ void twiddles(const float2* __restrict__ tw, int base, float2 (&w)[R]) {
  w[1] = tw_at(tw, base);
  if constexpr (R >= 3) w[2] = cmul(w[1], w[1]);
  if constexpr (R >= 4) w[3] = cmul(w[2], w[1]);
  if constexpr (R >= 5) w[4] = cmul(w[2], w[2]);
  if constexpr (R >= 8) {
    w[5] = cmul(w[4], w[1]);
    w[6] = cmul(w[4], w[2]);
    w[7] = cmul(w[4], w[3]);
  }
  if constexpr (R == 16) {  // second lookup keeps the product chains at depth <= 3
    w[8] = tw_at(tw, 8 * base);
#pragma unroll
    for (int r = 1; r < 8; ++r) w[8 + r] = cmul(w[8], w[r]);
  }
}

// Threads per FFT-pair block: the smallest of {128, 256, 384, 512} >= P/16 (one radix-16
// butterfly of both FFTs per thread).
__host__ __device__ constexpr int fft_threads_c(int P) {
  return P <= 2048 ? 128 : P <= 4096 ? 256 : P <= 6144 ? 384 : P <= 8192 ? 512 : 1024;
}

// Blocks per SM the register cap aims for.
template <int T>
constexpr int kMinBlocks = T == 128 ? 5 : T == 256 ? 3 : T == 384 ? 2 : 1;

// FFT flags: inputs zero at index >= N/2 (first stage skips them); only outputs < N/2 needed
// (last stage stores half).
enum { kZeroUpper = 1, kLowOut = 2 };

// In-place Stockham autosort stage (Govindaraju et al. 2008 formulation): radix R, size N,
// sub-transform size Ns (1 for the first stage, else a multiple of 16 since N % 256 == 0 and
// the first stage is radix 16).  Loads + butterflies into registers, barrier, stores, barrier.
// The last stage (Ns R = N) reads and writes the same elements per butterfly, so it needs no
// barrier between its loads and stores and streams one butterfly at a time.
// I/O fusion: the first stage takes its inputs from src(e) (element e in natural order) and
// the last stage hands its outputs to dst(e, v) unless they are SmemIO — so a kernel reads its
// global inputs straight into the first butterflies and writes its global outputs straight
// from the last ones, without a shared-memory round trip for either.
struct SmemIO {};

template <int T, int R, int N, int Ns, bool ZERO_UPPER, bool LOW_OUT, class Src, class Dst>
__device__ __forceinline__ void stage(float4* buf, const float2* __restrict__ tw, int tid,
                                      const Src& src, const Dst& dst) {
  constexpr int nb = N / R;
  constexpr int MB = (nb + T - 1) / T;  // butterflies per thread
  constexpr int step = nb / Ns;         // N / (Ns R)
  constexpr int sin_ = nb + (nb >> 4);  // padded stride of the loads (nb % 16 == 0)
  constexpr int sout = Ns == 1 ? 1 : Ns + (Ns >> 4);
  constexpr bool p2 = (Ns & (Ns - 1)) == 0;
  constexpr bool first = Ns == 1;
  constexpr bool last = Ns * R == N;
  constexpr bool src_smem = !first || std::is_same<Src, SmemIO>::value;
  constexpr bool dst_smem = !last || std::is_same<Dst, SmemIO>::value;
  auto butterfly = [&](int j, C2 (&v)[R]) {
    const int pj = j + (j >> 4);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (ZERO_UPPER && 2 * r >= R) v[r] = zero2();
      else if constexpr (src_smem) v[r] = ld(buf + pj + r * sin_);
      else v[r] = src(j + r * nb);
    }
    if constexpr (Ns > 1) {
      const int k = p2 ? (j & (Ns - 1)) : (j % Ns);
      float2 w[R];
      twiddles<R>(tw, k * step, w);
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = mulw(v[r], w[r].x, w[r].y);
    }
    if constexpr (ZERO_UPPER && R == 16) dft16<true>(v);
    else dft<R>(v);
  };
  if constexpr (last && Ns > 1) {
    // d = j: in place per butterfly
#pragma unroll 1
    for (int b = 0; b < MB; ++b) {
      const int j = tid + b * T;
      if (nb % T == 0 || j < nb) {
        C2 v[R];
        butterfly(j, v);
        const int pd = j + (j >> 4);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!LOW_OUT || 2 * r < R) {
            if constexpr (dst_smem) st(buf + pd + r * sout, v[r]);
            else dst(j + r * Ns, v[r]);
          }
        }
      }
    }
    if constexpr (dst_smem) __syncthreads();
  } else {
    C2 v[MB][R];
#pragma unroll
    for (int b = 0; b < MB; ++b) {
      const int j = tid + b * T;
      if (nb % T == 0 || j < nb) butterfly(j, v[b]);
    }
    if constexpr (src_smem) __syncthreads();
#pragma unroll
    for (int b = 0; b < MB; ++b) {
      const int j = tid + b * T;
      if (nb % T == 0 || j < nb) {
        const int k = Ns == 1 ? 0 : (p2 ? (j & (Ns - 1)) : (j % Ns));
        const int d = (j - k) * R + k;
        const int pd = d + (d >> 4);
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (!LOW_OUT || 2 * r < R) st(buf + pd + r * sout, v[b][r]);
      }
    }
    __syncthreads();
  }
}

__host__ __device__ constexpr int next_radix(int rem) {
  return rem % 16 == 0 ? 16 : rem % 8 == 0 ? 8 : rem % 4 == 0 ? 4 : rem % 2 == 0 ? 2
       : rem % 3 == 0 ? 3 : 5;
}

template <int T, int N, int FLAGS, int Ns, int REM, class Src, class Dst>
__device__ __forceinline__ void fft_rec(float4* buf, const float2* __restrict__ tw, int tid,
                                        const Src& src, const Dst& dst) {
  if constexpr (REM > 1) {
    constexpr int R = next_radix(REM);
    constexpr bool first = Ns == 1, last = REM == R;
    stage<T, R, N, Ns, first && (FLAGS & kZeroUpper) != 0,
          last && (FLAGS & kLowOut) != 0 && R % 2 == 0>(buf, tw, tid, src, dst);
    fft_rec<T, N, FLAGS, Ns * R, REM / R>(buf, tw, tid, src, dst);
  }
}

// ---- convolution column: forward FFT -> x K^ -> inverse FFT with the forward's last stage
// and the inverse's first stage fused in registers.  With radix 16 at both ends, the thread
// that finishes forward butterfly j holds the outputs X[j + r N/16], r = 0..15 — exactly the
// inputs x[j + r nb] (nb = N/16) of inverse first-stage butterfly j — so the product with
// K^ and the first inverse butterfly need no shared-memory round trip (two of the ~14 passes
// of a column pair).  The forward plan keeps a radix 16 for its last stage (16, ..., 16).
template <int REM, bool FIRST>
__host__ __device__ constexpr int radix_last16() {
  return (FIRST || REM == 16) ? 16 : next_radix(REM / 16);
}

// forward stages while more than the final radix-16 stage remains (first stage: ZU, src)
template <int T, int N, int Ns, int REM, class Src>
__device__ __forceinline__ void fwd_head(float4* buf, const float2* __restrict__ tw, int tid,
                                         const Src& src) {
  if constexpr (REM > 16) {
    constexpr int R = radix_last16<REM, Ns == 1>();
    stage<T, R, N, Ns, Ns == 1, false>(buf, tw, tid, src, SmemIO{});
    fwd_head<T, N, Ns * R, REM / R>(buf, tw, tid, src);
  }
}

// forward last stage (radix 16, Ns = N/16) -> kmul(u, X[u]) (= conj(X K^)) -> inverse first
// stage (radix 16, Ns = 1) -> shared memory
template <int T, int N, class KMul>
__device__ __forceinline__ void fused_mid(float4* buf, const float2* __restrict__ tw, int tid,
                                          const KMul& kmul) {
  constexpr int R = 16, nb = N / R, MB = (nb + T - 1) / T;
  constexpr int sin_ = nb + (nb >> 4);
  C2 v[MB][R];
#pragma unroll
  for (int b = 0; b < MB; ++b) {
    const int j = tid + b * T;
    if (nb % T == 0 || j < nb) {
      const int pj = j + (j >> 4);
#pragma unroll
      for (int r = 0; r < R; ++r) v[b][r] = ld(buf + pj + r * sin_);
      float2 w[R];
      twiddles<R>(tw, j, w);  // Ns = nb: k = j, step = 1
#pragma unroll
      for (int r = 1; r < R; ++r) v[b][r] = mulw(v[b][r], w[r].x, w[r].y);
      dft16<false>(v[b]);
#pragma unroll
      for (int r = 0; r < R; ++r) v[b][r] = kmul(j + r * nb, v[b][r]);
      dft16<false>(v[b]);  // inverse first stage: inputs at j + r nb
    }
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < MB; ++b) {
    const int j = tid + b * T;
    if (nb % T == 0 || j < nb) {
      const int d = j * R;  // first-stage outputs: d = j R + r
#pragma unroll
      for (int r = 0; r < R; ++r) st(buf + (d + r) + ((d + r) >> 4), v[b][r]);
    }
  }
  __syncthreads();
}

// Forward complex FFTs (both lanes) of N elements, N = 2^a 3^b 5^c, N % 256 == 0, in the
// padded shared buffer (in place) — inputs from src / outputs to dst when those are not
// SmemIO.  Radix 16 first (so Ns is a multiple of 16 afterwards), then 16/8/4/2, then 3, 5.
// Called by the whole block (T >= N/16 threads); a shared-memory source must be complete
// (barrier) before the call; ends with a barrier unless the outputs go to dst.
template <int T, int N, int FLAGS, class Src = SmemIO, class Dst = SmemIO>
__device__ __forceinline__ void fft_smem(float4* buf, const float2* __restrict__ tw,
                                         const Src& src = Src{}, const Dst& dst = Dst{}) {
  static_assert(N % 256 == 0 && T * 16 >= N, "FFT plan");
  fft_rec<T, N, FLAGS, 1, N>(buf, tw, threadIdx.x, src, dst);
}

__global__ void twiddle_kernel(float2* tw, int N) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= tw_len(N)) return;
  const int t = i < 64 ? i : 64 * (i - 64);
  double s, c;
  sincospi(2.0 * (double)t / (double)N, &s, &c);
  tw[i] = make_float2((float)c, (float)-s);
}

__device__ __forceinline__ void load_tw(float2* dst, const float2* __restrict__ src, int N) {
  for (int i = threadIdx.x; i < tw_len(N); i += blockDim.x) dst[i] = src[i];
}

// t-kernel sample (1 + d^2)^-gamma with the integer-gamma fast paths (uniform branch).
__device__ __forceinline__ float ksample(float s, float neg_gamma, int gi) {
  switch (gi) {
    case 1: return pow_neg<1>(s, neg_gamma);
    case 2: return pow_neg<2>(s, neg_gamma);
    case 3: return pow_neg<3>(s, neg_gamma);
    case 4: return pow_neg<4>(s, neg_gamma);
    case 8: return pow_neg<8>(s, neg_gamma);
    default: return pow_neg<0>(s, neg_gamma);
  }
}

// Slab-mode output of the column pass (out of line: keeps the one-GPU column pass's register
// allocation unchanged): rows u of columns (chA, qA), (chB, qB) into the row owner's CA.
__device__ __noinline__ void route_store_cols(const PeerRoute* __restrict__ rt, int u, int H,
                                              int chA, int qA, int chB, int qB, bool hB,
                                              float2 re, float2 im) {
  float2* ca = rt->ca[route_owner(rt->row0, rt->world, u)];
  const int64_t o = ca_row_off(u, H);
  ca[ca_col_base(chA, qA, H, rt->ca_pitch) + o] = make_float2(re.x, -im.x);
  if (hB) ca[ca_col_base(chB, qB, H, rt->ca_pitch) + o] = make_float2(re.y, -im.y);
}

#define TFDP_FFT_KERNEL(name) \
  template <int P>            \
  __global__ void __launch_bounds__(fft_threads_c(P), kMinBlocks<fft_threads_c(P)>) name

// Common prologue: smem = [padded_len(P)] float4 + the twiddle table.
#define TFDP_FFT_PROLOGUE                                              \
  constexpr int T = fft_threads_c(P);                                  \
  extern __shared__ float4 sm4[];                                      \
  float4* a = sm4;                                                     \
  float2* tws = reinterpret_cast<float2*>(sm4 + padded_len(P));        \
  load_tw(tws, tw, P); /* constant since the plan: before the wait */ \
  pdl_wait();                                                          \
  pdl_trigger();

// ---------------------------------------------------------------- K spectrum: rows
// The kernel is sampled over the whole periodic P x P range, K(h d(x), h d(y)) with
// d(x) = x for x <= P/2 and x - P above: the kept outputs of the circular convolution only
// ever use offsets |d| <= M - 1 (charges and outputs both live in [0, M), P >= 2M - 1, R9),
// so the other samples are free — and with them K^ depends on (P, h, gamma) alone, not on
// M: setup decides (geom->kspec) whether the spectrum held in KH is still the right one.
// four rows dy0..dy0+3 (dy <= P/2; rows P - dy are the same by evenness) per block: lane A =
// row dy0 + i row dy0+1, lane B = rows dy0+2, +3; the real-even row spectra (q <= P/2) leave
// from the last stage
TFDP_FFT_KERNEL(kspec_rows_kernel)(const GridGeom* __restrict__ geom, float neg_gamma, int gi,
                                   const float2* __restrict__ tw, float* __restrict__ KA) {
  if (!geom->kspec) return;  // spectrum of this (P, h, gamma) already in KH
  TFDP_FFT_PROLOGUE
  constexpr int half = P / 2;
  constexpr int ka_pitch = half + 1;
  const float h = geom->h;
  const int dy0 = 4 * blockIdx.x;
  if (dy0 > half) return;
  const float h2 = h * h;
  const float scale = 1.0f / ((float)P * (float)P);
  for (int x = threadIdx.x; x < P; x += T) {
    const int dx = x <= half ? x : x - P;
    const float dx2 = (float)(dx * dx);
    float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int dy = dy0 + c;
      if (dy <= half) v[c] = ksample(fmaf(h2, dx2 + (float)(dy * dy), 1.0f), neg_gamma, gi) * scale;
    }
    a[pad(x)] = make_float4(v[0], v[2], v[1], v[3]);
  }
  __syncthreads();
  auto dst = [&](int q, C2 z) {  // real-even rows: Re = even row, Im = odd row
    if (q > half) return;
    float* o = KA + (int64_t)q * ka_pitch + dy0;
    const float r4[4] = {z.re.x, z.im.x, z.re.y, z.im.y};
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (dy0 + c <= half) o[c] = r4[c];
  };
  fft_smem<T, P, 0>(a, tws, SmemIO{}, dst);
}

// ---------------------------------------------------------------- K spectrum: columns
// four columns q0..q0+3 per block (lane A = q0 + i q0+1, lane B = q0+2 + i q0+3), each the
// real-even mirror of dy = 0..P/2, read by the first stage; KH written by the last
TFDP_FFT_KERNEL(kspec_cols_kernel)(const GridGeom* __restrict__ geom,
                                   const float* __restrict__ KA, const float2* __restrict__ tw,
                                   float* __restrict__ KH) {
  if (!geom->kspec) return;  // (geom was written by setup, before kspec_rows started)
  TFDP_FFT_PROLOGUE
  constexpr int half = P / 2;
  constexpr int ka_pitch = half + 1;
  const int q0 = 4 * blockIdx.x;
  __syncthreads();  // twiddle table
  auto src = [&](int u) {
    const int dy = u <= half ? u : P - u;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (q0 + c <= half) v[c] = KA[(int64_t)(q0 + c) * ka_pitch + dy];
    return C2{make_float2(v[0], v[2]), make_float2(v[1], v[3])};
  };
  auto dst = [&](int u, C2 z) {
    const float r4[4] = {z.re.x, z.im.x, z.re.y, z.im.y};
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (q0 + c <= half) KH[(int64_t)(q0 + c) * P + u] = r4[c];
  };
  fft_smem<T, P, 0>(a, tws, src, dst);
}

// ---------------------------------------------------------------- columns
// Two (channel, column) items per block, three blocks per two columns q = 2u, 2u+1:
//   sub 0: (ch 0, 2u) and (ch 0, 2u+1);  sub 1: (ch 1, 2u), (ch 2, 2u);  sub 2: (ch 1, 2u+1),
//   (ch 2, 2u+1) — the blocks of a column pair are adjacent (K^ columns shared in L2).
// The forward FFT reads the columns in its first stage and multiplies by K^ (conjugated for
// the inverse) in its last; the inverse FFT writes rows 0..M-1 from its last stage.
TFDP_FFT_KERNEL(cols_kernel)(const GridGeom* __restrict__ geom, float2* __restrict__ CA,
                             int ca_pitch, const float* __restrict__ KH,
                             const float2* __restrict__ tw, int q_base, int Hl,
                             const PeerRoute* __restrict__ rt) {
  TFDP_FFT_PROLOGUE
  const int M = geom->M;
  constexpr int half = P / 2;
  // columns [q_base, q_base + Hl) live in CA (q_base even; the whole half spectrum on one
  // GPU, a column chunk of it per rank in the multi-GPU slab mode)
  const int u2 = q_base / 2 + blockIdx.x / 3, sub = blockIdx.x % 3;
  int chA, qA, chB, qB;
  if (sub == 0) {
    chA = 0, qA = 2 * u2, chB = 0, qB = 2 * u2 + 1;
  } else {
    const int q = 2 * u2 + sub - 1;
    chA = 1, qA = q, chB = 2, qB = q;
  }
  if (qA > half || qA >= q_base + Hl) return;
  const bool hB = qB <= half && qB < q_base + Hl;
  const int H = Hl;
  float2* colA = CA + ca_col_base(chA, qA - q_base, H, ca_pitch);
  float2* colB = CA + ca_col_base(chB, (hB ? qB : qA) - q_base, H, ca_pitch);
  const float* khA = KH + (int64_t)qA * P;
  const float* khB = KH + (int64_t)(hB ? qB : qA) * P;
  __syncthreads();  // twiddle table
  auto src = [&](int u) {  // u < P/2 (ZU)
    float2 va = make_float2(0.f, 0.f), vb = va;
    if (u < M) {
      const int64_t o = ca_row_off(u, H);
      va = colA[o];
      if (hB) vb = colB[o];
    }
    return C2{make_float2(va.x, vb.x), make_float2(va.y, vb.y)};
  };
  auto kmul = [&](int u, C2 z) {  // x K^ (real), conjugated for the inverse
    const float2 k = make_float2(__ldg(khA + u), __ldg(khB + u));
    return C2{__fmul2_rn(z.re, k), __fmul2_rn(z.im, neg2(k))};
  };
  auto out = [&](int u, C2 z) {  // u < P/2 (LowOut)
    if (u < M) {
      if (rt) {  // slab mode, fused transpose back: into the row owner's half spectra
        route_store_cols(rt, u, half + 1, chA, qA, chB, qB, hB, z.re, z.im);
      } else {
        const int64_t o = ca_row_off(u, H);
        colA[o] = make_float2(z.re.x, -z.im.x);
        if (hB) colB[o] = make_float2(z.re.y, -z.im.y);
      }
    }
  };
  // Fused only where it measured faster (C4, us per launch, separate / fused): P = 2048
  // 31.1 / 29.1; P = 4096 120.1 / 127.3 and P = 6144 346.4 / 348.6 — there the fused middle
  // holds both radix-16 butterflies and the K^ loads live at the 80-register cap (spills).
  if constexpr (P <= 2048) {
    fwd_head<T, P, 1, P>(a, tws, threadIdx.x, src);  // forward stages but the last
    fused_mid<T, P>(a, tws, threadIdx.x, kmul);       // last forward, x K^, first inverse
    fft_rec<T, P, kLowOut, 16, P / 16>(a, tws, threadIdx.x, SmemIO{}, out);
  } else {
    auto mult = [&](int u, C2 z) { st(a + pad(u), kmul(u, z)); };
    fft_smem<T, P, kZeroUpper>(a, tws, src, mult);
    __syncthreads();
    fft_smem<T, P, kLowOut>(a, tws, SmemIO{}, out);
  }
}

// ================================================================ AoS core (row passes)
// The row passes keep one complex FFT per group of T threads in AoS (float2) layout with RB
// groups per block: the transposed half-spectrum accesses of a row pass are latency-bound,
// and the AoS form needs ~60 registers (radix-16 butterfly of one FFT) against ~84 for the
// SoA pair, i.e. 32 instead of 24 warps per SM (C4 k = 1: rows_fwd 23.0 vs 28.8 us, rows_inv
// 20.9 vs 23.0 us; k = 3: 158 vs 214 us).
namespace aos {

template <int T>
constexpr int kMinBlocksA = T == 128 ? 8 : T == 256 ? 4 : T == 384 ? 3 : T == 512 ? 2 : 1;

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
  return __ffma2_rn(b, make_float2(-1.0f, -1.0f), a);
}
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }  // * (-i)

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
  const float c1 = 0.30901699437494742f, c2 = -0.80901699437494742f;
  const float s1 = -0.95105651629515357f, s2 = -0.58778525229247313f;
  const float2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
  const float2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
  const float2 x0 = v[0];
  const float2 m1 = make_float2(x0.x + c1 * a1.x + c2 * a2.x, x0.y + c1 * a1.y + c2 * a2.y);
  const float2 m2 = make_float2(x0.x + c2 * a1.x + c1 * a2.x, x0.y + c2 * a1.y + c1 * a2.y);
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
  const float2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
  const float2 s13 = cadd(v[1], v[3]), d13 = mul_mi(csub(v[1], v[3]));
  v[0] = cadd(s02, s13);
  v[2] = csub(s02, s13);
  v[1] = cadd(d02, d13);
  v[3] = csub(d02, d13);
}

template <>
__device__ __forceinline__ void dft<8>(float2 (&v)[8]) {
  float2 e[4] = {v[0], v[2], v[4], v[6]};
  float2 o[4] = {v[1], v[3], v[5], v[7]};
  dft<4>(e);
  dft<4>(o);
  const float h = 0.70710678118654752f;
  const float2 o1 = make_float2(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));  // W8
  const float2 o2 = mul_mi(o[2]);                                               // W8^2
  const float2 o3 = make_float2(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y)); // W8^3
  v[0] = cadd(e[0], o[0]);
  v[4] = csub(e[0], o[0]);
  v[1] = cadd(e[1], o1);
  v[5] = csub(e[1], o1);
  v[2] = cadd(e[2], o2);
  v[6] = csub(e[2], o2);
  v[3] = cadd(e[3], o3);
  v[7] = csub(e[3], o3);
}

// DFT-16 as 4 x 4 (Cooley-Tukey, r = 4 r1 + r2, s = s1 + 4 s2): DFT-4 over r1, twiddle
// W16^(r2 s1), DFT-4 over r2; outputs written back in natural order.
// ZU: inputs v[8..15] are zero (first stage of a zero-padded forward FFT): the first-level
// DFT-4s of (a, b, 0, 0) reduce to (a + b, a - i b, a - b, a + i b).  (The compiler cannot
// fold x + 0 in IEEE arithmetic, hence the explicit variant.)
template <bool ZU = false>
__device__ __forceinline__ void dft16(float2 (&v)[16]) {
  float2 y[4][4];  // y[r2][s1]
#pragma unroll
  for (int r2 = 0; r2 < 4; ++r2) {
    if constexpr (ZU) {
      const float2 a = v[r2], b = v[r2 + 4], ib = mul_mi(b);  // -i b
      y[r2][0] = cadd(a, b);
      y[r2][1] = cadd(a, ib);
      y[r2][2] = csub(a, b);
      y[r2][3] = csub(a, ib);
    } else {
      float2 t[4] = {v[r2], v[r2 + 4], v[r2 + 8], v[r2 + 12]};
      dft<4>(t);
#pragma unroll
      for (int s1 = 0; s1 < 4; ++s1) y[r2][s1] = t[s1];
    }
  }
  const float h = 0.70710678118654752f;
  const float c1 = 0.92387953251128674f, s1_ = 0.38268343236508978f;  // cos, sin(pi/8)
  // W16^e = exp(-2 pi i e / 16) for the products e = r2 * s1
  const float2 W1 = make_float2(c1, -s1_), W2 = make_float2(h, -h), W3 = make_float2(s1_, -c1);
  const float2 W6 = make_float2(-h, -h), W9 = make_float2(-c1, s1_);
  y[1][1] = cmul(y[1][1], W1);
  y[1][2] = cmul(y[1][2], W2);
  y[1][3] = cmul(y[1][3], W3);
  y[2][1] = cmul(y[2][1], W2);
  y[2][2] = mul_mi(y[2][2]);  // W16^4 = -i
  y[2][3] = cmul(y[2][3], W6);
  y[3][1] = cmul(y[3][1], W3);
  y[3][2] = cmul(y[3][2], W6);
  y[3][3] = cmul(y[3][3], W9);
#pragma unroll
  for (int s1 = 0; s1 < 4; ++s1) {
    float2 t[4] = {y[0][s1], y[1][s1], y[2][s1], y[3][s1]};
    dft<4>(t);
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) v[s1 + 4 * s2] = t[s2];
  }
}

template <>
__device__ __forceinline__ void dft<16>(float2 (&v)[16]) {
  dft16<false>(v);
}

// In-place Stockham autosort stage (Govindaraju et al. 2008 formulation): radix R, size N,
// sub-transform size Ns (1 for the first stage, else a multiple of 16 since N % 256 == 0 and
// the first stage is radix 16).  Loads + butterflies into registers, barrier, stores, barrier.
// I/O fusion as in the SoA core: the first stage takes its inputs from src(x) and the last
// hands its outputs to dst(x, v) (natural order) unless they are SmemIO — no shared-memory
// round trip (and no barrier) for the kernel's global loads / stores.
template <int T, int R, int N, int Ns, bool ZERO_UPPER, bool LOW_OUT, class Src, class Dst>
__device__ __forceinline__ void stage(float2* buf, const float2* __restrict__ tw, int tid,
                                      const Src& src, const Dst& dst) {
  constexpr int nb = N / R;
  constexpr int MB = (nb + T - 1) / T;  // butterflies per thread
  constexpr int step = nb / Ns;         // N / (Ns R)
  constexpr int sin_ = nb + (nb >> 4);  // padded stride of the loads (nb % 16 == 0)
  constexpr int sout = Ns == 1 ? 1 : Ns + (Ns >> 4);
  constexpr bool p2 = (Ns & (Ns - 1)) == 0;
  constexpr bool first = Ns == 1;
  constexpr bool last = Ns * R == N;
  constexpr bool src_smem = !first || std::is_same<Src, SmemIO>::value;
  constexpr bool dst_smem = !last || std::is_same<Dst, SmemIO>::value;
  float2 v[MB][R];
#pragma unroll
  for (int b = 0; b < MB; ++b) {
    const int j = tid + b * T;
    if (nb % T == 0 || j < nb) {
      const int pj = j + (j >> 4);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (ZERO_UPPER && 2 * r >= R) v[b][r] = make_float2(0.f, 0.f);
        else if constexpr (src_smem) v[b][r] = buf[pj + r * sin_];
        else v[b][r] = src(j + r * nb);
      }
      if constexpr (Ns > 1) {
        const int k = p2 ? (j & (Ns - 1)) : (j % Ns);
        float2 w[R];
        twiddles<R>(tw, k * step, w);
#pragma unroll
        for (int r = 1; r < R; ++r) v[b][r] = cmul(v[b][r], w[r]);
      }
      if constexpr (ZERO_UPPER && R == 16) dft16<true>(v[b]);
      else dft<R>(v[b]);
    }
  }
  if constexpr (src_smem && dst_smem) __syncthreads();
#pragma unroll
  for (int b = 0; b < MB; ++b) {
    const int j = tid + b * T;
    if (nb % T == 0 || j < nb) {
      const int k = Ns == 1 ? 0 : (p2 ? (j & (Ns - 1)) : (j % Ns));
      const int d = (j - k) * R + k;
      const int pd = d + (d >> 4);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!LOW_OUT || 2 * r < R) {
          if constexpr (dst_smem) buf[pd + r * sout] = v[b][r];
          else dst(d + r * Ns, v[b][r]);
        }
      }
    }
  }
  if constexpr (dst_smem) __syncthreads();
}


template <int T, int N, int FLAGS, int Ns, int REM, class Src, class Dst>
__device__ __forceinline__ void fft_rec(float2* buf, const float2* __restrict__ tw, int tid,
                                        const Src& src, const Dst& dst) {
  if constexpr (REM > 1) {
    constexpr int R = next_radix(REM);
    constexpr bool first = Ns == 1, last = REM == R;
    stage<T, R, N, Ns, first && (FLAGS & kZeroUpper) != 0,
          last && (FLAGS & kLowOut) != 0 && R % 2 == 0>(buf, tw, tid, src, dst);
    fft_rec<T, N, FLAGS, Ns * R, REM / R>(buf, tw, tid, src, dst);
  }
}

// Forward complex FFT of buf[0..N) in place (padded layout), N = 2^a 3^b 5^c, N % 256 == 0.
// Radix 16 first (so Ns is a multiple of 16 afterwards), then 16/8/4/2, then 3, 5.  Called
// by the whole block after a barrier (threads tid = 0..T-1 of each group of T own one FFT;
// the barriers are block-wide, so every group runs the same plan); ends with a barrier.
template <int T, int N, int FLAGS, class Src = SmemIO, class Dst = SmemIO>
__device__ __forceinline__ void fft_smem(float2* buf, const float2* __restrict__ tw,
                                         int tid = threadIdx.x, const Src& src = Src{},
                                         const Dst& dst = Dst{}) {
  static_assert(N % 256 == 0 && T * 16 >= N, "FFT plan");
  fft_rec<T, N, FLAGS, 1, N>(buf, tw, tid, src, dst);
}

// ---------------------------------------------------------------- forward rows
// RB row pairs per block (RB groups of T threads, one FFT each): the block's 2 RB rows are
// consecutive in the column-major half spectra, so the transposed stores write 16 RB
// contiguous bytes per q (RB = 1: half a sector).
template <int P, int RB>
constexpr int rows_min_blocks() {
  // P = 2048 (k = 1 at C4): a 48-register cap (5 blocks of 2 x 128 threads per SM instead of
  // 4; 4 B spills) leaves room for the K-spectrum side stream; k = 1 wall 118.6 -> 115.8 us.
  // 6 blocks (40 registers, 8 B spills) measured 118.9 (tools/rows_ab.sh, profiles/r1_rows_ab.txt).
#ifdef TFDP_ROWS_MINB2048
  if (P == 2048) return TFDP_ROWS_MINB2048;
#else
  if (P == 2048 && RB == 2) return 5;
#endif
  // P = 4096 (k = 2): 3 blocks of 2 x 256 threads per SM (40 registers, 12-20 B spills)
  // instead of 2; k = 2 wall 371.4 -> 354.1 us.  P = 6144 at 4 blocks measured 872 -> 906
  // (36 B spills), kept at 3 (tools/rows_ab23.sh, profiles/r1_rows_ab23.txt).
#ifdef TFDP_ROWS_MINB4096
  if (P == 4096) return TFDP_ROWS_MINB4096;
#else
  if (P == 4096 && RB == 2) return 3;
#endif
#ifdef TFDP_ROWS_MINB6144
  if (P == 6144) return TFDP_ROWS_MINB6144;
#endif
  return kMinBlocksA<fft_threads_c(P)> / RB > 0 ? kMinBlocksA<fft_threads_c(P)> / RB : 1;
}

// First-stage global loads (rows_fwd) and last-stage global stores (rows_inv) fused into
// the FFT: C4 rows_fwd k = 1 23.0 -> 18.9 us, k = 3 156.7 -> 140.5; rows_inv k = 3 146.0 ->
// 142.3 (k = 1 unchanged).  Not at P = 4096, whose 40-register cap (3 blocks per SM) it
// overflows: rows_fwd 65.7 -> 67.9, rows_inv 70.0 -> 73.8 us.  rows_inv's transposed
// half-spectrum loads fused into its first stage too (each entry read twice, for q and its
// mirror P - q) measured slower: k = 1 20.9 -> 25.0 us, k = 3 142.4 -> 154.5.
template <int P>
__host__ __device__ constexpr bool rows_fuse_io() {
  return P != 4096;
}

template <int P, int RB>
__global__ void __launch_bounds__(fft_threads_c(P) * RB, (rows_min_blocks<P, RB>()))
rows_fwd_kernel(const GridGeom* __restrict__ geom, const float4* __restrict__ C, int cpitch,
                const float2* __restrict__ tw, float2* __restrict__ CA, int ca_pitch, int row0,
                const PeerRoute* __restrict__ rt) {
  constexpr int T = fft_threads_c(P);
  constexpr int NT = T * RB;
  constexpr int PL = padded_len(P);
  extern __shared__ float2 sm[];
  float2* tws = sm + RB * PL;
  load_tw(tws, tw, P);  // constant since the plan: safe before the wait
  pdl_wait();
  pdl_trigger();
  const int M = geom->M;
  // the three channel blocks of a row group are adjacent in launch order: they read the
  // same interleaved charge sectors close together in time (L2 hits)
  const int ch = blockIdx.x % 3;
  const int p0 = row0 / 2 + (blockIdx.x / 3) * RB;  // first row pair of the block
  if (2 * p0 >= M) return;
  const int g = threadIdx.x / T, lt = threadIdx.x - g * T;
  const int ra = 2 * (p0 + g), rb = ra + 1;
  const bool ha = ra < M, hb = rb < M;
  float2* a = sm + g * PL;
  // channel ch of the interleaved charges (stride 4 floats; the three channel blocks of a
  // row pair read the same sectors, from L2)
  const float* rowa = reinterpret_cast<const float*>(C + (int64_t)ra * cpitch) + ch;
  const float* rowb = rowa + 4 * (int64_t)cpitch;
  constexpr int half = P / 2;
  auto src = [&](int x) {  // [P/2, P) is zero and never read
    float va = 0.f, vb = 0.f;
    if (x < M) {
      if (ha) va = rowa[4 * x];
      if (hb) vb = rowb[4 * x];
    }
    return make_float2(va, vb);
  };
  if constexpr (rows_fuse_io<P>()) {
    // the first stage reads the two rows straight from global memory
    fft_smem<T, P, kZeroUpper>(a, tws, lt, src);
  } else {
#pragma unroll
    for (int x = lt; x < half; x += T) a[pad(x)] = src(x);
    __syncthreads();
    fft_smem<T, P, kZeroUpper>(a, tws, lt);
  }
  const int rows_here = min(2 * RB, M - 2 * p0);
  constexpr int H = half + 1;
  for (int f = threadIdx.x; f < (half + 1) * RB; f += NT) {
    const int q = f / RB, gg = f - q * RB;
    if (2 * gg >= rows_here) continue;
    const float2* ag = sm + gg * PL;
    const float2 z = ag[pad(q)];
    const float2 zc = conjf2(ag[pad(q == 0 ? 0 : P - q)]);
    const float2 xa = make_float2(0.5f * (z.x + zc.x), 0.5f * (z.y + zc.y));
    const float2 xb = mul_mi(make_float2(0.5f * (z.x - zc.x), 0.5f * (z.y - zc.y)));
    float2* o;
    if (rt) {  // slab mode, fused transpose: straight into the column owner's receive buffer
      const int r = 2 * p0 + 2 * gg, s = route_owner(rt->q0, rt->world, q);
      const int nq = rt->q0[s + 1] - rt->q0[s];
      o = rt->xb[s] + (((int64_t)ch * (rt->R / kCaTile) + r / kCaTile) * nq + (q - rt->q0[s])) * kCaTile +
          r % kCaTile;
    } else {
      o = CA + ca_col_base(ch, q, H, ca_pitch) + ca_row_off(2 * p0 + 2 * gg, H);
    }
    if (2 * gg + 1 < rows_here) *reinterpret_cast<float4*>(o) = make_float4(xa.x, xa.y, xb.x, xb.y);
    else *o = xa;
  }
}

// ---------------------------------------------------------------- inverse rows
// RB row pairs per block as in rows_fwd: the transposed loads read 16 RB contiguous bytes
// per q, each half-spectrum entry once (it feeds q and its Hermitian mirror P - q).
template <int P, int RB>
__global__ void __launch_bounds__(fft_threads_c(P) * RB, (rows_min_blocks<P, RB>()))
rows_inv_kernel(const GridGeom* __restrict__ geom, const float2* __restrict__ CA, int ca_pitch,
                const float2* __restrict__ tw, float* __restrict__ Phi, int cpitch,
                float4* __restrict__ C, int row0, const PeerRoute* __restrict__ rt) {
  constexpr int T = fft_threads_c(P);
  constexpr int NT = T * RB;
  constexpr int PL = padded_len(P);
  extern __shared__ float2 sm[];
  float2* tws = sm + RB * PL;
  load_tw(tws, tw, P);  // constant since the plan: safe before the wait
  pdl_wait();
  pdl_trigger();
  const int M = geom->M;
  const int ch = blockIdx.x % 3;  // channel blocks of a row group adjacent (as rows_fwd)
  const int p0 = row0 / 2 + (blockIdx.x / 3) * RB;
  if (2 * p0 >= M) return;
  const int rows_here = min(2 * RB, M - 2 * p0);
  constexpr int half = P / 2;
  constexpr int H = half + 1;
  // Z[q] = Xa[q] + i Xb[q] over the full circle (Hermitian extension), stored conjugated so
  // that the forward FFT computes the inverse.
#pragma unroll 4
  for (int f = threadIdx.x; f < (half + 1) * RB; f += NT) {
    const int q = f / RB, gg = f - q * RB;
    float2 xa = make_float2(0.f, 0.f), xb = make_float2(0.f, 0.f);
    const float2* p = CA + ca_col_base(ch, q, H, ca_pitch) + ca_row_off(2 * p0 + 2 * gg, H);
    if (2 * gg + 1 < rows_here) {
      const float4 v = *reinterpret_cast<const float4*>(p);
      xa = make_float2(v.x, v.y);
      xb = make_float2(v.z, v.w);
    } else if (2 * gg < rows_here) {
      xa = *p;
    }
    float2* ag = sm + gg * PL;
    ag[pad(q)] = conjf2(make_float2(xa.x - xb.y, xa.y + xb.x));  // conj(xa + i xb)
    if (q > 0 && q < half)  // mirror P - q: conj(conj(xa) + i conj(xb))
      ag[pad(P - q)] = make_float2(xa.x + xb.y, xa.y - xb.x);
  }
  // rows_fwd (a previous kernel) consumed these charge rows: leave them zero for the next
  // spread, the three channel blocks of the row group taking a third of the columns each
  // (measured cheaper than zeroing in rows_fwd after its last channel block or in cols)
  {
    const int x0 = ch * M / 3, x1 = (ch + 1) * M / 3;
    float4* c0 = C + (int64_t)(2 * p0) * cpitch;
    for (int r = 0; r < rows_here; ++r)
      for (int x = x0 + threadIdx.x; x < x1; x += NT) c0[(int64_t)r * cpitch + x] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  const int g = threadIdx.x / T, lt = threadIdx.x - g * T;
  float2* a = sm + g * PL;
  const int ra = 2 * (p0 + g), rb = ra + 1;
  const bool ha = ra < M, hb = rb < M;
  float* pa = Phi + ((int64_t)ch * cpitch + (ha ? ra : 0)) * cpitch;
  float* pb = pa + cpitch;
  auto dst = [&](int x, float2 z) {  // conj(result) = xa + i xb
    if (ha && x < M) {
      pa[x] = z.x;
      if (hb) pb[x] = -z.y;
      if (rt) {  // slab mode, fused potential exchange: the same rows into every other rank
        const int64_t off = pa - Phi;
        for (int j = 0; j < rt->world; ++j) {
          if (j == rt->rank) continue;
          float* qa = rt->phi[j] + off;
          qa[x] = z.x;
          if (hb) qa[cpitch + x] = -z.y;
        }
      }
    }
  };
  if constexpr (rows_fuse_io<P>()) {
    // the last stage writes the potential rows straight to global memory (x < M <= P/2)
    fft_smem<T, P, kLowOut>(a, tws, lt, SmemIO{}, dst);
  } else {
    fft_smem<T, P, kLowOut>(a, tws, lt);
    if (!ha) return;
    for (int x = lt; x < M; x += T) {
      const float2 z = a[pad(x)];
      pa[x] = z.x;
      if (hb) pb[x] = -z.y;
    }
    if (rt) {
      const int64_t off = pa - Phi;
      for (int j = 0; j < rt->world; ++j) {
        if (j == rt->rank) continue;
        float* qa = rt->phi[j] + off;
        for (int x = lt; x < M; x += T) {
          const float2 z = a[pad(x)];
          qa[x] = z.x;
          if (hb) qa[cpitch + x] = -z.y;
        }
      }
    }
  }
}

// ---------------------------------------------------------------- P > 8192 (AoS, one FFT)
// The SoA pair core needs 16 B of shared memory per point (> 227 KB beyond P = 12288) and
// ~80 registers at 1024 threads; above P = 8192 the kernel spectrum and the column pass run
// one complex FFT per block in the AoS core (8 B per point: 139 KB at P = 16384, ~60
// registers), reading and writing through shared memory.  These sizes serve layouts whose
// span needs N_int k > 4096 (e.g. 4M-node unit-density layouts at k = 3).
template <int P>
__global__ void __launch_bounds__(fft_threads_c(P), 1)
kspec_rows1_kernel(const GridGeom* __restrict__ geom, float neg_gamma, int gi,
                   const float2* __restrict__ tw, float* __restrict__ KA) {
  if (!geom->kspec) return;
  constexpr int T = fft_threads_c(P), half = P / 2, ka_pitch = half + 1;
  extern __shared__ float2 sm[];
  float2* a = sm;
  float2* tws = sm + padded_len(P);
  load_tw(tws, tw, P);
  const float h = geom->h, h2 = h * h, scale = 1.0f / ((float)P * (float)P);
  const int dy0 = 2 * blockIdx.x;  // rows dy0 (real part) and dy0 + 1 (imaginary part)
  for (int x = threadIdx.x; x < P; x += T) {
    const int dx = x <= half ? x : x - P;
    const float dx2 = (float)dx * (float)dx;
    float v[2] = {0.f, 0.f};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int dy = dy0 + c;
      if (dy <= half) v[c] = ksample(fmaf(h2, dx2 + (float)dy * (float)dy, 1.0f), neg_gamma, gi) * scale;
    }
    a[pad(x)] = make_float2(v[0], v[1]);
  }
  __syncthreads();
  fft_smem<T, P, 0>(a, tws);
  for (int q = threadIdx.x; q <= half; q += T) {  // real-even rows: real spectra
    const float2 z = a[pad(q)];
    KA[(int64_t)q * ka_pitch + dy0] = z.x;
    if (dy0 + 1 <= half) KA[(int64_t)q * ka_pitch + dy0 + 1] = z.y;
  }
}

template <int P>
__global__ void __launch_bounds__(fft_threads_c(P), 1)
kspec_cols1_kernel(const GridGeom* __restrict__ geom, const float* __restrict__ KA,
                   const float2* __restrict__ tw, float* __restrict__ KH) {
  if (!geom->kspec) return;
  constexpr int T = fft_threads_c(P), half = P / 2, ka_pitch = half + 1;
  extern __shared__ float2 sm[];
  float2* a = sm;
  float2* tws = sm + padded_len(P);
  load_tw(tws, tw, P);
  pdl_wait();
  const int q0 = 2 * blockIdx.x;  // columns q0 (real part) and q0 + 1 (imaginary part)
  for (int u = threadIdx.x; u < P; u += T) {
    const int dy = u <= half ? u : P - u;
    const float va = KA[(int64_t)q0 * ka_pitch + dy];
    const float vb = q0 + 1 <= half ? KA[(int64_t)(q0 + 1) * ka_pitch + dy] : 0.f;
    a[pad(u)] = make_float2(va, vb);
  }
  __syncthreads();
  fft_smem<T, P, 0>(a, tws);
  for (int u = threadIdx.x; u < P; u += T) {
    const float2 z = a[pad(u)];
    KH[(int64_t)q0 * P + u] = z.x;
    if (q0 + 1 <= half) KH[(int64_t)(q0 + 1) * P + u] = z.y;
  }
}

// one (channel, column) per block: FFT (inputs below P/2) -> x K^ -> inverse FFT (outputs
// below P/2), rows 0..M-1 kept; columns [q_base, q_base + Hl) held in CA (as cols_kernel)
template <int P>
__global__ void __launch_bounds__(fft_threads_c(P), 1)
cols1_kernel(const GridGeom* __restrict__ geom, float2* __restrict__ CA, int ca_pitch,
             const float* __restrict__ KH, const float2* __restrict__ tw, int q_base, int Hl,
             const PeerRoute* __restrict__ rt) {
  constexpr int T = fft_threads_c(P), half = P / 2;
  extern __shared__ float2 sm[];
  float2* a = sm;
  float2* tws = sm + padded_len(P);
  load_tw(tws, tw, P);
  pdl_wait();
  pdl_trigger();
  const int M = geom->M;
  const int ch = blockIdx.x % 3, q = q_base + blockIdx.x / 3;
  if (q > half || q >= q_base + Hl) return;
  float2* col = CA + ca_col_base(ch, q - q_base, Hl, ca_pitch);
  for (int u = threadIdx.x; u < half; u += T)  // [P/2, P) is zero and never read
    a[pad(u)] = u < M ? col[ca_row_off(u, Hl)] : make_float2(0.f, 0.f);
  __syncthreads();
  fft_smem<T, P, kZeroUpper>(a, tws);
  const float* kh = KH + (int64_t)q * P;
  for (int u = threadIdx.x; u < P; u += T) {  // x K^ (real), conjugated for the inverse
    const float2 z = a[pad(u)];
    const float k = __ldg(kh + u);
    a[pad(u)] = make_float2(z.x * k, -z.y * k);
  }
  __syncthreads();
  fft_smem<T, P, kLowOut>(a, tws);
  for (int u = threadIdx.x; u < M; u += T) {
    const float2 z = a[pad(u)];
    if (rt)  // slab mode: into the row owner's half spectra (as cols_kernel)
      rt->ca[route_owner(rt->row0, rt->world, u)][ca_col_base(ch, q, half + 1, rt->ca_pitch) +
                                                  ca_row_off(u, half + 1)] = make_float2(z.x, -z.y);
    else
      col[ca_row_off(u, Hl)] = make_float2(z.x, -z.y);
  }
}

}  // namespace aos

// ================================================================ register core (columns)
// One warp per (channel, column) item, the FFT of P = 32 A points held in registers as a
// four-step transform (lane b owns the residue class n = b mod 32):
//   1. lane b: DFT_A over a of x[b + 32 a] (in registers; a >= A/2 is zero padding)
//   2. twiddle W_P^(b k1)
//   3. transpose through shared memory (lane L gets k1 = L + 32 kk, all b)
//   4. lane L: DFT_32 over b -> X[k1 + A k2]
// then x conj(K^) and the inverse as the same steps in reverse order (DFT_32 in registers,
// twiddle, transpose, DFT_A with only its low half of outputs kept).  Two shared-memory
// round trips per FFT instead of one per radix-16 stage, no block barrier, and every lane
// holds 32-64 independent values (the radix-16 column pass is bound by shared-memory
// wavefronts and barrier stalls).  Sub-DFTs use compile-time twiddles.
namespace reg {

constexpr double kPiD = 3.14159265358979323846;
constexpr double cx_sin(double x) {  // |x| <= 3 pi / 2 after cx_red
  double t = x, s = x;
  for (int i = 1; i < 30; ++i) {
    t *= -x * x / ((2.0 * i) * (2.0 * i + 1));
    s += t;
  }
  return s;
}
constexpr double cx_red(double x) {
  while (x > kPiD) x -= 2 * kPiD;
  while (x < -kPiD) x += 2 * kPiD;
  return x;
}
// W_N^e = exp(-2 pi i e / N), e = 0..N-1, rounded from double
template <int N>
struct WTab {
  float c[N], s[N];
  constexpr WTab() : c(), s() {
    for (int e = 0; e < N; ++e) {
      const double a = -2.0 * kPiD * e / N;
      s[e] = (float)cx_sin(cx_red(a));
      c[e] = (float)cx_sin(cx_red(a + kPiD / 2));
    }
  }
};
template <int N>
__device__ constexpr WTab<N> kW{};

// In-register DFT of N = 16 A' values, natural order in and out: n = n1 + A' n2, k = k2 + 16 k1
// (DFT_16 over n2, twiddle W_N^(n1 k2), DFT_A' over n1).  ZU: inputs n >= N/2 are zero
// (never read).  Outputs the caller never uses are dead code to the compiler.
template <int N, bool ZU>
__device__ __forceinline__ void dftr(float2 (&v)[N]) {
  if constexpr (N == 16) {
    aos::dft16<ZU>(v);
  } else {
    static_assert(N == 32 || N == 64, "register DFT size");
    constexpr int A1 = N / 16;
    float2 t[A1][16];
#pragma unroll
    for (int n1 = 0; n1 < A1; ++n1) {
#pragma unroll
      for (int n2 = 0; n2 < 16; ++n2)
        t[n1][n2] = (ZU && n2 >= 8) ? make_float2(0.f, 0.f) : v[n1 + A1 * n2];
      aos::dft16<ZU>(t[n1]);
#pragma unroll
      for (int k2 = 1; k2 < 16; ++k2)
        if (n1 > 0) t[n1][k2] = cmul(t[n1][k2], make_float2(kW<N>.c[n1 * k2], kW<N>.s[n1 * k2]));
    }
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
      float2 u[A1];
#pragma unroll
      for (int n1 = 0; n1 < A1; ++n1) u[n1] = t[n1][k2];
      aos::dft<A1>(u);
#pragma unroll
      for (int k1 = 0; k1 < A1; ++k1) v[k2 + 16 * k1] = u[k1];
    }
  }
}

// slab mode: the lane's outputs G[lane + 32 nb] (staged in buf[nb * 32 + lane]) into the
// row owners' half spectra, conjugated (out of line: keeps the kernel's allocation)
__device__ __noinline__ void route_store_col(const PeerRoute* __restrict__ rt,
                                             const float2* buf, int lane, int nbs, int M,
                                             int ch, int qg, int H) {
  for (int nb = 0; nb < nbs; ++nb) {
    const int u = lane + 32 * nb;
    if (u >= M) break;
    const float2 z = buf[nb * 32 + lane];
    rt->ca[route_owner(rt->row0, rt->world, u)][ca_col_base(ch, qg, H, rt->ca_pitch) +
                                                ca_row_off(u, H)] = make_float2(z.x, -z.y);
  }
}

// v[8 i + j] *= W_P^(m (8 i + j)) from the two-level table (short product chains)
template <int P, int NV>
__device__ __forceinline__ void twiddle_row(const float2* __restrict__ tws, int m, float2 (&v)[NV]) {
  float2 p[8];
  p[0] = make_float2(1.f, 0.f);
#pragma unroll
  for (int j = 1; j < 8; ++j) p[j] = tw_at(tws, (m * j) % P);
#pragma unroll
  for (int i = 0; i < NV / 8; ++i) {
    const float2 qi = i == 0 ? make_float2(1.f, 0.f) : tw_at(tws, (8 * m * i) % P);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (i == 0 && j == 0) continue;
      v[8 * i + j] = cmul(v[8 * i + j], i == 0 ? p[j] : j == 0 ? qi : cmul(qi, p[j]));
    }
  }
}

constexpr int kWarps = 4;  // items (warps) per block
template <int P>
__host__ __device__ constexpr int xbuf_len() {
  return (P / 32) * 33;
}
template <int P>
__host__ __device__ constexpr size_t smem_bytes() {
  return (size_t)(kWarps * xbuf_len<P>() + tw_len(P)) * sizeof(float2);
}

template <int P, int MINB>
__global__ void __launch_bounds__(32 * kWarps, MINB)
cols_reg_kernel(const GridGeom* __restrict__ geom, float2* __restrict__ CA, int ca_pitch,
                const float* __restrict__ KH, const float2* __restrict__ tw, int q_base, int Hl,
                const PeerRoute* __restrict__ rt) {
  constexpr int A = P / 32, KPL = A / 32, SA = 33;
  constexpr int half = P / 2;
  extern __shared__ float2 sm[];
  float2* tws = sm + kWarps * xbuf_len<P>();
  load_tw(tws, tw, P);
  pdl_wait();
  pdl_trigger();
  __syncthreads();
  const int M = geom->M;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float2* xb = sm + wid * xbuf_len<P>();
  const int items = 3 * Hl;
  for (int it = blockIdx.x * kWarps + wid; it < items; it += gridDim.x * kWarps) {
    const int ql = it / 3, ch = it - 3 * ql, qg = q_base + ql;
    const float2* col = CA + ca_col_base(ch, ql, Hl, ca_pitch);
    // 1. DFT_A over a of x[lane + 32 a] (a < A/2; the rest is zero padding, M <= P/2)
    // rows u = lane + 32 a sit at ca_row_off(lane, Hl) + a * 32 Hl (kCaTile divides 32)
    const int64_t rstride = (int64_t)(32 / kCaTile) * kCaTile * Hl;
    float2 v[A];
    {
      const float2* pl = col + ca_row_off(lane, Hl);
#pragma unroll
      for (int a = 0; a < A / 2; ++a)
        v[a] = lane + 32 * a < M ? pl[a * rstride] : make_float2(0.f, 0.f);
    }
    dftr<A, true>(v);
    // 2. twiddle W_P^(lane k1);  3. transpose: row k1 of the buffer (stride 33) = (b -> Y[b][k1])
    twiddle_row<P, A>(tws, lane, v);
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) xb[k1 * SA + lane] = v[k1];
    __syncwarp();
    const float* kh = KH + (int64_t)qg * P;
    // lane L owns rows k1 = L + 32 kk: reads its row, writes the inverse's row back in place
    // (row k1 = (n_a -> S[k1][n_a])), so no lane touches another lane's row in between
#pragma unroll 1
    for (int kk = 0; kk < KPL; ++kk) {
      const int k1 = lane + 32 * kk;
      float2 w[32];
#pragma unroll
      for (int b = 0; b < 32; ++b) w[b] = xb[k1 * SA + b];
      // 4. DFT_32 over b -> X[k1 + A k2];  x K^ (real), conjugated for the inverse
      dftr<32, false>(w);
#pragma unroll
      for (int k2 = 0; k2 < 32; ++k2) {
        const float kv = __ldg(kh + k1 + A * k2);
        w[k2] = make_float2(w[k2].x * kv, -w[k2].y * kv);
      }
      // inverse: DFT_32 over k2 -> S[k1][n_a], twiddle W_P^(n_a k1)
      dftr<32, false>(w);
      twiddle_row<P, 32>(tws, k1, w);
#pragma unroll
      for (int na = 0; na < 32; ++na) xb[k1 * SA + na] = w[na];
    }
    __syncwarp();
    float2 y[A];
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) y[k1] = xb[k1 * SA + lane];
    __syncwarp();
    // DFT_A over k1 -> G[lane + 32 n_b]; rows u < M <= P/2 kept (n_b < A/2), conjugated
    dftr<A, false>(y);
    if (rt) {  // slab mode, fused transpose back: via the warp's buffer, out of line
#pragma unroll
      for (int nb = 0; nb < A / 2; ++nb) xb[nb * 32 + lane] = y[nb];
      __syncwarp();
      route_store_col(rt, xb, lane, A / 2, M, ch, qg, half + 1);
      __syncwarp();
    } else {
      // the store addresses recomputed (opaque stride): the load phase's do not stay live
      int64_t rs;
      asm volatile("mov.b64 %0, %1;" : "=l"(rs) : "l"(rstride));
      float2* pl = CA + ca_col_base(ch, ql, Hl, ca_pitch) + ca_row_off(lane, Hl);
#pragma unroll
      for (int nb = 0; nb < A / 2; ++nb)
        if (lane + 32 * nb < M) pl[nb * rs] = make_float2(y[nb].x, -y[nb].y);
    }
  }
}

// sizes with a register column kernel
template <int P>
constexpr bool has() {
  return P == 2048;
}

template <int P>
cudaError_t prepare() {
  if constexpr (has<P>()) {
    cudaError_t e = cudaFuncSetAttribute(cols_reg_kernel<P, 3>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem_bytes<P>());
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(cols_reg_kernel<P, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem_bytes<P>());
    return e;
  } else
    return cudaSuccess;
}

template <int P>
bool launch(const GridGeom* geom, float2* CA, int ca_pitch, const float* KH, const float2* tw,
            int q0, int q1, cudaStream_t s, const PeerRoute* route) {
  if constexpr (has<P>()) {
    // persistent: one wave of MINB blocks per SM, items strided over the warps.  MINB = 3
    // (168 registers, ~200 B of spills) or 2 (255 registers): TFDP_COLS_MINB
    static const int minb = [] {
      const char* e = std::getenv("TFDP_COLS_MINB");
      return e && e[0] == '2' ? 2 : 3;
    }();
    const int items = 3 * (q1 - q0);
    const int blocks = std::min((items + kWarps - 1) / kWarps, 148 * minb);
    if (minb == 2)
      cols_reg_kernel<P, 2><<<(unsigned)blocks, 32 * kWarps, smem_bytes<P>(), s>>>(
          geom, CA, ca_pitch, KH, tw, q0, q1 - q0, route);
    else
      cols_reg_kernel<P, 3><<<(unsigned)blocks, 32 * kWarps, smem_bytes<P>(), s>>>(
          geom, CA, ca_pitch, KH, tw, q0, q1 - q0, route);
    return true;
  } else {
    return false;
  }
}

}  // namespace reg

}  // namespace

// Supported FFT sizes: P = 256 q, q = 2^a 3^b 5^c with b <= 2, c <= 1, P <= 16384.  The SoA
// kernels (kernel spectrum, column pass) up to 8192; above, their AoS one-FFT variants.
#define TFDP_FFT_SIZES(X) \
  X(256) X(512) X(768) X(1024) X(1280) X(1536) X(2048) X(2304) X(2560) X(3072) X(3840) \
  X(4096) X(4608) X(5120) X(6144) X(7680) X(8192)
#define TFDP_FFT_SIZES_BIG(X) X(9216) X(10240) X(11520) X(12288) X(15360) X(16384)
#define TFDP_FFT_SIZES_ALL(X) TFDP_FFT_SIZES(X) TFDP_FFT_SIZES_BIG(X)

bool fft_size_supported(int P) {
#define TFDP_CASE(S) if (P == S) return true;
  TFDP_FFT_SIZES_ALL(TFDP_CASE)
#undef TFDP_CASE
  return false;
}

size_t fftconv_smem_bytes(int P) {
  return (size_t)padded_len(P) * sizeof(float4) + (size_t)tw_len(P) * sizeof(float2);
}

// Row pairs per block of the AoS row passes: 2 up to 512-thread blocks (P <= 4096; C4 k = 1:
// rows_fwd 27.0 -> 23.0 us, k = 2: 94.8 -> 77.3 us), else 1 (P = 6144 at RB = 2 holds one
// 768-thread block per SM: 217 -> 232 us).  TFDP_ROWS_RB = 1, 2, 4 overrides (A/B runs),
// limited to blocks of <= 1024 threads.
int rows_rb(int P) {
  static const int env = [] {
    const char* e = std::getenv("TFDP_ROWS_RB");
    return e ? std::atoi(e) : 0;
  }();
  int rb = env == 4 ? 4 : env == 1 ? 1 : env == 2 ? 2 : (fft_threads_c(P) * 2 <= 512 ? 2 : 1);
  while (rb > 1 && fft_threads_c(P) * rb > 1024) rb /= 2;
  return rb;
}

size_t rows_smem_bytes(int P, int groups) {
  return (size_t)(groups * padded_len(P) + tw_len(P)) * sizeof(float2);
}

cudaError_t fftconv_prepare(int P) {
  const int b = (int)fftconv_smem_bytes(P);
  const int rb = rows_rb(P);
  const int br = (int)rows_smem_bytes(P, rb);
  cudaError_t e = cudaErrorInvalidValue;
#define TFDP_PREP_ROWS(S, RB)                                                                  \
  if constexpr (fft_threads_c(S) * RB <= 1024) {                                             \
    if (e == cudaSuccess && rb == RB) {                                                        \
      e = cudaFuncSetAttribute(aos::rows_fwd_kernel<S, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, br); \
      if (e == cudaSuccess)                                                                    \
        e = cudaFuncSetAttribute(aos::rows_inv_kernel<S, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, br); \
    }                                                                                          \
  }
#define TFDP_PREP(S)                                                                          \
  case S:                                                                                     \
    e = cudaFuncSetAttribute(kspec_rows_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, b); \
    if (e == cudaSuccess)                                                                     \
      e = cudaFuncSetAttribute(kspec_cols_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, b); \
    if (e == cudaSuccess)                                                                     \
      e = cudaFuncSetAttribute(cols_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, b); \
    if (e == cudaSuccess) e = reg::prepare<S>();                                              \
    TFDP_PREP_ROWS(S, 1)                                                                      \
    TFDP_PREP_ROWS(S, 2)                                                                      \
    TFDP_PREP_ROWS(S, 4)                                                                      \
    break;
#define TFDP_PREP_BIG(S)                                                                      \
  case S:                                                                                     \
    e = cudaFuncSetAttribute(aos::kspec_rows1_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, br1); \
    if (e == cudaSuccess)                                                                     \
      e = cudaFuncSetAttribute(aos::kspec_cols1_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, br1); \
    if (e == cudaSuccess)                                                                     \
      e = cudaFuncSetAttribute(aos::cols1_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, br1); \
    TFDP_PREP_ROWS(S, 1)                                                                      \
    break;
  const int br1 = (int)rows_smem_bytes(P, 1);
  switch (P) {
    TFDP_FFT_SIZES(TFDP_PREP)
    TFDP_FFT_SIZES_BIG(TFDP_PREP_BIG)
    default: break;
  }
#undef TFDP_PREP_BIG
#undef TFDP_PREP
#undef TFDP_PREP_ROWS
  return e;
}

void launch_twiddles(float2* tw, int P, cudaStream_t s) {
  twiddle_kernel<<<(tw_len(P) + 255) / 256, 256, 0, s>>>(tw, P);
}

void launch_kspec(const GridGeom* geom, int P, ForceArgs fa, const float2* tw, float* KA,
                  float* KH, cudaStream_t s) {
  const size_t sm = fftconv_smem_bytes(P);
#define TFDP_KS(S)                                                                          \
  case S:                                                                                   \
    kspec_rows_kernel<S><<<(unsigned)((S / 2 + 4) / 4), fft_threads_c(S), sm, s>>>(         \
        geom, -fa.gamma, fa.gamma_int, tw, KA);                                             \
    launch_chained(kspec_cols_kernel<S>, (unsigned)((S / 2 + 4) / 4), fft_threads_c(S), sm, s, \
                   geom, KA, tw, KH);                                                       \
    break;
#define TFDP_KS_BIG(S)                                                                      \
  case S:                                                                                   \
    aos::kspec_rows1_kernel<S><<<(unsigned)((S / 2 + 2) / 2), fft_threads_c(S), smb1, s>>>( \
        geom, -fa.gamma, fa.gamma_int, tw, KA);                                             \
    launch_chained(aos::kspec_cols1_kernel<S>, (unsigned)((S / 2 + 2) / 2), fft_threads_c(S), \
                   smb1, s, geom, KA, tw, KH);                                              \
    break;
  const size_t smb1 = rows_smem_bytes(P, 1);
  switch (P) {
    TFDP_FFT_SIZES(TFDP_KS)
    TFDP_FFT_SIZES_BIG(TFDP_KS_BIG)
    default: break;
  }
#undef TFDP_KS_BIG
#undef TFDP_KS
}

// launches one AoS row-pass instantiation per (P, RB) with RB a compile-time constant
#define TFDP_ROWS_DISPATCH(S, KERN, ...)                                                       \
  {                                                                                           \
    const int rb = rows_rb(S);                                                                \
    const size_t smb = rows_smem_bytes(S, rb);                                                \
    const dim3 grid((unsigned)(3 * (((row1 - row0 + 1) / 2 + rb - 1) / rb)));                 \
    if (rb == 4) {                                                                            \
      if constexpr (fft_threads_c(S) * 4 <= 1024)                                             \
        launch_chained(KERN<S, 4>, grid, fft_threads_c(S) * 4, smb, s, __VA_ARGS__);          \
    } else if (rb == 2) {                                                                     \
      if constexpr (fft_threads_c(S) * 2 <= 1024)                                             \
        launch_chained(KERN<S, 2>, grid, fft_threads_c(S) * 2, smb, s, __VA_ARGS__);          \
    } else {                                                                                  \
      launch_chained(KERN<S, 1>, grid, fft_threads_c(S), smb, s, __VA_ARGS__);                \
    }                                                                                         \
  }

void launch_rows_fwd(const GridGeom* geom, const float4* C, int cpitch, int P, int row0,
                     int row1, const float2* tw, float2* CA, int ca_pitch, cudaStream_t s,
                     const PeerRoute* route) {
  if (row1 <= row0) return;
#define TFDP_RF(S)                                                                          \
  case S:                                                                                   \
    TFDP_ROWS_DISPATCH(S, aos::rows_fwd_kernel, geom, C, cpitch, tw, CA, ca_pitch, row0, route) \
    break;
  switch (P) { TFDP_FFT_SIZES_ALL(TFDP_RF) default: break; }
#undef TFDP_RF
}

// Column pass core: the radix-16 shared-memory kernel; TFDP_COLS=reg selects the register
// four-step kernel where it exists (P = 2048), measured slower and kept as an A/B variant
// (C4 k = 1: 39.4 / 37.7 us at 3 / 2 blocks per SM against 30.0 us).
static bool cols_reg() {
  static const bool on = [] {
    const char* e = std::getenv("TFDP_COLS");
    return e && std::string(e) == "reg";
  }();
  return on;
}

void launch_cols(const GridGeom* geom, float2* CA, int ca_pitch, const float* KH, int P,
                 const float2* tw, int q0, int q1, cudaStream_t s, const PeerRoute* route) {
  if (q1 <= q0) return;
  const size_t sm = fftconv_smem_bytes(P);
#define TFDP_CO(S)                                                                          \
  case S:                                                                                   \
    if (cols_reg() && reg::launch<S>(geom, CA, ca_pitch, KH, tw, q0, q1, s, route)) break;  \
    cols_kernel<S><<<(unsigned)(3 * ((q1 - q0 + 1) / 2)), fft_threads_c(S), sm, s>>>(      \
        geom, CA, ca_pitch, KH, tw, q0, q1 - q0, route);                                    \
    break;
#define TFDP_CO_BIG(S)                                                                      \
  case S:                                                                                   \
    launch_chained(aos::cols1_kernel<S>, (unsigned)(3 * (q1 - q0)), fft_threads_c(S), smb1, s, \
                   geom, CA, ca_pitch, KH, tw, q0, q1 - q0, route);                         \
    break;
  const size_t smb1 = rows_smem_bytes(P, 1);
  switch (P) {
    TFDP_FFT_SIZES(TFDP_CO)
    TFDP_FFT_SIZES_BIG(TFDP_CO_BIG)
    default: break;
  }
#undef TFDP_CO_BIG
#undef TFDP_CO
}

void launch_rows_inv(const GridGeom* geom, const float2* CA, int ca_pitch, int P, int row0,
                     int row1, const float2* tw, float* Phi, int cpitch, float4* C,
                     cudaStream_t s, const PeerRoute* route) {
  if (row1 <= row0) return;
#define TFDP_RI(S)                                                                          \
  case S:                                                                                   \
    TFDP_ROWS_DISPATCH(S, aos::rows_inv_kernel, geom, CA, ca_pitch, tw, Phi, cpitch, C, row0, \
                       route)                                                               \
    break;
  switch (P) { TFDP_FFT_SIZES_ALL(TFDP_RI) default: break; }
#undef TFDP_RI
}

}  // namespace tfdp
