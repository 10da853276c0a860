// Micro-benchmark of inner-loop variants of the exact all-pairs t-force (gamma = 2).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/mbench_exact.cu
// Each variant: TPT targets per thread in registers, sources broadcast from shared memory.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int TPB = 256, TILE = 1024;
using u64 = unsigned long long;

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(unsigned long long v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b,
                                                   unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long sub2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// V0: scalar (production kernel)
template <int TPT>
__global__ void __launch_bounds__(TPB) v0(const float2* __restrict__ xy, int n, float2* out) {
  __shared__ float2 tile[TILE];
  float tx[TPT], ty[TPT], ax[TPT], ay[TPT];
  for (int r = 0; r < TPT; ++r) {
    float2 p = xy[(blockIdx.x * TPB * TPT + threadIdx.x + r * TPB) % n];
    tx[r] = p.x; ty[r] = p.y; ax[r] = ay[r] = 0.f;
  }
  for (int base = 0; base < n; base += TILE) {
    __syncthreads();
    for (int j = threadIdx.x; j < TILE; j += TPB) tile[j] = xy[base + j];
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < TILE; ++j) {
      const float2 q = tile[j];
#pragma unroll
      for (int r = 0; r < TPT; ++r) {
        const float dx = tx[r] - q.x, dy = ty[r] - q.y;
        const float s = fmaf(dx, dx, fmaf(dy, dy, 1.f));
        const float w = rcp_approx(s);
        const float w2 = w * w;
        ax[r] = fmaf(w2, dx, ax[r]);
        ay[r] = fmaf(w2, dy, ay[r]);
      }
    }
  }
  for (int r = 0; r < TPT; ++r) out[blockIdx.x * TPB * TPT + threadIdx.x + r * TPB] = make_float2(ax[r], ay[r]);
}

// V1: packed f32x2 over the (x, y) components: d = t - q (FADD2 as sub2), acc += w2 * d (FFMA2)
template <int TPT>
__global__ void __launch_bounds__(TPB) v1(const float2* __restrict__ xy, int n, float2* out) {
  __shared__ float2 tile[TILE];
  unsigned long long t[TPT], acc[TPT];
  for (int r = 0; r < TPT; ++r) {
    float2 p = xy[(blockIdx.x * TPB * TPT + threadIdx.x + r * TPB) % n];
    t[r] = pk(p.x, p.y); acc[r] = pk(0.f, 0.f);
  }
  for (int base = 0; base < n; base += TILE) {
    __syncthreads();
    for (int j = threadIdx.x; j < TILE; j += TPB) tile[j] = xy[base + j];
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < TILE; ++j) {
      const float2 qq = tile[j];
      const unsigned long long q = pk(qq.x, qq.y);
#pragma unroll
      for (int r = 0; r < TPT; ++r) {
        const unsigned long long d = sub2(t[r], q);
        float dx, dy;
        upk(d, dx, dy);
        const float s = fmaf(dx, dx, fmaf(dy, dy, 1.f));
        const float w = rcp_approx(s);
        const float w2 = w * w;
        acc[r] = fma2(pk(w2, w2), d, acc[r]);
      }
    }
  }
  for (int r = 0; r < TPT; ++r) {
    float a, b;
    upk(acc[r], a, b);
    out[blockIdx.x * TPB * TPT + threadIdx.x + r * TPB] = make_float2(a, b);
  }
}

// V2: packed over two sources j, j+1 for one target: (dx1,dx2), (dy1,dy2), (s1,s2) as f32x2;
// reciprocals: fraction of pairs share one MUFU (1/(s1 s2)), the rest 2 MUFU.
template <int TPT, bool PAIRED>
__global__ void __launch_bounds__(TPB) v2(const float2* __restrict__ xy, int n, float2* out) {
  __shared__ float xs[TILE], ys[TILE];
  unsigned long long tx[TPT], ty[TPT], ax[TPT], ay[TPT];
  for (int r = 0; r < TPT; ++r) {
    float2 p = xy[(blockIdx.x * TPB * TPT + threadIdx.x + r * TPB) % n];
    tx[r] = pk(p.x, p.x); ty[r] = pk(p.y, p.y); ax[r] = ay[r] = pk(0.f, 0.f);
  }
  const unsigned long long one = pk(1.f, 1.f);
  for (int base = 0; base < n; base += TILE) {
    __syncthreads();
    for (int j = threadIdx.x; j < TILE; j += TPB) {
      const float2 p = xy[base + j];
      xs[j] = p.x; ys[j] = p.y;
    }
    __syncthreads();
#pragma unroll 2
    for (int j = 0; j < TILE; j += 2) {
      const unsigned long long qx = *reinterpret_cast<const unsigned long long*>(xs + j);
      const unsigned long long qy = *reinterpret_cast<const unsigned long long*>(ys + j);
#pragma unroll
      for (int r = 0; r < TPT; ++r) {
        const unsigned long long dx = sub2(tx[r], qx), dy = sub2(ty[r], qy);
        const unsigned long long s = fma2(dy, dy, fma2(dx, dx, one));
        float s1, s2;
        upk(s, s1, s2);
        float w1, w2;
        if (PAIRED) {
          const float rr = rcp_approx(s1 * s2);
          w1 = rr * s2;
          w2 = rr * s1;
        } else {
          w1 = rcp_approx(s1);
          w2 = rcp_approx(s2);
        }
        const unsigned long long w = pk(w1, w2);
        const unsigned long long q2 = mul2(w, w);
        ax[r] = fma2(q2, dx, ax[r]);
        ay[r] = fma2(q2, dy, ay[r]);
      }
    }
  }
  for (int r = 0; r < TPT; ++r) {
    float a1, a2, b1, b2;
    upk(ax[r], a1, a2);
    upk(ay[r], b1, b2);
    out[blockIdx.x * TPB * TPT + threadIdx.x + r * TPB] = make_float2(a1 + a2, b1 + b2);
  }
}

// V3: as V2 (unpaired), but one source pair in every NE uses an FMA-pipe reciprocal:
// -y0 from an integer magic (one 64-bit subtract on the packed bits, no borrow since
// bits(s) < magic for s >= 1), then a cubic and a quadratic Newton step on the negated
// iterate (5 FFMA2, rel. error ~4e-6), moving work from the MUFU pipe to the FMA pipe.
__device__ __forceinline__ u64 rcp_neg_newton2(u64 s) {
  const u64 one = pk(1.f, 1.f);
  u64 z = 0xFEF311C3FEF311C3ull - s;  // -y0 per lane (sign bit set by the magic)
  u64 e = fma2(s, z, one);            // 1 - s y0
  u64 t = fma2(e, e, e);              // e + e^2
  z = fma2(z, t, z);                  // -(y0 (1 + e + e^2))
  e = fma2(s, z, one);
  z = fma2(z, e, z);                  // -y2
  return z;
}
template <int TPT, int NE>
__global__ void __launch_bounds__(TPB) v3(const float2* __restrict__ xy, int n, float2* out) {
  __shared__ float xs[TILE], ys[TILE];
  u64 tx[TPT], ty[TPT], ax[TPT], ay[TPT];
  for (int r = 0; r < TPT; ++r) {
    float2 p = xy[(blockIdx.x * TPB * TPT + threadIdx.x + r * TPB) % n];
    tx[r] = pk(p.x, p.x); ty[r] = pk(p.y, p.y); ax[r] = ay[r] = pk(0.f, 0.f);
  }
  const u64 one = pk(1.f, 1.f);
  for (int base = 0; base < n; base += TILE) {
    __syncthreads();
    for (int j = threadIdx.x; j < TILE; j += TPB) {
      const float2 p = xy[base + j];
      xs[j] = p.x; ys[j] = p.y;
    }
    __syncthreads();
    for (int j0 = 0; j0 + 2 * NE <= TILE; j0 += 2 * NE) {  // (remainder of the tile skipped)
#pragma unroll
      for (int jj = 0; jj < NE; ++jj) {
        const int j = j0 + 2 * jj;
        const u64 qx = *reinterpret_cast<const u64*>(xs + j);
        const u64 qy = *reinterpret_cast<const u64*>(ys + j);
#pragma unroll
        for (int r = 0; r < TPT; ++r) {
          const u64 dx = sub2(tx[r], qx), dy = sub2(ty[r], qy);
          const u64 s = fma2(dy, dy, fma2(dx, dx, one));
          u64 w;
          if (jj == NE - 1) {
            w = rcp_neg_newton2(s);
          } else {
            float s1, s2;
            upk(s, s1, s2);
            w = pk(rcp_approx(s1), rcp_approx(s2));
          }
          const u64 q2 = mul2(w, w);
          ax[r] = fma2(q2, dx, ax[r]);
          ay[r] = fma2(q2, dy, ay[r]);
        }
      }
    }
  }
  for (int r = 0; r < TPT; ++r) {
    float a1, a2, b1, b2;
    upk(ax[r], a1, a2);
    upk(ay[r], b1, b2);
    out[blockIdx.x * TPB * TPT + threadIdx.x + r * TPB] = make_float2(a1 + a2, b1 + b2);
  }
}

__global__ void check_newton(float* out) {
  float worst = 0.f, at = 0.f;
  for (float s = 1.0f; s < 1e7f; s *= 1.0001f) {
    float a, b;
    upk(rcp_neg_newton2(pk(s, s * 1.37f)), a, b);
    const float ea = fabsf(-a * s - 1.0f), eb = fabsf(-b * (s * 1.37f) - 1.0f);
    if (ea > worst) { worst = ea; at = s; }
    if (eb > worst) { worst = eb; at = s * 1.37f; }
  }
  out[0] = worst;
  out[1] = at;
}

template <typename K>
double run(K kern, int grid, const float2* xy, int n, float2* out, const char* name, int tpt) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<grid, TPB>>>(xy, n, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) kern<<<grid, TPB>>>(xy, n, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double pairs = 5.0 * grid * TPB * tpt * (double)n;
  const double rate = pairs / (ms / 1e3);
  printf("%-22s %8.3f ms  %.3e pairs/s  %s\n", name, ms / 5, rate, cudaGetErrorString(cudaGetLastError()));
  return rate;
}

int main() {
  const int n = 1 << 17;
  float2* xy;
  float2* out;
  cudaMalloc(&xy, n * sizeof(float2));
  cudaMalloc(&out, (1 << 22) * sizeof(float2));
  float2* h = (float2*)malloc(n * sizeof(float2));
  srand(1);
  for (int i = 0; i < n; ++i) h[i] = make_float2(rand() / (float)RAND_MAX * 300.f, rand() / (float)RAND_MAX * 300.f);
  cudaMemcpy(xy, h, n * sizeof(float2), cudaMemcpyHostToDevice);
  const int grid4 = 148 * 4 * 4;  // targets: grid * 256 * 4
  run(v0<4>, grid4, xy, n, out, "v0 scalar tpt4", 4);
  run(v0<8>, grid4 / 2, xy, n, out, "v0 scalar tpt8", 8);
  run(v1<4>, grid4, xy, n, out, "v1 f32x2(xy) tpt4", 4);
  run(v2<4, false>, grid4, xy, n, out, "v2 f32x2(jj) tpt4", 4);
  run(v2<4, true>, grid4, xy, n, out, "v2 paired tpt4", 4);
  run(v2<8, false>, grid4 / 2, xy, n, out, "v2 f32x2(jj) tpt8", 8);
  run(v2<8, true>, grid4 / 2, xy, n, out, "v2 paired tpt8", 8);
  run(v3<4, 16>, grid4, xy, n, out, "v3 newton 1/16 tpt4", 4);
  run(v3<4, 12>, grid4, xy, n, out, "v3 newton 1/12 tpt4", 4);
  run(v3<4, 8>, grid4, xy, n, out, "v3 newton 1/8 tpt4", 4);
  run(v3<4, 6>, grid4, xy, n, out, "v3 newton 1/6 tpt4", 4);
  run(v3<4, 4>, grid4, xy, n, out, "v3 newton 1/4 tpt4", 4);
  run(v3<4, 32>, grid4, xy, n, out, "v3 newton 1/32 tpt4", 4);
  {  // accuracy of the Newton reciprocal over s in [1, 1e7]
    float* d;
    cudaMalloc(&d, 2 * sizeof(float));
    check_newton<<<1, 1>>>(d);
    float h2[2];
    cudaMemcpy(h2, d, sizeof(h2), cudaMemcpyDeviceToHost);
    printf("newton rcp max rel err over s in [1, 1e7]: %.3e (at s = %.6g)\n", h2[0], h2[1]);
  }
  return 0;
}
