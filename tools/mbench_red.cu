// Micro-benchmark: L2 RED throughput for scalar / float2 / float4 fp32 adds (sm_100a).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_red tools/mbench_red.cu
#include <cstdio>
#include <cuda_runtime.h>

// each thread: R ops to pseudo-random 16B-aligned slots within a 'span' floats window
template <int V>
__global__ void red_kernel(float* g, int span_quads, int R, int local) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned h = t * 2654435761u;
  for (int r = 0; r < R; ++r) {
    h = h * 1664525u + 1013904223u;
    unsigned q = local ? ((t + r * 32) % span_quads) : (h % span_quads);
    float* p = g + 4 * (size_t)q;
    if constexpr (V == 1) atomicAdd(p, 1.0f);
    else if constexpr (V == 2) atomicAdd(reinterpret_cast<float2*>(p), make_float2(1.f, 1.f));
    else if constexpr (V == 4) atomicAdd(reinterpret_cast<float4*>(p), make_float4(1.f, 1.f, 1.f, 1.f));
    else {  // 3 scalar REDs into three planes (the direct spread pattern)
      atomicAdd(p, 1.0f);
      atomicAdd(p + 1, 1.0f);
      atomicAdd(p + 2, 1.0f);
    }
  }
}

int main() {
  const int span_quads = 1 << 22;  // 64 MB of floats window
  float* g;
  cudaMalloc(&g, (size_t)span_quads * 16);
  cudaMemset(g, 0, (size_t)span_quads * 16);
  const int blocks = 148 * 8, threads = 256, R = 64;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int local = 0; local < 2; ++local) {
    for (int v : {1, 2, 4, 3}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (v == 1) red_kernel<1><<<blocks, threads>>>(g, span_quads, R, local);
        if (v == 2) red_kernel<2><<<blocks, threads>>>(g, span_quads, R, local);
        if (v == 4) red_kernel<4><<<blocks, threads>>>(g, span_quads, R, local);
        if (v == 3) red_kernel<3><<<blocks, threads>>>(g, span_quads, R, local);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = (double)blocks * threads * R * (v == 3 ? 3 : 1);
        if (rep) printf("%s V=%d  %.3f ms  %.1f G RED instr/s  %.1f G floats/s\n",
                        local ? "coalesced" : "random   ", v, ms, ops / ms / 1e6,
                        ops * (v == 3 ? 1 : v) / ms / 1e6);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
