// Multi-GPU slab mode of the ibFFT grid convolution — sm_100a.
//
// The zero-padded 2-D convolution is the only super-linear step of an
// iteration; across p GPUs it is split like a slab-decomposed 2-D FFT: rank r runs the row
// passes on its grid-row slab and the column pass on its chunk of half-spectrum columns,
// with two all-to-all transposes in between (api.cpp: NCCL send/recv between processes, or
// device copies between the virtual ranks of one process).  These kernels move a rank's
// slab rows of the row-tiled half spectra CA ([ch][ca_pitch / 8][H][8] float2, see
// kernels_fftconv.cu) into / out of the per-destination segments of the exchange buffer
// xa = [s][ch][rt - rt0][q - q0(s)][8]: the column chunk of rank s is one contiguous block
// per channel, so every transfer is a single contiguous message.
#include <algorithm>

#include "tfdp_internal.h"

namespace tfdp {

void slab_plan(int world, int rank, int rows, int P, SlabPlan* pl) {
  pl->world = world;
  pl->rank = rank;
  pl->R = (rows + 23) / 24 * 24;
  pl->H = P / 2 + 1;
  const int64_t units = pl->R / 24, pairs = (pl->H + 1) / 2;
  for (int r = 0; r <= world; ++r) {
    pl->row0[r] = (int)(24 * (r * units / world));
    pl->q0[r] = (int)std::min<int64_t>(2 * (r * pairs / world), pl->H);
  }
}

namespace {

// owner of half-spectrum column q
__device__ __forceinline__ int col_owner(const SlabPlan& pl, int q) {
  int s = (int)((int64_t)q * pl.world / pl.H);
  s = min(max(s, 0), pl.world - 1);
  while (s > 0 && q < pl.q0[s]) --s;
  while (s < pl.world - 1 && q >= pl.q0[s + 1]) ++s;
  return s;
}

// element f of this rank's slab region of CA: (ch, rt, q, e) -> (CA offset, xa offset)
template <bool PACK>
__global__ void __launch_bounds__(256)
slab_copy_kernel(const float2* __restrict__ src, float2* __restrict__ dst, int ca_pitch,
                 SlabPlan pl) {
  const int me = pl.rank;
  const int rt0 = pl.row0[me] / 8, nrt = (pl.row0[me + 1] - pl.row0[me]) / 8;
  const int H = pl.H;
  const int64_t total = 3LL * nrt * H * 8;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(f & 7);
    const int64_t t = f >> 3;
    const int q = (int)(t % H);
    const int64_t u = t / H;
    const int rt = (int)(u % nrt), ch = (int)(u / nrt);
    const int64_t ca = (((int64_t)ch * (ca_pitch / 8) + rt0 + rt) * H + q) * 8 + e;
    const int s = col_owner(pl, q);
    const int nq = pl.q0[s + 1] - pl.q0[s];
    const int64_t xa = 3LL * nrt * 8 * pl.q0[s] + (((int64_t)ch * nrt + rt) * nq + (q - pl.q0[s])) * 8 + e;
    if (PACK) dst[xa] = src[ca];
    else dst[ca] = src[xa];
  }
}

unsigned copy_blocks(const SlabPlan& pl) {
  const int64_t nrt = (pl.row0[pl.rank + 1] - pl.row0[pl.rank]) / 8;
  const int64_t total = 3 * nrt * pl.H * 8;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16));
}

}  // namespace

void launch_pack_slab(const float2* CA, int ca_pitch, const SlabPlan& pl, float2* xa,
                      cudaStream_t s) {
  if (pl.row0[pl.rank + 1] <= pl.row0[pl.rank]) return;
  slab_copy_kernel<true><<<copy_blocks(pl), 256, 0, s>>>(CA, xa, ca_pitch, pl);
}

void launch_unpack_slab(const float2* xa, const SlabPlan& pl, float2* CA, int ca_pitch,
                        cudaStream_t s) {
  if (pl.row0[pl.rank + 1] <= pl.row0[pl.rank]) return;
  slab_copy_kernel<false><<<copy_blocks(pl), 256, 0, s>>>(xa, CA, ca_pitch, pl);
}

}  // namespace tfdp
