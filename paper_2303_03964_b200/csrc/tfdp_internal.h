// Internal declarations shared by the host runtime (api.cpp) and the sm_100a kernels.
// See DESIGN.md §Kernels for the roofline of each kernel.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tfdp {

constexpr int kExactThreads = 256;  // exact kernel block
constexpr int kExactTPT = 4;        // targets per thread (register blocking)
constexpr int kExactTargetsPerBlock = kExactThreads * kExactTPT;
constexpr int kExactTile = 1024;    // sources per smem tile (fp32 partial sum length)
constexpr int kNodeThreads = 256;   // per-node kernels

// Geometry of one ibFFT evaluation, computed on the device from the box (no host sync).
struct GridGeom {
  float lo_x, lo_y;  // lower-left corner of the bounding square (R6)
  float L;           // side (R6)
  float w;           // interval width L / N_int (fp32, R19)
  float h;           // grid spacing w / k
  float cx, cy;      // centre lo + L/2 (R11)
  int n_int;         // intervals per axis (R5)
  int k;             // nodes per interval (1..3)
  int M;             // grid points per axis = n_int * k
  int P;             // FFT size (>= 2M - 1, R9)
  int capped;        // 1 if n_int was clamped to the allocated grid (warning)
  int pitch;         // row pitch (floats) of the compact charge / potential planes
  int kspec;         // 1: the kernel spectrum must be (re)computed this evaluation
};

// Key of the kernel spectrum currently held in KH: K^ depends only on (P, h, gamma) (the
// kernel is sampled over the whole periodic P x P range, kernels_fftconv.cu), so setup
// compares the new geometry against it and the K-spectrum kernels skip when it matches.
struct KspecKey {
  int P;
  unsigned h_bits, gamma_bits;
  int valid;
};

// Box as order-preserving uint keys so atomicMin/atomicMax give the exact fp32 min/max.
struct BoxKeys {
  unsigned int minx, miny, maxx, maxy;
};

// High-degree rows (degree skew, power-law graphs): a row with more than kHeavyDeg edges is
// not walked by one thread; its attraction sum comes in chunks of kHeavyChunk edges, one
// warp per chunk (kernels_heavy.cu), summed by the row's thread in chunk order
// (deterministic, R15).  hv_first[i] = first chunk of row i (exclusive scan over rows).
constexpr int kHeavyDeg = 128;
constexpr int kHeavyChunk = 256;

// Kernel-side parameters of the force law.
struct ForceArgs {
  float alpha, beta, gamma, rho;
  int gamma_int;  // 1..8 if gamma is that integer, else 0 (general path)
  const long long* hv_first;  // [n + 1] or nullptr (no heavy rows)
  const float2* hv_part;      // chunk sums of the heavy rows (sum (1 + beta/s)(x_i - x_j))
};

// Local (fisheye) refinement mask (SPEC RefinementMask): label[i] = 1 for the focal
// region F u N(F) (internal slot order), s1 = exact repulsion sum over the region's sources
// for the shard's targets (focus_s1 kernel, unscaled by rho).  Repulsion weight w(i,j) = lf
// if both in the region, ls if both outside, else 1; attraction weight la if both in the
// region.  R_i = rho [w0(i) (S_all - S1_i) + w1(i) S1_i] (R23).  label == nullptr:
// no mask (the unmasked kernels' arithmetic, bit for bit).
struct FocusArgs {
  const unsigned char* label;
  const float2* s1;
  float la, lf, ls;
};

// ---- programmatic dependent launch (PDL) for the per-iteration kernel chain -----------
// Chain kernels are launched with programmatic stream serialization: a kernel may be
// scheduled while its predecessor's last wave is still running, does its independent
// prologue (twiddle table -> smem), then blocks in griddepcontrol.wait (pdl_wait in
// device_math.cuh) until the predecessor grid has completed and its writes are visible.
// Every chain kernel calls pdl_wait() before touching any buffer another kernel writes, so
// the ordering is the plain stream order.  TFDP_PDL=0 disables the attribute (A/B runs).
bool pdl_enabled();
// Per-iteration switch (host thread): the ibFFT chain uses PDL only up to P = kPdlMaxFft.
// Round 1 (then-current kernels): P = 4096 / 6144 slower with PDL (C4 k = 2: 405 vs 385 us,
// k = 3: 1091 vs 973 us per iteration), P = 2048 faster (122.6 vs 124.5 us).
// Round 2 re-measured (bench per-k): P = 4096 324.4 -> 314.2 us with PDL, P = 6144 751.9 ->
// 773.0 us: the threshold is 4096.
constexpr int kPdlMaxFft = 4096;
void set_pdl_active(bool on);
template <typename... KArgs, typename... Args>
inline void launch_chained(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                           cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- launchers (kernels.cu / kernels_fft.cu); all enqueue on `s` ---------------------
// exact path
void launch_exact_partial(const float2* xy, int64_t n, int64_t lo, int64_t n_local,
                          int64_t chunk, int n_chunks, ForceArgs fa, double2* part,
                          cudaStream_t s);
// finish: sum partials (fixed chunk order) + CSR attraction + (update | write forces)
void launch_exact_finish(const float2* xy, float2* xy_next, int64_t lo, int64_t n_local,
                         int n_chunks, const double2* part, const int64_t* row_ptr,
                         const int32_t* col, ForceArgs fa, FocusArgs fo, float eta, int iter,
                         int update, float2* rep_out, float2* att_out,
                         unsigned long long* diverge, cudaStream_t s,
                         const struct PeerRoute* route = nullptr, int next_buf = 0);

// ibFFT path
// Box: producers merge one block-reduced BoxKeys per block into kBoxSlots slots (atomic
// min/max); the consumer (one block) reduces the slots and resets them to the identity.
constexpr int kBoxSlots = 64;
int bbox_blocks(int64_t n);
void launch_reset_slots(BoxKeys* slots, cudaStream_t s);
int launch_bbox(const float2* xy, int64_t n, BoxKeys* slots, cudaStream_t s);  // -> n_part
void launch_box_reduce(BoxKeys* slots, int n_part, BoxKeys* keys, cudaStream_t s,
                       bool reset = true);
// rule: 0 = unit-width intervals when ceil L >= n_int_min (R5'), 1 = w = L / N_int (R5)
void launch_setup(BoxKeys* slots, int n_part, BoxKeys* keys, GridGeom* geom, int k,
                  int n_int_min, int n_int_fixed, int n_int_cap, int P, int pitch,
                  int* capped_flag, int rule, float gamma, KspecKey* kkey, cudaStream_t s);
// charges: float4 {C_1, C_x~, C_y~, 0} per grid node, row pitch = GridGeom::pitch float4s
// per-node (warp-aggregated for k >= 2) v4 REDs; TFDP_SPREAD=tile: the shared-memory
// privatised tile kernel (measured slower, kernels_fft.cu)
// [by_lo, by_hi): only nodes whose interval row lies in it are spread (slab mode)
void launch_spread(const float2* xy, int64_t lo, int64_t cnt, const GridGeom* geom, int k,
                   float4* grid, cudaStream_t s, int by_lo = 0, int by_hi = 0x7fffffff);

// multi-GPU slab mode (kernels_dist.cu): rank r owns grid rows
// [row0[r], row0[r+1]) of the row passes (multiples of 24: whole CA row tiles of 8 and whole
// intervals at every k) and half-spectrum columns [q0[r], q0[r+1]) of the column pass (even
// starts: the column pass works on column pairs).
constexpr int kMaxWorld = 64;
struct SlabPlan {
  int world, rank;
  int R;  // rows of the slab domain (cap_k k rounded up to 24)
  int H;  // half-spectrum columns P/2 + 1
  int row0[kMaxWorld + 1];
  int q0[kMaxWorld + 1];
};
void slab_plan(int world, int rank, int rows, int P, SlabPlan* pl);

// Peer routing of the slab mode's fused exchanges: the producing kernels store
// straight into the buffers of the ranks that consume the data — rows_fwd into the column
// owners' receive buffers xb, cols into the row owners' half spectra CA, rows_inv its
// potential rows and gather_update the new positions into every rank's copy.  Between
// processes the pointers are CUDA IPC mappings (NVLink P2P stores); between the virtual ranks
// of one device they are the other contexts' buffers.  One route per k (the plan's slabs);
// kept in device memory, nullptr on one GPU.
struct PeerRoute {
  int world, rank;
  int R;         // rows of the xb layout ([ch][R / 8][nq][8])
  int ca_pitch;  // rows of the full CA layout ([ch][ca_pitch / 8][P/2 + 1][8]), every rank
  int row0[kMaxWorld + 1];
  int q0[kMaxWorld + 1];
  float2* xb[kMaxWorld];
  float2* ca[kMaxWorld];
  float* phi[kMaxWorld];
  float2* xy[2][kMaxWorld];
};
__host__ __device__ inline int route_owner(const int* b, int world, int v) {
  int s = 0;
  while (s < world - 1 && v >= b[s + 1]) ++s;
  return s;
}
// exchange-1 send / exchange-2 receive layout: [s][ch][rt - rt0(me)][q - q0(s)][8] float2,
// i.e. segment (s, ch) starts at 3 * nrt * 8 * q0[s] + ch * nrt * nq(s) * 8
// pack: this rank's slab rows of CA ([ch][ca_pitch / 8][H][8]) -> xa;  unpack: xa -> CA
void launch_pack_slab(const float2* CA, int ca_pitch, const SlabPlan& pl, float2* xa,
                      cudaStream_t s);
void launch_unpack_slab(const float2* xa, const SlabPlan& pl, float2* CA, int ca_pitch,
                        cudaStream_t s);

// hand-written FFT convolution (kernels_fftconv.cu)
bool fft_size_supported(int P);  // P = 256 q, q = 2^a 3^b 5^c (b <= 2, c <= 1), P <= 8192
cudaError_t fftconv_prepare(int P);
void launch_twiddles(float2* tw, int P, cudaStream_t s);
// KA: (P/2 + 1) x (P/2 + 1) floats (pitch P/2 + 1); KH: (P/2 + 1) x P floats.  No-op
// (early exit) unless geom->kspec.
void launch_kspec(const GridGeom* geom, int P, ForceArgs fa, const float2* tw, float* KA,
                  float* KH, cudaStream_t s);
// row passes over grid rows [row0, row1) (row0 even; rows >= M are skipped on the device)
void launch_rows_fwd(const GridGeom* geom, const float4* C, int cpitch, int P, int row0,
                     int row1, const float2* tw, float2* CA, int ca_pitch, cudaStream_t s,
                     const PeerRoute* route = nullptr);
// column pass over half-spectrum columns [q0, q1) (q0 even), which CA holds as columns
// 0 .. q1 - q0 - 1 (the whole half spectrum on one GPU: q0 = 0, q1 = P/2 + 1)
void launch_cols(const GridGeom* geom, float2* CA, int ca_pitch, const float* KH, int P,
                 const float2* tw, int q0, int q1, cudaStream_t s,
                 const PeerRoute* route = nullptr);
// rows_inv also re-zeroes the charge rows it covers (consumed by rows_fwd)
void launch_rows_inv(const GridGeom* geom, const float2* CA, int ca_pitch, int P, int row0,
                     int row1, const float2* tw, float* Phi, int cpitch, float4* C,
                     cudaStream_t s, const PeerRoute* route = nullptr);
// internal node renumbering (kernels_reorder.cu)
size_t reorder_scratch_bytes(int64_t n);
void launch_iota(int* perm, int* inv, int64_t n, cudaStream_t s);
// new permutation (Morton order of the box): perm_new[new slot] = caller id
int launch_reorder_perm(const float2* xy_old, const BoxKeys* box, const int* perm_old,
                        int* perm_new, int64_t n, void* scratch, cudaStream_t s);
// positions, inverse and CSR in the new order (every rank, from the same perm_new)
int launch_reorder_apply(const float2* xy_old, float2* xy_new, const int* inv_old,
                         const int* perm_new, int* inv_new, const int64_t* row_ptr_o,
                         const int32_t* col_o, int64_t* row_ptr_p, int32_t* col_p, int64_t n,
                         void* scratch, cudaStream_t s);
void launch_unpermute(const float2* in, const int* perm, int64_t n, float2* out, cudaStream_t s);
void launch_permute(const float2* in, const int* perm, int64_t n, float2* out, cudaStream_t s);

// NP1 of the layout (kernels_np.cu): hits[q] = |N_G(t) ∩ N_L(t, deg t)| for t = lo + q;
// *np_sum = sum over the shard of (deg == 0 ? 1 : h / (2 deg - h)) / n (fixed-order sum).
// ids = caller node id per internal slot (tie rule), NULL = identity.  Returns launches.
int np_grid_side(int64_t n);
size_t np_scratch_bytes(int64_t n, int64_t n_local);
int launch_np1(const float2* xy, int64_t n, int64_t lo, int64_t n_local, const int64_t* row_ptr,
               const int32_t* col, const int* ids, const BoxKeys* box_keys, void* scratch,
               int* hits, double* np_sum, cudaStream_t s);
void launch_unpermute_int(const int* in, const int* perm, int64_t n, int* out, cudaStream_t s);
void exclusive_scan_ll(const long long* in, long long* out, int64_t n, long long* sums,
                       cudaStream_t s);

void launch_gather_update(const float2* xy, float2* xy_next, int64_t lo, int64_t n_local,
                          const GridGeom* geom, int k, const float* phi,
                          const int64_t* row_ptr, const int32_t* col, ForceArgs fa,
                          FocusArgs fo, float eta, int iter, int update, float2* rep_out,
                          float2* att_out, unsigned long long* diverge, BoxKeys* next_part,
                          cudaStream_t s, const PeerRoute* route = nullptr, int next_buf = 0,
                          const float2* A_pre = nullptr);
// attraction of the shard's nodes into A (gather_update's A_pre)
void launch_attraction(const float2* xy, int64_t lo, int64_t n_local, const int64_t* row_ptr,
                       const int32_t* col, ForceArgs fa, float2* A, cudaStream_t s,
                       int blocks = 0);

// heavy rows (kernels_heavy.cu): build the chunk index of the current CSR (scratch: 8 (n+1)
// + sums bytes, heavy_scratch_bytes), then the chunk sums for the rows [lo, hi)
size_t heavy_scratch_bytes(int64_t n);
void launch_heavy_build(const int64_t* row_ptr, int64_t n, long long* first, void* scratch,
                        cudaStream_t s);
void launch_heavy_attr(const float2* xy, const int64_t* row_ptr, const int32_t* col,
                       const long long* first, int64_t lo, int64_t hi, int64_t n_items_max,
                       float beta, float2* part, cudaStream_t s);

// PivotMDS initialisation (kernels_pmds.cu): caller-order CSR, p <= pmds_max_pivots();
// xy (device, n) receives the layout, pivots_out (host, p) the pivots.
int pmds_max_pivots();
size_t pmds_scratch_bytes(int64_t n, int p);
cudaError_t launch_pmds(const int64_t* rp, const int32_t* col, int64_t n, int64_t nnz, int p,
                        unsigned long long seed_pivot, void* scratch, float2* xy,
                        int* pivots_out, int64_t* launches, const char** stage,
                        cudaStream_t s);

// local refinement (kernels_focus.cu)
void launch_mark_focus(const int* focal, int n_focal, const int64_t* row_ptr_caller,
                       const int32_t* col_caller, unsigned char* label_caller, cudaStream_t s);
void launch_focus_slots(const unsigned char* label_caller, const int* perm, const int* inv,
                        int64_t n, const int* region_caller, int m, unsigned char* label_slot,
                        int* region_slot, cudaStream_t s);
void launch_focus_s1(const float2* xy, int64_t lo, int64_t n_local, const int* region_slot,
                     int m, ForceArgs fa, float2* s1, cudaStream_t s);

}  // namespace tfdp
