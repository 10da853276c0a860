// libtfdp host runtime: the C ABI of include/tfdp.h.
//
// Owns device memory, the per-iteration schedule (k_t, eta_t), the FFT geometry, the NCCL
// communicator and the CSR/shard indexing.  Every force evaluation is enqueued as sm_100a
// kernels (kernels_exact.cu, kernels_fft.cu, kernels_fftconv.cu) on the context stream;
// there is no host compute path and no library FFT.  Citations as in include/tfdp.h.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/tfdp.h"
#include "nccl_shim.h"
#include "tfdp_internal.h"

using tfdp::BoxKeys;
using tfdp::ForceArgs;
using tfdp::GridGeom;

namespace {

enum Kind {
  K_EXACT_PARTIAL = 0,
  K_EXACT_FINISH,
  K_BBOX,
  K_SETUP,
  K_REORDER,
  K_SPREAD,
  K_KSPEC,
  K_ROWS_FWD,
  K_COLS,
  K_ROWS_INV,
  K_GATHER_UPDATE,
  K_COMM,
  K_HEAVY,
  K_ATTR,
  K_COUNT
};
const char* kKindNames[K_COUNT] = {"exact_partial", "exact_finish", "bbox",     "setup",
                                   "reorder",       "spread",       "kspec_rows", "rows_fwd",
                                   "cols",          "rows_inv",     "gather_update", "nccl",
                                   "heavy_rows", "attraction"};
const bool kOwnKernel[K_COUNT] = {true, true, true, true, true, true,
                                  true, true, true, true, true, false, true, true};

}  // namespace

struct tfdp_ctx {
  int64_t n = 0, lo = 0, hi = 0;
  tfdp_params p{};
  int rank = 0, world = 1, device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // side stream: the kernel spectrum (depends only on the grid geometry) runs concurrently
  // with spread + rows_fwd; fork/join with events, so the ctx stream order is preserved
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_join2 = nullptr;  // after the side stream's heavy rows + attraction
  // attraction on the side stream (TFDP_ATTR_SIDE=0: walked inside gather_update)
  bool attr_side = true;
  bool attr_pre = false;  // this evaluation's attraction is in attr
  float2* attr = nullptr;
  bool kspec_overlap = true;  // env TFDP_KSPEC_OVERLAP=0 runs it in line (tuning / A-B)
  // where the side stream's attraction forks off the FFT chain (TFDP_ATTR_AT): 0 after setup,
  // 1 after rows_fwd, 2 after cols; its grid (TFDP_ATTR_BLOCKS: 0 = one thread per node)
  int attr_at = 0;
  int attr_blocks = 0;
  bool attr_deferred = false;
  cudaEvent_t ev_fork2 = nullptr;
  float2* xy[2] = {nullptr, nullptr};
  int cur = 0;
  int64_t* row_ptr = nullptr;
  int32_t* col = nullptr;
  int64_t nnz = 0;
  // exact path
  double2* part = nullptr;
  int n_chunks = 1;
  int64_t chunk = 0;
  // outputs of tfdp_forces
  float2* rep = nullptr;
  float2* att = nullptr;
  // status words
  unsigned long long* diverge = nullptr;
  int* capped = nullptr;
  unsigned long long* h_status = nullptr;  // pinned [2 + sizeof(GridGeom)/8]
  BoxKeys* keys = nullptr;      // reduced box of the last geometry setup
  BoxKeys* box_part = nullptr;  // per-block partial boxes (bbox / fused update epilogue)
  int n_part = 0;               // partials written by the last producer
  GridGeom* geom = nullptr;
  tfdp::KspecKey* kkey = nullptr;  // [4]: (P, h, gamma) of the spectrum held in kh[k] (device)
  bool box_valid = false;
  // ibFFT
  int nint_cap = 0;
  int P_of_k[4] = {0, 0, 0, 0};
  int cap_of_k[4] = {0, 0, 0, 0};
  int cpitch = 0;        // row pitch of the charges (float4) and the potential planes
  int ca_pitch = 0;      // rows of the half-spectra CA (multiple of 32; kernels_fftconv.cu)
  int64_t alloc_planes = 0, alloc_ca = 0, alloc_ka = 0;
  float* grid = nullptr;  // charges C (spread target): float4 {C_1, C_x~, C_y~, 0} per node
  float* phi = nullptr;   // potentials Phi (gather source)
  float2* ca = nullptr;   // row half-spectra, transformed in place by the column pass
  float* ka = nullptr;    // kernel row spectra KA[q][dy]
  // kernel spectrum columns KH[q][u] (real), one per k: K^ is a plan constant of (P_k, h, gamma)
  // under R5', so each order keeps its own across the k switches of the schedule
  float* kh[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t alloc_kh[4] = {0, 0, 0, 0};
  float2* tw[4] = {nullptr, nullptr, nullptr, nullptr};  // twiddles per k (length P_k)
  int tw_P[4] = {0, 0, 0, 0};
  // multi-GPU slab mode (TFDP_DIST_SLAB, kernels_dist.cu): per-k row slabs / column chunks,
  // xa = exchange-1 send / exchange-2 receive, xb = exchange-1 receive (column pass in place)
  bool slab = false;
  tfdp::SlabPlan plan[4];
  float2* xa = nullptr;
  float2* xb = nullptr;
  int64_t alloc_xa = 0, alloc_xb = 0;
  float2* fbuf = nullptr;  // n float2: forces of all ranks (tfdp_forces of a reordered shard)
  // slab mode with fused exchanges (peer routes, tfdp_internal.h PeerRoute): one route per k
  // in device memory; NCCL contexts map the peers' buffers with CUDA IPC (re-mapped after any
  // re-allocation), virtual ranks get the other contexts' pointers from the group call
  bool p2p = false;
  bool route_dirty = true;
  tfdp::PeerRoute* d_route = nullptr;  // [4]
  int* bar = nullptr;                  // barrier word of the NCCL phase barriers
  std::vector<void*> ipc_open;         // peer mappings to close
  // heavy rows (kernels_heavy.cu): chunk index of the current CSR and the chunk sums
  int64_t hv_items = 0;
  long long* hv_first = nullptr;
  float2* hv_part = nullptr;
  void* hv_scratch = nullptr;
  // schedule
  int t = 0;
  std::vector<int32_t> ksched;
  ForceArgs fa{};
  // state
  uint32_t warnings = 0;
  bool errored = false;
  std::string err;
  // NCCL
  const tfdp::NcclApi* nccl = nullptr;
  ncclComm_t comm = nullptr;
  // profiling
  uint32_t prof_mask = 0;  // kernel kinds timed with CUDA events (bit = kind)
  // internal node order (kernels_reorder.cu): internal slot i holds caller node perm[i]
  bool reorder = false;
  int64_t iters_run = 0, reordered_at = -1;
  int* perm = nullptr;
  int* inv = nullptr;
  int* perm2 = nullptr;
  int* inv2 = nullptr;
  int64_t* row_ptr_o = nullptr;  // caller-order CSR (source of every rebuild)
  int32_t* col_o = nullptr;
  void* rscratch = nullptr;
  float2* iobuf = nullptr;  // n float2 staging for (un)permuted inputs / outputs
  // NP1 metric (kernels_np.cu), allocated at the first tfdp_np1 call
  void* np_scratch = nullptr;
  int* np_hits = nullptr;    // [n_local] slot order
  int* np_hits2 = nullptr;   // [n] caller order (reordered contexts)
  BoxKeys* np_slots = nullptr;
  BoxKeys* np_keys = nullptr;
  double* np_sum = nullptr;
  // local refinement mask (kernels_focus.cu), tfdp_set_focus
  bool focus_on = false;
  float fo_la = 1.f, fo_lf = 1.f, fo_ls = 1.f;
  unsigned char* label_caller = nullptr;
  unsigned char* label_slot = nullptr;
  int* region_caller = nullptr;
  int* region_slot = nullptr;
  int region_m = 0, region_cap = 0;
  float2* s1 = nullptr;
  struct Pend {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Pend> pend;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[K_COUNT] = {};
  int64_t prof_n[K_COUNT] = {};
  int64_t launches = 0;
};

namespace {

thread_local std::string g_noctx_err;

tfdp_status fail(tfdp_ctx* c, tfdp_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  else g_noctx_err = buf;
  return s;
}

#define CUDA_TRY(c, call)                                                                  \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(c, e_ == cudaErrorMemoryAllocation ? TFDP_ERR_OOM : TFDP_ERR_CUDA,       \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);    \
  } while (0)

#define NCCL_TRY(c, call)                                                                  \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess)                                                                 \
      return fail(c, TFDP_ERR_NCCL, "%s: %s", #call, (c)->nccl->GetErrorString(r_));      \
  } while (0)

#define TRY(x)                          \
  do {                                  \
    tfdp_status s_ = (x);               \
    if (s_ != TFDP_OK) return s_;       \
  } while (0)

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ---------------------------------------------------------------- profiling
cudaEvent_t ev_get(tfdp_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct Scope {
  tfdp_ctx* c;
  int kind;
  cudaEvent_t a = nullptr;
  bool on;
  cudaStream_t st;
  Scope(tfdp_ctx* c_, int k, cudaStream_t s = nullptr, int n_launch = 1)
      : c(c_), kind(k), on((c_->prof_mask >> k) & 1u), st(s ? s : c_->stream) {
    if (on) {
      a = ev_get(c);
      cudaEventRecord(a, st);
    }
    if (kOwnKernel[k]) c->launches += n_launch;
  }
  ~Scope() {
    if (on) {
      cudaEvent_t b = ev_get(c);
      cudaEventRecord(b, st);
      c->pend.push_back({kind, a, b});
    }
  }
};

void prof_collect(tfdp_ctx* c) {
  if (c->pend.empty()) return;
  cudaStreamSynchronize(c->stream);
  for (auto& q : c->pend) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, q.a, q.b);
    c->prof_ms[q.kind] += ms;
    c->prof_n[q.kind] += 1;
    c->ev_pool.push_back(q.a);
    c->ev_pool.push_back(q.b);
  }
  c->pend.clear();
}

// ---------------------------------------------------------------- helpers
// Largest FFT of the shared-memory kernels (1024 threads, one radix-16 butterfly each; the
// AoS one-FFT-per-block kernels above 8192, kernels_fftconv.cu).
constexpr int kMaxFftSize = 16384;

// Smallest m >= target with m % 256 == 0 and m = 2^a 3^b 5^c, b <= 2, c <= 1 (the radices
// of kernels_fftconv.cu; the first two stages are radix 16, all strides multiples of 16).
int nice_fft_size(int64_t target) {
  for (int64_t m = std::max<int64_t>((target + 255) / 256 * 256, 256);; m += 256) {
    int64_t r = m;
    int b = 0, c5 = 0;
    while (r % 2 == 0) r /= 2;
    while (r % 3 == 0) { r /= 3; ++b; }
    while (r % 5 == 0) { r /= 5; ++c5; }
    if (r == 1 && b <= 2 && c5 <= 1) return (int)m;
  }
}

int gamma_int_of(double g) {
  for (int q : {1, 2, 3, 4, 8})
    if (g == (double)q) return q;
  return 0;
}

std::vector<int32_t> k_schedule(int T) {
  // P:545 / S:303 (reading R4): ceil(0.9T) x k1, ceil(0.05T) x k2, rest k3; T < 20 -> all 3
  std::vector<int32_t> ks(T, 3);
  if (T < 20) return ks;
  int n1 = (int)std::ceil(0.9 * T - 1e-9);
  int n2 = (int)std::ceil(0.05 * T - 1e-9);
  n1 = std::min(n1, T);
  n2 = std::min(n2, T - n1);
  for (int i = 0; i < T; ++i) ks[i] = i < n1 ? 1 : (i < n1 + n2 ? 2 : 3);
  return ks;
}

bool finite_d(double x) { return std::isfinite(x); }

tfdp_status validate_params(const tfdp_params* p, uint32_t* warn, std::string* msg) {
  char b[256];
  if (p->dim != 2) {
    *msg = "dim must be 2 (P:410)";
    return TFDP_ERR_UNSUPPORTED;
  }
  if (!finite_d(p->alpha) || !finite_d(p->beta) || !finite_d(p->gamma) || !finite_d(p->rho) ||
      !finite_d(p->step0)) {
    *msg = "non-finite parameter";
    return TFDP_ERR_ARG;
  }
  if (p->gamma <= 0 || p->rho <= 0 || p->alpha < 0 || p->beta < 0 || p->step0 <= 0 ||
      p->iterations < 1 || p->t0 < 0) {
    snprintf(b, sizeof b, "invalid parameter (need gamma>0, rho>0, alpha>=0, beta>=0, eta0>0, T>=1, t0>=0)");
    *msg = b;
    return TFDP_ERR_ARG;
  }
  if (p->solver != TFDP_EXACT && p->solver != TFDP_IBFFT) {
    *msg = "unknown solver";
    return TFDP_ERR_ARG;
  }
  if (p->k < 0 || p->k > 3) {
    *msg = "k must be 0 (dynamic) or 1..3";
    return TFDP_ERR_ARG;
  }
  if (p->cooling != TFDP_COOL_LINEAR && p->cooling != TFDP_COOL_CONSTANT) {
    *msg = "unknown cooling";
    return TFDP_ERR_ARG;
  }
  if (p->dist_mode != TFDP_DIST_SPREAD_ALL && p->dist_mode != TFDP_DIST_GRID_ALLREDUCE &&
      p->dist_mode != TFDP_DIST_SLAB) {
    *msg = "unknown dist_mode";
    return TFDP_ERR_ARG;
  }
  if (p->interval_rule != TFDP_RULE_UNIT && p->interval_rule != TFDP_RULE_SPAN) {
    *msg = "unknown interval_rule";
    return TFDP_ERR_ARG;
  }
  if (p->n_int_min < 1 || p->n_int_fixed < 0 || p->fft_size < 0) {
    *msg = "n_int_min >= 1, n_int_fixed >= 0, fft_size >= 0";
    return TFDP_ERR_ARG;
  }
  uint32_t w = 0;
  if (p->alpha * (1.0 + p->beta) >= 1.0) w |= TFDP_WARN_ALPHA_BETA;  // Eq. limitweight
  if (p->gamma <= 1.0) w |= TFDP_WARN_GAMMA;                          // Eq. exponentcondiction
  *warn = w;
  return TFDP_OK;
}

// O(m log d) check of the CSR invariants.
bool validate_csr(int64_t n, const int64_t* rp, const int32_t* col, std::string* msg) {
  char b[256];
  if (rp[0] != 0) {
    *msg = "row_ptr[0] != 0";
    return false;
  }
  for (int64_t i = 0; i < n; ++i) {
    if (rp[i + 1] < rp[i]) {
      snprintf(b, sizeof b, "row_ptr not monotone at %lld", (long long)i);
      *msg = b;
      return false;
    }
  }
  bool ok = true;
  int64_t bad = -1;
#pragma omp parallel for schedule(dynamic, 4096) reduction(&& : ok)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const int64_t j = col[e];
      bool good = j >= 0 && j < n && j != i && (e == rp[i] || col[e - 1] < col[e]);
      if (good) {  // symmetric: i in row j
        const int32_t* a = col + rp[j];
        const int32_t* z = col + rp[j + 1];
        good = std::binary_search(a, z, (int32_t)i);
      }
      if (!good) {
        ok = false;
#pragma omp critical
        bad = i;
      }
    }
  }
  if (!ok) {
    snprintf(b, sizeof b,
             "CSR invalid at row %lld (need sorted, symmetric, no self-loop/duplicate, in range)",
             (long long)bad);
    *msg = b;
  }
  return ok;
}

void host_box(const float* xy, int64_t n, float* L) {
  float mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    mnx = std::min(mnx, xy[2 * i]);
    mxx = std::max(mxx, xy[2 * i]);
    mny = std::min(mny, xy[2 * i + 1]);
    mxy = std::max(mxy, xy[2 * i + 1]);
  }
  *L = std::max(mxx - mnx, mxy - mny);
}

// ---------------------------------------------------------------- FFT resources
void free_fft_buffers(tfdp_ctx* c) {
  cudaFree(c->grid);
  cudaFree(c->phi);
  cudaFree(c->ca);
  cudaFree(c->ka);
  c->grid = c->phi = c->ka = nullptr;
  c->ca = nullptr;
  c->alloc_planes = c->alloc_ca = c->alloc_ka = 0;
  for (int k = 0; k < 4; ++k) {
    cudaFree(c->kh[k]);
    c->kh[k] = nullptr;
    c->alloc_kh[k] = 0;
  }
  for (int k = 0; k < 4; ++k) {
    cudaFree(c->tw[k]);
    c->tw[k] = nullptr;
    c->tw_P[k] = 0;
  }
}

bool k_used(const tfdp_ctx* c, int k) { return c->p.k == 0 || c->p.k == k; }

// Row pitch of the charge / potential planes at order k: the grid points the plan holds,
// cap_k k (the buffers are sized for the largest k; a per-k pitch keeps the planes of the
// smaller grids compact, and their slab rows contiguous for the potential exchange).
int pitch_k(const tfdp_ctx* c, int k) { return c->cap_of_k[k] * k; }

// Grid sizing: N_need = ceil(L) + 8 (or the forced N_int);
// P_k = smallest 2^a3^b5^c >= 2 N_need k - 1 (R9: any such P is exact); the grid then
// holds N_int <= cap_k = floor((P_k + 1) / 2k).  Re-planned when the layout outgrows it.
tfdp_status configure_fft(tfdp_ctx* c, float L) {
  const tfdp_params& p = c->p;
  int need;
  if (p.n_int_fixed > 0) need = p.n_int_fixed;
  else need = std::max<int>(p.n_int_min, (int)std::min<double>(std::ceil((double)L) + 8.0, 1e6));
  int mcap = 0;
  for (int k = 1; k <= 3; ++k) {
    int P = p.fft_size > 0 ? p.fft_size : nice_fft_size(2LL * need * k - 1);
    if (P > kMaxFftSize && p.fft_size == 0) P = kMaxFftSize;  // grid capped (warning bit)
    int cap = (P + 1) / (2 * k);
    if (p.n_int_fixed > 0 && k_used(c, k)) {
      if (cap < p.n_int_fixed)
        return fail(c, TFDP_ERR_ARG, "fft_size %d < 2*N_int*k-1 = %d (k=%d)", P,
                    2 * p.n_int_fixed * k - 1, k);
      cap = p.n_int_fixed;
    }
    if (!tfdp::fft_size_supported(P))
      return fail(c, TFDP_ERR_UNSUPPORTED,
                  "FFT size %d unsupported (256 q, q = 2^a 3^b 5^c, b <= 2, c <= 1, <= %d)", P,
                  kMaxFftSize);
    c->P_of_k[k] = P;
    c->cap_of_k[k] = cap;
    if (k_used(c, k)) mcap = std::max(mcap, cap * k);
  }
  c->nint_cap = need;
  const int cpitch = mcap;
  // CA rows: a multiple of the CA row tile (kernels_fftconv.cu); slab mode: of 96 (whole
  // 24-row slab units of every k, kernels_dist.cu)
  const int capitch = c->slab ? (mcap + 95) / 96 * 96 : (mcap + 31) & ~31;
  // charges: one float4 {C_1, C_x~, C_y~, 0} per grid node; potentials: 3 planes
  int64_t planes = 4LL * cpitch * cpitch, ca = 0, ka = 0;
  for (int k = 1; k <= 3; ++k) {
    if (!k_used(c, k)) continue;
    ca = std::max<int64_t>(ca, 3LL * (c->P_of_k[k] / 2 + 1) * capitch);
    ka = std::max<int64_t>(ka, (int64_t)(c->P_of_k[k] / 2 + 1) * (c->P_of_k[k] / 2 + 1));
  }
  if (planes > c->alloc_planes || ca > c->alloc_ca || ka > c->alloc_ka) {
    cudaStreamSynchronize(c->stream);
    cudaFree(c->grid);
    cudaFree(c->phi);
    cudaFree(c->ca);
    cudaFree(c->ka);
    c->grid = c->phi = c->ka = nullptr;
    c->ca = nullptr;
    CUDA_TRY(c, cudaMalloc(&c->grid, planes * sizeof(float)));
    // invariant: the charge planes are zero between iterations (rows_inv re-zeroes)
    CUDA_TRY(c, cudaMemsetAsync(c->grid, 0, planes * sizeof(float), c->stream));
    CUDA_TRY(c, cudaMalloc(&c->phi, (planes / 4) * 3 * sizeof(float)));
    CUDA_TRY(c, cudaMalloc(&c->ca, ca * sizeof(float2)));
    CUDA_TRY(c, cudaMalloc(&c->ka, ka * sizeof(float)));
    c->alloc_planes = planes;
    c->alloc_ca = ca;
    c->alloc_ka = ka;
    c->route_dirty = true;
  }
  for (int k = 1; k <= 3; ++k) {
    if (!k_used(c, k)) continue;
    const int64_t kh = (int64_t)(c->P_of_k[k] / 2 + 2) * c->P_of_k[k];
    if (kh > c->alloc_kh[k]) {
      cudaStreamSynchronize(c->stream);
      cudaFree(c->kh[k]);
      c->kh[k] = nullptr;
      CUDA_TRY(c, cudaMalloc(&c->kh[k], kh * sizeof(float)));
      c->alloc_kh[k] = kh;
      // a new buffer holds no spectrum (the key also carries P, so a same-buffer re-plan to
      // another P invalidates itself)
      CUDA_TRY(c, cudaMemsetAsync(c->kkey + k, 0, sizeof(tfdp::KspecKey), c->stream));
    }
  }
  c->cpitch = cpitch;
  c->ca_pitch = capitch;
  int Pmax = 0;
  for (int k = 1; k <= 3; ++k) {
    if (!k_used(c, k)) continue;
    const int P = c->P_of_k[k];
    Pmax = std::max(Pmax, P);
    if (c->tw_P[k] != P) {
      cudaFree(c->tw[k]);
      c->tw[k] = nullptr;
      CUDA_TRY(c, cudaMalloc(&c->tw[k], (size_t)(P + 128) * sizeof(float2)));  // >= tw_len
      tfdp::launch_twiddles(c->tw[k], P, c->stream);
      c->tw_P[k] = P;
    }
  }
  for (int k = 1; k <= 3; ++k)
    if (k_used(c, k)) CUDA_TRY(c, tfdp::fftconv_prepare(c->P_of_k[k]));
  if (c->slab) {  // per-k slabs over [0, cap_k k) and column chunks of P_k / 2 + 1
    int64_t xa = 1, xb = 1;
    for (int k = 1; k <= 3; ++k) {
      if (!k_used(c, k)) continue;
      tfdp::SlabPlan& pl = c->plan[k];
      tfdp::slab_plan(c->world, c->rank, c->cap_of_k[k] * k, c->P_of_k[k], &pl);
      const int64_t rows_me = pl.row0[c->rank + 1] - pl.row0[c->rank];
      const int64_t nq_me = pl.q0[c->rank + 1] - pl.q0[c->rank];
      xa = std::max<int64_t>(xa, 3 * rows_me * pl.H);
      xb = std::max<int64_t>(xb, 3LL * pl.R * nq_me);
    }
    if (xa > c->alloc_xa || xb > c->alloc_xb) {
      cudaStreamSynchronize(c->stream);
      cudaFree(c->xa);
      cudaFree(c->xb);
      c->xa = c->xb = nullptr;
      CUDA_TRY(c, cudaMalloc(&c->xa, xa * sizeof(float2)));
      CUDA_TRY(c, cudaMalloc(&c->xb, xb * sizeof(float2)));
      c->alloc_xa = xa;
      c->alloc_xb = xb;
      c->route_dirty = true;
    }
  }
  CUDA_TRY(c, cudaGetLastError());
  return TFDP_OK;
}

// ---------------------------------------------------------------- groups of ranks
// A Group is the set of ranks one call drives: {self} for a normal context (one process per
// GPU), whose exchanges are NCCL calls; or all p virtual ranks of one process on one device
// (tfdp_group_step / tfdp_group_forces), whose exchanges are device copies on their shared
// stream.  Either way the same kernels run in the same phases.
struct Group {
  tfdp_ctx** c;
  int p;
  tfdp_ctx* operator[](int i) const { return c[i]; }
  bool virt() const { return p > 1; }
};

// d2d copy on the ctx stream (virtual exchanges; NCCL self-messages)
tfdp_status dcopy(tfdp_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return TFDP_OK;
  CUDA_TRY(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
  return TFDP_OK;
}

// Position all-gather: every rank's own slice [lo, hi) of xy (the update's output buffer)
// to every other rank.
tfdp_status phase_barrier(const Group& G);

tfdp_status exchange_positions(const Group& G, int buf) {
  tfdp_ctx* c = G[0];
  if (c->world == 1) return TFDP_OK;
  if (c->p2p && (c->slab || c->p.solver == TFDP_EXACT))  // the update stored into every rank
    return phase_barrier(G);
  if (G.virt()) {
    for (int r = 0; r < G.p; ++r)
      for (int s = 0; s < G.p; ++s)
        if (s != r)
          TRY(dcopy(G[s], G[s]->xy[buf] + G[r]->lo, G[r]->xy[buf] + G[r]->lo,
                    (G[r]->hi - G[r]->lo) * sizeof(float2)));
    return TFDP_OK;
  }
  if (!c->comm)
    return fail(c, TFDP_ERR_UNSUPPORTED,
                "virtual shard context (no NCCL id): use tfdp_group_step / tfdp_group_forces");
  float2* xy = c->xy[buf];
  Scope sc(c, K_COMM);
  NCCL_TRY(c, c->nccl->GroupStart());
  for (int r = 0; r < c->world; ++r) {
    int64_t lo, hi;
    tfdp_shard_range(c->n, c->world, r, &lo, &hi);
    if (hi > lo)
      NCCL_TRY(c, c->nccl->Broadcast(xy + lo, xy + lo, (size_t)(hi - lo) * 2, ncclFloat, r,
                                     c->comm, c->stream));
  }
  NCCL_TRY(c, c->nccl->GroupEnd());
  return TFDP_OK;
}

// Same for an int array (the new permutation of a renumbering, root rank 0 only).
tfdp_status exchange_perm(const Group& G) {
  tfdp_ctx* c = G[0];
  if (c->world == 1) return TFDP_OK;
  if (G.virt()) {
    for (int s = 1; s < G.p; ++s) TRY(dcopy(G[s], G[s]->perm2, G[0]->perm2, c->n * sizeof(int)));
    return TFDP_OK;
  }
  Scope sc(c, K_COMM);
  NCCL_TRY(c, c->nccl->Broadcast(c->perm2, c->perm2, (size_t)c->n, ncclInt32, 0, c->comm, c->stream));
  return TFDP_OK;
}

// ---- slab mode layout helpers (kernels_dist.cu): float2 offsets
int64_t slab_nrt(const tfdp::SlabPlan& pl, int r) { return (pl.row0[r + 1] - pl.row0[r]) / 8; }
int64_t slab_nq(const tfdp::SlabPlan& pl, int s) { return pl.q0[s + 1] - pl.q0[s]; }
// xa segment (dest s, channel ch) of a rank whose slab has nrt row tiles
int64_t xa_seg(const tfdp::SlabPlan& pl, int64_t nrt, int s, int ch) {
  return 3 * nrt * 8 * pl.q0[s] + ch * nrt * slab_nq(pl, s) * 8;
}
// xb block (rows of rank r, channel ch) of column-chunk owner me
int64_t xb_blk(const tfdp::SlabPlan& pl, int me, int r, int ch) {
  return ((int64_t)ch * (pl.R / 8) + pl.row0[r] / 8) * slab_nq(pl, me) * 8;
}

// Exchange 1 (dir = 0): row-pass output segments xa -> column-chunk blocks xb.
// Exchange 2 (dir = 1): column-pass output blocks xb -> segments xa of the row owners.
// Message (src r -> dst s, channel ch) holds nrt(row rank) x nq(column rank) x 8 float2.
tfdp_status exchange_slabs(const Group& G, int k, int dir) {
  tfdp_ctx* c = G[0];
  const int p = c->world;
  auto msg = [&](tfdp_ctx* cr, tfdp_ctx* cs, int r, int s, int ch, float2** src, float2** dst,
                 int64_t* cnt) {
    const tfdp::SlabPlan& pl = c->plan[k];
    if (dir == 0) {  // r = row owner, s = column owner
      *cnt = slab_nrt(pl, r) * slab_nq(pl, s) * 8;
      *src = cr ? cr->xa + xa_seg(pl, slab_nrt(pl, r), s, ch) : nullptr;
      *dst = cs ? cs->xb + xb_blk(pl, s, r, ch) : nullptr;
    } else {  // r = column owner, s = row owner
      *cnt = slab_nrt(pl, s) * slab_nq(pl, r) * 8;
      *src = cr ? cr->xb + xb_blk(pl, r, s, ch) : nullptr;
      *dst = cs ? cs->xa + xa_seg(pl, slab_nrt(pl, s), r, ch) : nullptr;
    }
  };
  if (G.virt()) {
    for (int r = 0; r < p; ++r)
      for (int s = 0; s < p; ++s)
        for (int ch = 0; ch < 3; ++ch) {
          float2 *src, *dst;
          int64_t cnt;
          msg(G[r], G[s], r, s, ch, &src, &dst, &cnt);
          TRY(dcopy(G[s], dst, src, cnt * sizeof(float2)));
        }
    return TFDP_OK;
  }
  const int me = c->rank;
  Scope sc(c, K_COMM);
  for (int ch = 0; ch < 3; ++ch) {  // self-message: a device copy
    float2 *src, *dst;
    int64_t cnt;
    msg(c, c, me, me, ch, &src, &dst, &cnt);
    TRY(dcopy(c, dst, src, cnt * sizeof(float2)));
  }
  NCCL_TRY(c, c->nccl->GroupStart());
  for (int o = 0; o < p; ++o) {
    if (o == me) continue;
    for (int ch = 0; ch < 3; ++ch) {
      float2 *src, *dst;
      int64_t cnt;
      msg(c, nullptr, me, o, ch, &src, &dst, &cnt);  // me -> o
      if (cnt > 0) NCCL_TRY(c, c->nccl->Send(src, (size_t)cnt * 2, ncclFloat, o, c->comm, c->stream));
      msg(nullptr, c, o, me, ch, &src, &dst, &cnt);  // o -> me
      if (cnt > 0) NCCL_TRY(c, c->nccl->Recv(dst, (size_t)cnt * 2, ncclFloat, o, c->comm, c->stream));
    }
  }
  NCCL_TRY(c, c->nccl->GroupEnd());
  return TFDP_OK;
}

// Exchange 3: every rank's slab rows of the three potential planes to every rank (the
// gather of a rank's nodes may read any row).
tfdp_status exchange_phi(const Group& G, int k) {
  tfdp_ctx* c = G[0];
  const tfdp::SlabPlan& pl = c->plan[k];
  const int pk = pitch_k(c, k);
  const int64_t plane = (int64_t)pk * pk;
  auto rows = [&](int r) {
    return std::max<int64_t>(0, std::min<int64_t>(pl.row0[r + 1], pk) - pl.row0[r]);
  };
  if (G.virt()) {
    for (int r = 0; r < G.p; ++r)
      for (int s = 0; s < G.p; ++s)
        if (s != r)
          for (int ch = 0; ch < 3; ++ch) {
            const int64_t off = ch * plane + (int64_t)pl.row0[r] * pk;
            TRY(dcopy(G[s], G[s]->phi + off, G[r]->phi + off, rows(r) * pk * sizeof(float)));
          }
    return TFDP_OK;
  }
  Scope sc(c, K_COMM);
  NCCL_TRY(c, c->nccl->GroupStart());
  for (int r = 0; r < c->world; ++r)
    for (int ch = 0; ch < 3; ++ch) {
      const int64_t cnt = rows(r) * pk;
      float* b = c->phi + ch * plane + (int64_t)pl.row0[r] * pk;
      if (cnt > 0) NCCL_TRY(c, c->nccl->Broadcast(b, b, (size_t)cnt, ncclFloat, r, c->comm, c->stream));
    }
  NCCL_TRY(c, c->nccl->GroupEnd());
  return TFDP_OK;
}

// chunk sums of this shard's heavy rows (before the finishing kernel that adds them)
void heavy_rows(tfdp_ctx* c, cudaStream_t st) {
  if (!c->hv_items) return;
  Scope sc(c, K_HEAVY, st);
  tfdp::launch_heavy_attr(c->xy[c->cur], c->row_ptr, c->col, c->hv_first, c->lo, c->hi,
                          c->hv_items, c->fa.beta, c->hv_part, st);
}

int pdl_max_fft() {
  static const int v = [] {  // TFDP_PDL_MAX_FFT overrides the threshold (A/B runs)
    const char* e = getenv("TFDP_PDL_MAX_FFT");
    return e ? atoi(e) : tfdp::kPdlMaxFft;
  }();
  return v;
}

// bbox (when the box is not known) + setup + the kernel spectrum forked on the side stream
// heavy-row chunks + the per-node attraction on stream st; the join event for gather_update
void side_attraction(tfdp_ctx* c, cudaStream_t st, bool overlap) {
  heavy_rows(c, st);
  if (c->attr_pre) {
    Scope sc(c, K_ATTR, st);
    tfdp::launch_attraction(c->xy[c->cur], c->lo, c->hi - c->lo, c->row_ptr, c->col, c->fa,
                            c->attr, st, c->attr_blocks);
  }
  if (overlap) cudaEventRecord(c->ev_join2, st);
}

// the deferred side-stream attraction, forked at this point of the main stream
void fork_attraction(tfdp_ctx* c, bool overlap, int at) {
  if (!c->attr_deferred || c->attr_at != at) return;
  c->attr_deferred = false;
  cudaEventRecord(c->ev_fork2, c->stream);
  cudaStreamWaitEvent(c->side, c->ev_fork2, 0);
  side_attraction(c, c->side, overlap);
}

void fft_prologue(tfdp_ctx* c, int k, bool* overlap, bool allow_defer = false) {
  const int P = c->P_of_k[k];
  tfdp::set_pdl_active(P <= pdl_max_fft());
  if (!c->box_valid || c->world > 1) {
    Scope sc(c, K_BBOX, nullptr, 2);  // reset_slots + bbox
    tfdp::launch_reset_slots(c->box_part, c->stream);
    c->n_part = tfdp::launch_bbox(c->xy[c->cur], c->n, c->box_part, c->stream);
  }
  {
    Scope sc(c, K_SETUP);
    tfdp::launch_setup(c->box_part, c->n_part, c->keys, c->geom, k, c->p.n_int_min,
                       c->p.n_int_fixed, c->cap_of_k[k], P, pitch_k(c, k), c->capped,
                       c->p.interval_rule, c->fa.gamma, c->kkey + k, c->stream);
  }
  // The kernel spectrum needs only the geometry: fork it onto the side stream so it overlaps
  // spread + rows_fwd (both latency-bound); cols joins on it.  Its kernels exit at once
  // unless setup found the held spectrum stale (a new P, h or gamma: under R5' h = 1/k,
  // so a run recomputes it when k switches or the grid is re-planned).
  // (in line while kspec itself is being timed, so that its events measure the kernel
  // rather than its wait for SMs)
  *overlap = c->kspec_overlap && !((c->prof_mask >> K_KSPEC) & 1u);
  cudaStream_t ks = *overlap ? c->side : c->stream;
  if (*overlap) {
    cudaEventRecord(c->ev_fork, c->stream);
    cudaStreamWaitEvent(c->side, c->ev_fork, 0);
  }
  {
    Scope sc(c, K_KSPEC, ks, 2);  // kspec_rows + kspec_cols
    tfdp::launch_kspec(c->geom, P, c->fa, c->tw[k], c->ka, c->kh[k], ks);
  }
  if (*overlap) cudaEventRecord(c->ev_join, c->side);  // cols joins here
  // the attraction depends only on the positions: heavy-row chunks and the per-node sums also
  // run beside spread + FFT passes; gather_update joins after them (ev_join2)
  c->attr_pre = c->attr_side && !c->focus_on && c->attr;
  c->attr_deferred = allow_defer && *overlap && c->attr_at > 0;
  if (!c->attr_deferred) side_attraction(c, ks, *overlap);
}

tfdp::FocusArgs focus_prologue(tfdp_ctx* c) {
  tfdp::FocusArgs fo{nullptr, nullptr, 1.f, 1.f, 1.f};
  if (c->focus_on) {  // exact repulsion sum over the focal region's sources (R23)
    tfdp::launch_focus_s1(c->xy[c->cur], c->lo, c->hi - c->lo, c->region_slot, c->region_m, c->fa,
                          c->s1, c->stream);
    c->launches++;
    fo = tfdp::FocusArgs{c->label_slot, c->s1, c->fo_la, c->fo_lf, c->fo_ls};
  }
  return fo;
}

// ---------------------------------------------------------------- one evaluation, one rank
// update = 1: x_{t+1} into xy[cur^1] (own shard); update = 0: forces to rep/att.  (The
// position exchange and the buffer flip are the caller's, evaluate().)
tfdp_status evaluate_one(tfdp_ctx* c, int update, float eta, int k) {
  const int64_t n_local = c->hi - c->lo;
  float2* xy = c->xy[c->cur];
  float2* xyn = c->xy[c->cur ^ 1];
  const tfdp::FocusArgs fo = focus_prologue(c);
  if (c->p.solver == TFDP_EXACT) {
    {
      Scope sc(c, K_EXACT_PARTIAL);
      tfdp::launch_exact_partial(xy, c->n, c->lo, n_local, c->chunk, c->n_chunks, c->fa, c->part,
                                 c->stream);
    }
    heavy_rows(c, c->stream);
    {
      Scope sc(c, K_EXACT_FINISH);
      tfdp::launch_exact_finish(xy, xyn, c->lo, n_local, c->n_chunks, c->part, c->row_ptr,
                                c->col, c->fa, fo, eta, c->t, update, c->rep, c->att, c->diverge,
                                c->stream, update && c->p2p && c->world > 1 ? c->d_route : nullptr,
                                c->cur ^ 1);
    }
  } else {
    const bool allreduce = c->world > 1 && c->p.dist_mode == TFDP_DIST_GRID_ALLREDUCE;
    if (allreduce && !c->comm)  // before any charge is spread (the grid stays all-zero)
      return fail(c, TFDP_ERR_UNSUPPORTED, "grid all-reduce needs an NCCL communicator");
    const int P = c->P_of_k[k];
    const int mcap = c->cap_of_k[k] * k;
    const float2* tw = c->tw[k];
    bool overlap;
    fft_prologue(c, k, &overlap, true);
    // The charges are all-zero here: they start zeroed and rows_inv clears the rows rows_fwd
    // consumed (no separate zeroing pass).
    float4* grid4 = reinterpret_cast<float4*>(c->grid);
    {
      Scope sc(c, K_SPREAD);
      if (allreduce)
        tfdp::launch_spread(xy, c->lo, n_local, c->geom, k, grid4, c->stream);
      else
        tfdp::launch_spread(xy, 0, c->n, c->geom, k, grid4, c->stream);
    }
    if (allreduce) {
      Scope sc(c, K_COMM);
      // rows [0, M_cap) of the interleaved charges (they live in [0, M) x [0, M)); a failed
      // reduction leaves charges in the grid: the context is errored (no zero-grid invariant)
      ncclResult_t r = c->nccl->AllReduce(c->grid, c->grid, (size_t)mcap * pitch_k(c, k) * 4,
                                          ncclFloat, ncclSum, c->comm, c->stream);
      if (r != ncclSuccess) {
        c->errored = true;
        return fail(c, TFDP_ERR_NCCL, "grid all-reduce: %s", c->nccl->GetErrorString(r));
      }
    }
    {
      Scope sc(c, K_ROWS_FWD);
      tfdp::launch_rows_fwd(c->geom, grid4, pitch_k(c, k), P, 0, mcap, tw, c->ca, c->ca_pitch,
                            c->stream);
    }
    fork_attraction(c, overlap, 1);
    if (overlap) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    {
      Scope sc(c, K_COLS);
      tfdp::launch_cols(c->geom, c->ca, c->ca_pitch, c->kh[k], P, tw, 0, P / 2 + 1, c->stream);
    }
    fork_attraction(c, overlap, 2);
    {
      Scope sc(c, K_ROWS_INV);
      tfdp::launch_rows_inv(c->geom, c->ca, c->ca_pitch, P, 0, mcap, tw, c->phi, pitch_k(c, k),
                            grid4, c->stream);
    }
    if (overlap) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_join2, 0));
    {
      Scope sc(c, K_GATHER_UPDATE);
      BoxKeys* nk = (update && c->world == 1) ? c->box_part : nullptr;
      if (nk) c->n_part = tfdp::kBoxSlots;
      tfdp::launch_gather_update(xy, xyn, c->lo, n_local, c->geom, k, c->phi, c->row_ptr, c->col,
                                 c->fa, fo, eta, c->t, update, c->rep, c->att, c->diverge, nk,
                                 c->stream, nullptr, 0, c->attr_pre ? c->attr : nullptr);
    }
    c->box_valid = update && c->world == 1;
  }
  CUDA_TRY(c, cudaGetLastError());
  return TFDP_OK;
}

// ---------------------------------------------------------------- slab mode: peer routes
// Phase barrier of the fused exchanges: NCCL contexts order the ranks with a one-word
// all-reduce on the ctx stream (every rank's previous kernels, and so its peer stores, have
// completed before any rank passes it); the virtual ranks of one device share a stream.
tfdp_status phase_barrier(const Group& G) {
  tfdp_ctx* c = G[0];
  if (G.virt() || c->world == 1) return TFDP_OK;
  Scope sc(c, K_COMM);
  NCCL_TRY(c, c->nccl->AllReduce(c->bar, c->bar, 1, ncclInt32, ncclMax, c->comm, c->stream));
  return TFDP_OK;
}

void fill_route(tfdp_ctx* c, int k, tfdp::PeerRoute* r, void* const* xb, void* const* ca,
                void* const* phi, void* const* xy0, void* const* xy1) {
  memset(r, 0, sizeof(*r));
  r->world = c->world;
  r->rank = c->rank;
  if (k > 0) {  // (route 0: positions only — the exact path)
    const tfdp::SlabPlan& pl = c->plan[k];
    r->R = pl.R;
    r->ca_pitch = c->ca_pitch;
    for (int j = 0; j <= c->world; ++j) {
      r->row0[j] = pl.row0[j];
      r->q0[j] = pl.q0[j];
    }
  }
  for (int j = 0; j < c->world; ++j) {
    r->xb[j] = static_cast<float2*>(xb[j]);
    r->ca[j] = static_cast<float2*>(ca[j]);
    r->phi[j] = static_cast<float*>(phi[j]);
    r->xy[0][j] = static_cast<float2*>(xy0[j]);
    r->xy[1][j] = static_cast<float2*>(xy1[j]);
  }
}

// Routes of every rank of the group: the virtual ranks' own pointers, or the peers' buffers
// mapped with CUDA IPC (handles exchanged with NCCL broadcasts; collective, and repeated after
// a re-allocation, which every rank makes at the same call since the plans are identical).
tfdp_status setup_routes(const Group& G) {
  tfdp_ctx* c0 = G[0];
  const int p = c0->world;
  tfdp::PeerRoute h[4];
  if (G.virt()) {
    std::vector<void*> xb(p), ca(p), phi(p), xy0(p), xy1(p);
    for (int j = 0; j < p; ++j) {
      xb[j] = G[j]->xb;
      ca[j] = G[j]->ca;
      phi[j] = G[j]->phi;
      xy0[j] = G[j]->xy[0];
      xy1[j] = G[j]->xy[1];
    }
    for (int i = 0; i < G.p; ++i) {
      tfdp_ctx* c = G[i];
      fill_route(c, 0, &h[0], xb.data(), ca.data(), phi.data(), xy0.data(), xy1.data());
      if (c->p.solver == TFDP_IBFFT)
        for (int k = 1; k <= 3; ++k)
          if (k_used(c, k)) fill_route(c, k, &h[k], xb.data(), ca.data(), phi.data(), xy0.data(), xy1.data());
      CUDA_TRY(c, cudaMemcpyAsync(c->d_route, h, sizeof h, cudaMemcpyHostToDevice, c->stream));
      c->route_dirty = false;
    }
    return TFDP_OK;
  }
  tfdp_ctx* c = c0;
  if (!c->route_dirty) return TFDP_OK;
  for (void* q : c->ipc_open) cudaIpcCloseMemHandle(q);
  c->ipc_open.clear();
  constexpr int kB = 5;  // buffers per rank: xb, ca, phi, xy0, xy1
  std::vector<cudaIpcMemHandle_t> mine(kB);
  void* bufs[kB] = {c->xb, c->ca, c->phi, c->xy[0], c->xy[1]};
  // TFDP_IPC_LOOPBACK=1 (tests only: the ranks are threads of one process, whose own
  // allocations CUDA IPC cannot open): the exchanged "handles" carry the raw device pointers
  static const bool loopback = [] {
    const char* e = getenv("TFDP_IPC_LOOPBACK");
    return e && e[0] == '1';
  }();
  int got = 1;  // a failure here must not leave the other ranks in the handle broadcast alone
  for (int b = 0; b < kB; ++b)
    if (!bufs[b]) {  // (the exact path exchanges positions only)
      memset(&mine[b], 0, sizeof(cudaIpcMemHandle_t));
    } else if (loopback) {
      memset(&mine[b], 0, sizeof(cudaIpcMemHandle_t));
      memcpy(&mine[b], &bufs[b], sizeof(void*));
    } else if (cudaIpcGetMemHandle(&mine[b], bufs[b]) != cudaSuccess) {
      cudaGetLastError();
      memset(&mine[b], 0, sizeof(cudaIpcMemHandle_t));
      got = 0;
    }
  const size_t hs = sizeof(cudaIpcMemHandle_t) * kB;
  unsigned char* dh = nullptr;
  CUDA_TRY(c, cudaMalloc(&dh, hs * p));
  std::vector<unsigned char> all(hs * p);
  CUDA_TRY(c, cudaMemcpyAsync(dh + hs * c->rank, mine.data(), hs, cudaMemcpyHostToDevice, c->stream));
  NCCL_TRY(c, c->nccl->GroupStart());
  for (int r = 0; r < p; ++r)
    NCCL_TRY(c, c->nccl->Broadcast(dh + hs * r, dh + hs * r, hs, ncclChar, r, c->comm, c->stream));
  NCCL_TRY(c, c->nccl->GroupEnd());
  CUDA_TRY(c, cudaMemcpyAsync(all.data(), dh, hs * p, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  cudaFree(dh);
  std::vector<void*> ptr[kB];
  for (int b = 0; b < kB; ++b) ptr[b].resize(p);
  for (int r = 0; r < p; ++r)
    for (int b = 0; b < kB; ++b) {
      if (r == c->rank || !bufs[b]) {
        ptr[b][r] = r == c->rank ? bufs[b] : nullptr;
        continue;
      }
      cudaIpcMemHandle_t hh, zero;
      memcpy(&hh, all.data() + hs * r + sizeof(cudaIpcMemHandle_t) * b, sizeof hh);
      memset(&zero, 0, sizeof zero);
      void* q = nullptr;
      if (loopback) {
        memcpy(&q, &hh, sizeof(void*));
      } else if (memcmp(&hh, &zero, sizeof hh) != 0 &&
                 cudaIpcOpenMemHandle(&q, hh, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
        c->ipc_open.push_back(q);
      } else {
        cudaGetLastError();
        q = nullptr;
      }
      ptr[b][r] = q;
    }
  // every rank must be able to map every peer, else all fall back to the copy exchanges
  int ok = got;
  for (int b = 0; b < kB; ++b)
    for (int r = 0; r < p; ++r) ok &= !bufs[b] || ptr[b][r] != nullptr;
  CUDA_TRY(c, cudaMemcpyAsync(c->bar, &ok, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  NCCL_TRY(c, c->nccl->AllReduce(c->bar, c->bar, 1, ncclInt32, ncclMin, c->comm, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(&ok, c->bar, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (!ok) {
    for (void* q : c->ipc_open) cudaIpcCloseMemHandle(q);
    c->ipc_open.clear();
    c->p2p = false;
    return TFDP_OK;
  }
  fill_route(c, 0, &h[0], ptr[0].data(), ptr[1].data(), ptr[2].data(), ptr[3].data(), ptr[4].data());
  if (c->p.solver == TFDP_IBFFT)
    for (int k = 1; k <= 3; ++k)
      if (k_used(c, k))
        fill_route(c, k, &h[k], ptr[0].data(), ptr[1].data(), ptr[2].data(), ptr[3].data(), ptr[4].data());
  CUDA_TRY(c, cudaMemcpyAsync(c->d_route, h, sizeof h, cudaMemcpyHostToDevice, c->stream));
  c->route_dirty = false;
  return TFDP_OK;
}

// Slab mode with the exchanges fused into the producing kernels (p2p): rows_fwd stores into
// the column owners' receive buffers, cols into the row owners' half spectra, rows_inv its
// potential rows and gather_update the new positions into every rank — no pack / unpack, no
// separate transfers; three phase barriers per evaluation (plus the position barrier).
tfdp_status evaluate_slab_p2p(const Group& G, int update, float eta, int k) {
  bool overlap[tfdp::kMaxWorld];
  for (int i = 0; i < G.p; ++i) {  // phase A: spread of the slab, row FFTs -> peers' xb
    tfdp_ctx* c = G[i];
    const tfdp::SlabPlan& pl = c->plan[k];
    const int r = c->rank;
    fft_prologue(c, k, &overlap[i]);
    float4* grid4 = reinterpret_cast<float4*>(c->grid);
    {
      Scope sc(c, K_SPREAD);
      tfdp::launch_spread(c->xy[c->cur], 0, c->n, c->geom, k, grid4, c->stream,
                          pl.row0[r] / k, pl.row0[r + 1] / k);
    }
    Scope sc(c, K_ROWS_FWD);
    tfdp::launch_rows_fwd(c->geom, grid4, pitch_k(c, k), c->P_of_k[k], pl.row0[r], pl.row0[r + 1],
                          c->tw[k], c->ca, c->ca_pitch, c->stream, c->d_route + k);
  }
  TRY(phase_barrier(G));
  for (int i = 0; i < G.p; ++i) {  // phase B: column pass of the chunk -> row owners' CA
    tfdp_ctx* c = G[i];
    const tfdp::SlabPlan& pl = c->plan[k];
    if (overlap[i]) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    Scope sc(c, K_COLS);
    tfdp::launch_cols(c->geom, c->xb, pl.R, c->kh[k], c->P_of_k[k], c->tw[k], pl.q0[c->rank],
                      pl.q0[c->rank + 1], c->stream, c->d_route + k);
  }
  TRY(phase_barrier(G));
  for (int i = 0; i < G.p; ++i) {  // phase C: inverse rows of the slab -> every rank's Phi
    tfdp_ctx* c = G[i];
    const tfdp::SlabPlan& pl = c->plan[k];
    Scope sc(c, K_ROWS_INV);
    tfdp::launch_rows_inv(c->geom, c->ca, c->ca_pitch, c->P_of_k[k], pl.row0[c->rank],
                          pl.row0[c->rank + 1], c->tw[k], c->phi, pitch_k(c, k),
                          reinterpret_cast<float4*>(c->grid), c->stream, c->d_route + k);
  }
  TRY(phase_barrier(G));
  for (int i = 0; i < G.p; ++i) {  // phase D: own nodes -> every rank's next positions
    tfdp_ctx* c = G[i];
    const tfdp::FocusArgs fo = focus_prologue(c);
    if (overlap[i]) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_join2, 0));
    Scope sc(c, K_GATHER_UPDATE);
    tfdp::launch_gather_update(c->xy[c->cur], c->xy[c->cur ^ 1], c->lo, c->hi - c->lo, c->geom, k,
                               c->phi, c->row_ptr, c->col, c->fa, fo, eta, c->t, update, c->rep,
                               c->att, c->diverge, nullptr, c->stream,
                               update ? c->d_route + k : nullptr, c->cur ^ 1,
                               c->attr_pre ? c->attr : nullptr);
    c->box_valid = false;
    CUDA_TRY(c, cudaGetLastError());
  }
  return TFDP_OK;
}

// ---------------------------------------------------------------- slab mode (p > 1, ibFFT)
// Per iteration, every rank r: box + setup from the full positions; spread of
// the nodes in its grid-row slab; row FFTs of that slab; transpose 1; column pass on its
// column chunk; transpose 2; inverse row FFTs of its slab -> potentials of its slab rows;
// potential exchange; gather + attraction + update of its own node shard; position
// all-gather.  Each phase runs on every rank of the group before the next exchange.
tfdp_status evaluate_slab(const Group& G, int update, float eta, int k) {
  bool overlap[tfdp::kMaxWorld];
  for (int i = 0; i < G.p; ++i) {  // phase A: ... rows_fwd of the slab, pack
    tfdp_ctx* c = G[i];
    const tfdp::SlabPlan& pl = c->plan[k];
    const int P = c->P_of_k[k], r = c->rank;
    fft_prologue(c, k, &overlap[i]);
    float4* grid4 = reinterpret_cast<float4*>(c->grid);
    {
      Scope sc(c, K_SPREAD);
      tfdp::launch_spread(c->xy[c->cur], 0, c->n, c->geom, k, grid4, c->stream,
                          pl.row0[r] / k, pl.row0[r + 1] / k);
    }
    {
      Scope sc(c, K_ROWS_FWD);
      tfdp::launch_rows_fwd(c->geom, grid4, pitch_k(c, k), P, pl.row0[r], pl.row0[r + 1], c->tw[k],
                            c->ca, c->ca_pitch, c->stream);
      tfdp::launch_pack_slab(c->ca, c->ca_pitch, pl, c->xa, c->stream);
      c->launches++;
    }
  }
  TRY(exchange_slabs(G, k, 0));
  for (int i = 0; i < G.p; ++i) {  // phase B: column pass on the chunk (in place in xb)
    tfdp_ctx* c = G[i];
    const tfdp::SlabPlan& pl = c->plan[k];
    if (overlap[i]) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    Scope sc(c, K_COLS);
    tfdp::launch_cols(c->geom, c->xb, pl.R, c->kh[k], c->P_of_k[k], c->tw[k], pl.q0[c->rank],
                      pl.q0[c->rank + 1], c->stream);
  }
  TRY(exchange_slabs(G, k, 1));
  for (int i = 0; i < G.p; ++i) {  // phase C: unpack, inverse rows of the slab -> Phi rows
    tfdp_ctx* c = G[i];
    const tfdp::SlabPlan& pl = c->plan[k];
    const int r = c->rank;
    Scope sc(c, K_ROWS_INV);
    tfdp::launch_unpack_slab(c->xa, pl, c->ca, c->ca_pitch, c->stream);
    c->launches++;
    tfdp::launch_rows_inv(c->geom, c->ca, c->ca_pitch, c->P_of_k[k], pl.row0[r], pl.row0[r + 1],
                          c->tw[k], c->phi, pitch_k(c, k), reinterpret_cast<float4*>(c->grid),
                          c->stream);
  }
  TRY(exchange_phi(G, k));
  for (int i = 0; i < G.p; ++i) {  // phase D: gather + attraction + update of the own nodes
    tfdp_ctx* c = G[i];
    const tfdp::FocusArgs fo = focus_prologue(c);
    if (overlap[i]) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_join2, 0));
    Scope sc(c, K_GATHER_UPDATE);
    tfdp::launch_gather_update(c->xy[c->cur], c->xy[c->cur ^ 1], c->lo, c->hi - c->lo, c->geom, k,
                               c->phi, c->row_ptr, c->col, c->fa, fo, eta, c->t, update, c->rep,
                               c->att, c->diverge, nullptr, c->stream, nullptr, 0,
                               c->attr_pre ? c->attr : nullptr);
    c->box_valid = false;
    CUDA_TRY(c, cudaGetLastError());
  }
  return TFDP_OK;
}

// One evaluation of the whole group (+ the position exchange and buffer flip on update).
tfdp_status evaluate(const Group& G, int update, float eta, int k) {
  tfdp_ctx* c0 = G[0];
  if (c0->p.solver == TFDP_IBFFT && c0->slab) {
    if (!G.virt() && !c0->comm)
      return fail(c0, TFDP_ERR_UNSUPPORTED,
                  "slab mode of a virtual shard context: use tfdp_group_step / tfdp_group_forces");
    // the routes first: a rank that cannot map a peer turns every rank to the copy path
    if (c0->p2p) TRY(setup_routes(G));
    TRY(c0->p2p ? evaluate_slab_p2p(G, update, eta, k) : evaluate_slab(G, update, eta, k));
  } else {
    if (update && c0->p.solver == TFDP_EXACT && c0->p2p && c0->world > 1) {
      if (!G.virt() && !c0->comm)
        return fail(c0, TFDP_ERR_UNSUPPORTED,
                    "virtual shard context (no NCCL id): use tfdp_group_step / tfdp_group_forces");
      TRY(setup_routes(G));
    }
    for (int i = 0; i < G.p; ++i) TRY(evaluate_one(G[i], update, eta, k));
  }
  if (update) {
    TRY(exchange_positions(G, c0->cur ^ 1));
    for (int i = 0; i < G.p; ++i) G[i]->cur ^= 1;
  }
  return TFDP_OK;
}

int k_at(const tfdp_ctx* c, int t) {
  if (c->p.k != 0) return c->p.k;
  const int T = c->p.iterations;
  return c->ksched[std::min(std::max(t, 0), T - 1)];
}

// Reads the divergence word, the grid-cap flag and the last grid geometry (the only host
// sync of a step call).
tfdp_status check_status(tfdp_ctx* c, bool* capped) {
  // p > 1: every rank sees the smallest divergence word of all ranks, so that all of them
  // stop at the same block instead of one blocking in the next exchange
  if (c->world > 1 && c->comm)
    NCCL_TRY(c, c->nccl->AllReduce(c->diverge, c->diverge, 1, ncclUint64, ncclMin, c->comm,
                                   c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->h_status, c->diverge, sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->h_status + 1, c->capped, sizeof(int), cudaMemcpyDeviceToHost,
                              c->stream));
  if (c->p.solver == TFDP_IBFFT)
    CUDA_TRY(c, cudaMemcpyAsync(c->h_status + 2, c->geom, sizeof(GridGeom), cudaMemcpyDeviceToHost,
                                c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  const unsigned long long d = c->h_status[0];
  *capped = (int)(c->h_status[1] & 0xffffffffu) != 0;
  if (d != ~0ULL) {
    c->errored = true;
    unsigned node = (unsigned)(d & 0xffffffffu);
    if (c->reorder) {  // internal slot -> caller's node id
      int orig = -1;
      cudaMemcpy(&orig, c->perm + node, sizeof(int), cudaMemcpyDeviceToHost);
      node = (unsigned)orig;
    }
    return fail(c, TFDP_ERR_DIVERGED, "diverged at iter %u node %u", (unsigned)(d >> 32), node);
  }
  return TFDP_OK;
}

// Internal Morton renumbering of the nodes (kernels_reorder.cu): box -> keys -> counting
// sort -> the new permutation (rank 0; broadcast at p > 1 so that every rank holds the same
// internal order) -> positions, inverse and CSR rebuilt in the new order.  Stream-ordered.
tfdp_status reorder_nodes(const Group& G) {
  for (int i = 0; i < G.p; ++i) {
    tfdp_ctx* c = G[i];
    if (c->rank != 0) continue;
    Scope sc(c, K_REORDER);
    if (!c->box_valid) {  // else the slots already hold the box of the current positions
      tfdp::launch_reset_slots(c->box_part, c->stream);
      tfdp::launch_bbox(c->xy[c->cur], c->n, c->box_part, c->stream);
      c->launches += 2;
    }
    // reduce without consuming: the box is permutation invariant, the next setup reuses it
    tfdp::launch_box_reduce(c->box_part, tfdp::kBoxSlots, c->keys, c->stream, /*reset=*/false);
    c->launches += tfdp::launch_reorder_perm(c->xy[c->cur], c->keys, c->perm, c->perm2, c->n,
                                             c->rscratch, c->stream);
  }
  TRY(exchange_perm(G));
  for (int i = 0; i < G.p; ++i) {
    tfdp_ctx* c = G[i];
    Scope sc(c, K_REORDER, nullptr, 0);
    c->launches += tfdp::launch_reorder_apply(c->xy[c->cur], c->xy[c->cur ^ 1], c->inv, c->perm2,
                                              c->inv2, c->row_ptr_o, c->col_o, c->row_ptr, c->col,
                                              c->n, c->rscratch, c->stream);
    std::swap(c->perm, c->perm2);
    std::swap(c->inv, c->inv2);
    c->cur ^= 1;
    if (c->hv_items) {  // chunk index of the renumbered CSR
      tfdp::launch_heavy_build(c->row_ptr, c->n, c->hv_first, c->hv_scratch, c->stream);
      c->launches += 4;
    }
    if (c->focus_on) {  // the mask follows the renumbering
      tfdp::launch_focus_slots(c->label_caller, c->perm, c->inv, c->n, c->region_caller,
                               c->region_m, c->label_slot, c->region_slot, c->stream);
      c->launches += c->region_m > 0 ? 2 : 1;
    }
    c->box_valid = c->world == 1 && c->rank == 0;
    c->n_part = tfdp::kBoxSlots;
    CUDA_TRY(c, cudaGetLastError());
  }
  return TFDP_OK;
}

// Copies n_rows float2 rows from internal order (src, device) to the caller's order (dst,
// host or device).  Without reordering this is a plain copy.
tfdp_status copy_out(tfdp_ctx* c, const float2* src, float* dst, int64_t n_rows) {
  const bool d = is_device_ptr(dst);
  const float2* from = src;
  if (c->reorder) {
    tfdp::launch_unpermute(src, c->perm, n_rows, c->iobuf, c->stream);
    c->launches++;
    from = c->iobuf;
  }
  CUDA_TRY(c, cudaMemcpyAsync(dst, from, n_rows * sizeof(float2),
                              d ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
  if (!d) CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TFDP_OK;
}

// Box of the current device layout -> configure_fft.  The slots keep the box (no reset), so
// the next setup can consume it without another bbox pass.
tfdp_status replan_from_device(tfdp_ctx* c) {
  tfdp::launch_reset_slots(c->box_part, c->stream);
  c->n_part = tfdp::launch_bbox(c->xy[c->cur], c->n, c->box_part, c->stream);
  tfdp::launch_box_reduce(c->box_part, c->n_part, c->keys, c->stream, /*reset=*/false);
  c->launches += 3;
  BoxKeys hk;
  CUDA_TRY(c, cudaMemcpyAsync(&hk, c->keys, sizeof hk, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  auto k2f = [](unsigned k) {
    unsigned u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    float f;
    memcpy(&f, &u, 4);
    return f;
  };
  const float L = std::max(k2f(hk.maxx) - k2f(hk.minx), k2f(hk.maxy) - k2f(hk.miny));
  c->box_valid = c->world == 1;
  return configure_fft(c, L);
}

// Re-sizes the grid when an iteration ran capped, or when the last N_int came within 4
// intervals of the cap (so the next block of iterations does not run capped).
tfdp_status maybe_replan(tfdp_ctx* c, bool capped) {
  if (c->p.solver != TFDP_IBFFT) return TFDP_OK;
  if (capped) {
    c->warnings |= TFDP_WARN_NINT_CAPPED;
    CUDA_TRY(c, cudaMemsetAsync(c->capped, 0, sizeof(int), c->stream));
  }
  if (c->p.n_int_fixed > 0) return TFDP_OK;
  GridGeom last;
  memcpy(&last, c->h_status + 2, sizeof last);
  int mincap = INT32_MAX;
  for (int k = 1; k <= 3; ++k)
    if (k_used(c, k)) mincap = std::min(mincap, c->cap_of_k[k]);
  if (!capped && last.n_int + 4 <= mincap) return TFDP_OK;
  if (!capped && c->P_of_k[3] >= kMaxFftSize) return TFDP_OK;  // already at the largest grid
  return replan_from_device(c);
}

// ---------------------------------------------------------------- step / forces of a group
// The iteration loop of tfdp_step (one context) and tfdp_group_step (the virtual ranks of
// one process): the ranks advance in lockstep; every rank holds the same t and schedule.
tfdp_status step_impl(const Group& G, int32_t n_iters) {
  tfdp_ctx* c = G[0];
  const int T = c->p.iterations;
  if (c->p.cooling == TFDP_COOL_LINEAR && c->t + n_iters > T)
    return fail(c, TFDP_ERR_STATE, "iteration %d + %d exceeds T = %d under linear cooling",
                c->t, n_iters, T);
  // locality: renumber at the first call, then whenever 64 iterations ran since the last one
  if (c->reorder && n_iters >= 8 && (c->reordered_at < 0 || c->iters_run - c->reordered_at >= 64)) {
    TRY(reorder_nodes(G));
    for (int i = 0; i < G.p; ++i) G[i]->reordered_at = c->iters_run;
  }
  for (int i = 0; i < G.p; ++i) G[i]->iters_run += n_iters;
  int done = 0;
  while (done < n_iters) {
    const int block = std::min(n_iters - done, 32);  // host check every 32 iterations
    for (int b = 0; b < block; ++b) {
      const double eta = c->p.cooling == TFDP_COOL_LINEAR
                             ? c->p.step0 * (1.0 - (double)c->t / T)  // R2
                             : c->p.step0;                            // R2'
      TRY(evaluate(G, 1, (float)eta, k_at(c, c->t)));
      for (int i = 0; i < G.p; ++i) G[i]->t++;
    }
    done += block;
    for (int i = 0; i < G.p; ++i) {
      bool capped = false;
      TRY(check_status(G[i], &capped));
      TRY(maybe_replan(G[i], capped));
    }
  }
  return TFDP_OK;
}

// Forces of every rank's shard to outs[i] (host or device, caller order).  A renumbered
// multi-rank context computes the internal slots [lo, hi); the caller's nodes [lo, hi) are
// spread over all ranks: gather all shards, un-permute, cut the caller range.
tfdp_status shard_out(const Group& G, bool att, float* const* outs) {
  tfdp_ctx* c0 = G[0];
  if (!(c0->reorder && c0->world > 1)) {
    for (int i = 0; i < G.p; ++i)
      if (outs[i]) TRY(copy_out(G[i], att ? G[i]->att : G[i]->rep, outs[i], G[i]->hi - G[i]->lo));
    return TFDP_OK;
  }
  for (int i = 0; i < G.p; ++i)
    if (!G[i]->fbuf) CUDA_TRY(G[i], cudaMalloc(&G[i]->fbuf, G[i]->n * sizeof(float2)));
  if (G.virt()) {
    for (int r = 0; r < G.p; ++r)
      for (int s = 0; s < G.p; ++s)
        TRY(dcopy(G[s], G[s]->fbuf + G[r]->lo, att ? G[r]->att : G[r]->rep,
                  (G[r]->hi - G[r]->lo) * sizeof(float2)));
  } else {
    tfdp_ctx* c = c0;
    TRY(dcopy(c, c->fbuf + c->lo, att ? c->att : c->rep, (c->hi - c->lo) * sizeof(float2)));
    NCCL_TRY(c, c->nccl->GroupStart());
    for (int r = 0; r < c->world; ++r) {
      int64_t lo, hi;
      tfdp_shard_range(c->n, c->world, r, &lo, &hi);
      if (hi > lo)
        NCCL_TRY(c, c->nccl->Broadcast(c->fbuf + lo, c->fbuf + lo, (size_t)(hi - lo) * 2, ncclFloat,
                                       r, c->comm, c->stream));
    }
    NCCL_TRY(c, c->nccl->GroupEnd());
  }
  for (int i = 0; i < G.p; ++i) {
    tfdp_ctx* c = G[i];
    if (!outs[i]) continue;
    tfdp::launch_unpermute(c->fbuf, c->perm, c->n, c->iobuf, c->stream);
    c->launches++;
    const bool d = is_device_ptr(outs[i]);
    CUDA_TRY(c, cudaMemcpyAsync(outs[i], c->iobuf + c->lo, (c->hi - c->lo) * sizeof(float2),
                                d ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
    if (!d) CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  }
  return TFDP_OK;
}

tfdp_status forces_impl(const Group& G, float* const* rep, float* const* att) {
  tfdp_ctx* c = G[0];
  TRY(evaluate(G, 0, 0.f, k_at(c, c->t)));
  for (int i = 0; i < G.p; ++i) G[i]->box_valid = false;  // setup consumed the box keys
  TRY(shard_out(G, false, rep));
  TRY(shard_out(G, true, att));
  for (int i = 0; i < G.p; ++i) {
    bool capped = false;
    TRY(check_status(G[i], &capped));
    TRY(maybe_replan(G[i], capped));
    G[i]->box_valid = false;
  }
  return TFDP_OK;
}

// Validates the virtual ranks of a group call: all contexts of one world, in rank order,
// without a communicator, on one stream, of one problem.
tfdp_status group_check(tfdp_ctx* const* ctxs, int32_t p) {
  if (!ctxs || p < 1 || p > tfdp::kMaxWorld || !ctxs[0])
    return fail(nullptr, TFDP_ERR_ARG, "group: need 1 <= p <= %d contexts", tfdp::kMaxWorld);
  for (int i = 0; i < p; ++i) {
    tfdp_ctx* c = ctxs[i];
    if (!c) return fail(ctxs[0], TFDP_ERR_ARG, "group: context %d is NULL", i);
    if (c->errored) return fail(ctxs[0], TFDP_ERR_STATE, "context %d is errored: %s", i, c->err.c_str());
    if (c->world != p || c->rank != i || c->comm)
      return fail(ctxs[0], TFDP_ERR_ARG, "group: context %d must be virtual rank %d of world %d", i, i, p);
    if (c->stream != ctxs[0]->stream || c->n != ctxs[0]->n || c->p.solver != ctxs[0]->p.solver ||
        c->p.dist_mode != ctxs[0]->p.dist_mode || c->t != ctxs[0]->t)
      return fail(ctxs[0], TFDP_ERR_ARG, "group: contexts must share stream, n, solver, dist_mode, t");
  }
  return TFDP_OK;
}

}  // namespace

// =============================================================================== C ABI
extern "C" {

tfdp_status tfdp_params_default(tfdp_params* p) {
  if (!p) return TFDP_ERR_ARG;
  memset(p, 0, sizeof(*p));
  p->dim = 2;
  p->alpha = 0.1;
  p->beta = 8.0;
  p->gamma = 2.0;
  p->rho = 1.0;
  p->solver = TFDP_EXACT;
  p->k = 0;
  p->n_int_min = 50;
  p->n_int_fixed = 0;
  p->fft_size = 0;
  p->step0 = 0.1;
  p->iterations = 300;
  p->t0 = 0;
  p->cooling = TFDP_COOL_LINEAR;
  p->dist_mode = TFDP_DIST_SLAB;
  p->node_order = TFDP_ORDER_AUTO;
  return TFDP_OK;
}

tfdp_status tfdp_shard_range(int64_t n, int32_t world, int32_t rank, int64_t* lo, int64_t* hi) {
  if (n < 0 || world < 1 || rank < 0 || rank >= world || !lo || !hi) return TFDP_ERR_ARG;
  *lo = (int64_t)((__int128)rank * n / world);
  *hi = (int64_t)((__int128)(rank + 1) * n / world);
  return TFDP_OK;
}

tfdp_status tfdp_csr_build(int64_t n, int64_t m, const int32_t* u, const int32_t* v,
                           int64_t* row_ptr, int32_t* col, int64_t* nnz) {
  if (n < 1 || m < 0 || !row_ptr || !nnz || (m > 0 && (!u || !v || !col)))
    return fail(nullptr, TFDP_ERR_ARG, "tfdp_csr_build: bad arguments");
  for (int64_t e = 0; e < m; ++e)
    if (u[e] < 0 || u[e] >= n || v[e] < 0 || v[e] >= n)
      return fail(nullptr, TFDP_ERR_ARG, "tfdp_csr_build: endpoint out of range at pair %lld",
                  (long long)e);
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t e = 0; e < m; ++e)
    if (u[e] != v[e]) {
      cnt[u[e] + 1]++;
      cnt[v[e] + 1]++;
    }
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  std::vector<int32_t> tmp((size_t)cnt[n]);
  {
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (int64_t e = 0; e < m; ++e)
      if (u[e] != v[e]) {
        tmp[pos[u[e]]++] = v[e];
        tmp[pos[v[e]]++] = u[e];
      }
  }
  std::vector<int64_t> len(n, 0);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i) {
    int32_t* a = tmp.data() + cnt[i];
    int32_t* z = tmp.data() + cnt[i + 1];
    std::sort(a, z);
    len[i] = std::unique(a, z) - a;  // duplicate unordered pairs collapse
  }
  row_ptr[0] = 0;
  for (int64_t i = 0; i < n; ++i) row_ptr[i + 1] = row_ptr[i] + len[i];
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i)
    memcpy(col + row_ptr[i], tmp.data() + cnt[i], (size_t)len[i] * sizeof(int32_t));
  *nnz = row_ptr[n];
  return TFDP_OK;
}

tfdp_status tfdp_init(tfdp_ctx** out, int64_t n, const int64_t* row_ptr, const int32_t* col,
                      const float* xy0, const tfdp_params* pin, const tfdp_dist* dist,
                      void* stream) {
  if (!out) return fail(nullptr, TFDP_ERR_ARG, "ctx out-pointer is NULL");
  *out = nullptr;
  if (n < 1 || n > (int64_t)INT32_MAX || !row_ptr || !xy0)
    return fail(nullptr, TFDP_ERR_ARG, "need 1 <= n <= 2^31-1, row_ptr and xy0");
  tfdp_params p;
  if (pin) p = *pin;
  else tfdp_params_default(&p);
  uint32_t warn = 0;
  std::string msg;
  tfdp_status st = validate_params(&p, &warn, &msg);
  if (st != TFDP_OK) return fail(nullptr, st, "%s", msg.c_str());
  const int64_t nnz = row_ptr[n];
  if (nnz > 0 && !col) return fail(nullptr, TFDP_ERR_ARG, "col is NULL");
  if (!validate_csr(n, row_ptr, col, &msg)) return fail(nullptr, TFDP_ERR_ARG, "%s", msg.c_str());

  tfdp_ctx* c = new tfdp_ctx();
  c->n = n;
  c->p = p;
  c->warnings = warn;
  c->nnz = nnz;
  c->t = p.t0;
  c->ksched = k_schedule(p.iterations);
  c->fa.alpha = (float)p.alpha;
  c->fa.beta = (float)p.beta;
  c->fa.gamma = (float)p.gamma;
  c->fa.rho = (float)p.rho;
  c->fa.gamma_int = gamma_int_of(p.gamma);
  if (dist) {
    if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world) {
      delete c;
      return fail(nullptr, TFDP_ERR_ARG, "bad dist rank/world");
    }
    c->rank = dist->rank;
    c->world = dist->world;
    c->device = dist->device;
  } else {
    cudaGetDevice(&c->device);
  }
  auto bail = [&](tfdp_status s) {
    g_noctx_err = c->err;
    tfdp_destroy(c);
    return s;
  };
  if (cudaSetDevice(c->device) != cudaSuccess)
    return bail(fail(c, TFDP_ERR_CUDA, "cudaSetDevice(%d) failed (no GPU?)", c->device));
  tfdp_shard_range(n, c->world, c->rank, &c->lo, &c->hi);
  if (stream) {
    c->stream = (cudaStream_t)stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
      return bail(fail(c, TFDP_ERR_CUDA, "cudaStreamCreate failed"));
    c->own_stream = true;
  }
  if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join2, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork2, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(c, TFDP_ERR_CUDA, "side stream / events"));
  if (const char* e = getenv("TFDP_KSPEC_OVERLAP")) c->kspec_overlap = atoi(e) != 0;
  if (const char* e = getenv("TFDP_ATTR_AT")) c->attr_at = std::max(0, std::min(2, atoi(e)));
  if (const char* e = getenv("TFDP_ATTR_BLOCKS")) c->attr_blocks = std::max(0, atoi(e));
  const bool xy_dev = is_device_ptr(xy0);
  float L0 = 1.f;
  if (!xy_dev) {
    for (int64_t i = 0; i < 2 * n; ++i)
      if (!std::isfinite(xy0[i]))
        return bail(fail(c, TFDP_ERR_ARG, "xy0 non-finite at node %lld", (long long)(i / 2)));
    host_box(xy0, n, &L0);
  }
  const int64_t n_local = c->hi - c->lo;
#define ALLOC(ptr, bytes)                                                           \
  if (cudaMalloc((void**)&(ptr), (bytes)) != cudaSuccess) {                         \
    cudaGetLastError();                                                             \
    return bail(fail(c, TFDP_ERR_OOM, "cudaMalloc(%zu) failed", (size_t)(bytes)));  \
  }
  ALLOC(c->xy[0], n * sizeof(float2));
  ALLOC(c->xy[1], n * sizeof(float2));
  ALLOC(c->row_ptr, (n + 1) * sizeof(int64_t));
  ALLOC(c->col, std::max<int64_t>(nnz, 1) * sizeof(int32_t));
  ALLOC(c->rep, std::max<int64_t>(n_local, 1) * sizeof(float2));
  if (const char* e = getenv("TFDP_ATTR_SIDE")) c->attr_side = e[0] != '0';
  if (p.solver == TFDP_IBFFT && c->attr_side)
    ALLOC(c->attr, std::max<int64_t>(n_local, 1) * sizeof(float2));
  ALLOC(c->att, std::max<int64_t>(n_local, 1) * sizeof(float2));
  ALLOC(c->diverge, sizeof(unsigned long long));
  ALLOC(c->capped, sizeof(int));
  ALLOC(c->keys, sizeof(BoxKeys));
  ALLOC(c->box_part, tfdp::kBoxSlots * sizeof(BoxKeys));
  ALLOC(c->geom, sizeof(GridGeom));
  ALLOC(c->kkey, 4 * sizeof(tfdp::KspecKey));
  ALLOC(c->d_route, 4 * sizeof(tfdp::PeerRoute));
  ALLOC(c->bar, sizeof(int));
  if (cudaMemsetAsync(c->kkey, 0, 4 * sizeof(tfdp::KspecKey), c->stream ? c->stream : 0) != cudaSuccess)
    return bail(fail(c, TFDP_ERR_CUDA, "kkey memset"));
  if (cudaMallocHost((void**)&c->h_status, 2 * sizeof(unsigned long long) + sizeof(GridGeom)) !=
      cudaSuccess)
    return bail(fail(c, TFDP_ERR_OOM, "cudaMallocHost failed"));
  if (p.solver == TFDP_EXACT) {
    // source chunks depend on n only (bitwise-identical results for any shard count, R15)
    int64_t ch = std::max<int64_t>(1024, (n + 31) / 32);
    ch = (ch + tfdp::kExactTile - 1) / tfdp::kExactTile * tfdp::kExactTile;
    c->chunk = ch;
    c->n_chunks = (int)((n + ch - 1) / ch);
    ALLOC(c->part, (size_t)c->n_chunks * std::max<int64_t>(n_local, 1) * sizeof(double2));
  }
  c->slab = c->world > 1 && p.solver == TFDP_IBFFT && p.dist_mode == TFDP_DIST_SLAB;
  if (c->slab && c->world > tfdp::kMaxWorld)
    return bail(fail(c, TFDP_ERR_ARG, "slab mode supports world <= %d", tfdp::kMaxWorld));
  if (c->slab || (c->world > 1 && p.solver == TFDP_EXACT)) {
    // fused exchanges (peer stores) unless TFDP_P2P=0 (the NCCL / copy path)
    const char* e = getenv("TFDP_P2P");
    c->p2p = !(e && e[0] == '0');
  }
  // internal renumbering: one GPU, or the slab mode (every rank renumbers identically: rank
  // 0's permutation is broadcast)
  c->reorder = p.solver == TFDP_IBFFT && p.node_order == TFDP_ORDER_AUTO && n >= 65536 &&
               (c->world == 1 || c->slab);
  if (c->reorder) {
    ALLOC(c->perm, n * sizeof(int));
    ALLOC(c->inv, n * sizeof(int));
    ALLOC(c->perm2, n * sizeof(int));
    ALLOC(c->inv2, n * sizeof(int));
    ALLOC(c->row_ptr_o, (n + 1) * sizeof(int64_t));
    ALLOC(c->col_o, std::max<int64_t>(nnz, 1) * sizeof(int32_t));
    ALLOC(c->rscratch, tfdp::reorder_scratch_bytes(n));
    ALLOC(c->iobuf, n * sizeof(float2));
    tfdp::launch_iota(c->perm, c->inv, n, c->stream);
    c->launches++;
  }
#undef ALLOC
  cudaStream_t s = c->stream;
  if (cudaMemcpyAsync(c->xy[0], xy0, n * sizeof(float2),
                      xy_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(c->row_ptr, row_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s) !=
          cudaSuccess ||
      (nnz > 0 && cudaMemcpyAsync(c->col, col, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s) !=
                      cudaSuccess) ||
      cudaMemsetAsync(c->diverge, 0xff, sizeof(unsigned long long), s) != cudaSuccess ||
      cudaMemsetAsync(c->capped, 0, sizeof(int), s) != cudaSuccess)
    return bail(fail(c, TFDP_ERR_CUDA, "initial copies failed: %s", cudaGetErrorString(cudaGetLastError())));
  if (c->reorder &&
      (cudaMemcpyAsync(c->row_ptr_o, c->row_ptr, (n + 1) * sizeof(int64_t),
                       cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
       (nnz > 0 && cudaMemcpyAsync(c->col_o, c->col, nnz * sizeof(int32_t),
                                   cudaMemcpyDeviceToDevice, s) != cudaSuccess)))
    return bail(fail(c, TFDP_ERR_CUDA, "CSR copy failed"));
#define ALLOC2(ptr, bytes)                                                          \
  if (cudaMalloc((void**)&(ptr), (bytes)) != cudaSuccess) {                         \
    cudaGetLastError();                                                             \
    return bail(fail(c, TFDP_ERR_OOM, "cudaMalloc(%zu) failed", (size_t)(bytes)));  \
  }
  {  // heavy rows: chunk count from the host CSR (permutation invariant)
    int64_t items = 0;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t d = row_ptr[i + 1] - row_ptr[i];
      if (d > tfdp::kHeavyDeg) items += (d + tfdp::kHeavyChunk - 1) / tfdp::kHeavyChunk;
    }
    if (const char* e = getenv("TFDP_HEAVY"))  // TFDP_HEAVY=0: one thread per row (A/B runs)
      if (e[0] == '0') items = 0;
    if (items > 0) {
      ALLOC2(c->hv_first, (n + 1) * sizeof(long long));
      ALLOC2(c->hv_part, items * sizeof(float2));
      ALLOC2(c->hv_scratch, tfdp::heavy_scratch_bytes(n));
      c->hv_items = items;
      tfdp::launch_heavy_build(c->row_ptr, n, c->hv_first, c->hv_scratch, s);
      c->launches += 4;
      c->fa.hv_first = c->hv_first;
      c->fa.hv_part = c->hv_part;
    }
  }
#undef ALLOC2
  tfdp::launch_reset_slots(c->box_part, s);
  if (p.solver == TFDP_IBFFT) {
    if (xy_dev) {  // box of a device layout: one bbox pass
      c->n_part = tfdp::launch_bbox(c->xy[0], n, c->box_part, s);
      tfdp::launch_box_reduce(c->box_part, c->n_part, c->keys, s);
      BoxKeys hk;
      cudaMemcpyAsync(&hk, c->keys, sizeof hk, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      auto k2f = [](unsigned k) {
        unsigned u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
        float f;
        memcpy(&f, &u, 4);
        return f;
      };
      L0 = std::max(k2f(hk.maxx) - k2f(hk.minx), k2f(hk.maxy) - k2f(hk.miny));
    }
    st = configure_fft(c, L0);
    if (st != TFDP_OK) return bail(st);
  }
  if (c->world > 1 && dist->nccl_uid) {
    const char* e = nullptr;
    c->nccl = tfdp::nccl_api(&e);
    if (!c->nccl) return bail(fail(c, TFDP_ERR_NCCL, "%s", e));
  }
  if (c->world > 1 && dist->nccl_uid) {
    ncclUniqueId uid;
    memcpy(&uid, dist->nccl_uid, sizeof uid);
    ncclResult_t r = c->nccl->CommInitRank(&c->comm, c->world, uid, c->rank);
    if (r != ncclSuccess)
      return bail(fail(c, TFDP_ERR_NCCL, "ncclCommInitRank: %s", c->nccl->GetErrorString(r)));
  }
  if (cudaStreamSynchronize(s) != cudaSuccess)
    return bail(fail(c, TFDP_ERR_CUDA, "init sync: %s", cudaGetErrorString(cudaGetLastError())));
  *out = c;
  return TFDP_OK;
}

tfdp_status tfdp_step(tfdp_ctx* c, int32_t n_iters) {
  if (!c) return fail(nullptr, TFDP_ERR_ARG, "ctx is NULL");
  if (c->errored) return fail(c, TFDP_ERR_STATE, "context is errored: %s", c->err.c_str());
  if (n_iters < 0) return fail(c, TFDP_ERR_ARG, "n_iters < 0");
  cudaSetDevice(c->device);
  tfdp_ctx* one[1] = {c};
  return step_impl(Group{one, 1}, n_iters);
}

tfdp_status tfdp_forces(tfdp_ctx* c, float* rep_xy, float* att_xy) {
  if (!c) return fail(nullptr, TFDP_ERR_ARG, "ctx is NULL");
  if (c->errored) return fail(c, TFDP_ERR_STATE, "context is errored: %s", c->err.c_str());
  cudaSetDevice(c->device);
  tfdp_ctx* one[1] = {c};
  float* r[1] = {rep_xy};
  float* a[1] = {att_xy};
  return forces_impl(Group{one, 1}, r, a);
}

tfdp_status tfdp_group_step(tfdp_ctx* const* ctxs, int32_t p, int32_t n_iters) {
  TRY(group_check(ctxs, p));
  if (n_iters < 0) return fail(ctxs[0], TFDP_ERR_ARG, "n_iters < 0");
  cudaSetDevice(ctxs[0]->device);
  return step_impl(Group{const_cast<tfdp_ctx**>(ctxs), p}, n_iters);
}

tfdp_status tfdp_group_forces(tfdp_ctx* const* ctxs, int32_t p, float* const* rep_xy,
                              float* const* att_xy) {
  TRY(group_check(ctxs, p));
  cudaSetDevice(ctxs[0]->device);
  std::vector<float*> r(p, nullptr), a(p, nullptr);
  for (int i = 0; i < p; ++i) {
    if (rep_xy) r[i] = rep_xy[i];
    if (att_xy) a[i] = att_xy[i];
  }
  return forces_impl(Group{const_cast<tfdp_ctx**>(ctxs), p}, r.data(), a.data());
}

tfdp_status tfdp_slab_plan(int32_t rows, int32_t fft_size, int32_t world, int32_t* row0,
                           int32_t* q0) {
  if (rows < 1 || fft_size < 2 || fft_size % 2 || world < 1 || world > tfdp::kMaxWorld || !row0 || !q0)
    return fail(nullptr, TFDP_ERR_ARG, "tfdp_slab_plan: bad arguments");
  tfdp::SlabPlan pl;
  tfdp::slab_plan(world, 0, rows, fft_size, &pl);
  for (int r = 0; r <= world; ++r) {
    row0[r] = pl.row0[r];
    q0[r] = pl.q0[r];
  }
  return TFDP_OK;
}

tfdp_status tfdp_layout(tfdp_ctx* c, float* xy_out) {
  if (!c || !xy_out) return fail(c, TFDP_ERR_ARG, "NULL argument");
  cudaSetDevice(c->device);
  return copy_out(c, c->xy[c->cur], xy_out, c->n);
}

tfdp_status tfdp_set_layout(tfdp_ctx* c, const float* xy) {
  if (!c || !xy) return fail(c, TFDP_ERR_ARG, "NULL argument");
  cudaSetDevice(c->device);
  const bool d = is_device_ptr(xy);
  if (!d) {
    // the H2D copy goes to a staging buffer first, so the argument check of the host buffer
    // (all cores: first non-finite node) runs while the DMA is in flight; a failed
    // check leaves the layout untouched
    if (!c->iobuf) CUDA_TRY(c, cudaMalloc(&c->iobuf, c->n * sizeof(float2)));
    CUDA_TRY(c, cudaMemcpyAsync(c->iobuf, xy, c->n * sizeof(float2), cudaMemcpyHostToDevice,
                                c->stream));
    const int64_t m = 2 * c->n;
    int64_t first = m;
#pragma omp parallel for schedule(static) reduction(min : first)
    for (int64_t i = 0; i < m; ++i)
      if (!std::isfinite(xy[i]) && i < first) first = i;
    if (first < m) {
      cudaStreamSynchronize(c->stream);  // the caller may free xy on return
      return fail(c, TFDP_ERR_ARG, "layout non-finite at node %lld", (long long)(first / 2));
    }
    if (c->reorder) {  // caller order -> internal order
      tfdp::launch_permute(c->iobuf, c->perm, c->n, c->xy[c->cur], c->stream);
      c->launches++;
    } else {
      CUDA_TRY(c, cudaMemcpyAsync(c->xy[c->cur], c->iobuf, c->n * sizeof(float2),
                                  cudaMemcpyDeviceToDevice, c->stream));
    }
  } else {
    float2* dst = c->reorder ? c->iobuf : c->xy[c->cur];
    CUDA_TRY(c, cudaMemcpyAsync(dst, xy, c->n * sizeof(float2), cudaMemcpyDeviceToDevice,
                                c->stream));
    if (c->reorder) {  // caller order -> internal order
      tfdp::launch_permute(c->iobuf, c->perm, c->n, c->xy[c->cur], c->stream);
      c->launches++;
    }
  }
  c->box_valid = false;
  // a new layout may need a larger grid: re-plan now (one bbox + a host sync) rather than
  // run up to 32 iterations below the N_int rule (R5) before the in-step check
  if (c->p.solver == TFDP_IBFFT && c->p.n_int_fixed == 0) return replan_from_device(c);
  if (!d) CUDA_TRY(c, cudaStreamSynchronize(c->stream));  // the host buffer is free on return
  return TFDP_OK;
}

tfdp_status tfdp_set_iteration(tfdp_ctx* c, int32_t t) {
  if (!c || t < 0) return fail(c, TFDP_ERR_ARG, "bad iteration");
  c->t = t;
  return TFDP_OK;
}

int32_t tfdp_iteration(const tfdp_ctx* c) { return c ? c->t : -1; }

tfdp_status tfdp_set_params(tfdp_ctx* c, const tfdp_params* p) {
  if (!c || !p) return fail(c, TFDP_ERR_ARG, "NULL argument");
  if (c->errored) return fail(c, TFDP_ERR_STATE, "context is errored: %s", c->err.c_str());
  uint32_t warn = 0;
  std::string msg;
  tfdp_status st = validate_params(p, &warn, &msg);
  if (st != TFDP_OK) return fail(c, st, "%s", msg.c_str());
  if (p->solver != c->p.solver || p->dist_mode != c->p.dist_mode || p->node_order != c->p.node_order)
    return fail(c, TFDP_ERR_ARG, "solver, dist_mode and node_order are fixed at tfdp_init");
  cudaSetDevice(c->device);
  const bool replan = p->solver == TFDP_IBFFT &&
                      (p->k != c->p.k || p->n_int_min != c->p.n_int_min ||
                       p->n_int_fixed != c->p.n_int_fixed || p->fft_size != c->p.fft_size);
  const tfdp_params old = c->p;
  c->p = *p;
  if (replan) {
    tfdp_status r = replan_from_device(c);
    if (r != TFDP_OK) {  // keep the context usable with its previous plan
      c->p = old;
      const std::string m = c->err;
      replan_from_device(c);
      return fail(c, r, "%s", m.c_str());
    }
  }
  c->warnings = (c->warnings & TFDP_WARN_NINT_CAPPED) | warn;
  c->t = p->t0;
  c->ksched = k_schedule(p->iterations);
  c->fa.alpha = (float)p->alpha;
  c->fa.beta = (float)p->beta;
  c->fa.gamma = (float)p->gamma;
  c->fa.rho = (float)p->rho;
  c->fa.gamma_int = gamma_int_of(p->gamma);
  return TFDP_OK;
}

tfdp_status tfdp_np1(tfdp_ctx* c, double* np1, int32_t* hits) {
  if (!c) return fail(nullptr, TFDP_ERR_ARG, "ctx is NULL");
  if (c->errored) return fail(c, TFDP_ERR_STATE, "context is errored: %s", c->err.c_str());
  cudaSetDevice(c->device);
  const int64_t n_local = c->hi - c->lo;
  if (!c->np_scratch) {
    CUDA_TRY(c, cudaMalloc(&c->np_scratch, tfdp::np_scratch_bytes(c->n, n_local)));
    CUDA_TRY(c, cudaMalloc(&c->np_hits, std::max<int64_t>(n_local, 1) * sizeof(int)));
    if (c->reorder) CUDA_TRY(c, cudaMalloc(&c->np_hits2, c->n * sizeof(int)));
    CUDA_TRY(c, cudaMalloc(&c->np_slots, tfdp::kBoxSlots * sizeof(BoxKeys)));
    CUDA_TRY(c, cudaMalloc(&c->np_keys, sizeof(BoxKeys)));
    CUDA_TRY(c, cudaMalloc(&c->np_sum, sizeof(double)));
  }
  if (hits && c->reorder && c->world > 1 && !c->comm)
    return fail(c, TFDP_ERR_UNSUPPORTED, "per-node hits of a renumbered virtual rank");
  const float2* xy = c->xy[c->cur];
  tfdp::launch_reset_slots(c->np_slots, c->stream);
  const int np = tfdp::launch_bbox(xy, c->n, c->np_slots, c->stream);
  tfdp::launch_box_reduce(c->np_slots, np, c->np_keys, c->stream);
  c->launches += 3;
  c->launches += tfdp::launch_np1(xy, c->n, c->lo, n_local, c->row_ptr, c->col,
                                  c->reorder ? c->perm : nullptr, c->np_keys, c->np_scratch,
                                  c->np_hits, c->np_sum, c->stream);
  if (c->world > 1 && c->comm)
    NCCL_TRY(c, c->nccl->AllReduce(c->np_sum, c->np_sum, 1, ncclDouble, ncclSum, c->comm,
                                   c->stream));
  CUDA_TRY(c, cudaGetLastError());
  if (hits) {
    const int* src = c->np_hits;
    if (c->reorder && c->world > 1) {
      // the shard's internal slots hold caller nodes spread over all ranks: gather every
      // rank's hits (internal order), un-permute, cut the caller range [lo, hi)
      int* full = reinterpret_cast<int*>(c->iobuf);  // n float2 >= n ints
      CUDA_TRY(c, cudaMemcpyAsync(full + c->lo, c->np_hits, n_local * sizeof(int),
                                  cudaMemcpyDeviceToDevice, c->stream));
      NCCL_TRY(c, c->nccl->GroupStart());
      for (int r = 0; r < c->world; ++r) {
        int64_t lo, hi;
        tfdp_shard_range(c->n, c->world, r, &lo, &hi);
        if (hi > lo)
          NCCL_TRY(c, c->nccl->Broadcast(full + lo, full + lo, (size_t)(hi - lo), ncclInt32, r,
                                         c->comm, c->stream));
      }
      NCCL_TRY(c, c->nccl->GroupEnd());
      tfdp::launch_unpermute_int(full, c->perm, c->n, c->np_hits2, c->stream);
      c->launches++;
      src = c->np_hits2 + c->lo;
    } else if (c->reorder) {  // internal slot -> caller order
      tfdp::launch_unpermute_int(c->np_hits, c->perm, c->n, c->np_hits2, c->stream);
      c->launches++;
      src = c->np_hits2;
    }
    const bool d = is_device_ptr(hits);
    CUDA_TRY(c, cudaMemcpyAsync(hits, src, n_local * sizeof(int),
                                d ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
  }
  if (np1) CUDA_TRY(c, cudaMemcpyAsync(np1, c->np_sum, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TFDP_OK;
}

tfdp_status tfdp_set_focus(tfdp_ctx* c, const int32_t* focal, int64_t n_focal, double la,
                           double lf, double ls) {
  if (!c) return fail(nullptr, TFDP_ERR_ARG, "ctx is NULL");
  if (c->errored) return fail(c, TFDP_ERR_STATE, "context is errored: %s", c->err.c_str());
  if (n_focal < 0 || (n_focal > 0 && !focal)) return fail(c, TFDP_ERR_ARG, "bad focal list");
  if (n_focal == 0) {
    c->focus_on = false;
    return TFDP_OK;
  }
  if (!std::isfinite(la) || !std::isfinite(lf) || !std::isfinite(ls) || la < 1.0 || lf < 1.0 ||
      ls < 1.0)
    return fail(c, TFDP_ERR_ARG, "boosts must be finite and >= 1 (S:156), got %g %g %g", la, lf, ls);
  if (n_focal > c->n) return fail(c, TFDP_ERR_ARG, "more focal nodes than nodes");
  for (int64_t i = 0; i < n_focal; ++i)
    if (focal[i] < 0 || focal[i] >= c->n)
      return fail(c, TFDP_ERR_ARG, "focal node %lld out of range", (long long)focal[i]);
  cudaSetDevice(c->device);
  const int64_t n_local = c->hi - c->lo;
  if (!c->label_caller) {
    CUDA_TRY(c, cudaMalloc(&c->label_caller, c->n));
    CUDA_TRY(c, cudaMalloc(&c->label_slot, c->n));
    CUDA_TRY(c, cudaMalloc(&c->s1, std::max<int64_t>(n_local, 1) * sizeof(float2)));
  }
  int* dfocal = nullptr;
  CUDA_TRY(c, cudaMalloc(&dfocal, n_focal * sizeof(int)));
  cudaMemcpyAsync(dfocal, focal, n_focal * sizeof(int), cudaMemcpyHostToDevice, c->stream);
  cudaMemsetAsync(c->label_caller, 0, c->n, c->stream);
  const int64_t* rp = c->reorder ? c->row_ptr_o : c->row_ptr;  // caller-order CSR
  const int32_t* cl = c->reorder ? c->col_o : c->col;
  tfdp::launch_mark_focus(dfocal, (int)n_focal, rp, cl, c->label_caller, c->stream);
  std::vector<unsigned char> lab(c->n);
  cudaMemcpyAsync(lab.data(), c->label_caller, c->n, cudaMemcpyDeviceToHost, c->stream);
  const cudaError_t e = cudaStreamSynchronize(c->stream);
  cudaFree(dfocal);
  CUDA_TRY(c, e);
  std::vector<int> region;  // caller ids of F u N(F), ascending (fixed source order of S1)
  for (int64_t i = 0; i < c->n; ++i)
    if (lab[i]) region.push_back((int)i);
  if ((int)region.size() > c->region_cap) {
    cudaFree(c->region_caller);
    cudaFree(c->region_slot);
    c->region_caller = c->region_slot = nullptr;
    CUDA_TRY(c, cudaMalloc(&c->region_caller, region.size() * sizeof(int)));
    CUDA_TRY(c, cudaMalloc(&c->region_slot, region.size() * sizeof(int)));
    c->region_cap = (int)region.size();
  }
  c->region_m = (int)region.size();
  CUDA_TRY(c, cudaMemcpyAsync(c->region_caller, region.data(), region.size() * sizeof(int),
                              cudaMemcpyHostToDevice, c->stream));
  tfdp::launch_focus_slots(c->label_caller, c->reorder ? c->perm : nullptr,
                           c->reorder ? c->inv : nullptr, c->n, c->region_caller, c->region_m,
                           c->label_slot, c->region_slot, c->stream);
  c->launches += 3;
  CUDA_TRY(c, cudaGetLastError());
  c->fo_la = (float)la;
  c->fo_lf = (float)lf;
  c->fo_ls = (float)ls;
  // the identity mask changes nothing: run the unmasked kernels, bit for bit
  c->focus_on = !(la == 1.0 && lf == 1.0 && ls == 1.0);
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TFDP_OK;
}

tfdp_status tfdp_local_refine(tfdp_ctx* c, const int32_t* focal, int64_t n_focal, double la,
                              double lf, double ls, int32_t iterations) {
  if (!c) return fail(nullptr, TFDP_ERR_ARG, "ctx is NULL");
  if (n_focal < 1) return fail(c, TFDP_ERR_ARG, "empty focal set (S:372)");
  if (iterations < 1) return fail(c, TFDP_ERR_ARG, "iterations must be >= 1");
  TRY(tfdp_set_focus(c, focal, n_focal, la, lf, ls));
  tfdp_params p = c->p;
  p.iterations = iterations;
  p.t0 = 0;
  TRY(tfdp_set_params(c, &p));
  return tfdp_step(c, iterations);
}

tfdp_status tfdp_pivot_mds(tfdp_ctx* c, int32_t n_pivots, uint64_t seed, int32_t* pivots) {
  if (!c) return fail(nullptr, TFDP_ERR_ARG, "ctx is NULL");
  if (c->errored) return fail(c, TFDP_ERR_STATE, "context is errored: %s", c->err.c_str());
  if (n_pivots < 1 || n_pivots > tfdp::pmds_max_pivots())
    return fail(c, TFDP_ERR_ARG, "pivot count must be in 1..%d (S:117)", tfdp::pmds_max_pivots());
  cudaSetDevice(c->device);
  const int p = (int)std::min<int64_t>(n_pivots, c->n);
  // splitmix64(seed): the first pivot (the counter-based generator the oracle implements too)
  uint64_t z = seed + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  void* scratch = nullptr;
  CUDA_TRY(c, cudaMalloc(&scratch, tfdp::pmds_scratch_bytes(c->n, p)));
  std::vector<int> piv(p);
  const int64_t* rp = c->reorder ? c->row_ptr_o : c->row_ptr;  // caller order
  const int32_t* cl = c->reorder ? c->col_o : c->col;
  float2* out = c->reorder ? c->iobuf : c->xy[c->cur];
  const char* stage = "";
  const cudaError_t e = tfdp::launch_pmds(rp, cl, c->n, c->nnz, p, z, scratch, out, piv.data(),
                                          &c->launches, &stage, c->stream);
  if (e == cudaSuccess && c->reorder) {  // caller order -> internal order
    tfdp::launch_permute(c->iobuf, c->perm, c->n, c->xy[c->cur], c->stream);
    c->launches++;
  }
  const cudaError_t e2 = cudaStreamSynchronize(c->stream);
  cudaFree(scratch);
  if (e != cudaSuccess || e2 != cudaSuccess)
    return fail(c, TFDP_ERR_CUDA, "pivot_mds (%s): %s", stage,
                cudaGetErrorString(e != cudaSuccess ? e : e2));
  c->box_valid = false;
  if (pivots)
    for (int j = 0; j < p; ++j) pivots[j] = piv[j];
  if (c->p.solver == TFDP_IBFFT && c->p.n_int_fixed == 0) return replan_from_device(c);  // as set_layout
  return TFDP_OK;
}

tfdp_status tfdp_global_refine(tfdp_ctx* c, double gamma, double rho, int32_t iterations) {
  if (!c) return fail(nullptr, TFDP_ERR_ARG, "ctx is NULL");
  if (!std::isfinite(gamma) || gamma <= 1.0)
    return fail(c, TFDP_ERR_ARG, "global refinement needs gamma > 1 (S:362), got %g", gamma);
  if (!std::isfinite(rho) || rho <= 0.0)
    return fail(c, TFDP_ERR_ARG, "global refinement needs rho > 0, got %g", rho);
  if (iterations < 1) return fail(c, TFDP_ERR_ARG, "iterations must be >= 1");
  tfdp_params p = c->p;
  p.gamma = gamma;
  p.rho = rho;
  p.iterations = iterations;
  p.t0 = 0;
  TRY(tfdp_set_params(c, &p));
  return tfdp_step(c, iterations);
}

tfdp_status tfdp_shard(const tfdp_ctx* c, int64_t* lo, int64_t* hi) {
  if (!c || !lo || !hi) return TFDP_ERR_ARG;
  *lo = c->lo;
  *hi = c->hi;
  return TFDP_OK;
}

tfdp_status tfdp_fft_geometry(tfdp_ctx* c, float* box4, int32_t* n_int, int32_t* k,
                              int32_t* fft_size) {
  if (!c) return TFDP_ERR_ARG;
  if (c->p.solver != TFDP_IBFFT) return fail(c, TFDP_ERR_STATE, "not an ibFFT context");
  GridGeom g;
  CUDA_TRY(c, cudaMemcpyAsync(&g, c->geom, sizeof g, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (box4) {
    box4[0] = g.lo_x;
    box4[1] = g.lo_y;
    box4[2] = g.L;
    box4[3] = g.w;
  }
  if (n_int) *n_int = g.n_int;
  if (k) *k = g.k;
  if (fft_size) *fft_size = g.P;
  return TFDP_OK;
}

tfdp_status tfdp_fft_plan(const tfdp_ctx* c, int32_t k, int32_t* fft_size, int32_t* n_int_cap) {
  if (!c || k < 1 || k > 3) return TFDP_ERR_ARG;
  if (c->p.solver != TFDP_IBFFT) return TFDP_ERR_STATE;
  if (fft_size) *fft_size = c->P_of_k[k];
  if (n_int_cap) *n_int_cap = c->cap_of_k[k];
  return TFDP_OK;
}

tfdp_status tfdp_profile(tfdp_ctx* c, int32_t enable) {
  return tfdp_profile_mask(c, enable ? 0xffffffffu : 0u);
}

tfdp_status tfdp_profile_mask(tfdp_ctx* c, uint32_t kinds) {
  if (!c) return TFDP_ERR_ARG;
  prof_collect(c);
  for (int i = 0; i < K_COUNT; ++i) {
    c->prof_ms[i] = 0;
    c->prof_n[i] = 0;
  }
  c->prof_mask = kinds;
  return TFDP_OK;
}

tfdp_status tfdp_profile_select(tfdp_ctx* c, uint32_t kinds) {
  if (!c) return TFDP_ERR_ARG;
  c->prof_mask = kinds;
  return TFDP_OK;
}

int32_t tfdp_profile_read(tfdp_ctx* c, const char** names, double* ms, int64_t* launches,
                          int32_t cap) {
  if (!c) return -1;
  prof_collect(c);
  for (int i = 0; i < K_COUNT && i < cap; ++i) {
    if (names) names[i] = kKindNames[i];
    if (ms) ms[i] = c->prof_ms[i];
    if (launches) launches[i] = c->prof_n[i];
  }
  return K_COUNT;
}

int64_t tfdp_launch_count(const tfdp_ctx* c) { return c ? c->launches : -1; }

uint32_t tfdp_warnings(const tfdp_ctx* c) { return c ? c->warnings : 0u; }

const char* tfdp_last_error(const tfdp_ctx* c) {
  return c ? c->err.c_str() : g_noctx_err.c_str();
}

const char* tfdp_status_string(tfdp_status s) {
  switch (s) {
    case TFDP_OK: return "TFDP_OK";
    case TFDP_ERR_ARG: return "TFDP_ERR_ARG";
    case TFDP_ERR_CUDA: return "TFDP_ERR_CUDA";
    case TFDP_ERR_OOM: return "TFDP_ERR_OOM";
    case TFDP_ERR_DIVERGED: return "TFDP_ERR_DIVERGED";
    case TFDP_ERR_STATE: return "TFDP_ERR_STATE";
    case TFDP_ERR_NCCL: return "TFDP_ERR_NCCL";
    case TFDP_ERR_UNSUPPORTED: return "TFDP_ERR_UNSUPPORTED";
  }
  return "TFDP_ERR_UNKNOWN";
}

void tfdp_destroy(tfdp_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& q : c->pend) {
    cudaEventDestroy(q.a);
    cudaEventDestroy(q.b);
  }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  free_fft_buffers(c);
  cudaFree(c->xy[0]);
  cudaFree(c->xy[1]);
  cudaFree(c->row_ptr);
  cudaFree(c->col);
  cudaFree(c->part);
  cudaFree(c->rep);
  cudaFree(c->att);
  cudaFree(c->attr);
  cudaFree(c->diverge);
  cudaFree(c->capped);
  cudaFree(c->keys);
  cudaFree(c->box_part);
  cudaFree(c->perm);
  cudaFree(c->inv);
  cudaFree(c->perm2);
  cudaFree(c->inv2);
  cudaFree(c->row_ptr_o);
  cudaFree(c->col_o);
  cudaFree(c->rscratch);
  cudaFree(c->iobuf);
  cudaFree(c->label_caller);
  cudaFree(c->label_slot);
  cudaFree(c->region_caller);
  cudaFree(c->region_slot);
  cudaFree(c->s1);
  cudaFree(c->xa);
  cudaFree(c->xb);
  cudaFree(c->fbuf);
  for (void* q : c->ipc_open) cudaIpcCloseMemHandle(q);
  cudaFree(c->d_route);
  cudaFree(c->bar);
  cudaFree(c->hv_first);
  cudaFree(c->hv_part);
  cudaFree(c->hv_scratch);
  cudaFree(c->np_scratch);
  cudaFree(c->np_hits);
  cudaFree(c->np_hits2);
  cudaFree(c->np_slots);
  cudaFree(c->np_keys);
  cudaFree(c->np_sum);
  cudaFree(c->geom);
  cudaFree(c->kkey);
  if (c->h_status) cudaFreeHost(c->h_status);
  if (c->comm && c->nccl) c->nccl->CommDestroy(c->comm);
  if (c->side) {
    cudaStreamSynchronize(c->side);
    cudaStreamDestroy(c->side);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->ev_join2) cudaEventDestroy(c->ev_join2);
  if (c->ev_fork2) cudaEventDestroy(c->ev_fork2);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

tfdp_status tfdp_nccl_unique_id(unsigned char* uid128) {
  if (!uid128) return TFDP_ERR_ARG;
  const char* e = nullptr;
  const tfdp::NcclApi* api = tfdp::nccl_api(&e);
  if (!api) return fail(nullptr, TFDP_ERR_NCCL, "%s", e);
  ncclUniqueId id;
  ncclResult_t r = api->GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, TFDP_ERR_NCCL, "ncclGetUniqueId: %s", api->GetErrorString(r));
  memcpy(uid128, &id, sizeof id);
  return TFDP_OK;
}

}  // extern "C"
