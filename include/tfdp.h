/*
 * tfdp.h — C ABI of libtfdp.so, the B200-native t-FDP force step.
 *
 * t-FDP: Zhong et al., "Force-directed graph layouts revisited: a new force based on the
 * t-Distribution", arXiv 2303.03964.  Citations: P:n = /root/reference/PAPER.md line n,
 * S:n = /root/reference/SPEC.md line n, R<k> = reading k of DESIGN.md (§Readings).
 *
 * What one iteration computes, for x_i in R^2:
 *   R_i = rho * sum_j (x_i - x_j) (1 + |x_i - x_j|^2)^-gamma      repulsion
 *         exact all-pairs (TFDP_EXACT) or interpolation+FFT (TFDP_IBFFT)
 *   A_i = -alpha * sum_{j in adj(i)} (1 + beta / (1 + d_ij^2)) (x_i - x_j)
 *   x_i <- x_i + eta_t (R_i + A_i)                                 P:412, S:352 (R1, R2)
 *
 * Conventions for every entry point:
 *   - Positions and forces are float32, 2 per node, node-major (x0,y0,x1,y1,...).
 *   - Returned status: TFDP_OK or an error code; nothing aborts or throws across the ABI.
 *     The message of the last error is kept per context (tfdp_last_error).
 *   - Pointers marked "host or device" are classified with cudaPointerGetAttributes; all
 *     work is ordered on the context stream; calls that write HOST memory synchronize
 *     that stream before returning, calls that write DEVICE memory do not.
 *   - The context owns every device buffer it allocates; callers own their pointers.
 *   - There is no CPU fallback: every force evaluation runs in sm_100a kernels.
 */
#ifndef TFDP_H_
#define TFDP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TFDP_VERSION_MAJOR 0
#define TFDP_VERSION_MINOR 1

typedef struct tfdp_ctx tfdp_ctx; /* opaque; owns all device memory and FFT buffers */

typedef enum {
  TFDP_OK = 0,
  TFDP_ERR_ARG = 1,         /* invalid argument (see each call)                          */
  TFDP_ERR_CUDA = 2,        /* CUDA runtime failure                                       */
  TFDP_ERR_OOM = 3,         /* device allocation failed                                   */
  TFDP_ERR_DIVERGED = 4,    /* non-finite position after a step; ctx -> errored   */
  TFDP_ERR_STATE = 5,       /* ctx is errored, or iteration t >= T under linear cooling   */
  TFDP_ERR_NCCL = 6,        /* NCCL failure (multi-GPU)                                   */
  TFDP_ERR_UNSUPPORTED = 7  /* dim != 2, or a feature not built                           */
} tfdp_status;

enum { TFDP_EXACT = 0, TFDP_IBFFT = 1 };                 /* repulsion path (P:454 / P:488) */
enum { TFDP_COOL_LINEAR = 0, TFDP_COOL_CONSTANT = 1 };    /* integrator readings R2 / R2'   */
/* FFT path at p > 1:
 *   TFDP_DIST_SLAB (default): the grid convolution is distributed like a slab-decomposed
 *     2-D FFT — every rank spreads the nodes of its grid-row slab (from the full positions),
 *     transforms those rows, transposes (NCCL send/recv), runs the column pass on its chunk
 *     of half-spectrum columns, transposes back, inverse-transforms its rows and broadcasts
 *     its potential rows; gather / attraction / update of its own node shard, position
 *     all-gather.  Nodes are renumbered in Morton order identically on every rank.
 *   TFDP_DIST_SPREAD_ALL: every rank spreads all nodes and runs the whole convolution.
 *   TFDP_DIST_GRID_ALLREDUCE: own nodes spread, charge grid all-reduced, whole convolution. */
enum { TFDP_DIST_SPREAD_ALL = 0, TFDP_DIST_GRID_ALLREDUCE = 1, TFDP_DIST_SLAB = 2 };
enum { TFDP_ORDER_AUTO = 0, TFDP_ORDER_KEEP = 1 };        /* internal node renumbering      */
enum { TFDP_RULE_UNIT = 0, TFDP_RULE_SPAN = 1 };          /* interval width readings R5'/R5 */

/* Warning bits (returned by tfdp_warnings; the call itself returns TFDP_OK). */
enum {
  TFDP_WARN_ALPHA_BETA = 1u,  /* alpha (1 + beta) >= 1 violates Eq. limitweight      */
  TFDP_WARN_GAMMA = 2u,       /* gamma <= 1 violates Eq. exponentcondiction          */
  TFDP_WARN_NINT_CAPPED = 4u  /* an FFT iteration ran with N_int below the rule (grid cap);
                                 the next tfdp_step call re-plans a larger grid            */
};

typedef struct {
  int32_t dim;         /* must be 2; else TFDP_ERR_UNSUPPORTED              */
  double alpha;        /* attraction weight, default 0.1                           */
  double beta;         /* short-range attraction weight, default 8                 */
  double gamma;        /* repulsion exponent, default 2; integer 1..8 fast paths   */
  double rho;          /* repulsion scale, default 1 (global refinement P:13-18)    */
  int32_t solver;      /* TFDP_EXACT | TFDP_IBFFT                                          */
  int32_t k;           /* interpolation nodes per interval: 1,2,3; 0 = dynamic 90/5/5 */
  int32_t n_int_min;   /* 50                                                       */
  int32_t n_int_fixed; /* 0 = rule N_int = max(n_int_min, ceil L) (R5); > 0 forces N_int  */
  int32_t fft_size;    /* 0 = automatic P; > 0 forces P (must be >= 2 N_int k - 1, R9)     */
  double step0;        /* eta_0, default 0.1                                       */
  int32_t iterations;  /* T >= 1 (cooling + dynamic-k length), default 300 (R3)            */
  int32_t t0;          /* first iteration index (resume), default 0                        */
  int32_t cooling;     /* TFDP_COOL_LINEAR (eta_t = eta0 (1 - t/T), R2, default) |
                          TFDP_COOL_CONSTANT (eta_t = eta0, R2')                           */
  int32_t dist_mode;   /* TFDP_DIST_SLAB (default) | TFDP_DIST_SPREAD_ALL |
                          TFDP_DIST_GRID_ALLREDUCE (ibFFT path at p > 1)                   */
  int32_t node_order;  /* TFDP_ORDER_AUTO (default): the ibFFT path renumbers nodes internally
                          in Morton order of the layout (single GPU, n >= 65536) at the start
                          of each tfdp_step call; all inputs/outputs stay in the caller's
                          order.  TFDP_ORDER_KEEP: never renumber                          */
  int32_t interval_rule; /* TFDP_RULE_UNIT (R5', default): when ceil L >= n_int_min the
                          N_int = ceil L intervals have unit width (square of side N_int);
                          the grid spacing h = 1/k is then constant and the kernel spectrum
                          is recomputed only when P, k or gamma change.  TFDP_RULE_SPAN (R5):
                          w = L / N_int always (K^ recomputed every iteration).  With
                          n_int_fixed > 0, or N_int = n_int_min > ceil L, both use L / N_int */
} tfdp_params;

/* Multi-GPU description: one process per GPU.  nccl_uid = 128 bytes from
 * tfdp_nccl_unique_id() on rank 0, broadcast by the caller (e.g. over torch.distributed).
 * nccl_uid == NULL with world > 1 is a "virtual rank": no communicator.  Alone it evaluates
 * its shard [lo, hi) on one GPU with tfdp_forces (exact path and the SPREAD_ALL mode;
 * tfdp_step returns TFDP_ERR_UNSUPPORTED); all p virtual ranks of a world together run
 * every mode, tfdp_step included, through tfdp_group_step / tfdp_group_forces, with device
 * copies on their shared stream in place of NCCL — the same kernels, phases, layouts and
 * message boundaries as the NCCL path (one device: correctness, not scaling). */
typedef struct {
  int32_t rank, world, device;
  const unsigned char* nccl_uid;
} tfdp_dist;

/* Fills *p with the defaults above.  TFDP_ERR_ARG if p == NULL. */
tfdp_status tfdp_params_default(tfdp_params* p);

/* Host-side symmetric CSR build of an undirected simple graph:
 * self-loops dropped, duplicate unordered pairs collapsed, columns of each row sorted.
 *   n        node count (>= 1);  m  number of input pairs (>= 0)
 *   u, v     host int32[m] endpoints in [0, n)
 *   row_ptr  host int64[n+1] out;  col  host int32[capacity 2m] out;  *nnz = row_ptr[n]
 * TFDP_ERR_ARG on n < 1, m < 0, NULL pointers (when m > 0) or endpoints out of range.
 * Deterministic; bit-identical to the oracle's csr_build. */
tfdp_status tfdp_csr_build(int64_t n, int64_t m, const int32_t* u, const int32_t* v,
                           int64_t* row_ptr, int32_t* col, int64_t* nnz);

/* Shard rule: rank r of p owns targets [floor(r n / p), floor((r+1) n / p)).
 * TFDP_ERR_ARG unless n >= 0, 0 <= rank < world. */
tfdp_status tfdp_shard_range(int64_t n, int32_t world, int32_t rank, int64_t* lo, int64_t* hi);

/* Creates a context on the current (or dist->device) GPU.
 *   n        node count >= 1
 *   row_ptr  host int64[n+1], col host int32[row_ptr[n]]: a symmetric CSR as produced by
 *            tfdp_csr_build (validated in O(m log d): symmetric, sorted, no self-loop, no
 *            duplicate, in range; else TFDP_ERR_ARG)
 *   xy0      host or device float32[2n] starting layout (finite; else TFDP_ERR_ARG)
 *   p        parameters (NULL = defaults).  TFDP_ERR_ARG if T < 1, eta0 <= 0, gamma <= 0,
 *            rho <= 0, alpha < 0, beta < 0, any value non-finite, k not in 0..3,
 *            solver/cooling/dist_mode unknown.  TFDP_ERR_UNSUPPORTED if dim != 2.
 *            Parameter-validity violations only set warning bits.
 *   dist     NULL = single GPU; else rank/world/device + NCCL unique id
 *   stream   cudaStream_t to order all work on (NULL = the context creates its own)
 * The context copies the CSR and xy0; the caller may free them on return. */
tfdp_status tfdp_init(tfdp_ctx** ctx, int64_t n, const int64_t* row_ptr, const int32_t* col,
                      const float* xy0, const tfdp_params* p, const tfdp_dist* dist,
                      void* stream);

/* Runs n_iters >= 0 iterations t = t_cur .. t_cur + n_iters - 1 of the layout loop:
 * k_t and eta_t from the schedules (R2/R2'), repulsion + attraction from the
 * snapshot (Jacobi), position update, and (p > 1) the position exchange.
 * Reads one 8-byte divergence word back at the end (the only host sync).
 * TFDP_ERR_DIVERGED with "diverged at iter t node i"; TFDP_ERR_STATE if the ctx
 * is errored or, under linear cooling, t would reach T. */
tfdp_status tfdp_step(tfdp_ctx* ctx, int32_t n_iters);

/* Evaluates R (rep_xy) and A (att_xy) at the current layout for this rank's shard
 * [lo, hi) without updating; rep_xy / att_xy are host or device float32[2 (hi - lo)]
 * (either may be NULL).  The ibFFT path uses k = params.k, or the schedule's k at the
 * current iteration when params.k == 0.  Parity entry point of the tests. */
tfdp_status tfdp_forces(tfdp_ctx* ctx, float* rep_xy, float* att_xy);

/* The virtual ranks 0..p-1 of one world (contexts created with tfdp_dist {r, p, device,
 * NULL}, one stream, one problem, same iteration t), driven in lockstep on one device:
 * tfdp_group_step = tfdp_step of every rank, tfdp_group_forces = tfdp_forces of every rank
 * (rep_xy[r] / att_xy[r]: rank r's output, host or device float32[2 (hi_r - lo_r)], arrays
 * or entries may be NULL).  Every exchange of the multi-GPU path (position all-gather,
 * renumbering broadcast, slab transposes, potential rows) is a device copy between the
 * contexts' buffers.  TFDP_ERR_ARG if the contexts do not form such a group (1 <= p <= 64);
 * otherwise the errors of tfdp_step / tfdp_forces. */
tfdp_status tfdp_group_step(tfdp_ctx* const* ctxs, int32_t p, int32_t n_iters);
tfdp_status tfdp_group_forces(tfdp_ctx* const* ctxs, int32_t p, float* const* rep_xy,
                              float* const* att_xy);

/* Slab plan of the TFDP_DIST_SLAB mode (host only, no GPU): for `rows` grid rows
 * (N_int cap x k) and FFT size fft_size split over world ranks, rank r owns grid rows
 * [row0[r], row0[r+1]) (multiples of 24, row0[world] = rows rounded up to 24) and
 * half-spectrum columns [q0[r], q0[r+1]) (even starts, q0[world] = fft_size/2 + 1).
 * row0, q0: host int32[world + 1].  TFDP_ERR_ARG unless rows >= 1, fft_size even >= 2,
 * 1 <= world <= 64. */
tfdp_status tfdp_slab_plan(int32_t rows, int32_t fft_size, int32_t world, int32_t* row0,
                           int32_t* q0);

/* Copies the full current layout (all n nodes, every rank) to xy_out (host or device
 * float32[2n]). */
tfdp_status tfdp_layout(tfdp_ctx* ctx, float* xy_out);

/* Replaces the full layout with xy (host or device float32[2n], finite).  With
 * tfdp_set_iteration this is the resume path (checkpoint = tfdp_layout + iteration). */
tfdp_status tfdp_set_layout(tfdp_ctx* ctx, const float* xy);
tfdp_status tfdp_set_iteration(tfdp_ctx* ctx, int32_t t);
int32_t tfdp_iteration(const tfdp_ctx* ctx);

/* Replaces the parameters of a live context (the layout is kept).  Validated like tfdp_init
 * (same errors, same warning bits, which replace the previous ones; TFDP_WARN_NINT_CAPPED
 * is kept).  solver, dist_mode and node_order are fixed at tfdp_init (TFDP_ERR_ARG if they
 * differ).  The iteration counter is set to p->t0 and the k schedule rebuilt for
 * p->iterations.  On the ibFFT path a change of k, n_int_min, n_int_fixed or fft_size
 * re-plans the grid from the current layout (one bbox pass and a sync); on failure the
 * previous parameters stay in force.  Used by global refinement. */
tfdp_status tfdp_set_params(tfdp_ctx* ctx, const tfdp_params* p);

/* Global refinement (SPEC global_refine S:359-366): taking the current layout as
 * the initialization, re-runs the layout loop for `iterations` iterations t = 0 .. T-1
 * (T = iterations, schedules rebuilt for T) with repulsion exponent gamma and scale rho
 * ("a large repulsive t-force will distribute nearby nodes evenly"; "a repulsive force
 * with a shorter range (larger gamma)" shows the skeleton).  alpha, beta, eta0, cooling,
 * solver and k are kept; gamma and rho stay set afterwards.  Errors: TFDP_ERR_ARG if
 * gamma <= 1 or non-finite, rho <= 0 or non-finite, iterations < 1; otherwise the
 * errors of tfdp_step. */
tfdp_status tfdp_global_refine(tfdp_ctx* ctx, double gamma, double rho, int32_t iterations);

/* PivotMDS initialisation ("we use the same PMDS layout as initialization"; SPEC
 * init_pivot_mds S:110-118; Brandes & Pich 2006), computed on the device; replaces the
 * context's layout (the paper's evaluation protocol: PMDS, then t-FDP).
 *   p = min(n_pivots, n) pivots by max-min farthest-point BFS selection, the first one
 *   splitmix64(seed) mod n, ties by the lowest node id; hop distances D (n x p; unreachable
 *   = that pivot's eccentricity + 1, R24); C = double-centred -D^2/2; the top-2
 *   eigenvectors v_1, v_2 of C^T C (power iteration, fp64; sign: largest-|.| component
 *   positive); positions C v_k, centred, scaled to mean edge length 1 (rank < 2: the
 *   second axis is 0).
 *   pivots  host int32[min(n_pivots, n)] (may be NULL): the chosen pivots (caller ids)
 * TFDP_ERR_ARG unless 1 <= n_pivots <= 64.  Syncs once per pivot.  Scratch (~4 p + 60 B per
 * node) is allocated for the call and freed. */
tfdp_status tfdp_pivot_mds(tfdp_ctx* ctx, int32_t n_pivots, uint64_t seed, int32_t* pivots);

/* Local (fisheye) refinement mask (SPEC RefinementMask S:155-158).  The region
 * F u N(F) = the focal nodes and their graph neighbours.  Forces with the mask:
 *   repulsion pair weight  lf if both ends are in the region, ls if both are outside, else 1
 *   attraction edge weight la if both ends are in the region, else 1
 * ("we enhance the attractive forces between the focal nodes and their neighbors ... while
 * exerting repulsive forces to highlight them ... large repulsive forces between other
 * nodes").  The exact path applies the weights exactly; the ibFFT path computes the unmasked
 * grid sum S_all plus an exact sum S1 over the region's sources and combines
 * rho [w0 (S_all - S1) + w1 S1] (R23).  The mask stays active for every later
 * tfdp_step / tfdp_forces until replaced; n_focal = 0 clears it; boosts (1, 1, 1) are the
 * identity (the unmasked kernels run).
 *   focal   host int32[n_focal] caller node ids (duplicates allowed)
 *   la, lf, ls  boosts >= 1, finite
 * TFDP_ERR_ARG on an id out of range, a boost < 1 or non-finite.  Syncs the stream.  Cost per
 * iteration: one n_local x |region| exact pass. */
tfdp_status tfdp_set_focus(tfdp_ctx* ctx, const int32_t* focal, int64_t n_focal, double la,
                           double lf, double ls);

/* Local refinement (SPEC local_refine S:368-372): tfdp_set_focus, then `iterations`
 * iterations t = 0 .. T-1 from the current layout (T = iterations, schedules rebuilt, as in
 * tfdp_global_refine).  TFDP_ERR_ARG on an empty focal set or iterations < 1; else
 * the errors of tfdp_set_focus and tfdp_step.  The mask stays set afterwards. */
tfdp_status tfdp_local_refine(tfdp_ctx* ctx, const int32_t* focal, int64_t n_focal, double la,
                              double lf, double ls, int32_t iterations);

/* Neighbourhood preservation NP1 of the current layout, computed on
 * the device (NEXT-3: per-iteration convergence traces):
 *   NP1 = (1/n) sum_i |N_G(i) ∩ N_L(i, k_i)| / |N_G(i) ∪ N_L(i, k_i)|,  k_i = deg(i),
 * N_L(i, k) = the k nearest other nodes in the layout, equal distances broken by the lower
 * node id; a degree-0 node contributes 1.  Distances are compared as d^2 = (dx dx) + (dy dy)
 * with each operation rounded in IEEE fp32 (R22), so the set decisions are exact
 * and deterministic.
 *   np1   host double* (may be NULL): the full-graph value on every rank (NCCL sum over the
 *         ranks); for a virtual shard (no communicator) this shard's share sum_{i in shard}/n
 *   hits  host or device int32[hi - lo] (may be NULL): |N_G(i) ∩ N_L(i, k_i)| for the
 *         shard's nodes in the caller's order
 * Syncs the stream.  Cost: O(n + sum_i c_i) with c_i the nodes in the cells around i that
 * hold its k_i nearest (uniform cell grid of ~2 nodes per cell over the bounding square).
 * Scratch (~8 B x cells + 24 B x n) is allocated at the first call and kept. */
tfdp_status tfdp_np1(tfdp_ctx* ctx, double* np1, int32_t* hits);

/* This rank's target shard. */
tfdp_status tfdp_shard(const tfdp_ctx* ctx, int64_t* lo, int64_t* hi);

/* Geometry of the most recent ibFFT evaluation (diagnostics; syncs the stream):
 * box4 = {lo_x, lo_y, L, w} (fp32, R6/R19), *n_int, *k, *fft_size (any may be NULL). */
tfdp_status tfdp_fft_geometry(tfdp_ctx* ctx, float* box4, int32_t* n_int, int32_t* k,
                              int32_t* fft_size);

/* FFT plan for interpolation order k (1..3): *fft_size = P_k, *n_int_cap = largest N_int
 * the allocated grid holds at that k (TFDP_ERR_STATE unless an ibFFT context). */
tfdp_status tfdp_fft_plan(const tfdp_ctx* ctx, int32_t k, int32_t* fft_size, int32_t* n_int_cap);

/* Per-kernel device timing (CUDA events around each launch on the ctx stream).
 * tfdp_profile(ctx, 1) resets and times every kernel kind, 0 disables.
 * tfdp_profile_mask(ctx, kinds) resets and times only the kinds whose bit is set (bit i =
 * entry i of tfdp_profile_read), so a timed region can be instrumented around its dominant
 * kernel alone.  tfdp_profile_read fills up to cap entries: names (static strings), total
 * milliseconds and launch counts; returns the number of kernel kinds (or -1 on error).
 * Syncs the stream. */
tfdp_status tfdp_profile(tfdp_ctx* ctx, int32_t enable);
tfdp_status tfdp_profile_mask(tfdp_ctx* ctx, uint32_t kinds);
/* Sets the timed kinds WITHOUT resetting the accumulated times or syncing (a host-side
 * switch): a timed region can instrument a sample of its launches — e.g. every fourth step —
 * and read the sample's total with tfdp_profile_read at the end. */
tfdp_status tfdp_profile_select(tfdp_ctx* ctx, uint32_t kinds);
int32_t tfdp_profile_read(tfdp_ctx* ctx, const char** names, double* ms, int64_t* launches,
                          int32_t cap);

/* Number of kernel launches this library has issued on the ctx (its own kernels, not
 * NCCL).  For the bench's gpu_launches claim. */
int64_t tfdp_launch_count(const tfdp_ctx* ctx);

uint32_t tfdp_warnings(const tfdp_ctx* ctx);
const char* tfdp_last_error(const tfdp_ctx* ctx); /* "" if none; never NULL            */
const char* tfdp_status_string(tfdp_status s);
void tfdp_destroy(tfdp_ctx* ctx);                 /* NULL is a no-op                   */

/* NCCL bootstrap for multi-GPU: writes a 128-byte ncclUniqueId.  Resolves NCCL from the
 * process (libnccl.so.2, e.g. the one torch loaded).  TFDP_ERR_NCCL if unavailable. */
tfdp_status tfdp_nccl_unique_id(unsigned char* uid128);

#ifdef __cplusplus
}
#endif
#endif /* TFDP_H_ */
