/* A plain C client of libtfdp.so (include/tfdp.h only; no Python, no torch): builds the
 * symmetric CSR of a grid graph, initialises it with PivotMDS and lays it out with the
 * paper's dynamic schedule, checks the status of every call, and prints the NP1 of the
 * result.
 *   usage: tfdp_layout [side = 100] [iterations = 300] [solver: 0 exact | 1 ibfft]
 * Exit status 0 on success. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "tfdp.h"

#define CHECK(call)                                                                       \
  do {                                                                                    \
    tfdp_status s_ = (call);                                                              \
    if (s_ != TFDP_OK) {                                                                  \
      fprintf(stderr, "%s failed: %s (%s)\n", #call, tfdp_status_string(s_),              \
              tfdp_last_error(ctx));                                                      \
      return 1;                                                                           \
    }                                                                                     \
  } while (0)

int main(int argc, char** argv) {
  const int side = argc > 1 ? atoi(argv[1]) : 100;
  const int T = argc > 2 ? atoi(argv[2]) : 300;
  const int solver = argc > 3 ? atoi(argv[3]) : TFDP_IBFFT;
  const int64_t n = (int64_t)side * side;
  tfdp_ctx* ctx = NULL;
  /* grid graph: right and down neighbours */
  int64_t m = 0;
  int32_t* u = malloc(sizeof(int32_t) * 2 * n);
  int32_t* v = malloc(sizeof(int32_t) * 2 * n);
  for (int r = 0; r < side; ++r)
    for (int c = 0; c < side; ++c) {
      const int32_t i = r * side + c;
      if (c + 1 < side) { u[m] = i; v[m] = i + 1; ++m; }
      if (r + 1 < side) { u[m] = i; v[m] = i + side; ++m; }
    }
  int64_t* row_ptr = malloc(sizeof(int64_t) * (n + 1));
  int32_t* col = malloc(sizeof(int32_t) * 2 * m);
  int64_t nnz = 0;
  CHECK(tfdp_csr_build(n, m, u, v, row_ptr, col, &nnz));
  /* starting layout: a seeded uniform square (LCG), side sqrt(n) */
  float* xy = malloc(sizeof(float) * 2 * n);
  uint64_t st = 12345;
  for (int64_t i = 0; i < 2 * n; ++i) {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    xy[i] = (float)((st >> 40) * (1.0 / 16777216.0)) * (float)side;
  }
  tfdp_params p;
  CHECK(tfdp_params_default(&p));
  p.solver = solver;
  p.k = 0; /* dynamic 90/5/5 */
  p.iterations = T;
  CHECK(tfdp_init(&ctx, n, row_ptr, col, xy, &p, NULL, NULL));
  CHECK(tfdp_pivot_mds(ctx, 50, 0, NULL)); /* the paper's initialisation */
  CHECK(tfdp_step(ctx, T));
  CHECK(tfdp_layout(ctx, xy));
  double np1 = 0.0;
  CHECK(tfdp_np1(ctx, &np1, NULL));
  for (int64_t i = 0; i < 2 * n; ++i)
    if (!isfinite(xy[i])) {
      fprintf(stderr, "non-finite position\n");
      return 1;
    }
  printf("n=%lld nnz=%lld T=%d solver=%d np1=%.4f warnings=%u\n", (long long)n, (long long)nnz, T,
         solver, np1, tfdp_warnings(ctx));
  tfdp_destroy(ctx);
  free(u); free(v); free(row_ptr); free(col); free(xy);
  return 0;
}
