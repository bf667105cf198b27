/* A plain C consumer of libditer.so (include/diter.h), no Python involved:
 * PageRank (d = 0.85, B = (1-d)/n) on the directed cycle i -> i+1 mod n, whose
 * fixed point is X_i = 1/n exactly (every column of P = dQ sums to d and Q is a
 * permutation, so X = B / (1-d)).  With no dangling node the error bound of
 * PAPER.md:104-107 holds with equality: |X - H|_1 = |F|_1 / (1-d).  Also checks
 * that a non-monotone col_ptr is rejected with a message and no context.
 * Exit 0 when every check holds; prints one summary line.  Test infrastructure
 * (tests/test_c_abi.py builds and runs it). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "diter.h"

int main(int argc, char **argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 100000;
  const double d = 0.85, target = 1e-10;
  int64_t *cp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int32_t *ri = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  double *H = (double *)malloc(sizeof(double) * (size_t)n);
  if (!cp || !ri || !H) return 3;
  for (int64_t i = 0; i < n; ++i) {
    cp[i] = i;
    ri[i] = (int32_t)((i + 1) % n);
  }
  cp[n] = n;

  di_options o;
  di_default_options(&o);
  di_ctx *ctx = NULL;
  di_status st = di_create(&ctx, n, cp, ri, NULL, NULL, d, &o);
  if (st != DI_OK) {
    fprintf(stderr, "di_create: %d %s\n", (int)st, di_last_error(NULL));
    return 2;
  }
  st = di_run(ctx, target);
  if (st != DI_OK) {
    fprintf(stderr, "di_run: %d %s\n", (int)st, di_last_error(ctx));
    return 2;
  }
  double r = -1.0;
  di_stats s;
  if (di_get_history(ctx, H) != DI_OK || di_get_residual(ctx, &r) != DI_OK || di_get_stats(ctx, &s) != DI_OK) {
    fprintf(stderr, "getters: %s\n", di_last_error(ctx));
    return 2;
  }
  di_destroy(ctx);

  double err = 0.0;
  for (int64_t i = 0; i < n; ++i) err += fabs(H[i] - 1.0 / (double)n);
  const double bound = r / (1.0 - d);
  const int ok_bound = r < target && fabs(err - bound) <= 1e-9 * bound + 1e-15;

  /* invalid input: col_ptr not non-decreasing */
  cp[1] = 5;
  cp[2] = 1;
  di_ctx *bad = (di_ctx *)0x1;
  const di_status sb = di_create(&bad, n, cp, ri, NULL, NULL, d, &o);
  const int ok_reject = sb == DI_ERR_INVALID_ARG && bad == NULL && di_last_error(NULL)[0] != '\0';

  printf("n=%lld passes=%lld edges=%lld r=%.6e err=%.6e bound=%.6e reject=%d ok=%d\n", (long long)n,
         (long long)s.passes, (long long)s.edges, r, err, bound, (int)sb, ok_bound && ok_reject);
  free(cp);
  free(ri);
  free(H);
  return ok_bound && ok_reject ? 0 : 1;
}
