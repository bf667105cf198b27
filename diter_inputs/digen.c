/*
 * digen.c -- seeded synthetic input generators for the D-iteration hot path.
 *
 * This module is SHARED INPUT PLUMBING: it is the only code used by both the
 * CPU oracle (oracle/) and the CUDA path (paper_1202_6168_b200/).  It holds
 * none of the method's arithmetic (no fluid, no history, no diffusion, no
 * CSC construction from COO, no partitioning): it only draws graphs and
 * right-hand sides from the recipes of BASELINE.json configs[0..4] and
 * SURVEY.md Appendix C.
 *
 * RNG: counter-based.  Every random number is mix64(stream key, node/edge id,
 * counter), so generation is order-independent, OpenMP-parallel and
 * bit-reproducible.  Floating point appears only in the host-side draws
 * (pow/exp for the degree law and the Zipf-over-id destination); the CUDA
 * path never re-generates, it receives these arrays through di_create.
 *
 * Recipes (DESIGN.md §"Input recipe"):
 *   kind 1 "uniform"  (configs[0], C1): outdeg ~ U{deg_lo..deg_hi}, destinations
 *                     distinct, uniform on [0,N)\{i}; no dangling nodes.
 *   kind 2 "web"      (configs[1]/[3], C2/C4): dangling w.p. p_dangling;
 *                     otherwise Pareto-floor degree
 *                     deg = min(max_deg, max(1, floor(x_min * u^(-1/1.1)))) (tail
 *                     exponent 2.1); per slot: local w.p. p_local
 *                     (offset uniform in +-[1,window], wrapped mod N) else global
 *                     Zipf(1) over id, j = min(N-1, floor((N+1)^u) - 1); a draw
 *                     equal to i is re-drawn; then the column is sorted + deduped.
 *   kind 3 "rmat"     (configs[2], C3): edge_factor * 2^scale COO samples, 2 bits per
 *                     level from quadrant cut-points (a, a+b, a+b+c), ids then
 *                     permuted by a seeded Fisher-Yates permutation.  Duplicates are
 *                     KEPT here: dropping them is CSC construction (method side).
 *   kind 5 "signed"   (configs[4], C5): nnz_per_col distinct rows uniform on [0,N),
 *                     values U[-1,1] scaled so each column's |.|-sum = col_abs_sum;
 *                     B_i ~ U[-1,1].
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <omp.h>

#include "digen.h"

static inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* stream key from (config kind, seed, sub-stream) */
static inline uint64_t stream_key(const dg_params *p, uint64_t sub) {
  return mix64(mix64(((uint64_t)p->kind << 48) ^ p->seed) ^ (sub * 0xd1b54a32d192ed03ULL));
}

static inline uint64_t draw(uint64_t key, uint64_t id, uint64_t ctr) {
  return mix64(mix64(key ^ mix64(id)) + ctr * 0x9e3779b97f4a7c15ULL);
}

/* uniform double in [0,1) with 53 random bits */
static inline double u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

/* uniform integer in [0, m) (multiply-high, negligible bias for m << 2^64) */
static inline uint64_t below(uint64_t h, uint64_t m) {
  return (uint64_t)(((unsigned __int128)h * m) >> 64);
}

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* insertion sort for short columns, qsort for long ones */
static void sort_i32(int32_t *a, int64_t n) {
  if (n > 48) { qsort(a, (size_t)n, sizeof(int32_t), cmp_i32); return; }
  for (int64_t i = 1; i < n; ++i) {
    int32_t v = a[i]; int64_t j = i - 1;
    while (j >= 0 && a[j] > v) { a[j + 1] = a[j]; --j; }
    a[j + 1] = v;
  }
}

static int64_t unique_i32(int32_t *a, int64_t n) {
  if (n == 0) return 0;
  int64_t w = 1;
  for (int64_t i = 1; i < n; ++i) if (a[i] != a[w - 1]) a[w++] = a[i];
  return w;
}

/* ---------------------------------------------------------------- params -- */

int dg_validate(const dg_params *p) {
  if (!p || p->n < 1 || p->n > 2147483647LL) return DG_ERR_ARG;
  switch (p->kind) {
    case DG_UNIFORM:
      if (p->deg_lo < 1 || p->deg_hi < p->deg_lo || p->deg_hi > p->n - 1) return DG_ERR_ARG;
      return DG_OK;
    case DG_WEB:
      if (p->n < 2 || p->max_deg < 1 || p->x_min < 1.0 || p->window < 1) return DG_ERR_ARG;
      if (p->max_deg > p->n - 1) return DG_ERR_ARG;
      return DG_OK;
    case DG_RMAT:
      if (p->scale < 1 || p->scale > 30 || p->edge_factor < 1) return DG_ERR_ARG;
      if (p->n != (1LL << p->scale)) return DG_ERR_ARG;
      return DG_OK;
    case DG_SIGNED:
      if (p->nnz_per_col < 1 || p->nnz_per_col > p->n || !(p->col_abs_sum > 0)) return DG_ERR_ARG;
      return DG_OK;
    default:
      return DG_ERR_ARG;
  }
}

/* ------------------------------------------------------- column drawing -- */

/* Draw column i (sorted, unique rows) into rows[]; optional values into vals[].
 * Returns the column length.  rows/vals must hold max_raw_degree(p) entries. */
static int64_t max_raw_degree(const dg_params *p) {
  switch (p->kind) {
    case DG_UNIFORM: return p->deg_hi;
    case DG_WEB: return p->max_deg;
    case DG_SIGNED: return p->nnz_per_col;
    default: return 0;
  }
}

static int64_t web_degree(const dg_params *p, uint64_t key, int64_t i) {
  double u0 = u01(draw(key, (uint64_t)i, 0));
  if (u0 < p->p_dangling) return 0;
  double u1 = u01(draw(key, (uint64_t)i, 1));
  if (u1 <= 0.0) return p->max_deg;                     /* u^(-1/1.1) -> inf */
  double x = p->x_min * pow(u1, -1.0 / 1.1);
  if (!(x < (double)p->max_deg)) return p->max_deg;
  int64_t d = (int64_t)floor(x);
  return d < 1 ? 1 : d;
}

static int64_t draw_column(const dg_params *p, uint64_t key, int64_t i, int32_t *rows, double *vals) {
  const int64_t n = p->n;
  if (p->kind == DG_UNIFORM) {
    int64_t deg = p->deg_lo + (int64_t)below(draw(key, (uint64_t)i, 0), (uint64_t)(p->deg_hi - p->deg_lo + 1));
    int64_t got = 0; uint64_t ctr = 1;
    while (got < deg) {
      int64_t j = (int64_t)below(draw(key, (uint64_t)i, ctr++), (uint64_t)(n - 1));
      if (j >= i) ++j;                                  /* excludes the self-loop */
      int dup = 0;
      for (int64_t t = 0; t < got; ++t) if (rows[t] == (int32_t)j) { dup = 1; break; }
      if (!dup) rows[got++] = (int32_t)j;
    }
    sort_i32(rows, got);
    return got;
  }
  if (p->kind == DG_WEB) {
    int64_t deg = web_degree(p, key, i);
    uint64_t ctr = 2;
    for (int64_t s = 0; s < deg; ++s) {
      for (;;) {
        uint64_t h1 = draw(key, (uint64_t)i, ctr++);
        uint64_t h2 = draw(key, (uint64_t)i, ctr++);
        int64_t j;
        if (u01(h1) < p->p_local) {
          int64_t o = (int64_t)below(h2, (uint64_t)(2 * p->window));   /* 0..2w-1 */
          o = (o < p->window) ? (o - p->window) : (o - p->window + 1);  /* -w..-1, 1..w */
          j = (i + o) % n; if (j < 0) j += n;
        } else {
          double u3 = u01(h2);
          double y = floor(exp(u3 * log((double)n + 1.0))) - 1.0;
          j = (y < 0.0) ? 0 : (y > (double)(n - 1) ? n - 1 : (int64_t)y);
        }
        if (j != i) { rows[s] = (int32_t)j; break; }  /* re-draw self-loops */
      }
    }
    sort_i32(rows, deg);
    return unique_i32(rows, deg);
  }
  if (p->kind == DG_SIGNED) {
    int64_t k = p->nnz_per_col, got = 0; uint64_t ctr = 0;
    while (got < k) {
      int32_t j = (int32_t)below(draw(key, (uint64_t)i, ctr++), (uint64_t)n);
      int dup = 0;
      for (int64_t t = 0; t < got; ++t) if (rows[t] == j) { dup = 1; break; }
      if (!dup) rows[got++] = j;
    }
    sort_i32(rows, got);
    if (vals) {
      /* values keyed by (column, row) so they do not depend on draw order */
      uint64_t vkey = stream_key(p, 2);
      double s = 0.0;
      for (int64_t t = 0; t < got; ++t) {
        double u = 2.0 * u01(draw(vkey, (uint64_t)i, (uint64_t)rows[t])) - 1.0;
        vals[t] = u; s += fabs(u);
      }
      double scale = (s > 0.0) ? p->col_abs_sum / s : 0.0;
      for (int64_t t = 0; t < got; ++t) vals[t] *= scale;
    }
    return got;
  }
  return 0;
}

int dg_csc_count(const dg_params *p, int64_t *col_ptr) {
  int rc = dg_validate(p); if (rc) return rc;
  if (p->kind == DG_RMAT) return DG_ERR_ARG;
  const int64_t n = p->n, cap = max_raw_degree(p);
  const uint64_t key = stream_key(p, 1);
  int err = 0;
  #pragma omp parallel
  {
    int32_t *rows = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cap > 0 ? cap : 1));
    if (!rows) {
      #pragma omp atomic write
      err = 1;
    }
    #pragma omp for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
      if (rows) col_ptr[i + 1] = draw_column(p, key, i, rows, NULL);
    }
    free(rows);
  }
  if (err) return DG_ERR_OOM;
  col_ptr[0] = 0;
  for (int64_t i = 0; i < n; ++i) col_ptr[i + 1] += col_ptr[i];
  return DG_OK;
}

int dg_csc_fill(const dg_params *p, const int64_t *col_ptr, int32_t *row_idx, double *vals) {
  int rc = dg_validate(p); if (rc) return rc;
  if (p->kind == DG_RMAT) return DG_ERR_ARG;
  const int64_t n = p->n, cap = max_raw_degree(p);
  const uint64_t key = stream_key(p, 1);
  int err = 0;
  #pragma omp parallel
  {
    int32_t *rows = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cap > 0 ? cap : 1));
    double *vv = (double *)malloc(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
    if (!rows || !vv) {
      #pragma omp atomic write
      err = 1;
    }
    #pragma omp for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
      if (!rows || !vv) continue;
      int64_t len = draw_column(p, key, i, rows, (vals && p->kind == DG_SIGNED) ? vv : NULL);
      if (len != col_ptr[i + 1] - col_ptr[i]) {
        #pragma omp atomic write
        err = 2;
        continue;
      }
      memcpy(row_idx + col_ptr[i], rows, sizeof(int32_t) * (size_t)len);
      if (vals && p->kind == DG_SIGNED) memcpy(vals + col_ptr[i], vv, sizeof(double) * (size_t)len);
    }
    free(rows); free(vv);
  }
  return err == 1 ? DG_ERR_OOM : (err ? DG_ERR_ARG : DG_OK);
}

int dg_b_signed(const dg_params *p, double *b) {
  int rc = dg_validate(p); if (rc) return rc;
  const uint64_t key = stream_key(p, 3);
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < p->n; ++i) b[i] = 2.0 * u01(draw(key, (uint64_t)i, 0)) - 1.0;
  return DG_OK;
}

/* ------------------------------------------------------------------ R-MAT -- */

int64_t dg_rmat_edges(const dg_params *p) {
  if (dg_validate(p) || p->kind != DG_RMAT) return -1;
  return (int64_t)p->edge_factor << p->scale;
}

int dg_rmat_fill(const dg_params *p, int32_t *src, int32_t *dst) {
  int rc = dg_validate(p); if (rc) return rc;
  if (p->kind != DG_RMAT) return DG_ERR_ARG;
  const int64_t m = (int64_t)p->edge_factor << p->scale, n = p->n;
  const uint64_t key = stream_key(p, 1);
  /* cut points as 32-bit thresholds: one 32-bit half of a hash per level */
  const double ca = p->a, cb = p->a + p->b, cc = p->a + p->b + p->c;
  const uint64_t ta = (uint64_t)(ca * 4294967296.0), tb = (uint64_t)(cb * 4294967296.0),
                 tc = (uint64_t)(cc * 4294967296.0);
  #pragma omp parallel for schedule(static, 65536)
  for (int64_t e = 0; e < m; ++e) {
    uint64_t s = 0, t = 0, h = 0;
    for (int lvl = 0; lvl < p->scale; ++lvl) {
      uint64_t q;
      if ((lvl & 1) == 0) { h = draw(key, (uint64_t)e, (uint64_t)(lvl >> 1)); q = h & 0xffffffffULL; }
      else q = h >> 32;
      int sb, tbit;
      if (q < ta) { sb = 0; tbit = 0; }
      else if (q < tb) { sb = 0; tbit = 1; }
      else if (q < tc) { sb = 1; tbit = 0; }
      else { sb = 1; tbit = 1; }
      s = (s << 1) | (uint64_t)sb; t = (t << 1) | (uint64_t)tbit;
    }
    src[e] = (int32_t)s; dst[e] = (int32_t)t;
  }
  /* seeded Fisher-Yates permutation of the ids (sequential, O(n)) */
  int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  if (!perm) return DG_ERR_OOM;
  for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
  const uint64_t pkey = stream_key(p, 4);
  for (int64_t i = n - 1; i > 0; --i) {
    int64_t j = (int64_t)below(draw(pkey, 0, (uint64_t)i), (uint64_t)(i + 1));
    int32_t tmp = perm[i]; perm[i] = perm[j]; perm[j] = tmp;
  }
  #pragma omp parallel for schedule(static, 65536)
  for (int64_t e = 0; e < m; ++e) { src[e] = perm[src[e]]; dst[e] = perm[dst[e]]; }
  free(perm);
  return DG_OK;
}

int dg_num_threads(void) { return omp_get_max_threads(); }
void dg_set_threads(int n) { if (n > 0) omp_set_num_threads(n); }
