/*
 * oracle.c -- plain, slow, single-threaded fp64 CPU oracle of the D-iteration
 * diffusion sweep (D. Hong, arXiv 1202.6168, reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, constant or helper with the CUDA path
 * (paper_1202_6168_b200/); neither side includes or links the other.
 *
 * Every function cites the passage it follows ("P:n" = PAPER.md line n,
 * "S:n" = SPEC.md line n, "§8c" = SURVEY.md §8(c) readings, listed again in
 * DESIGN.md "Readings of the paper").  No blocking, fusion or reordering
 * beyond what the cited definition states.  fp64, round-to-nearest, built
 * with -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 *
 * Parity pins (tests/test_oracle_pins.py): every function below is pinned
 * against closed forms, brute force, SPEC worked examples, LAPACK (numpy) or
 * invariants that the paper states; none is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#include "oracle.h"

/* ------------------------------------------------------------------------ *
 * CSC construction from a COO edge list.                                    *
 * p_ij is the weight of the edge from j to i, so column j of P      *
 * holds the out-edges of j.  SURVEY §8a row a0 / §8c step 1: counting sort   *
 * by source, rows ascending within a column, duplicates dropped (configs[2]  *
 * "duplicate edges dropped").                                               *
 * ------------------------------------------------------------------------ */
static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

int orc_csc_from_coo(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                     int64_t *col_ptr, int32_t *row_idx, int64_t *nnz_out) {
  if (n < 1 || m < 0) return ORC_ERR_ARG;
  for (int64_t e = 0; e < m; ++e)
    if (src[e] < 0 || src[e] >= n || dst[e] < 0 || dst[e] >= n) return ORC_ERR_ARG;
  /* 1. histogram of sources */
  int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  if (!cnt) return ORC_ERR_OOM;
  for (int64_t e = 0; e < m; ++e) cnt[src[e] + 1] += 1;
  /* 2. exclusive prefix sum -> raw column starts */
  for (int64_t j = 0; j < n; ++j) cnt[j + 1] += cnt[j];
  /* 3. stable counting-sort placement of destinations */
  int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  if (!pos) { free(cnt); return ORC_ERR_OOM; }
  for (int64_t j = 0; j < n; ++j) pos[j] = cnt[j];
  for (int64_t e = 0; e < m; ++e) row_idx[pos[src[e]]++] = dst[e];
  free(pos);
  /* 4. per column: sort rows ascending, drop duplicates, compact to the left */
  int64_t w = 0;
  col_ptr[0] = 0;
  for (int64_t j = 0; j < n; ++j) {
    int64_t a = cnt[j], b = cnt[j + 1];
    qsort(row_idx + a, (size_t)(b - a), sizeof(int32_t), cmp_i32);
    for (int64_t e = a; e < b; ++e)
      if (e == a || row_idx[e] != row_idx[e - 1]) row_idx[w++] = row_idx[e];
    col_ptr[j + 1] = w;
  }
  free(cnt);
  *nnz_out = w;
  return ORC_OK;
}

/* ------------------------------------------------------------------------ *
 * Partitions.                                                    *
 * Uniform (garbled "N/K+1, 2, ..."; reading §8c-Q20):              *
 *   Omega_k = [floor(k N / K), floor((k+1) N / K)).                            *
 * Cost Balanced ("sum_{n in Omega_k} #out_n = L/K", unattainable   *
 * exactly; reading §8c-Q10): with C the prefix sum of a per-node cost,        *
 *   w_0 = 0, w_K = N, w_k = min{ i : C[i] >= ceil(k C[N] / K) },               *
 *   then w_k = max(w_k, w_{k-1} + 1) so that no range is empty, and           *
 *   w_k <= N - (K - k) so that the later ranges are not empty either.         *
 * ------------------------------------------------------------------------ */
int orc_partition_uniform(int64_t n, int32_t K, int64_t *bounds) {
  if (K < 1 || n < K) return ORC_ERR_ARG;
  for (int32_t k = 0; k <= K; ++k) bounds[k] = (int64_t)(((__int128)k * n) / K);
  return ORC_OK;
}

int orc_partition_cb(int64_t n, const int64_t *cost_prefix, int32_t K, int64_t *bounds) {
  if (K < 1 || n < K) return ORC_ERR_ARG;
  const int64_t total = cost_prefix[n];
  bounds[0] = 0;
  for (int32_t k = 1; k < K; ++k) {
    /* ceil(k * total / K) in exact integer arithmetic */
    __int128 num = (__int128)k * total;
    int64_t goal = (int64_t)((num + K - 1) / K);
    int64_t i = 0;
    while (i < n && cost_prefix[i] < goal) ++i;          /* linear scan: plain, slow */
    if (i < bounds[k - 1] + 1) i = bounds[k - 1] + 1;
    if (i > n - (K - k)) i = n - (K - k);
    bounds[k] = i;
  }
  bounds[K] = n;
  return ORC_OK;
}

/* ------------------------------------------------------------------------ *
 * Edge weight p_ji for the stored edge e of column i.                        *
 * PageRank (eq. pr2): P = dQ, q_ji = 1/#out_i, computed once per   *
 * column as w_i = d / #out_i (reading §8c-Q19); dangling columns (#out = 0)   *
 * hold no entries, their fluid leaves (BASELINE.json configs[1]).            *
 * Signed: p_ji = vals[e].                                          *
 * ------------------------------------------------------------------------ */
static inline double pagerank_w(const int64_t *col_ptr, int64_t i, double d) {
  int64_t deg = col_ptr[i + 1] - col_ptr[i];
  return deg > 0 ? d / (double)deg : 0.0;
}

/* One elementary D-iteration step on node i (eq. defF P:86-97 with
 * J_i; eq. defH):  sent := F[i]; H[i] += sent; F[i] := 0;
 * for every child j of i: F[j] += sent * p(j,i).  Returns #out_i.          */
int64_t orc_diffuse_node(int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                         const double *vals, double d, int64_t i, double *F, double *H) {
  (void)n;
  double sent = F[i];
  H[i] += sent;
  F[i] = 0.0;
  double w = vals ? 0.0 : pagerank_w(col_ptr, i, d);
  for (int64_t e = col_ptr[i]; e < col_ptr[i + 1]; ++e)
    F[row_idx[e]] += sent * (vals ? vals[e] : w);
  return col_ptr[i + 1] - col_ptr[i];
}

double orc_l1(int64_t n, const double *v) {
  double r = 0.0;
  for (int64_t i = 0; i < n; ++i) r += fabs(v[i]);       /* plain left-to-right */
  return r;
}

/* ------------------------------------------------------------------------ *
 * Selection key weights.  The paper picks                        *
 *   i_n = argmax_i (F_{n-1})_i / ((#in_i + 1) x (#out_i + 1))                 *
 * and approximates the argmax by a threshold on the same quantity (P:213-   *
 * 216).  key_i = |F_i| * w_i with                                            *
 *   ORC_KEY_RAW   w_i = 1                       (BASELINE north_star, R3)    *
 *   ORC_KEY_EDGE  w_i = 1 / (#out_i + 1)         *
 *   ORC_KEY_PAPER w_i = 1 / ((#in_i + 1)(#out_i + 1))   (f1 (i))      *
 * #out_i = stored entries of column i, #in_i = stored entries of row i      *
 * ("number of incoming (resp. outgoing) links").  w_i is computed  *
 * in fp64 and rounded once to fp32 (reading R20: the GPU keeps 4 B/node);    *
 * the test is |F_i| * (double)w_i > T in fp64.                               *
 * ------------------------------------------------------------------------ */
int orc_key_weights(int64_t n, const int64_t *col_ptr, const int32_t *row_idx, int32_t key, float *w) {
  if (n < 1 || key < ORC_KEY_RAW || key > ORC_KEY_PAPER) return ORC_ERR_ARG;
  int64_t *in = (int64_t *)calloc((size_t)n, sizeof(int64_t));
  if (!in) return ORC_ERR_OOM;
  for (int64_t e = 0; e < col_ptr[n]; ++e) in[row_idx[e]] += 1;
  for (int64_t i = 0; i < n; ++i) {
    const double out = (double)(col_ptr[i + 1] - col_ptr[i]);
    double x = 1.0;
    if (key == ORC_KEY_EDGE) x = 1.0 / (out + 1.0);
    else if (key == ORC_KEY_PAPER) x = 1.0 / (((double)in[i] + 1.0) * (out + 1.0));
    w[i] = (float)x;
  }
  free(in);
  return ORC_OK;
}

static inline double sel_key(const double *F, const float *kw, int64_t i) {
  return kw ? fabs(F[i]) * (double)kw[i] : fabs(F[i]);
}

/* Initialisation: H := 0, F := B.  T_0 = max_i key_i(B) / alpha
 * (reading §8c-Q5: the paper gives no T_0; with strict ">" the first pass
 * then selects every node of maximal key, e.g. every node of a uniform B
 * under the raw key).  kw = NULL is the raw key. */
double orc_init_key(int64_t n, const double *b, double alpha, const float *kw, double *F, double *H) {
  double mx = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    F[i] = b[i];
    H[i] = 0.0;
    const double k = sel_key(b, kw, i);
    if (k > mx) mx = k;
  }
  return mx / alpha;
}

double orc_init(int64_t n, const double *b, double alpha, double *F, double *H) {
  return orc_init_key(n, b, alpha, NULL, F, H);
}

/* ------------------------------------------------------------------------ *
 * Snapshot (block) pass mode -- the semantics the GPU path implements       *
 * (SURVEY §8a "Pass semantics", §8c step 3).  Pass p:                        *
 *   1. r_p = sum_i |F_i|  (|.| for signed P, reading §8c-Q9)    *
 *   2. stop if r_p < target (P:124 stops on r/(1-d) <= Target; BASELINE.json  *
 *      states the target on |F|_1 directly)                                  *
 *   3. S_p = [ i ascending : key_i > T_p ]  ("all i such that (F_n)_i *
 *      is above a threshold T_k are chosen"; strict, reading §8c-Q7; key_i =   *
 *      |F_i| w_i, see orc_key_weights; raw key |F_i| when kw = NULL)          *
 *   4. for i in S_p: s_i = F_i; F_i = 0; H_i += s_i                           *
 *   5. for i in S_p ascending, for each child j: F_j += s_i * p_ji            *
 *      (this is eq. defF with J_S = sum_{i in S_p} J_i, a valid D-iteration by  *
 *      P:93-94 since every node with fluid is selected as T_p -> 0)            *
 *   6. T_{p+1}: GEOM  T/alpha every pass ("scale down the threshold *
 *      progressively by a factor alpha", "T_k \= alpha" read as T_k /= alpha, *
 *      §8c-Q6);  HYBRID(f)  T/alpha iff |S_p| <= f N, else unchanged (§8c-Q4). *
 * The log records (p, T_p, r_p, |S_p|, E_p = sum_{i in S_p} #out_i, dangling   *
 * takes).  E_p counts elementary diffusions.                     *
 * ------------------------------------------------------------------------ */
int orc_dit_snapshot_key(int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                         const double *vals, double d, double target, int32_t policy,
                         double alpha, double hybrid_frac, int64_t max_passes, const float *kw,
                         double *F, double *H, double *T_io, int64_t *pass_io,
                         orc_pass_log *log, int64_t log_cap, int64_t *edges_io) {
  if (n < 1 || !(alpha > 1.0) || !(d > 0.0 && d < 1.0)) return ORC_ERR_ARG;
  int32_t *S = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  double *s = (double *)malloc(sizeof(double) * (size_t)n);
  if (!S || !s) { free(S); free(s); return ORC_ERR_OOM; }
  double T = *T_io;
  int64_t p = *pass_io;
  int rc = ORC_ERR_NOT_CONVERGED;
  for (int64_t it = 0; it < max_passes; ++it) {
    /* 1. residual */
    double r = orc_l1(n, F);
    /* 2. stop test */
    if (r < target) { rc = ORC_OK; break; }
    /* 3. selection */
    int64_t cnt = 0, E = 0, dang = 0;
    for (int64_t i = 0; i < n; ++i)
      if (sel_key(F, kw, i) > T) S[cnt++] = (int32_t)i;
    /* 4. take */
    for (int64_t k = 0; k < cnt; ++k) {
      int64_t i = S[k];
      s[k] = F[i];
      F[i] = 0.0;
      H[i] += s[k];
    }
    /* 5. push */
    for (int64_t k = 0; k < cnt; ++k) {
      int64_t i = S[k];
      int64_t deg = col_ptr[i + 1] - col_ptr[i];
      E += deg;
      if (deg == 0) ++dang;
      double w = vals ? 0.0 : pagerank_w(col_ptr, i, d);
      for (int64_t e = col_ptr[i]; e < col_ptr[i + 1]; ++e)
        F[row_idx[e]] += s[k] * (vals ? vals[e] : w);
    }
    if (log && p < log_cap) {
      log[p].pass = p; log[p].T = T; log[p].r = r;
      log[p].frontier = cnt; log[p].edges = E; log[p].dangling = dang;
    }
    *edges_io += E;
    /* 6. threshold */
    if (policy == ORC_GEOM) T = T / alpha;
    else if ((double)cnt <= hybrid_frac * (double)n) T = T / alpha;
    ++p;
  }
  *T_io = T;
  *pass_io = p;
  free(S); free(s);
  return rc;
}

int orc_dit_snapshot(int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                     const double *vals, double d, double target, int32_t policy,
                     double alpha, double hybrid_frac, int64_t max_passes,
                     double *F, double *H, double *T_io, int64_t *pass_io,
                     orc_pass_log *log, int64_t log_cap, int64_t *edges_io) {
  return orc_dit_snapshot_key(n, col_ptr, row_idx, vals, d, target, policy, alpha, hybrid_frac,
                              max_passes, NULL, F, H, T_io, pass_io, log, log_cap, edges_io);
}

/* ------------------------------------------------------------------------ *
 * Sequential (literal pseudo-code) mode: P:116-134 with the cyclic threshold   *
 * test of P:213-219: scan i = 0..N-1 cyclically, diffuse i at once when       *
 * |F_i| > T (later nodes see its pushes in the same cycle); after a full     *
 * cycle without any diffusion, T /= alpha.  r is recomputed once per  *
 * cycle ("we don't have to compute r in each step").  Used only to  *
 * show order-independence of the limit.                            *
 * ------------------------------------------------------------------------ */
int orc_dit_sequential(int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                       const double *vals, double d, double target, double alpha,
                       int64_t max_cycles, double *F, double *H, double *T_io,
                       int64_t *ops_io) {
  if (n < 1 || !(alpha > 1.0)) return ORC_ERR_ARG;
  double T = *T_io;
  for (int64_t c = 0; c < max_cycles; ++c) {
    double r = orc_l1(n, F);
    if (r < target) { *T_io = T; return ORC_OK; }
    int any = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (fabs(F[i]) > T) {
        *ops_io += orc_diffuse_node(n, col_ptr, row_idx, vals, d, i, F, H);
        any = 1;
      }
    }
    if (!any) T = T / alpha;
  }
  *T_io = T;
  return ORC_ERR_NOT_CONVERGED;
}

/* ------------------------------------------------------------------------ *
 * Fixed-point (Richardson / "Jacobi", reading §8c-Q16) iteration for          *
 * X = P X + B: X_0 = 0, X_{t+1} = P X_t + B, until                 *
 * |X_{t+1} - X_t|_1 <= tol.  Converges when rho(P) < 1.            *
 * ------------------------------------------------------------------------ */
int orc_jacobi(int64_t n, const int64_t *col_ptr, const int32_t *row_idx, const double *vals,
               double d, const double *b, double tol, int64_t max_iter, double *X,
               int64_t *iters_out) {
  double *Y = (double *)malloc(sizeof(double) * (size_t)n);
  if (!Y) return ORC_ERR_OOM;
  for (int64_t i = 0; i < n; ++i) X[i] = 0.0;
  int rc = ORC_ERR_NOT_CONVERGED;
  int64_t t;
  for (t = 0; t < max_iter; ++t) {
    for (int64_t i = 0; i < n; ++i) Y[i] = b[i];
    for (int64_t j = 0; j < n; ++j) {
      double w = vals ? 0.0 : pagerank_w(col_ptr, j, d);
      for (int64_t e = col_ptr[j]; e < col_ptr[j + 1]; ++e)
        Y[row_idx[e]] += (vals ? vals[e] : w) * X[j];
    }
    double delta = 0.0;
    for (int64_t i = 0; i < n; ++i) { delta += fabs(Y[i] - X[i]); X[i] = Y[i]; }
    if (delta <= tol) { ++t; rc = ORC_OK; break; }
  }
  if (iters_out) *iters_out = t;
  free(Y);
  return rc;
}

/* ------------------------------------------------------------------------ *
 * Dense solve of (I - P) X = B by Gaussian elimination with        *
 * partial pivoting (textbook; tiny N only).  A is built densely from CSC.    *
 * ------------------------------------------------------------------------ */
/* Gaussian elimination with partial pivoting on the dense n x n system A X = y
 * (A and y are overwritten). */
static int gauss_solve(int64_t n, double *A, double *y, double *X) {
  for (int64_t k = 0; k < n; ++k) {
    int64_t piv = k;
    for (int64_t i = k + 1; i < n; ++i)
      if (fabs(A[i * n + k]) > fabs(A[piv * n + k])) piv = i;
    if (A[piv * n + k] == 0.0) return ORC_ERR_SINGULAR;
    if (piv != k) {
      for (int64_t c = 0; c < n; ++c) { double t = A[k * n + c]; A[k * n + c] = A[piv * n + c]; A[piv * n + c] = t; }
      double t = y[k]; y[k] = y[piv]; y[piv] = t;
    }
    for (int64_t i = k + 1; i < n; ++i) {
      double f = A[i * n + k] / A[k * n + k];
      if (f == 0.0) continue;
      for (int64_t c = k; c < n; ++c) A[i * n + c] -= f * A[k * n + c];
      y[i] -= f * y[k];
    }
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double acc = y[i];
    for (int64_t c = i + 1; c < n; ++c) acc -= A[i * n + c] * X[c];
    X[i] = acc / A[i * n + i];
  }
  return ORC_OK;
}

int orc_dense_solve(int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                    const double *vals, double d, const double *b, double *X) {
  if (n < 1 || n > 4096) return ORC_ERR_ARG;
  double *A = (double *)calloc((size_t)(n * n), sizeof(double));
  double *y = (double *)malloc(sizeof(double) * (size_t)n);
  if (!A || !y) { free(A); free(y); return ORC_ERR_OOM; }
  for (int64_t i = 0; i < n; ++i) { A[i * n + i] = 1.0; y[i] = b[i]; }
  for (int64_t j = 0; j < n; ++j) {
    double w = vals ? 0.0 : pagerank_w(col_ptr, j, d);
    for (int64_t e = col_ptr[j]; e < col_ptr[j + 1]; ++e)
      A[(int64_t)row_idx[e] * n + j] -= (vals ? vals[e] : w);
  }
  int rc = gauss_solve(n, A, y, X);
  free(A); free(y);
  return rc;
}

/* Completed PageRank: the paper's "one may complete by 1/N" for a
 * node without out-link makes Q stochastic, Q' = Q + (1/N) 1 a^T (a marks the
 * dangling columns), and X' = d Q' X' + (1-d)/N 1 (eq. pr2 with V = 1/N).  Solved
 * here densely from that definition (n <= 4096); SURVEY App. A.4 shows
 * X' = X / |X|_1 for the fluid-leaves X the D-iteration computes. */
int orc_completed_pagerank_dense(int64_t n, const int64_t *col_ptr, const int32_t *row_idx, double d,
                                 double *X) {
  if (n < 1 || n > 4096 || !(d > 0.0 && d < 1.0)) return ORC_ERR_ARG;
  double *A = (double *)calloc((size_t)(n * n), sizeof(double));
  double *y = (double *)malloc(sizeof(double) * (size_t)n);
  if (!A || !y) { free(A); free(y); return ORC_ERR_OOM; }
  for (int64_t i = 0; i < n; ++i) { A[i * n + i] = 1.0; y[i] = (1.0 - d) / (double)n; }
  for (int64_t j = 0; j < n; ++j) {
    const int64_t deg = col_ptr[j + 1] - col_ptr[j];
    if (deg == 0) {
      for (int64_t i = 0; i < n; ++i) A[i * n + j] -= d / (double)n;     /* completion 1/N */
    } else {
      for (int64_t e = col_ptr[j]; e < col_ptr[j + 1]; ++e)
        A[(int64_t)row_idx[e] * n + j] -= d / (double)deg;
    }
  }
  int rc = gauss_solve(n, A, y, X);
  free(A); free(y);
  return rc;
}
