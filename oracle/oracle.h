/* oracle.h -- CPU oracle of the D-iteration sweep.  TEST INFRASTRUCTURE ONLY:
 * see the header of oracle.c.  Not included by, and does not include, any
 * file of the CUDA path. */
#ifndef DITER_ORACLE_H
#define DITER_ORACLE_H
#include <stdint.h>

enum { ORC_OK = 0, ORC_ERR_ARG = 1, ORC_ERR_OOM = 2, ORC_ERR_NOT_CONVERGED = 3, ORC_ERR_SINGULAR = 4 };
enum { ORC_GEOM = 0, ORC_HYBRID = 1 };
enum { ORC_KEY_RAW = 0, ORC_KEY_EDGE = 1, ORC_KEY_PAPER = 2 };

typedef struct {
  int64_t pass;      /* p */
  double T;          /* T_p */
  double r;          /* r_p = |F|_1 before the pass */
  int64_t frontier;  /* |S_p| */
  int64_t edges;     /* E_p = sum of #out over S_p */
  int64_t dangling;  /* dangling nodes in S_p */
} orc_pass_log;

int orc_csc_from_coo(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                     int64_t *col_ptr, int32_t *row_idx, int64_t *nnz_out);
int orc_partition_uniform(int64_t n, int32_t K, int64_t *bounds);
int orc_partition_cb(int64_t n, const int64_t *cost_prefix, int32_t K, int64_t *bounds);
int64_t orc_diffuse_node(int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                         const double *vals, double d, int64_t i, double *F, double *H);
double orc_l1(int64_t n, const double *v);
double orc_init(int64_t n, const double *b, double alpha, double *F, double *H);
int orc_key_weights(int64_t n, const int64_t *col_ptr, const int32_t *row_idx, int32_t key, float *w);
double orc_init_key(int64_t n, const double *b, double alpha, const float *kw, double *F, double *H);
int orc_dit_snapshot_key(int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                         const double *vals, double d, double target, int32_t policy,
                         double alpha, double hybrid_frac, int64_t max_passes, const float *kw,
                         double *F, double *H, double *T_io, int64_t *pass_io,
                         orc_pass_log *log, int64_t log_cap, int64_t *edges_io);
int orc_dit_snapshot(int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                     const double *vals, double d, double target, int32_t policy,
                     double alpha, double hybrid_frac, int64_t max_passes,
                     double *F, double *H, double *T_io, int64_t *pass_io,
                     orc_pass_log *log, int64_t log_cap, int64_t *edges_io);
int orc_dit_sequential(int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                       const double *vals, double d, double target, double alpha,
                       int64_t max_cycles, double *F, double *H, double *T_io,
                       int64_t *ops_io);
int orc_jacobi(int64_t n, const int64_t *col_ptr, const int32_t *row_idx, const double *vals,
               double d, const double *b, double tol, int64_t max_iter, double *X,
               int64_t *iters_out);
int orc_dense_solve(int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                    const double *vals, double d, const double *b, double *X);
int orc_completed_pagerank_dense(int64_t n, const int64_t *col_ptr, const int32_t *row_idx, double d,
                                 double *X);
#endif
