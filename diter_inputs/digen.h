/* digen.h -- seeded synthetic input generators (shared input plumbing only).
 * See digen.c for the recipes; DESIGN.md "Input recipe" for the citations. */
#ifndef DIGEN_H
#define DIGEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { DG_OK = 0, DG_ERR_ARG = 1, DG_ERR_OOM = 2 };
enum { DG_UNIFORM = 1, DG_WEB = 2, DG_RMAT = 3, DG_SIGNED = 5 };

typedef struct {
  int32_t kind;          /* DG_* */
  int32_t _pad0;
  int64_t n;             /* number of nodes */
  uint64_t seed;
  /* DG_UNIFORM */
  int32_t deg_lo, deg_hi;
  /* DG_WEB */
  double x_min, p_dangling, p_local;
  int32_t window, max_deg;
  /* DG_SIGNED */
  int32_t nnz_per_col, _pad1;
  double col_abs_sum;
  /* DG_RMAT */
  int32_t scale, edge_factor;
  double a, b, c;
} dg_params;

int dg_validate(const dg_params *p);
/* CSC kinds (uniform, web, signed): pass 1 fills col_ptr[n+1]; pass 2 fills
 * row_idx[col_ptr[n]] (and vals for DG_SIGNED, may be NULL otherwise). */
int dg_csc_count(const dg_params *p, int64_t *col_ptr);
int dg_csc_fill(const dg_params *p, const int64_t *col_ptr, int32_t *row_idx, double *vals);
/* DG_SIGNED right-hand side B_i ~ U[-1,1] */
int dg_b_signed(const dg_params *p, double *b);
/* R-MAT raw COO samples (duplicates kept): src[m], dst[m], m = dg_rmat_edges(p) */
int64_t dg_rmat_edges(const dg_params *p);
int dg_rmat_fill(const dg_params *p, int32_t *src, int32_t *dst);
int dg_num_threads(void);
void dg_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
