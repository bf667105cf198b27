// types.cuh -- plain data shared between the host code and the kernels.
#pragma once
#include <cstdint>

namespace diter {

// Degree bins (edges of the column = #out_i).
constexpr int kLowMax = 32;      // 1..32     : thread per node
constexpr int kMidMax = 2048;    // 33..2048  : warp per node
constexpr int kHubChunk = 2048;  // > 2048    : one CTA per 2048-edge chunk of the column

constexpr int kSelectThreads = 256;
constexpr int kScatterThreads = 256;
constexpr int kFinalizeThreads = 512;

// Device-resident control block of one context.
struct Ctl {
  double T;            // current threshold T_p
  double r;            // r_p measured by the last executed pass
  double r_pred;       // upper bound on the current |F|_1 (exact before the first pass)
  double target;       // residual target of the current di_run
  double alpha;
  double hybrid_frac;
  double n_total;      // N as a double, for the HYBRID rule |S_p| <= f N
  long long pass;      // passes executed since create
  long long max_pass;  // run stops with done = 2 when pass reaches this
  long long edges;     // cumulative E_p
  long long nodes;     // cumulative |S_p|
  int done;            // 0 running, 1 converged, 2 max passes reached
  int policy;          // DI_POLICY_*
  unsigned n_low;      // per-pass bin counters (reset by k_finalize)
  unsigned n_mid;
  unsigned long long hub_packed;  // (hub slots << 32) | hub chunks
  long long log_cap;
};

struct Partial {
  double r;       // sum |F_i| over the block's nodes (before the take)
  double loss;    // guaranteed |F|_1 decrease: sum (1 - c_i)|s_i|
  long long edges;
  int cnt;
  int dang;
};

struct Graph {
  const long long *col_ptr;  // [n+1]
  const int *row_idx;        // [nnz]
  const double *vals;        // [nnz] or nullptr (PageRank)
  long long n;
  double d;
};

struct Bins {
  int *low_idx;
  double *low_w;
  int *mid_idx;
  double *mid_w;
  int *hub_idx;
  double *hub_w;
  unsigned *hub_chunk;
};

// Validation + degree-bin census in one pass over the columns.
struct Census {
  unsigned long long bad_ptr;     // non-monotone col_ptr
  unsigned long long bad_row;     // row out of range
  unsigned long long n_low, n_mid, n_hub, n_dang;
  unsigned long long bad_contraction;  // signed: column |.|-sum > d
  double max_abs_b;
};

}  // namespace diter
