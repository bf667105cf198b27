// types.cuh -- plain data shared between the host code and the kernels.
#pragma once
#include <cstdint>
#include <vector_types.h>

namespace diter {

// Degree classes (edges of the column = #out_i).
constexpr int kLowMax = 32;      // 1..32     : "low"  (statistics only; same warp path as mid)
constexpr int kMidMax = 8192;    // 33..8192  : "mid"  -- both: 32 selected nodes per warp,
                                 //             lanes over the group's concatenated edges
constexpr int kHubChunk = 2048;  // > 8192    : "hub"  -- one CTA per 2048-edge chunk
constexpr int kHot = 2048;       // rows staged in shared memory by each scatter CTA

constexpr int kSelectThreads = 256;
constexpr int kSelectItems = 8;                      // 32-node words per warp iteration
constexpr int kScatterThreads = 256;
constexpr int kFinalizeThreads = 512;
constexpr int kWordsPerSuper = 32;                   // bitmap words per scatter superword (1024 nodes)

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
  unsigned long long hub_packed;  // (hub slots << 32) | hub chunks; reset by k_finalize
  long long log_cap;
  unsigned sc_next;    // next superword chunk for the scatter's dynamic schedule (reset per pass)
  int _pad;
  double t_sel_us;     // fused kernel: accumulated select / scatter phase time (%globaltimer)
  double t_sc_us;
};

// k_select partials (one per CTA): r_p and |S_p|.
struct SelPartial {
  double r;
  long long cnt;
};

// k_scatter partials (one per CTA): guaranteed |F|_1 drop and frontier census.
struct ScPartial {
  double loss;      // sum over taken nodes of (1 - c_i)|s_i|, c_i = d (0 if dangling)
  long long edges;  // E_p
  int dang, n_low, n_mid, n_hub;
};

struct Graph {
  const long long *col_ptr;  // [n+1] owned columns, local (starting at 0)
  const int *row_idx;        // [nnz] GLOBAL row ids
  const double *vals;        // [nnz] or nullptr (PageRank)
  long long n;               // owned nodes (n_local)
  double d;
  int hot_lo;                // global id of the shared-memory hot window start
  long long lo;              // first owned global id (0 on one GPU)
  double *G;                 // remote outbox over global ids, or nullptr on one GPU
  unsigned char *dflags;     // dirty flag per 32-row block of G
};

// Frontier of one pass: selection bitmap (bit i%32 of word i/32) and the taken
// values s_i (valid where the bit is set); hubs go to a separate list.
struct Frontier {
  unsigned *bits;        // [n_words_pad]
  double *S;             // [n]
  long long n_words;     // ceil(n / 32)
  double *hub_w;         // push value per edge of the hub (s d/#out or s)
  long long *hub_b0;
  long long *hub_deg;
  unsigned *hub_chunk;   // first 2048-edge chunk id of the hub (prefix in slot order)
};

// Validation + degree census in one pass over the columns.
struct Census {
  unsigned long long bad_ptr;     // non-monotone col_ptr
  unsigned long long bad_row;     // row out of range
  unsigned long long n_low, n_mid, n_hub, n_dang;
  unsigned long long bad_contraction;  // signed: column |.|-sum > d
  double max_abs_b;
};

}  // namespace diter
