// ctx.cuh -- the opaque di_ctx behind include/diter.h (host-side layout).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/diter.h"
#include "types.cuh"

struct DistState;  // dist.cu

// NVTX range over a host-side phase (create, run, exchange round, confirmation):
// visible in nsys / ncu timelines; free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

struct di_ctx {
  // problem
  long long n_rows = 0;     // N (global)
  long long n_local = 0;    // owned nodes (= N on one GPU)
  long long nnz_local = 0;  // stored edges of the owned columns
  long long lo = 0;         // first owned node id
  int hot_lo = 0;           // shared-memory hot window of the scatter (global row id)
  double d = 0.85;
  di_options opt{};
  int check_interval = 16;
  int device = -1;
  int rank = 0, world = 1;

  // device state (HBM)
  long long *col_ptr = nullptr;  // [n_local+1]
  int *row_idx = nullptr;        // [nnz_local] global row ids
  double *vals = nullptr;        // [nnz_local] signed mode only
  double *d_b = nullptr;         // B [n_local] when given (kept for di_reset)
  double *F = nullptr;           // fluid [n_local]
  double *G = nullptr;           // remote outbox over global ids (distributed only)
  unsigned char *dflags = nullptr;  // dirty flag per 32-row block of G
  double *H = nullptr;           // history [n_local]
  float *kw = nullptr;           // selection-key weights [n_local] (nullptr = raw key |F_i|)
  int *nloc = nullptr;           // distributed: local (owned-row) edges per column, stored first
  double *H_old = nullptr;       // DI_REMOTE_INCREMENT: H at the last push of the remote edges
  long long remote_pushes = 0;   // pushes into the outbox since create
  long long rebalances = 0;      // di_rebalance calls that moved ownership (distributed)
  diter::Frontier fr{};
  diter::Far far{};               // far-push bins (propagation blocking), 1 GPU
  long long *far_off = nullptr;   // [n_bins + 1] first chunk of each bin (device)
  long long far_cap = 0;          // total chunks
  long long l2_lo = 0, l2_bytes = 0;   // L2 persisting window over F (rows from l2_lo), 0 = none
  std::vector<unsigned> blk_hist; // sampled in-degree per 1024-row block (setup)
  int blk_stride = 1;
  unsigned long long cap_low = 0, cap_mid = 0, cap_hub = 0;
  diter::SelPartial *sel_part = nullptr;
  diter::ScPartial *sc_part = nullptr;
  double *l1_part = nullptr;
  double *l1_out = nullptr;
  diter::Ctl *ctl = nullptr;
  di_pass_log *log = nullptr;
  long long log_cap = 0;

  // launch
  cudaStream_t stream = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int num_sms = 0, grid_select = 0, grid_scatter = 0, grid_l1 = 0, grid_fused = 0, grid_hubs = 0;
  size_t scatter_smem = 0;  // dynamic shared memory of the scatter: group prefix over segments
  bool fused = false;
  void *h_ctl = nullptr;  // pinned mirror of Ctl
  diter::Ctl ctl_init{};  // control block right after create (di_reset restores it)
  double b_uniform = 0.0;
  std::vector<cudaEvent_t> prof_ev;  // profile=1: 4 events per captured pass

  // stats
  long long passes_done = 0, edges = 0, nodes = 0, dang = 0;
  long long graph_launches = 0, kernel_launches = 0;
  long long run_kernel_launches = 0;   // kernels launched by the last di_run
  long long exchanged_bytes = 0, exchanges = 0, alg_bytes_exchange = 0;
  double residual = 0.0, threshold = 0.0, run_ms = 0.0, run_ms_total = 0.0;
  double kt_ms[3] = {0.0, 0.0, 0.0};
  long long kt_passes = 0;
  std::vector<std::pair<double, double>> pass_us;  // profile=1: (select, scatter) us per pass

  // far-edge deferral (defer.cu; one GPU, PageRank): nloc = near edges per column
  int defer_m = 0;                // passes between flushes (0 = off)
  int sweep_on = 0;               // one-kernel async sweeps (options.sweep)
  int grid_sweep = 0;
  long long far_edges = 0;        // edges deferred to the flushes
  long long far_flushes = 0;

  DistState *dist = nullptr;
  std::string err;
};

void diter_set_err(di_ctx *ctx, const char *fmt, ...);
// local part of a create: upload, validation, buffers (no collective; may fail on
// one rank only)
di_status diter_setup(di_ctx *ctx, const int64_t *col_ptr, const int32_t *row_idx,
                      const double *values, const double *b, const di_options *opt);
// collective tail: paper-key in-degrees, T_0, control block, captured graph
di_status diter_setup_finish(di_ctx *ctx);
di_status diter_l1_launch(di_ctx *ctx);
di_status diter_l1_launch_of(di_ctx *ctx, const double *v);
diter::Graph diter_graph(const di_ctx *ctx);

// distributed hooks (dist.cu); identities / no-ops on single-GPU contexts
void diter_dist_free(di_ctx *ctx);
// the context's L2 persisting window (options.l2_persist) as its stream's access policy
di_status diter_set_l2_window(di_ctx *ctx);
// context device memory (per-device stream-ordered pool, ordered on ctx->stream)
di_status diter_alloc(di_ctx *ctx, void **p, size_t bytes);
void diter_free(di_ctx *ctx, void *p);
// max / sum of one host double over the ranks (identity when not distributed); collective
di_status diter_dist_max(di_ctx *ctx, double v, double *out);
di_status diter_dist_sum(di_ctx *ctx, double v, double *out);
di_status diter_dist_indegree(di_ctx *ctx, unsigned *indeg_local);   // DI_KEY_PAPER, collective
di_status diter_dist_run(di_ctx *ctx, double target);
void diter_dist_stats(const di_ctx *ctx, di_stats *s);   // collectives, confirmations, exchange memory
void diter_dist_pass_prologue(di_ctx *ctx);               // kernels before each pass (P2P: inbox merge)
di_status diter_capture_graph(di_ctx *ctx);               // (re)capture check_interval passes as a graph
di_status diter_dist_reset(di_ctx *ctx);
// far-edge deferral (defer.cu): setup after the upload, the flush pair of a pass, a
// host-driven flush
di_status diter_setup_defer(di_ctx *ctx);
void diter_defer_launch(di_ctx *ctx);
di_status diter_defer_flush_now(di_ctx *ctx, int done);
// per-CTA partial counts a pass's k_finalize reduces (the sweep grid when sweeps run)
inline int diter_n_sel_part(const di_ctx *ctx) { return ctx->sweep_on ? ctx->grid_sweep : ctx->grid_select; }
inline int diter_n_sc_part(const di_ctx *ctx) { return ctx->sweep_on ? ctx->grid_sweep : ctx->grid_scatter; }
// one sweep of a distributed rank (dist.cu's non-graph pass path)
void diter_launch_sweep(di_ctx *ctx);
