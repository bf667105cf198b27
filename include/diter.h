/*
 * diter.h -- C ABI of libditer.so, the B200 (sm_100a) D-iteration diffusion
 * sweep (D. Hong, "D-iteration: Evaluation of the Asynchronous Distributed
 * Computation", arXiv 1202.6168).
 *
 * Problem:  X = P X + B with spectral radius of P < 1.
 *   p_ij is the weight of the edge j -> i; column j of P holds the out-edges
 *   of j, stored as CSC.  PageRank: P = d Q,
 *   q_ij = 1/#out_j, B = (1-d) V, V uniform; a dangling column (#out_j = 0)
 *   stays zero, so its fluid leaves the system (BASELINE.json configs[1]).
 *
 * Method:  fluid F_0 = B, history H_0 = 0; a
 *   diffusion of node i does  sent = F_i; H_i += sent; F_i = 0;
 *   F_j += p_ji * sent  for every child j (eq. defF/defH).  The library runs
 *   it as snapshot passes: pass p selects S_p = {i : |F_i| > T_p} (cyclic
 *   threshold test), takes every i in S_p, then pushes
 *   their fluid (eq. defF with J_S = sum_{i in S_p} J_i), and lowers T by
 *   alpha per the threshold policy.  It stops when the
 *   residual |F|_1 falls below the caller's target; |X - H|_1 <= |F|_1/(1-d)
 *   (PAPER.md:104-107).
 *
 * Conventions (all functions):
 *   - Every function returns a di_status and never throws or aborts.
 *   - All array arguments of di_create / di_create_dist / helpers are HOST
 *     pointers, copied before the call returns; the caller keeps ownership.
 *     Output buffers are caller-owned (host unless the name says _device).
 *   - The library owns all device memory and its own CUDA stream.
 *   - A context is not thread-safe: one owner at a time.
 *   - Invalid inputs are rejected at create time (DI_ERR_INVALID_ARG /
 *     DI_ERR_CONTRACTION) and leave *out = NULL.
 *   - di_last_error(ctx) gives a message for the last failure on ctx, or on
 *     the calling thread when ctx == NULL.
 */
#ifndef DITER_H
#define DITER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define DI_API __attribute__((visibility("default")))
#else
#define DI_API
#endif

typedef struct di_ctx di_ctx;

typedef enum {
  DI_OK = 0,
  DI_ERR_INVALID_ARG = 1,   /* bad sizes, non-monotone col_ptr, row out of range, d not in (0,1) */
  DI_ERR_CONTRACTION = 2,   /* signed mode: some column has sum_i |p_ij| > d */
  DI_ERR_OOM = 3,           /* device or host allocation failed */
  DI_ERR_CUDA = 4,          /* CUDA runtime error (message in di_last_error) */
  DI_ERR_NCCL = 5,          /* NCCL error (distributed contexts) */
  DI_ERR_NOT_CONVERGED = 6, /* max_passes reached before the target; state stays valid and resumable */
  DI_ERR_STATE = 7,         /* call not valid in the context's current state */
  DI_ERR_UNSUPPORTED = 8    /* feature not built into this library */
} di_status;

/* Threshold policies for T_{p+1} (readings R4). */
enum {
  DI_POLICY_GEOM = 0,      /* T <- T/alpha after every pass (literal "scale down progressively") */
  DI_POLICY_HYBRID = 1     /* T <- T/alpha iff |S_p| <= hybrid_frac * N, else T unchanged */
};

/* Selection keys (readings R3, R20).  Pass p selects
   {i : |F_i| w_i > T_p} with fp32 weights w_i computed once at create in fp64 and
   rounded to nearest fp32; T_0 = max_i |B_i| w_i / alpha. */
enum {
  DI_KEY_RAW = 0,          /* w_i = 1 (BASELINE north_star "above a per-pass threshold") */
  DI_KEY_EDGE = 1,         /* w_i = 1 / (#out_i + 1): per-edge key, out-degree only */
  DI_KEY_PAPER = 2         /* w_i = 1 / ((#in_i + 1)(#out_i + 1)): the paper's argmax key
                              (PAPER.md:210); distributed ranks get the global in-degrees of
                              their rows by a reduce-scatter at create */
};

/* How a distributed rank pushes fluid along edges to rows it does not own. */
enum {
  DI_REMOTE_PER_DIFFUSION = 0,  /* every diffusion pushes its remote edges into the outbox
                                   (continuous s_k, PAPER.md:227 first bullet) */
  DI_REMOTE_INCREMENT = 1,      /* the scatter pushes local edges only; at an exchange round
                                   the remote edges get (H - H_old) p_ji and H_old := H
                                   (the paper's preferred variant) */
  DI_REMOTE_RECEIVER = 2        /* receiver computes: ship (j, H_j - H_old_j)
                                   once per peer owning rows of column j; receivers keep the
                                   remote in-edges of their rows (one setup all-to-all) and
                                   apply p_ij themselves; at most 64 ranks */
};

/* Exchange modes of distributed contexts. */
enum {
  DI_EXCHANGE_SYNC = 0,    /* exchange + merge after every pass (reproduces the 1-GPU passes) */
  DI_EXCHANGE_ASYNC = 1,   /* send when s_k > r_k / K (eq. send), shipped in a
                              bulk round every rank joins (counts, all-to-all-v, all-reduce) */
  DI_EXCHANGE_P2P = 2      /* the paper's asynchronous scheme without a barrier (PAPER.md:50-53,
                              223-256, 274-280, 516-521): each rank decides s_k > r_k / K on its
                              own and writes the records straight into its inbox ring in the
                              receiver's memory (CUDA IPC / NVLink, a system-scope release of the
                              ring head); receivers merge whatever has arrived at the start of
                              their next round.  Termination: a board of r_k + s_k + in-flight in
                              every rank's memory triggers a quiesce-then-reduce confirmation,
                              the only collectives of a run.  Needs remote_push =
                              DI_REMOTE_INCREMENT, adapt_rounds = 0, <= 64 ranks; di_rebalance is
                              not available.  Memory per rank: a compact outbox over the distinct
                              remote rows of its columns, and one inbox ring per peer holding one
                              message (the distinct rows that peer can send it) */
};

typedef struct {
  int32_t policy;          /* DI_POLICY_*; default HYBRID */
  int32_t check_interval;  /* passes per captured CUDA graph between host checks; default 16 */
  double alpha;            /* threshold factor alpha > 1; default 1.5 */
  double hybrid_frac;      /* HYBRID frontier fraction f; default 0.05 */
  double t0;               /* initial threshold; <= 0 means max_i |B_i| / alpha (reading R5) */
  int64_t max_passes;      /* guard -> DI_ERR_NOT_CONVERGED; default 1000000 */
  int32_t exchange_mode;   /* DI_EXCHANGE_*; distributed only; default ASYNC */
  int32_t device;          /* CUDA device ordinal; -1 = current device (default) */
  int32_t scatter_kernel;  /* reserved (0): the scatter grabs runs of frontier groups dynamically;
                              static CTA-tile and warp-interleave schedules measured 30 % slower */
  int32_t profile;         /* 1: time each kernel of each executed pass with CUDA events
                              recorded inside the captured graph (di_stats.kt_*); default 0 */
  int32_t pass_kernel;     /* 0 = auto (= 1), 1 = one kernel per phase, check_interval passes per captured
                              CUDA graph, 2 = one cooperative persistent kernel per 4 x check_interval
                              passes (grid barriers between phases; 1-GPU only) */
  int32_t hot_window;      /* 0 = stage the 2048 rows of largest in-degree in shared memory (default),
                              -1 = off (every push is an L2 RED) */
  int32_t scatter_run;     /* groups per dynamic grab of the scatter; 0 = default (2) */
  int32_t scatter_stripes; /* ticket stripes of the dynamic schedule, 1..32; 0 = default (8) */
  int32_t far_push;        /* far-push bins (propagation blocking, one GPU): 1 = on; 0 = auto (= off:
                              on C4 the record emission costs more than the L2-missing REDs it
                              removes; on a pure Zipf-over-id graph it wins, 18.2 -> 13.8 ms/pass);
                              -1 = off */
  int32_t far_warm_log2;   /* log2 of the warm row range kept on direct L2 REDs; 0 = default (21) */
  int32_t select_key;      /* DI_KEY_*; default DI_KEY_RAW */
  int32_t remote_push;     /* DI_REMOTE_*; distributed only; default DI_REMOTE_PER_DIFFUSION */
  int32_t receive_rescale; /* ASYNC only: after merging received fluid R, T_k <- T_k (r_k + R) / r_k
                              (reading R13); 1 = on (default), 0 = off */
  int32_t adapt_rounds;    /* ASYNC only: every adapt_rounds exchange rounds apply the paper's
                              partition adaptation (reading R22) -- a boundary
                              moves by 10 % of the busier side when its residual is > 2x and its
                              work since the last check > 1.2x the neighbour's; 0 = off (default) */
  int32_t l2_persist;      /* L2 persisting window over the rows of F that receive the most pushes
                              (from the create-time in-degree sample; the set-aside is per device,
                              refcounted over contexts): 0 = auto (off while F fits in 64 MB, else
                              28 MB when F <= 2x L2 and 20 MB above: C3 219 -> 184 ms, C4 265 ->
                              250 ms; with sweeps 36 / 28 MB), -1 = off, > 0 = a window of that
                              many MB */
  int32_t p2p_sleep;       /* DI_EXCHANGE_P2P: a rank whose local residual r_k is below target / K
                              sleeps: its rounds only merge, send and measure,
                              no local passes, until received fluid lifts r_k again; 0 = on
                              (default), -1 = off; k > 0 = also asleep while r_k is below k % of
                              the rank's even share (1 / K) of the fluid on the board (every
                              rank's r + s + in flight as last published) */
  int32_t far_defer;       /* one GPU, PageRank: far-edge deferral -- a column's
                              edges to rows more than 2048 ids away and outside the L2 persisting
                              window (else the shared-memory hot window) are pushed not at every
                              diffusion but every far_defer passes, as (H_i - H_old_i) p_ji (the
                              paper's increment push); a run stops on
                              |F|_1 + pending and only with nothing pending.  Same fixed point X
                              (P:93-94), another pass schedule.  0 = off (default: slower on C4 at
                              every cadence measured), > 0 = passes between flushes */
  int32_t sweep;           /* one GPU: 1 = one-kernel asynchronous sweeps (reading R26) --
                              the paper's cyclic scan with immediate diffusion (PAPER.md:116-134,
                              213-216) run by the whole grid: each node above T_p is taken
                              (atomic exchange of F_i) and diffused at once, its pushes visible to
                              nodes scanned later in the same sweep; no frontier list.  Same fixed
                              point X; the pass log is per sweep and not the snapshot
                              oracle's.  0 = snapshot passes (select, then scatter; default) */
  int32_t key_offset;      /* sweeps with select_key = DI_KEY_EDGE: the key the sweep derives from
                              col_ptr is |F_i| / (#out_i + c) with c = key_offset; 0 = default
                              (c = 1, the per-edge key).  A larger c charges a node's take like c
                              pushes (cost-aware variant of the weighting heuristic, PAPER.md:208-212;
                              DESIGN.md reading R27); any c reaches the same X */
} di_options;

/* One record per executed pass (device-logged, read with di_get_pass_log). */
typedef struct {
  int64_t pass;            /* p */
  double T;                /* T_p used for the selection */
  double r;                /* r_p = |F|_1 (local part if distributed) before the pass */
  int64_t frontier;        /* |S_p| (all bins, dangling included) */
  int64_t edges;           /* E_p = sum_{i in S_p} #out_i (elementary diffusions) */
  int64_t dangling;        /* nodes of S_p with #out = 0 */
  int64_t bin_low;         /* nodes of S_p with 1 <= #out <= 32      (32 per warp, edge-balanced) */
  int64_t bin_mid;         /* nodes of S_p with 33 <= #out <= 8192   (warp per node)    */
  int64_t bin_hub;         /* nodes of S_p with #out > 8192          (CTA per 2048-edge chunk) */
  double t_select_us;      /* profile=1: device time of k_select in this pass, else 0 */
  double t_scatter_us;     /* profile=1: device time of k_scatter in this pass, else 0 */
} di_pass_log;

typedef struct {
  int64_t passes;          /* passes executed since create */
  int64_t edges;           /* elementary diffusions since create (sum of E_p); distributed: this
                              rank's under ASYNC, all ranks' under SYNC (whose pass totals are
                              all-reduced every pass) -- likewise nodes */
  int64_t nodes;           /* node diffusions since create (sum of |S_p|) */
  double residual;         /* last measured/predicted |F|_1 (exact after di_get_residual) */
  double threshold;        /* current T */
  double run_ms;           /* device time of the last di_run (CUDA events on the library stream) */
  double run_ms_total;     /* summed over all di_run calls */
  int64_t alg_bytes;       /* algorithmic bytes moved since create: 8 N_scan + 40 |S| + 20 E (+8 E signed) */
  int64_t exchanged_bytes; /* payload bytes sent to peers since create (distributed) */
  int64_t exchanges;       /* number of outbox flushes (distributed) */
  int64_t n_local;         /* nodes owned by this context */
  int64_t nnz_local;       /* stored edges owned by this context */
  int64_t graph_launches;  /* CUDA graph launches by di_run since create */
  int64_t kernel_launches; /* kernels launched by the library since create (counting graph nodes) */
  double kt_select_ms;     /* profile=1: summed device time of k_select over executed passes */
  double kt_scatter_ms;    /* profile=1: summed device time of k_scatter over executed passes */
  double kt_finalize_ms;   /* profile=1: summed device time of k_finalize over executed passes */
  int64_t kt_passes;       /* profile=1: executed passes those sums cover */
  int64_t scatter_bytes;   /* algorithmic bytes of the scatter kernel since create: 20 E (28 E signed)
                              + 16 per non-dangling diffused node (its col_ptr pair) */
  int64_t remote_pushes;   /* distributed: pushes into the remote outbox since create (one RED per
                              remote edge per diffusion, or per column increment with
                              DI_REMOTE_INCREMENT; the receiver's in-edge adds with
                              DI_REMOTE_RECEIVER) */
  int64_t rebalances;      /* distributed: ownership changes (di_rebalance / adapt_rounds) */
  int64_t l2_window_bytes; /* L2 persisting window over F chosen at create (options.l2_persist), 0 = none */
  int64_t l2_window_row;   /* its first row (global id) */
  int64_t dangling;        /* dangling node diffusions since create (in nodes; taken by the select,
                              their fluid leaves; the scatter never reads their col_ptr) */
  int64_t run_kernel_launches; /* kernels launched by the last di_run (graph nodes counted, including
                              passes of a graph launch that return at once after convergence) */
  int64_t collectives;     /* distributed: fabric collectives (all-reduce, all-to-all, ...) since create,
                              setup included -- one or more per round under SYNC / ASYNC, only at
                              termination confirmations under P2P */
  int64_t confirms;        /* DI_EXCHANGE_P2P: quiesce-then-reduce confirmations run since create */
  int64_t exchange_bytes_resident; /* distributed: device bytes of the exchange state (outbox, flags,
                              record buffers or inbox rings) */
  int64_t sleep_rounds;    /* DI_EXCHANGE_P2P: rounds this rank spent asleep since create */
  int64_t far_flushes;     /* far-edge deferral: flushes of the far-edge increments since create */
  int64_t far_edges;       /* far-edge deferral: edges deferred to the flushes (0 = deferral off) */
} di_stats;

/* Fill *opt with the defaults above. */
DI_API void di_default_options(di_options *opt);

/* sizeof of the ABI structs as compiled into the library (which: 0 = di_options,
 * 1 = di_stats, 2 = di_pass_log; anything else returns 0), so a binding can check
 * its own layout against the library's. */
DI_API size_t di_struct_size(int32_t which);

/* Single-GPU context.  n nodes; col_ptr[n+1] (int64, col_ptr[0] = 0,
 * non-decreasing, col_ptr[n] = nnz); row_idx[nnz] (int32 in [0,n)).
 *  values == NULL -> PageRank mode: p_ji = d / #out_i for each stored edge,
 *                    derived on the device from col_ptr (never stored).
 *  values != NULL -> signed mode: p_ji = values[e]; d is the contraction
 *                    factor of the bound; validated: max_j sum_i |p_ij| <= d < 1.
 *  b == NULL -> B_i = (1-d)/n; else b[n] is copied.
 * Duplicate rows within a column are allowed (they add). */
DI_API di_status di_create(di_ctx **out, int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                    const double *values, const double *b, double d, const di_options *opt);

/* Distributed context, one call per rank (collective).  This rank owns the
 * node range [bounds[rank], bounds[rank+1]) (PID_k computes
 * [F]_k and [H]_k), and the columns of that range:
 * col_ptr_local[hi-lo+1] (starting at 0), row_idx_local with GLOBAL row ids.
 * bounds[world+1] must be identical on all ranks (di_partition_cb).
 * comm_id (128 bytes) selects the fabric of the collectives:
 *   - an ncclUniqueId created by rank 0 (di_get_unique_id) and broadcast by the
 *     caller: NCCL, one GPU per rank (DI_ERR_UNSUPPORTED if built without NCCL);
 *   - "DILOOP01" + key: K contexts of ONE process (host threads), host-side
 *     collectives, any devices (tests: K ranks on one GPU);
 *   - "DISHM001" + name: K processes of one host through POSIX shared memory,
 *     host-side collectives, no bulk all-to-all-v (use DI_EXCHANGE_P2P; its
 *     windows are mapped with CUDA IPC).
 * A failure of one rank inside a collective sequence releases its peers with
 * DI_ERR_STATE (loopback / shared memory) instead of leaving them waiting. */
DI_API di_status di_create_dist(di_ctx **out, int32_t rank, int32_t world, const void *comm_id,
                         const int64_t *bounds, int64_t n_global,
                         const int64_t *col_ptr_local, const int32_t *row_idx_local,
                         const double *values_local, const double *b_local, double d,
                         const di_options *opt);

/* 128-byte ncclUniqueId for di_create_dist (call on rank 0 only). */
DI_API di_status di_get_unique_id(void *comm_id_out);

/* Reset the state to F = B, H = 0, T = T_0 keeping the
 * uploaded graph, and clear the pass counters, the pass log and the stats, so
 * the next di_run solves from scratch.  Collective for distributed contexts. */
DI_API di_status di_reset(di_ctx *ctx);

/* Checkpoint / resume: load a state (F, H) -- host arrays of n (or hi-lo when
 * distributed) doubles, e.g. from di_get_fluid / di_get_history of an earlier run
 * on the same (P, B) -- and restart the schedule from it: the counters, pass log
 * and stats are cleared as by di_reset, T = max_i |F_i| w_i / alpha (reading R5
 * applied to the loaded F; a max over ranks when distributed), nothing in flight
 * (remote increments start from H).  The caller vouches that F = B - (I - P) H (the
 * identity every D-iteration state satisfies): the solve then
 * converges to the same X.  Collective for distributed contexts. */
DI_API di_status di_set_state(di_ctx *ctx, const double *f_in, const double *h_in);

/* Switch per-kernel timing on (1) or off (0) for the following di_run calls:
 * with it on, CUDA events recorded between the pass kernels give the select /
 * scatter / finalize durations in di_stats (kt_*_ms) and the pass log, at a cost
 * of ~25 us of device time per pass (the events split the captured pass graph);
 * the single-GPU pass graph is re-captured.  Same as options.profile at create.
 * Not collective. */
DI_API di_status di_set_profile(di_ctx *ctx, int32_t on);

/* Run passes until |F|_1 < residual_target (absolute; global if distributed).
 * Resumable: call again with a smaller target to continue from (F, H).
 * Collective for distributed contexts.  Returns DI_OK when the target is met,
 * DI_ERR_NOT_CONVERGED when max_passes was reached first. */
DI_API di_status di_run(di_ctx *ctx, double residual_target);

/* Copy H (n, or hi-lo when distributed) into the caller's host buffer. */
DI_API di_status di_get_history(const di_ctx *ctx, double *h_out);
/* Copy F likewise (for invariant checks, e.g. F = B - (I-P) H). */
DI_API di_status di_get_fluid(const di_ctx *ctx, double *f_out);
/* Device-to-device variants: d_out is a device pointer on the context's device. */
DI_API di_status di_get_history_device(const di_ctx *ctx, double *d_out);
DI_API di_status di_get_fluid_device(const di_ctx *ctx, double *d_out);
/* Completed PageRank ("one may complete by 1/N"):
 * with dangling fluid leaving, the completed solution is X' = X / |X|_1, so this
 * writes H_i / |H|_1 (|H|_1 by a deterministic reduction, global if distributed;
 * collective then) into the caller's host buffer (n, or hi-lo when distributed).
 * Defined for PageRank contexts with the default B = (1-d)/N (values == NULL and
 * b == NULL at create): A.4 needs B proportional to the completion vector V = 1/N;
 * any other context returns DI_ERR_STATE.  H approximates X within |F|_1/(1-d)
 * (P:104-107).  The device variant writes a device pointer. */
DI_API di_status di_get_pagerank(di_ctx *ctx, double *x_out);
DI_API di_status di_get_pagerank_device(di_ctx *ctx, double *d_out);
/* Exact |F|_1 by a deterministic two-level reduction (global if distributed;
 * collective then).  Also refreshes stats.residual. */
DI_API di_status di_get_residual(di_ctx *ctx, double *r_out);
DI_API di_status di_get_stats(const di_ctx *ctx, di_stats *s);
/* Distributed: move node ownership to new_bounds[world+1] (0 = b_0 < ... < b_world = N,
 * the same array on every rank; collective).  Everything in flight is delivered
 * first; each moved node's column (rows, values), F, H and B travel to its new owner,
 * which rebuilds its device state over the new range and keeps T, the pass counters
 * and the statistics ("we just need to transmit the information F_n
 * and H_n of the candidate nodes").  Call between di_run calls, or let di_run do it
 * with options.adapt_rounds. */
DI_API di_status di_rebalance(di_ctx *ctx, const int64_t *new_bounds);
/* Current ownership bounds: world+1 entries (distributed) or {0, N}. */
DI_API di_status di_get_bounds(const di_ctx *ctx, int64_t *out);
/* Copy pass records [first, first+count) into out; *n_copied receives the
 * number copied (passes beyond the log capacity are not recorded). */
DI_API di_status di_get_pass_log(const di_ctx *ctx, int64_t first, int64_t count, di_pass_log *out,
                          int64_t *n_copied);
DI_API const char *di_last_error(const di_ctx *ctx);
DI_API void di_destroy(di_ctx *ctx);

/* ---- setup helpers (integer work, bit-exact against the oracle) ---- */

/* COO (src[e] -> dst[e]) to CSC on the GPU: sort by (src, dst), drop
 * duplicates, histogram + scan -> col_ptr[n+1]; row_idx must hold m entries;
 * *nnz_out receives the deduplicated count.  Host pointers. (
 * BASELINE.json configs[2] "duplicate edges dropped") */
DI_API di_status di_csc_from_coo(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                          int64_t *col_ptr, int32_t *row_idx, int64_t *nnz_out);

/* Cost-balanced contiguous partition (reading R10):
 * bounds[0] = 0, bounds[K] = n, bounds[k] = min{i : C[i] >= ceil(k C[n] / K)}
 * forced strictly increasing, where C = cost_prefix[n+1] (e.g. col_ptr). */
DI_API di_status di_partition_cb(int64_t n, const int64_t *cost_prefix, int32_t K, int64_t *bounds);

#ifdef __cplusplus
}
#endif
#endif /* DITER_H */
