// types.cuh -- plain data shared between the host code and the kernels.
#pragma once
#include <cstdint>
#include <vector_types.h>

namespace diter {

// Degree classes (edges of the column = #out_i).
constexpr int kLowMax = 32;      // 1..32     : "low"  (statistics only; same warp path as mid)
#ifndef DITER_MID_MAX
#define DITER_MID_MAX 8192
#endif
constexpr int kMidMax = DITER_MID_MAX;    // 33..8192  : "mid"  -- both: 32 selected nodes per warp,
                                 //             lanes over the group's concatenated edges
constexpr int kHubChunk = 2048;  // > 8192    : "hub"  -- one CTA per 2048-edge chunk
#ifndef DITER_HOT_ROWS
#define DITER_HOT_ROWS 2048
#endif
constexpr int kHot = DITER_HOT_ROWS;        // rows staged in shared memory by each scatter CTA

constexpr int kSelectThreads = 256;
#ifndef DITER_SELECT_ITEMS
#define DITER_SELECT_ITEMS 16
#endif
#ifndef DITER_SELECT_CTAS
#define DITER_SELECT_CTAS 2
#endif
constexpr int kSelectItems = DITER_SELECT_ITEMS;     // 32-node words per warp iteration
constexpr int kSelectSpan = 32 * kSelectItems;       // nodes per warp iteration (segment granule)
constexpr int kScatterThreads = 256;
#ifndef DITER_HUB_CTAS_PER_SM
#define DITER_HUB_CTAS_PER_SM 0     // k_scatter_hubs CTAs per SM (0: as many as fit)
#endif
#ifndef DITER_SWEEP_HUBS
#define DITER_SWEEP_HUBS 1          // sweeps push hub chunks inside k_sweep (no k_scatter_hubs launch)
#endif
#ifndef DITER_SCATTER_MIN_BLOCKS
#define DITER_SCATTER_MIN_BLOCKS 3
#endif
constexpr int kScatterMinBlocks = DITER_SCATTER_MIN_BLOCKS;   // __launch_bounds__ min CTAs/SM of k_scatter
constexpr int kFinalizeThreads = 512;
constexpr int kSelectCtasPerSm = DITER_SELECT_CTAS;  // 16 select warps/SM x 16 x 256 B loads in flight
constexpr int kMaxSegments = 8192;                   // select warps (= frontier segments) per launch
constexpr int kStripes = 32;                         // max scatter ticket counters (contiguous group stripes)
constexpr int kMaxBins = 64;                         // far-push destination bins (propagation blocking)
constexpr int kNear = 2048;                          // pushes within +-kNear rows of the group are "near"
constexpr int kFarChunk = 128;                       // far-record slots per warp-owned chunk

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
  long long dang;      // cumulative dangling nodes of S_p (taken by the select, never scattered)
  int done;            // 0 running, 1 converged, 2 max passes reached
  int policy;          // DI_POLICY_*
  unsigned long long hub_packed;  // (hub slots << 32) | hub chunks; reset by k_finalize
  long long log_cap;
  int flush_now;       // far-edge deferral: k_far_flush delivers the increments after this pass
  unsigned long long remote_pushes;   // distributed: pushes into the outbox (one atomic per CTA per pass)
  double t_sel_us;     // fused kernel: accumulated select / scatter phase time (%globaltimer)
  double t_sc_us;
  double T_floor;      // P2P: the local schedule does not lower T below this (0 = no floor)
  // far-edge deferral (one GPU; defer.cu): the far edges of diffused nodes wait for a
  // flush that pushes (H_i - H_old_i) p_ji along them (PAPER.md:227-250 applied to the
  // rows far from their source); `pending` bounds the undelivered mass |D|_1
  double pending;
  int defer_m;         // passes between flushes (0 = deferral off)
  int stop_after_flush;   // the bound met the target with mass pending: stop once it is delivered
  long long flushes;   // flushes executed since create
  int sweep;           // one-kernel async sweeps (options.sweep): r_p is the carried bound r_pred
  float key_off;       // sweeps, derived per-edge key: |F_i| / (#out_i + key_off) (options.key_offset)
  // scatter tickets: one counter per stripe of the frontier groups, each on its
  // own 128-byte line (reset per pass)
  alignas(128) unsigned tickets[kStripes * 32];
  // far-push chunks opened per destination bin this pass, one counter per 128-byte line
  alignas(128) unsigned far_cnt[kMaxBins * 32];
  // sweeps with in-kernel hub chunks (DITER_SWEEP_HUBS): chunk claims and spans finished
  // this pass, each on its own 128-byte line (reset per pass)
  alignas(128) unsigned hub_take;
  alignas(128) unsigned long long spans_done;
};

// k_select partials (one per CTA): r_p and |S_p|.
struct SelPartial {
  double r;
  long long cnt;      // |S_p|, dangling nodes included
  double loss;        // sum |s_i| over the dangling nodes taken (their fluid leaves, App. A.2)
  long long dang;     // dangling nodes taken (they never reach the scatter)
};

// k_scatter partials (one per CTA): guaranteed |F|_1 drop and frontier census.
struct ScPartial {
  double loss;      // sum over taken nodes of (1 - c_i)|s_i|, c_i = d (0 if dangling)
  long long edges;  // E_p
  int dang, n_low, n_mid, n_hub;
  double pend;      // far-edge deferral: sum |s_i| d #far_i / #out_i (mass left for the flush)
};

// Far pushes (propagation blocking).  A push whose row lies outside the shared-
// memory hot window, outside the L2-resident "warm" row range [warm_lo, warm_lo +
// warm_len) and more than kNear rows away from its group's columns would miss L2
// (a random DRAM sector read-modify-write); it is appended instead as a (row,
// value) record to the bin of its row (row >> shift), and k_apply_far adds the
// records bin by bin, each bin's slice of F staying L2-resident while it is
// applied.  Records go to kFarChunk-slot chunks: each scatter warp owns one open
// chunk per bin (state in shared memory) and takes a new one with a single atomic
// on the bin's chunk counter; a closed chunk stores its fill count.  Bin b owns
// chunks [coff[b], coff[b+1]) (capacity from an exact census at create plus the
// per-warp waste bound), records at slot chunk * kFarChunk + k.
struct Far {
  int on;
  int warm_lo;
  unsigned warm_len;
  int shift;                 // bin = row >> shift
  int n_bins;
  int *rows;                 // [n_chunks * kFarChunk]
  double *vals;
  int *fill;                 // [n_chunks] records in each closed chunk
  const long long *coff;     // [n_bins + 1] first chunk of each bin
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
  Far far;
  const int *nloc;           // distributed: local edges of each column (stored first); one GPU with
                             // far-edge deferral: near edges of each column (stored first); else nullptr
  int local_only;            // DI_REMOTE_INCREMENT: the scatter pushes [b0, b0 + nloc) only
  int defer;                 // one GPU: far-edge deferral on (the scatter pushes [b0, b0 + nloc))
};

// Frontier of one pass, compacted per select warp: warp w scans the owned nodes
// [w seg_len, (w+1) seg_len) and writes its selected nodes in ascending order to
// ids/S[w seg_len + k], k < seg_cnt[w].  The scatter takes them 32 at a time
// ("groups") through a prefix over ceil(seg_cnt/32).  Hubs go to a separate list.
struct Frontier {
  int *ids;              // [n_seg * seg_len] local node ids
  double *S;             // [n_seg * seg_len] taken values s_i
  int *seg_cnt;          // [n_seg] selected nodes per segment (dangling ones excluded)
  const unsigned *dang_bits;   // [ceil(n/32)] bit i%32 of word i/32: column i has no out-edge
  long long seg_len;     // nodes per segment, a multiple of kSelectSpan
  int n_seg;             // select grid x warps per CTA (<= kMaxSegments)
  int run;               // groups per dynamic grab of the scatter
  int stripes;           // ticket stripes in use (<= kStripes)
  double *hub_w;         // push value per edge of the hub (s d/#out or s)
  long long *hub_b0;
  long long *hub_deg;
  unsigned *hub_chunk;   // first 2048-edge chunk id of the hub (prefix in slot order)
  unsigned *hub_cslot;   // sweeps: chunk -> hub slot + 1, 0 until published (cleared once pushed)
  const unsigned *cp32;  // sweeps: col_ptr as 32-bit values [n + 1] when the owned edges fit (the scan then
                         // reads 4 B per node instead of 8), else nullptr
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
