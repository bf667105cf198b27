// dist.cuh -- state of a distributed context shared by dist.cu (fabric, bulk
// exchanges, SYNC / ASYNC rounds, rebalance) and p2p.cu (the barrier-free
// exchange, DI_EXCHANGE_P2P).
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "../../include/diter.h"
#include "ctx.cuh"

// One exchanged record of the bulk (all-to-all-v) exchange: destination row (local
// to the receiver) and fluid.
struct Rec {
  long long row;
  double val;
};

// ------------------------------------------------------------------ fabric --
// Collectives between the ranks of a distributed context.  Every call is counted
// (`calls`): di_stats.collectives shows which exchange modes need one per round.
struct Fabric {
  long long calls = 0;
  virtual ~Fabric() {}
  // in-place sum over ranks of `count` (<= 8) doubles on the device
  virtual di_status allreduce_sum(di_ctx *ctx, double *dev, int count) = 0;
  // host-side exchange of per-peer record counts
  virtual di_status alltoall_counts(di_ctx *ctx, const long long *send, long long *recv) = 0;
  // records: send[soff[q] .. soff[q]+scnt[q]) to peer q, into recv[roff[q] ..]
  virtual di_status alltoallv(di_ctx *ctx, const Rec *send, const long long *soff, const long long *scnt,
                              Rec *recv, const long long *roff, const long long *rcnt) = 0;
  // max over ranks of one host double (setup: T_0, validation agreement)
  virtual di_status host_max(di_ctx *ctx, double v, double *out) = 0;
  // every rank's `bytes` host bytes, in rank order, into all[world * bytes] (setup)
  virtual di_status allgather(di_ctx *ctx, const void *mine, size_t bytes, void *all) = 0;
  // a rank failed mid-collective-sequence: release the peers (loopback) instead of
  // leaving them waiting
  virtual void abort() {}
};

// ------------------------------------------------------------- P2P exchange --
// DI_EXCHANGE_P2P (p2p.cu).  Every rank exposes one device window to its peers
// (CUDA IPC across processes, plain pointers between contexts of one process):
// a header of per-peer control words, then one inbox ring per peer.  A sender
// writes records straight into its ring in the receiver's window and then
// publishes the ring's new head with a system-scope release store; the receiver
// merges whatever has been published at the start of its next round and writes
// back (into the sender's window) how many records it consumed and their mass.
constexpr int kP2PMaxWorld = 64;
struct alignas(128) P2PHeader {
  unsigned long long head[kP2PMaxWorld];   // [q]: records q has published into my ring from q (written by q)
  unsigned long long tail[kP2PMaxWorld];   // [q]: records of MY ring at q that q has merged (written by q)
  double acked[kP2PMaxWorld];              // [q]: fluid mass of those records (written by q)
  double board[kP2PMaxWorld];              // [q]: q's latest r_q + s_q + in-flight_q (written by q)
  double tval[kP2PMaxWorld];               // [q]: q's current threshold T_q (written by q)
  unsigned long long quiesce;              // confirmation epoch requested by any rank
  unsigned long long pad[15];
};

// One peer as seen by this rank (device table, uploaded at setup).
struct P2PPeer {
  P2PHeader *hdr;        // the peer's window header
  int *out_rows;         // my ring in the peer's window
  double *out_vals;
  long long out_cap;     // its capacity in records
  int *in_rows;          // the peer's ring in my window
  double *in_vals;
  long long in_cap;
  long long slot_lo, slot_hi;   // my outbox slots of rows the peer owns
  long long row0;        // first global row the peer owns (records carry row - row0)
};

struct P2PState {
  bool on = false;
  // compact outbox: slot s of G stands for global row tgt[s] (sorted: the rows of
  // every peer form one contiguous slot range); remote row ids in row_idx are
  // rewritten to slots at create
  int *tgt = nullptr;
  long long m = 0;
  std::vector<long long> slot_off;         // [world + 1]
  // my window (cudaMalloc: IPC-exportable) and the peers' mappings
  char *win = nullptr;
  size_t win_bytes = 0;
  std::vector<char *> peer_win;            // [world]
  std::vector<bool> peer_ipc;              // opened with cudaIpcOpenMemHandle (closed at destroy)
  P2PPeer *d_peers = nullptr;              // [world]
  std::vector<P2PPeer> peers;
  // device-side progress (local memory)
  unsigned long long *d_head_out = nullptr;   // [world] records published into my ring at q
  unsigned long long *d_tail_in = nullptr;    // [world] records merged from q
  unsigned long long *d_snap = nullptr;       // [world] heads snapshot of the current merge
  double *d_sent = nullptr;                   // [world] mass published to q (cumulative)
  double *d_merged = nullptr;                 // [world] mass merged from q (cumulative)
  long long *d_cnt = nullptr;                 // [world] records compacted this send
  double *d_mass = nullptr;                   // [world] their mass
  double *d_round = nullptr;                  // [8] round scalars (s_k, r_k, r before merge, ...)
  void *h_round = nullptr;                    // pinned host copy of a round's header + scalars
  unsigned long long epoch = 0;               // confirmations completed
  long long confirms = 0;                     // confirmations run (stats)
  long long publishes = 0;
  long long sleep_rounds = 0;                 // rounds spent asleep (merge only, no local passes)
};

// ------------------------------------------------------------ dist state --
struct DistState {
  std::unique_ptr<Fabric> fabric;
  std::vector<long long> bounds;       // [world + 1]
  long long *d_bounds = nullptr;
  Rec *send = nullptr, *recv = nullptr;
  long long send_cap = 0, recv_cap = 0;
  long long *d_scnt = nullptr;         // [world] records compacted per peer
  double *d_sums = nullptr;            // [kSums + 3] + [world] long long (send offsets)
  std::vector<long long> soff, scnt, roff, rcnt;
  double s_k = 0.0;                    // outbox mass (ASYNC)
  // DI_REMOTE_RECEIVER (NEXT f3).  Sender: per peer q the local
  // columns with at least one row in Omega_q, cols[pair_off[q] ..).  Receiver: the
  // remote in-edges of the owned rows grouped by source column: ric_src sorted
  // global source ids, edges [ric_off[k], ric_off[k+1]) of (ric_row local row,
  // ric_p weight p_ij).
  int *cols = nullptr;
  long long *d_pair_off = nullptr;     // [world + 1]
  std::vector<long long> pair_off;
  long long *ric_src = nullptr, *ric_off = nullptr;
  int *ric_row = nullptr;
  double *ric_p = nullptr;
  long long ric_n = 0, ric_e = 0;
  P2PState p2p;
};

// p2p.cu
di_status p2p_setup(di_ctx *ctx);     // collective (create): outbox slots, windows, IPC
di_status p2p_run(di_ctx *ctx, double target);
di_status p2p_reset(di_ctx *ctx);     // every rank, before the next di_run
void p2p_pass_merge(di_ctx *ctx);     // merge + ack + rescale, enqueued before each pass (graph)
void p2p_free(di_ctx *ctx);
// dist.cu helpers used by p2p.cu
void dist_push_increment(di_ctx *ctx);
void dist_launch_pass_kernels(di_ctx *ctx, int slot);
void dist_pending_mass(di_ctx *ctx, double *out);              // += s_k of the pending increments
void dist_set_target(di_ctx *ctx, double target, long long max_pass);
