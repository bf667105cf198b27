// p2p.cu -- DI_EXCHANGE_P2P: the paper's asynchronous exchange without a barrier.
//
// PID k accumulates the fluid its diffusions owe to the nodes of
// other PIDs (s_k, here the pending remote increments H - H_old of
// DI_REMOTE_INCREMENT plus what is left in the outbox) and sends "when s_k > r_k/K"
// (eq. send); :274-280: the receiver adds the fluid to its nodes, and that
// reception "can be delayed"; :50-53, :516-521: no synchronisation constraint.
//
// Rank k owns a device window (P2PHeader + one inbox ring per peer).  A round of
// rank k, with no collective and no wait on any peer:
//   1-2. check_interval local passes (one captured CUDA graph), each preceded by a
//      merge: snapshot the heads peers published into k's header (acquire), add
//      every record in [tail, head) of each ring to F (RED), write the new tail and
//      the merged mass back into the sender's header, rescale T (reading R13);
//   3. s_k and r_k; the board value r_k + s_k + in-flight_k into every header;
//      one device->host copy of k's header and counters;
//   4. send rule: if s_k > r_k / K, push the remote increments into the compact
//      outbox, compact the outbox of every peer whose ring has room straight into
//      that ring (NVLink stores through the IPC mapping), fence, publish the head
//      (st.release.sys).
// Termination: the board sum (in k's own header) is only a
// trigger -- a message merged between two ranks' samples can be counted by nobody --
// so a rank that sees it below the target, or has run out of passes, raises the
// quiesce epoch in every header, and every rank, on seeing the epoch, runs the
// confirmation: push all increments, merge, barrier, merge (rings now empty),
// barrier, flush the whole outbox, barrier, merge, then one all-reduce of the exact
// r_k -- the only collectives of a run besides one all-reduce at its start.
//
// Contexts of one process (loopback tests, K contexts on one GPU) map each other's
// windows by pointer; other processes through cudaIpcOpenMemHandle.  No kernel ever
// waits on another rank: every wait is host-side, inside the fabric's collectives.
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/diter.h"
#include "ctx.cuh"
#include "dist.cuh"
#include "kernels.cuh"

#define CKP(call)                                                                      \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      diter_set_err(ctx, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),       \
                    __FILE__, __LINE__);                                               \
      return e_ == cudaErrorMemoryAllocation ? DI_ERR_OOM : DI_ERR_CUDA;               \
    }                                                                                  \
  } while (0)

#define TRYP(x)                     \
  do {                              \
    di_status s_ = (x);             \
    if (s_ != DI_OK) return s_;     \
  } while (0)

namespace diter {
namespace {

// round scalars in P2PState::d_round
enum { kRoundS = 0, kRoundR = 1, kRoundRBefore = 2, kRoundRecv = 3, kRoundKeyMax = 4, kRoundPend = 5, kRoundN = 8 };

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_volatile(double *p, double v) { *(volatile double *)p = v; }

// ------------------------------------------------------------ setup kernels --
// bit r of bits: global row r is the target of at least one remote edge of this rank
__global__ void k_p2p_mark(const long long *__restrict__ col_ptr, const int *__restrict__ nloc,
                           const int *__restrict__ ri, long long n, unsigned *bits) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    for (long long e = col_ptr[i] + nloc[i]; e < col_ptr[i + 1]; ++e) {
      const int r = ri[e];
      atomicOr(bits + (r >> 5), 1u << (r & 31));
    }
}

__global__ void k_p2p_popc(const unsigned *__restrict__ bits, long long nw, int *cnt) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += stride) cnt[w] = __popc(bits[w]);
}

__device__ __forceinline__ int slot_of(const unsigned *bits, const int *woff, int r) {
  return woff[r >> 5] + __popc(bits[r >> 5] & ((1u << (r & 31)) - 1u));
}

// tgt[slot] = row, slots in ascending row order
__global__ void k_p2p_targets(const unsigned *__restrict__ bits, const int *__restrict__ woff, long long nw, int *tgt) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += stride) {
    unsigned b = bits[w];
    int s = woff[w];
    while (b) {
      const int j = __ffs(b) - 1;
      b &= b - 1;
      tgt[s++] = (int)(w << 5) + j;
    }
  }
}

// remote entries of row_idx: global row -> outbox slot
__global__ void k_p2p_remap(const long long *__restrict__ col_ptr, const int *__restrict__ nloc, int *ri, long long n,
                            const unsigned *__restrict__ bits, const int *__restrict__ woff) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    for (long long e = col_ptr[i] + nloc[i]; e < col_ptr[i + 1]; ++e) ri[e] = slot_of(bits, woff, ri[e]);
}

// slot_off[q] = slots of rows below bounds[q]
__global__ void k_p2p_slot_bounds(const long long *bounds, int W, long long n_rows, long long m,
                                  const unsigned *__restrict__ bits, const int *__restrict__ woff, long long *out) {
  const int q = threadIdx.x;
  if (q > W) return;
  const long long r = bounds[q];
  out[q] = r >= n_rows ? m : slot_of(bits, woff, (int)r);
}

// ------------------------------------------------------------ round kernels --
// |outbox|_1 over dirty blocks (fluid pushed but not yet shipped, part of s_k)
__global__ void k_p2p_outbox_mass(const double *__restrict__ G, const unsigned char *__restrict__ dflags, long long m,
                                  double *out) {
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < m; t += stride)
    if (dflags[t >> 5]) s += fabs(G[t]);
  s = warp_sum(s);
  if (lane_id() == 0 && s != 0.0) atomicAdd(out, s);
}

// Compact the outbox slots of every peer in send_mask into that peer's ring (in its
// window): a warp reads 32 dirty flags (1024 slots), and for each dirty block the
// lanes keep the non-zero slots, take ring positions with one warp-aggregated atomic
// and store (row - row0, value) straight into the receiver's memory.
__global__ void k_p2p_compact(double *__restrict__ G, const unsigned char *__restrict__ dflags,
                              const int *__restrict__ tgt, const P2PPeer *__restrict__ peers, int W, int rank,
                              const unsigned long long *__restrict__ head_out, unsigned long long send_mask,
                              long long *cnt, double *mass) {
  const unsigned lane = lane_id();
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (int q = 0; q < W; ++q) {
    if (q == rank || !((send_mask >> q) & 1ull)) continue;
    const P2PPeer p = peers[q];
    const long long a = p.slot_lo, b = p.slot_hi;
    const long long blk0 = a >> 5, blk1 = (b + 31) >> 5;
    const unsigned long long h0 = head_out[q];
    double ms = 0.0;
    for (long long sb = blk0 + gw * 32; sb < blk1; sb += warps * 32) {
      const long long myblk = sb + lane;
      unsigned dm = __ballot_sync(0xffffffffu, myblk < blk1 && dflags[myblk]);
      while (dm) {
        const int j = __ffs(dm) - 1;
        dm &= dm - 1;
        const long long slot = ((sb + j) << 5) + lane;
        const bool in = slot >= a && slot < b;
        const double v = in ? G[slot] : 0.0;
        const bool keep = in && v != 0.0;
        const unsigned km = __ballot_sync(0xffffffffu, keep);
        if (km == 0u) continue;
        unsigned long long base = 0;
        if (lane == 0) base = (unsigned long long)atomicAdd((unsigned long long *)&cnt[q], (unsigned long long)__popc(km));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) {
          const long long pos = (long long)((h0 + base + __popc(km & lanemask_lt())) % (unsigned long long)p.out_cap);
          p.out_rows[pos] = tgt[slot] - (int)p.row0;
          p.out_vals[pos] = v;
          G[slot] = 0.0;
          ms += fabs(v);
        }
      }
    }
    ms = warp_sum(ms);
    if (lane == 0 && ms != 0.0) atomicAdd(&mass[q], ms);
  }
  __threadfence_system();   // the records reach the receiver before the publish kernel's release
}

// Publish: new head of each ring sent to (release, system scope: the receiver's
// acquire of the head orders its record reads after it)
__global__ void k_p2p_publish(const P2PPeer *__restrict__ peers, int W, int rank, unsigned long long send_mask,
                              unsigned long long *head_out, const long long *cnt, const double *mass, double *sent) {
  const int q = threadIdx.x;
  if (q >= W || q == rank || !((send_mask >> q) & 1ull) || cnt[q] == 0) return;
  __threadfence_system();
  const unsigned long long h = head_out[q] + (unsigned long long)cnt[q];
  head_out[q] = h;
  sent[q] += mass[q];
  st_release_sys(&peers[q].hdr->head[rank], h);
}

// Merge, step 1: snapshot the published heads (acquire)
__global__ void k_p2p_snap(const P2PHeader *hdr, int W, int rank, unsigned long long *snap) {
  const int q = threadIdx.x;
  if (q < W) snap[q] = q == rank ? 0ull : ld_acquire_sys(&hdr->head[q]);
}

// Merge, step 2: F[row] += val for every record in [tail, snap) of every inbox ring
// ("add them to existing fluids, node per node"); per-peer merged
// mass, total received mass and the largest merged key (the rescale's inputs)
__global__ void k_p2p_merge(double *__restrict__ F, const float *__restrict__ kw, const P2PPeer *__restrict__ peers,
                            int W, int rank, const unsigned long long *__restrict__ snap,
                            const unsigned long long *__restrict__ tail_in, double *round_mass, double *recv) {
  __shared__ long long s_pre[kP2PMaxWorld + 1];
  __shared__ double s_mass[kP2PMaxWorld];
  if (threadIdx.x == 0) {
    long long acc = 0;
    for (int q = 0; q < W; ++q) {
      s_pre[q] = acc;
      if (q != rank) acc += (long long)(snap[q] - tail_in[q]);
    }
    s_pre[W] = acc;
  }
  for (int q = threadIdx.x; q < W; q += blockDim.x) s_mass[q] = 0.0;
  __syncthreads();
  const long long total = s_pre[W];
  double m = 0.0, km = 0.0;
  int q = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
    while (s_pre[q + 1] <= t) ++q;
    const P2PPeer &p = peers[q];
    const long long pos = (long long)((tail_in[q] + (unsigned long long)(t - s_pre[q])) % (unsigned long long)p.in_cap);
    const int row = p.in_rows[pos];
    const double v = p.in_vals[pos];
    red_add(F + row, v);
    m += fabs(v);
    atomicAdd(&s_mass[q], fabs(v));
    km = fmax(km, fabs(v) * (kw ? (double)kw[row] : 1.0));
  }
  m = warp_sum(m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) km = fmax(km, __shfl_xor_sync(0xffffffffu, km, o));
  if (lane_id() == 0) {
    if (m != 0.0) atomicAdd(recv, m);
    if (km > 0.0)
      atomicMax(reinterpret_cast<unsigned long long *>(recv + 1), (unsigned long long)__double_as_longlong(km));
  }
  __syncthreads();
  for (int r = threadIdx.x; r < W; r += blockDim.x)
    if (s_mass[r] != 0.0) atomicAdd(&round_mass[r], s_mass[r]);
}

// Merge, step 3: consumed counts and merged mass back into each sender's header
__global__ void k_p2p_ack(const P2PPeer *__restrict__ peers, int W, int rank, const unsigned long long *snap,
                          unsigned long long *tail_in, double *round_mass, double *merged) {
  const int q = threadIdx.x;
  if (q >= W || q == rank) return;
  if (snap[q] == tail_in[q]) return;
  tail_in[q] = snap[q];
  merged[q] += round_mass[q];
  round_mass[q] = 0.0;
  P2PHeader *h = peers[q].hdr;
  st_volatile(&h->acked[rank], merged[q]);
  __threadfence_system();
  st_release_sys(&h->tail[rank], snap[q]);
}

// Receive-side rescale (reading R13) with r_k taken on the device before the merge
__global__ void k_p2p_rescale(Ctl *ctl, const double *round) {
  const double R = round[kRoundRecv], kmax = round[kRoundKeyMax], r_k = round[kRoundRBefore];
  if (!(R > 0.0)) return;
  if (r_k > 0.0) ctl->T = ctl->T * ((r_k + R) / r_k);
  else if (kmax > 0.0) ctl->T = kmax / ctl->alpha;
}

// The same before each pass inside the captured graph: r_k is the residual the last
// pass predicted (ctl->r_pred, r_p minus the pass's guaranteed drop, App. A.2);
// none yet (start of a run) -> no rescale
__global__ void k_p2p_rescale_ctl(Ctl *ctl, const double *round) {
  const double R = round[kRoundRecv], kmax = round[kRoundKeyMax], r_k = ctl->r_pred;
  if (!(R > 0.0) || !isfinite(r_k)) return;
  if (r_k > 0.0) ctl->T = ctl->T * ((r_k + R) / r_k);
  else if (kmax > 0.0) ctl->T = kmax / ctl->alpha;
}

// Board: r_k + s_k + in-flight_k (sent minus what the receivers acknowledged) into
// every rank's header; in-flight can be counted twice or not at all across ranks'
// samples, hence only a trigger for the confirmation
__global__ void k_p2p_board(const P2PPeer *__restrict__ peers, int W, int rank, const P2PHeader *my,
                            const double *round, const double *sent, const Ctl *ctl) {
  __shared__ double s_v;
  if (threadIdx.x == 0) {
    double inflight = 0.0;
    for (int q = 0; q < W; ++q)
      if (q != rank) inflight += sent[q] - *(volatile const double *)&my->acked[q];
    s_v = round[kRoundR] + round[kRoundS] + fmax(inflight, 0.0);
  }
  __syncthreads();
  const int q = threadIdx.x;
  if (q < W) {
    st_volatile(&peers[q].hdr->board[rank], s_v);
    st_volatile(&peers[q].hdr->tval[rank], ctl->T);
    __threadfence_system();
  }
}

// Threshold coupling (reading R25): the local schedule may not lower T_k below
// max_q T_q / alpha^2, the other ranks' thresholds as last published on the board
__global__ void k_p2p_floor(Ctl *ctl, const P2PHeader *my, int W, int rank) {
  double m = 0.0;
  for (int q = 0; q < W; ++q)
    if (q != rank) m = fmax(m, *(volatile const double *)&my->tval[q]);
#ifndef DITER_P2P_FLOOR_POW
#define DITER_P2P_FLOOR_POW 2
#endif
  ctl->T_floor = DITER_P2P_FLOOR_POW == 2 ? m / (ctl->alpha * ctl->alpha) : DITER_P2P_FLOOR_POW == 1 ? m / ctl->alpha : m;
}

// Quiesce request: epoch into every rank's header
__global__ void k_p2p_quiesce(const P2PPeer *__restrict__ peers, int W, unsigned long long epoch) {
  const int q = threadIdx.x;
  if (q < W) {
    st_release_sys(&peers[q].hdr->quiesce, epoch);
  }
}

__global__ void k_copy_double(double *dst, const double *src) { *dst = *src; }

// No board entry counts as low until its rank has written one.
__global__ void k_p2p_board_init(P2PHeader *hdr) {
  hdr->board[threadIdx.x] = INFINITY;
  hdr->tval[threadIdx.x] = 0.0;
}

}  // namespace
}  // namespace diter

using namespace diter;

// Host copy of what a round decides on (one device->host transfer per round).
struct RoundHost {
  P2PHeader hdr;
  double round[kRoundN];
  unsigned long long head_out[kP2PMaxWorld];
};

// ------------------------------------------------------------------- setup --
struct WinDesc {
  unsigned long long ptr;
  cudaIpcMemHandle_t handle;
  int pid;
  int device;
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

di_status p2p_setup(di_ctx *ctx) {
  NvtxRange nv("p2p setup");
  DistState *ds = ctx->dist;
  P2PState &P = ds->p2p;
  const int W = ctx->world, rank = ctx->rank;
  const long long n = ctx->n_local, n_rows = ctx->n_rows;
  const long long nw = (n_rows + 31) >> 5;
  // 1. distinct remote target rows -> compact outbox slots; remote row ids -> slots
  unsigned *bits = nullptr;
  int *cnt = nullptr, *woff = nullptr;
  void *tmp = nullptr;
  long long *d_so = nullptr;
  size_t tmp_bytes = 0;
  struct Temps {   // setup scratch, freed on every return path
    void **p[5];
    ~Temps() { for (void **q : p) if (*q) { cudaFree(*q); *q = nullptr; } }
  } temps{{(void **)&bits, (void **)&cnt, (void **)&woff, &tmp, (void **)&d_so}};
  CKP(cudaMalloc(&bits, sizeof(unsigned) * nw));
  CKP(cudaMalloc(&cnt, sizeof(int) * (nw + 1)));
  CKP(cudaMalloc(&woff, sizeof(int) * (nw + 1)));
  CKP(cudaMemsetAsync(bits, 0, sizeof(unsigned) * nw, ctx->stream));
  CKP(cudaMemsetAsync(cnt, 0, sizeof(int) * (nw + 1), ctx->stream));
  k_p2p_mark<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->col_ptr, ctx->nloc, ctx->row_idx, n, bits);
  k_p2p_popc<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(bits, nw, cnt);
  CKP(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, woff, (int)(nw + 1), ctx->stream));
  CKP(cudaMalloc(&tmp, std::max<size_t>(tmp_bytes, 1)));
  CKP(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, woff, (int)(nw + 1), ctx->stream));
  int m_host = 0;
  CKP(cudaMemcpyAsync(&m_host, woff + nw, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CKP(cudaStreamSynchronize(ctx->stream));
  P.m = m_host;
  TRYP(diter_alloc(ctx, (void **)&P.tgt, sizeof(int) * std::max(1LL, P.m)));
  TRYP(diter_alloc(ctx, (void **)&ctx->G, sizeof(double) * std::max(1LL, P.m)));
  TRYP(diter_alloc(ctx, (void **)&ctx->dflags, (size_t)((P.m + 31) >> 5) + 1));
  k_p2p_targets<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(bits, woff, nw, P.tgt);
  k_p2p_remap<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->col_ptr, ctx->nloc, ctx->row_idx, n, bits, woff);
  CKP(cudaMalloc(&d_so, sizeof(long long) * (W + 1)));
  k_p2p_slot_bounds<<<1, 128, 0, ctx->stream>>>(ds->d_bounds, W, n_rows, P.m, bits, woff, d_so);
  P.slot_off.assign(W + 1, 0);
  CKP(cudaMemcpyAsync(P.slot_off.data(), d_so, sizeof(long long) * (W + 1), cudaMemcpyDeviceToHost, ctx->stream));
  CKP(cudaStreamSynchronize(ctx->stream));
  // 2. ring capacities: a message to q holds at most one record per slot of q's rows;
  //    a ring holds one such message (a sender ships when the ring has room for it,
  //    receivers drain their rings every round).  Sized per sender: the Zipf-over-id
  //    head's owner receives from every peer, so its inbox grows with K while the
  //    mean per rank falls
  std::vector<long long> m_out(W, 0), m_in(W, 0), cap_in(W, 0), off_in(W, 0), off_out(W, 0);
  for (int q = 0; q < W; ++q) m_out[q] = q == rank ? 0 : P.slot_off[q + 1] - P.slot_off[q];
  TRYP(ds->fabric->alltoall_counts(ctx, m_out.data(), m_in.data()));
  auto ring_cap = [](long long msg) { return msg > 0 ? msg + 64 : 0; };
  size_t off = align_up(sizeof(P2PHeader), 256);
  for (int q = 0; q < W; ++q) {
    cap_in[q] = q == rank ? 0 : ring_cap(m_in[q]);
    off_in[q] = (long long)off;
    off += align_up(sizeof(int) * cap_in[q], 256) + align_up(sizeof(double) * cap_in[q], 256);
  }
  P.win_bytes = off;
  CKP(cudaMalloc(&P.win, P.win_bytes));                // plain cudaMalloc: IPC-exportable
  CKP(cudaMemsetAsync(P.win, 0, P.win_bytes, ctx->stream));
  TRYP(ds->fabric->alltoall_counts(ctx, off_in.data(), off_out.data()));   // where my ring lives at q
  // 3. map every peer's window
  WinDesc me{};
  me.ptr = (unsigned long long)(uintptr_t)P.win;
  me.pid = (int)getpid();
  me.device = ctx->device;
  if (W > 1 && cudaIpcGetMemHandle(&me.handle, P.win) != cudaSuccess) {
    cudaGetLastError();   // same-process peers do not need it
    std::memset(&me.handle, 0, sizeof(me.handle));
  }
  std::vector<WinDesc> all(W);
  TRYP(ds->fabric->allgather(ctx, &me, sizeof(WinDesc), all.data()));
  P.peer_win.assign(W, nullptr);
  P.peer_ipc.assign(W, false);
  for (int q = 0; q < W; ++q) {
    if (q == rank) { P.peer_win[q] = P.win; continue; }
    if (all[q].pid == me.pid) {
      P.peer_win[q] = reinterpret_cast<char *>((uintptr_t)all[q].ptr);
      if (all[q].device != ctx->device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(all[q].device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CKP(e);
        cudaGetLastError();
      }
    } else {
      void *p = nullptr;
      CKP(cudaIpcOpenMemHandle(&p, all[q].handle, cudaIpcMemLazyEnablePeerAccess));
      P.peer_win[q] = static_cast<char *>(p);
      P.peer_ipc[q] = true;
    }
  }
  // 4. the peer table
  P.peers.assign(W, P2PPeer{});
  for (int q = 0; q < W; ++q) {
    P2PPeer &p = P.peers[q];
    p.hdr = reinterpret_cast<P2PHeader *>(P.peer_win[q]);
    p.row0 = ds->bounds[q];
    p.slot_lo = P.slot_off[q];
    p.slot_hi = P.slot_off[q + 1];
    if (q == rank) continue;
    p.out_cap = ring_cap(m_out[q]);
    p.out_rows = reinterpret_cast<int *>(P.peer_win[q] + off_out[q]);
    p.out_vals = reinterpret_cast<double *>(P.peer_win[q] + off_out[q] + align_up(sizeof(int) * p.out_cap, 256));
    p.in_cap = cap_in[q];
    p.in_rows = reinterpret_cast<int *>(P.win + off_in[q]);
    p.in_vals = reinterpret_cast<double *>(P.win + off_in[q] + align_up(sizeof(int) * cap_in[q], 256));
  }
  CKP(cudaMalloc(&P.d_peers, sizeof(P2PPeer) * W));
  CKP(cudaMemcpyAsync(P.d_peers, P.peers.data(), sizeof(P2PPeer) * W, cudaMemcpyHostToDevice, ctx->stream));
  CKP(cudaMalloc(&P.d_head_out, sizeof(unsigned long long) * W));
  CKP(cudaMalloc(&P.d_tail_in, sizeof(unsigned long long) * W));
  CKP(cudaMalloc(&P.d_snap, sizeof(unsigned long long) * W));
  CKP(cudaMalloc(&P.d_sent, sizeof(double) * W));
  CKP(cudaMalloc(&P.d_merged, sizeof(double) * W));
  CKP(cudaMalloc(&P.d_cnt, sizeof(long long) * W));
  CKP(cudaMalloc(&P.d_mass, sizeof(double) * 2 * W));   // [W] per-send mass, [W] per-merge mass
  CKP(cudaMalloc(&P.d_round, sizeof(double) * kRoundN));
  CKP(cudaMallocHost(&P.h_round, sizeof(RoundHost)));
  TRYP(p2p_reset(ctx));
  // the pass graph again, now with the inbox merge before every pass
  if (ctx->graph_exec) TRYP(diter_capture_graph(ctx));
  // 5. the peers' windows are zeroed: nobody writes into another window before
  //    every rank is past this point
  TRYP(ds->fabric->allreduce_sum(ctx, ds->d_sums, 1));
  CKP(cudaStreamSynchronize(ctx->stream));
  return DI_OK;
}

di_status p2p_reset(di_ctx *ctx) {
  P2PState &P = ctx->dist->p2p;
  const int W = ctx->world;
  CKP(cudaMemsetAsync(ctx->G, 0, sizeof(double) * std::max(1LL, P.m), ctx->stream));
  CKP(cudaMemsetAsync(ctx->dflags, 0, (size_t)((P.m + 31) >> 5) + 1, ctx->stream));
  if (ctx->H_old) CKP(cudaMemsetAsync(ctx->H_old, 0, sizeof(double) * ctx->n_local, ctx->stream));
  CKP(cudaMemsetAsync(P.win, 0, sizeof(P2PHeader), ctx->stream));
  k_p2p_board_init<<<1, kP2PMaxWorld, 0, ctx->stream>>>(reinterpret_cast<P2PHeader *>(P.win));
  CKP(cudaMemsetAsync(P.d_head_out, 0, sizeof(unsigned long long) * W, ctx->stream));
  CKP(cudaMemsetAsync(P.d_tail_in, 0, sizeof(unsigned long long) * W, ctx->stream));
  CKP(cudaMemsetAsync(P.d_sent, 0, sizeof(double) * W, ctx->stream));
  CKP(cudaMemsetAsync(P.d_merged, 0, sizeof(double) * W, ctx->stream));
  CKP(cudaMemsetAsync(P.d_mass, 0, sizeof(double) * 2 * W, ctx->stream));
  CKP(cudaMemsetAsync(P.d_round, 0, sizeof(double) * kRoundN, ctx->stream));
  CKP(cudaStreamSynchronize(ctx->stream));
  P.epoch = 0;
  ctx->dist->s_k = 0.0;
  return DI_OK;
}

void p2p_free(di_ctx *ctx) {
  P2PState &P = ctx->dist->p2p;
  if (!P.on) return;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (size_t q = 0; q < P.peer_win.size(); ++q)
    if (P.peer_ipc[q] && P.peer_win[q]) cudaIpcCloseMemHandle(P.peer_win[q]);
  void *ptrs[] = {P.win, P.d_peers, P.d_head_out, P.d_tail_in, P.d_snap, P.d_sent, P.d_merged, P.d_cnt, P.d_mass,
                  P.d_round};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  if (P.h_round) cudaFreeHost(P.h_round);
  diter_free(ctx, P.tgt);
  P = P2PState{};
}

// -------------------------------------------------------------------- run --
static di_status merge_inbox(di_ctx *ctx, bool rescale) {
  DistState *ds = ctx->dist;
  P2PState &P = ds->p2p;
  const int W = ctx->world, rank = ctx->rank;
  if (rescale) {
    TRYP(diter_l1_launch(ctx));                              // r_k before the merge
    k_copy_double<<<1, 1, 0, ctx->stream>>>(P.d_round + kRoundRBefore, ctx->l1_out);
  }
  CKP(cudaMemsetAsync(P.d_round + kRoundRecv, 0, 2 * sizeof(double), ctx->stream));
  k_p2p_snap<<<1, kP2PMaxWorld, 0, ctx->stream>>>(reinterpret_cast<const P2PHeader *>(P.win), W, rank, P.d_snap);
  k_p2p_merge<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->F, ctx->kw, P.d_peers, W, rank, P.d_snap, P.d_tail_in,
                                                        P.d_mass + W, P.d_round + kRoundRecv);
  k_p2p_ack<<<1, kP2PMaxWorld, 0, ctx->stream>>>(P.d_peers, W, rank, P.d_snap, P.d_tail_in, P.d_mass + W, P.d_merged);
  ctx->kernel_launches += 3;
  if (rescale) {
    k_p2p_rescale<<<1, 1, 0, ctx->stream>>>(ctx->ctl, P.d_round);
    ctx->kernel_launches += 2;
  }
  CKP(cudaGetLastError());
  return DI_OK;
}

// Enqueued before every pass (captured in the context's pass graph): what peers have
// published is in F before the select looks at it ("can be delayed", by at
// most one pass), with the receive rescale of T.
void p2p_pass_merge(di_ctx *ctx) {
  P2PState &P = ctx->dist->p2p;
  const int W = ctx->world, rank = ctx->rank;
  cudaMemsetAsync(P.d_round + kRoundRecv, 0, 2 * sizeof(double), ctx->stream);
  k_p2p_snap<<<1, kP2PMaxWorld, 0, ctx->stream>>>(reinterpret_cast<const P2PHeader *>(P.win), W, rank, P.d_snap);
  k_p2p_merge<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->F, ctx->kw, P.d_peers, W, rank, P.d_snap, P.d_tail_in,
                                                        P.d_mass + W, P.d_round + kRoundRecv);
  k_p2p_ack<<<1, kP2PMaxWorld, 0, ctx->stream>>>(P.d_peers, W, rank, P.d_snap, P.d_tail_in, P.d_mass + W, P.d_merged);
  if (ctx->opt.receive_rescale) k_p2p_rescale_ctl<<<1, 1, 0, ctx->stream>>>(ctx->ctl, P.d_round);
  if (ctx->sweep_on) k_rpred_add<<<1, 1, 0, ctx->stream>>>(ctx->ctl, P.d_round + kRoundRecv);   // merged mass
}

// Compact the outbox into the rings of the peers in `mask` and publish.
static di_status send_outbox(di_ctx *ctx, unsigned long long mask) {
  NvtxRange nv("p2p send");
  DistState *ds = ctx->dist;
  P2PState &P = ds->p2p;
  const int W = ctx->world;
  if (!mask) return DI_OK;
  CKP(cudaMemsetAsync(P.d_cnt, 0, sizeof(long long) * W, ctx->stream));
  CKP(cudaMemsetAsync(P.d_mass, 0, sizeof(double) * W, ctx->stream));
  k_p2p_compact<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->G, ctx->dflags, P.tgt, P.d_peers, W, ctx->rank,
                                                          P.d_head_out, mask, P.d_cnt, P.d_mass);
  k_p2p_publish<<<1, kP2PMaxWorld, 0, ctx->stream>>>(P.d_peers, W, ctx->rank, mask, P.d_head_out, P.d_cnt, P.d_mass,
                                                     P.d_sent);
  ctx->kernel_launches += 2;
  P.publishes += 1;
  CKP(cudaGetLastError());
  return DI_OK;
}

static unsigned long long all_peers(const di_ctx *ctx) {
  unsigned long long m = 0;
  for (int q = 0; q < ctx->world; ++q)
    if (q != ctx->rank) m |= 1ull << q;
  return m;
}

// s_k (pending increments + unsent outbox) and r_k into d_round, the board, and
// one host copy of the header, the round scalars and the published heads
static di_status round_measure(di_ctx *ctx, RoundHost *hb) {
  DistState *ds = ctx->dist;
  P2PState &P = ds->p2p;
  const int W = ctx->world;
  CKP(cudaMemsetAsync(P.d_round + kRoundS, 0, sizeof(double), ctx->stream));
  CKP(cudaMemsetAsync(P.d_round + kRoundPend, 0, sizeof(double), ctx->stream));
  if (ctx->H_old) dist_pending_mass(ctx, P.d_round + kRoundPend);
  k_p2p_outbox_mass<<<ctx->num_sms * 2, 256, 0, ctx->stream>>>(ctx->G, ctx->dflags, P.m, P.d_round + kRoundS);
  TRYP(diter_l1_launch(ctx));
  k_copy_double<<<1, 1, 0, ctx->stream>>>(P.d_round + kRoundR, ctx->l1_out);
  if (ctx->sweep_on) k_rpred_set<<<1, 1, 0, ctx->stream>>>(ctx->ctl, ctx->l1_out);   // sweeps carry |F|_1
  k_p2p_board<<<1, kP2PMaxWorld, 0, ctx->stream>>>(P.d_peers, W, ctx->rank, reinterpret_cast<const P2PHeader *>(P.win),
                                                  P.d_round, P.d_sent, ctx->ctl);
  ctx->kernel_launches += 3;
#ifndef DITER_P2P_FLOOR
#define DITER_P2P_FLOOR 1
#endif
  if (DITER_P2P_FLOOR) {
    k_p2p_floor<<<1, 1, 0, ctx->stream>>>(ctx->ctl, reinterpret_cast<const P2PHeader *>(P.win), W, ctx->rank);
    ctx->kernel_launches += 1;
  }
  CKP(cudaMemcpyAsync(&hb->hdr, P.win, sizeof(P2PHeader), cudaMemcpyDeviceToHost, ctx->stream));
  CKP(cudaMemcpyAsync(hb->round, P.d_round, sizeof(double) * kRoundN, cudaMemcpyDeviceToHost, ctx->stream));
  CKP(cudaMemcpyAsync(hb->head_out, P.d_head_out, sizeof(unsigned long long) * W, cudaMemcpyDeviceToHost, ctx->stream));
  CKP(cudaMemcpyAsync(ctx->h_ctl, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
  CKP(cudaStreamSynchronize(ctx->stream));
  return DI_OK;
}

// Quiesce-then-reduce confirmation.  Collective: every rank runs it
// once it has seen the epoch.  Returns the exact global residual in *R and whether
// any rank ran out of passes in *oop.
static di_status confirm(di_ctx *ctx, bool my_oop, double *R, bool *oop) {
  NvtxRange nv("p2p confirm");
  DistState *ds = ctx->dist;
  P2PState &P = ds->p2p;
  Fabric &fab = *ds->fabric;
  P.confirms += 1;
  if (ctx->H_old) dist_push_increment(ctx);        // everything pending into the outbox
  TRYP(merge_inbox(ctx, false));
  TRYP(fab.allreduce_sum(ctx, ds->d_sums, 1));     // all publishes of the round loops done
  TRYP(merge_inbox(ctx, false));
  TRYP(fab.allreduce_sum(ctx, ds->d_sums, 1));     // every ring consumed, tails written back
  TRYP(send_outbox(ctx, all_peers(ctx)));          // flush: an empty ring holds any message
  CKP(cudaMemsetAsync(ctx->dflags, 0, (size_t)((P.m + 31) >> 5) + 1, ctx->stream));
  TRYP(fab.allreduce_sum(ctx, ds->d_sums, 1));     // the flushes published
  TRYP(merge_inbox(ctx, false));                   // nothing in flight from here on
  TRYP(diter_l1_launch(ctx));
  CKP(cudaMemcpyAsync(ds->d_sums, ctx->l1_out, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  const double flag = my_oop ? 1.0 : 0.0;
  CKP(cudaMemcpyAsync(ds->d_sums + 1, &flag, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  TRYP(fab.allreduce_sum(ctx, ds->d_sums, 2));
  double h[2];
  CKP(cudaMemcpyAsync(h, ds->d_sums, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CKP(cudaStreamSynchronize(ctx->stream));
  *R = h[0];
  *oop = h[1] > 0.0;
  P.epoch += 1;
  ds->s_k = 0.0;
  return DI_OK;
}

di_status p2p_run(di_ctx *ctx, double target) {
  DistState *ds = ctx->dist;
  P2PState &P = ds->p2p;
  const int W = ctx->world;
  CKP(cudaSetDevice(ctx->device));
  CKP(cudaEventRecord(ctx->ev0, ctx->stream));
  const long long launches0 = ctx->kernel_launches;
  const long long max_pass_abs = ctx->passes_done + ctx->opt.max_passes;
  Ctl *h = reinterpret_cast<Ctl *>(ctx->h_ctl);
  di_status st = DI_OK;
  RoundHost *hb = reinterpret_cast<RoundHost *>(P.h_round);   // pinned, allocated at setup
  // a run starts (and every run ended) with nothing in flight: the exact global
  // residual decides whether there is anything to do
  double R = 0.0;
  {
    TRYP(diter_l1_launch(ctx));
    CKP(cudaMemcpyAsync(ds->d_sums, ctx->l1_out, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    TRYP(ds->fabric->allreduce_sum(ctx, ds->d_sums, 1));
    CKP(cudaMemcpyAsync(&R, ds->d_sums, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CKP(cudaStreamSynchronize(ctx->stream));
  }
  ctx->residual = R;
  if (R >= target) {
    dist_set_target(ctx, 0.0, max_pass_abs);   // local passes never stop on their own
    const bool graph = ctx->graph_exec != nullptr && !ctx->opt.profile;
    bool asleep = false;
    const int kpp = (ctx->sweep_on ? 2 + 1 : 3) + (ctx->cap_hub > 0 && !(ctx->sweep_on && DITER_SWEEP_HUBS) ? 1 : 0) + 3 + (ctx->opt.receive_rescale ? 1 : 0);
    for (;;) {
      // 1-2. local passes, each after a merge of what has arrived (p2p_pass_merge) --
      //      or, asleep (r_k below this rank's share of the target), only the
      //      merge: the rank keeps receiving and answering, and wakes up when what it
      //      receives lifts r_k again
      if (asleep) {
        usleep(50);                           // nothing to diffuse: do not spin on the device
        p2p_pass_merge(ctx);
        ctx->kernel_launches += 3 + (ctx->opt.receive_rescale ? 1 : 0);
        P.sleep_rounds += 1;
      } else if (graph) {
        CKP(cudaGraphLaunch(ctx->graph_exec, ctx->stream));
        ctx->graph_launches += 1;
        ctx->kernel_launches += (long long)kpp * ctx->check_interval;
      } else {
        for (int k = 0; k < ctx->check_interval; ++k) {
          dist_launch_pass_kernels(ctx, k);   // the P2P merge first (diter_dist_pass_prologue)
          k_finalize<<<1, kFinalizeThreads, 0, ctx->stream>>>(ctx->ctl, ctx->sel_part, diter_n_sel_part(ctx),
                                                              ctx->sc_part, diter_n_sc_part(ctx), ctx->log);
          ctx->kernel_launches += 4 + (ctx->opt.receive_rescale ? 1 : 0);
        }
      }
      // 3. s_k, r_k, board; one host copy
      const bool slept = asleep;
      TRYP(round_measure(ctx, hb));
      if (ctx->opt.profile && !slept) {
        for (int k = 0; k < ctx->check_interval; ++k) {
          float a = 0.f, b = 0.f;
          CKP(cudaEventElapsedTime(&a, ctx->prof_ev[4 * k + 0], ctx->prof_ev[4 * k + 1]));
          CKP(cudaEventElapsedTime(&b, ctx->prof_ev[4 * k + 1], ctx->prof_ev[4 * k + 2]));
          ctx->kt_ms[0] += a;
          ctx->kt_ms[1] += b;
          ctx->pass_us.push_back({a * 1e3, b * 1e3});
        }
        ctx->kt_passes += ctx->check_interval;
      }
      ctx->passes_done = h->pass;
      const double s_k = hb->round[kRoundS] + hb->round[kRoundPend];
      const double r_k = hb->round[kRoundR];
      ds->s_k = s_k;
      double board = 0.0;
      for (int q = 0; q < W; ++q) board += hb->hdr.board[q];
      // sleep: r_k below this rank's share of the target, or (p2p_sleep = k > 0) below
      // k % of its even share of the fluid the board still holds -- a rank left with crumbs waits
      // for its peers' shipments instead of diffusing them at ever lower thresholds
      asleep = ctx->opt.p2p_sleep >= 0 &&
               (r_k < target / W || (ctx->opt.p2p_sleep > 0 && r_k < 0.01 * ctx->opt.p2p_sleep * board / W));
      const bool oop = h->pass >= max_pass_abs;
      // 4. termination: a trigger raises the epoch in every header; every rank confirms
      if (hb->hdr.quiesce > P.epoch || board < target || oop) {
        if (hb->hdr.quiesce <= P.epoch) {
          k_p2p_quiesce<<<1, kP2PMaxWorld, 0, ctx->stream>>>(P.d_peers, W, P.epoch + 1);
          ctx->kernel_launches += 1;
        }
        bool any_oop = false;
        TRYP(confirm(ctx, oop, &R, &any_oop));
        ctx->residual = R;
        if (R < target) break;
        if (any_oop) { st = DI_ERR_NOT_CONVERGED; break; }
        // not yet: fresh board entries before anyone can trigger again
        TRYP(round_measure(ctx, hb));
        continue;
      }
      // 5. send rule (eq. send, strict): push the increments, ship to every peer whose
      //    ring can take a whole message
      if (s_k > r_k / W || (r_k == 0.0 && s_k > 0.0)) {
        if (ctx->H_old) dist_push_increment(ctx);
        unsigned long long mask = 0;
        for (int q = 0; q < W; ++q) {
          if (q == ctx->rank) continue;
          const P2PPeer &p = P.peers[q];
          const long long used = (long long)(hb->head_out[q] - hb->hdr.tail[q]);
          if (p.slot_hi > p.slot_lo && p.out_cap - used >= p.slot_hi - p.slot_lo) mask |= 1ull << q;
        }
        TRYP(send_outbox(ctx, mask));
        if (mask == all_peers(ctx)) CKP(cudaMemsetAsync(ctx->dflags, 0, (size_t)((P.m + 31) >> 5) + 1, ctx->stream));
      }
    }
  }
  CKP(cudaEventRecord(ctx->ev1, ctx->stream));
  CKP(cudaEventSynchronize(ctx->ev1));
  {
    float ms = 0.f;
    CKP(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    ctx->run_ms = ms;
    ctx->run_ms_total += ms;
  }
  CKP(cudaMemcpyAsync(ctx->h_ctl, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
  CKP(cudaMemcpyAsync(hb->head_out, P.d_head_out, sizeof(unsigned long long) * W, cudaMemcpyDeviceToHost, ctx->stream));
  CKP(cudaStreamSynchronize(ctx->stream));
  long long recs = 0;
  for (int q = 0; q < W; ++q) recs += (long long)hb->head_out[q];
  ctx->exchanged_bytes = 12LL * recs;                // 4-byte row + 8-byte value per record
  ctx->alg_bytes_exchange = 12LL * recs + 20LL * recs;
  ctx->exchanges = P.publishes;
  ctx->passes_done = h->pass;
  ctx->edges = h->edges;
  ctx->nodes = h->nodes;
  ctx->dang = h->dang;
  ctx->threshold = h->T;
  ctx->remote_pushes = (long long)h->remote_pushes;
  ctx->run_kernel_launches = ctx->kernel_launches - launches0;
  if (st == DI_ERR_NOT_CONVERGED) diter_set_err(ctx, "max_passes reached before |F|_1 < %g", target);
  return st;
}
