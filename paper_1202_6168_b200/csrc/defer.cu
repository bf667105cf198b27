// defer.cu -- far-edge deferral (one GPU, PageRank contexts; options.far_defer).
//
// The paper's increment push (algorithm (*)): a PID does not push
// fluid to another PID's nodes at every diffusion; at send time it pushes, along
// those edges, the increment of its history since the last send,
//   sum_i p_ji (H_i - H_old_i),   H_old_i := H_i,
// which carries exactly the fluid of every diffusion of i in between (eq. defH:
// H_i grows by each sent amount).  Multi-GPU contexts use it for remote rows
// (DI_REMOTE_INCREMENT, dist.cu).  On one GPU the same bookkeeping pays for the
// edges whose row is far from their source (|j - i| > kNear): on the web-like
// configs those are the 30 % Zipf-over-id pushes, and their REDs are the costly
// ones (tail rows miss L2: a DRAM sector read-modify-write per push), while the
// +-1000-local pushes land in L2 lines the scatter's working window keeps hot.
// A node diffused several times between two flushes pushes its far edges once.
//
//   * setup: each column's edges re-ordered near first, far last; nloc_i = #near;
//   * scatter: pushes [b0, b0 + nloc_i) and adds |s_i| d #far_i / #out_i to the
//     pass's `pend` (an upper bound on the far mass it deferred);
//   * k_far_flush (every far_defer passes, and before the run stops): for every
//     column with H_i != H_old_i, push (H_i - H_old_i) d / #out_i along its far
//     edges, H_old_i := H_i; k_flush_end clears the pending bound.
// Invariant: F + D = B - (I - P) H, D = the undelivered far pushes, |D|_1 <=
// pending; k_finalize stops on r + pending (App. A.1-A.2), and never with D
// undelivered, so between di_run calls F = B - (I - P)H holds as without deferral.
// Only the order in which fluid reaches the far rows changes, so the limit is the
// same X; the pass schedule is not the snapshot oracle's, so the
// bit-exact frontier tests run with deferral off.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "../../include/diter.h"
#include "ctx.cuh"
#include "kernels.cuh"

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      diter_set_err(ctx, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),       \
                    __FILE__, __LINE__);                                               \
      return e_ == cudaErrorMemoryAllocation ? DI_ERR_OOM : DI_ERR_CUDA;               \
    }                                                                                  \
  } while (0)
#define TRY(x)                      \
  do {                              \
    di_status s_ = (x);             \
    if (s_ != DI_OK) return s_;     \
  } while (0)

namespace diter {
namespace {   // the same anonymous namespace as kernels.cuh's (one per translation unit)

constexpr int kSetupThreads = 256;

// An edge is deferred ("far") when its row is more than kNear ids from its column
// and outside the rows the scatter keeps on-chip or L2-resident ([keep_lo, keep_hi):
// the L2 persisting window, which holds the shared-memory hot window on the Zipf
// configs) -- those pushes are cheap, and their rows are the ones whose fluid the
// schedule needs early.
struct Keep { long long lo, hi; };

__device__ __forceinline__ bool is_near(int row, long long src, Keep k) {
  const long long dd = (long long)row - src;
  return (dd >= -kNear && dd <= kNear) || (row >= k.lo && row < k.hi);
}

// Warp-cooperative walk over the edges of 32 consecutive columns (lane = column):
// lanes take edges l, l+32, ... of the group's concatenated edge list; the owner
// column of an edge by a shuffle binary search over the degree prefix.
template <typename Fn>
__device__ __forceinline__ void for_group_edges(const long long *col_ptr, long long n, long long c0, Fn &&f) {
  const unsigned lane = lane_id();
  const long long c = c0 + lane;
  const long long b0 = c < n ? col_ptr[c] : 0;
  const long long deg = c < n ? col_ptr[c + 1] - b0 : 0;
  long long incl = deg;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if ((int)lane >= o) incl += t;
  }
  const long long excl = incl - deg;
  const long long total = __shfl_sync(0xffffffffu, incl, 31);
  for (long long base = 0; base < total; base += 32) {
    const long long e = base + lane;
    int lo = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int cand = lo + step;
      if (__shfl_sync(0xffffffffu, excl, cand) <= e) lo = cand;
    }
    const long long ob = __shfl_sync(0xffffffffu, b0, lo);
    const long long oe = __shfl_sync(0xffffffffu, excl, lo);
    if (e < total) f(lo, c0 + lo, ob + (e - oe), ob);
  }
}

// nloc[i] = near edges of column i; near_total += sum
__global__ void __launch_bounds__(kSetupThreads)
k_near_count(const long long *__restrict__ col_ptr, const int *__restrict__ row_idx, long long n,
             int *__restrict__ nloc, unsigned long long *near_total, Keep keep) {
  __shared__ int s_c[kSetupThreads];
  const int w0 = threadIdx.x & ~31;
  const long long groups = (n + 31) >> 5;
  unsigned long long tot = 0;
  for (long long g = (long long)blockIdx.x * (kSetupThreads / 32) + (threadIdx.x >> 5); g < groups;
       g += (long long)gridDim.x * (kSetupThreads / 32)) {
    s_c[threadIdx.x] = 0;
    __syncwarp();
    for_group_edges(col_ptr, n, g << 5, [&](int lo, long long col, long long e, long long) {
      if (is_near(row_idx[e], col, keep)) atomicAdd(&s_c[w0 + lo], 1);
    });
    __syncwarp();
    const long long c = (g << 5) + lane_id();
    if (c < n) {
      nloc[c] = s_c[threadIdx.x];
      tot += (unsigned long long)s_c[threadIdx.x];
    }
    __syncwarp();
  }
  tot = warp_sum(tot);
  if (lane_id() == 0 && tot) atomicAdd(near_total, tot);
}

// Columns re-ordered into rows_out: near edges first, far edges last.
__global__ void __launch_bounds__(kSetupThreads)
k_near_split(const long long *__restrict__ col_ptr, const int *__restrict__ row_idx, long long n,
             const int *__restrict__ nloc, int *__restrict__ rows_out, Keep keep) {
  __shared__ int s_near[kSetupThreads], s_far[kSetupThreads];
  const int w0 = threadIdx.x & ~31;
  const long long groups = (n + 31) >> 5;
  for (long long g = (long long)blockIdx.x * (kSetupThreads / 32) + (threadIdx.x >> 5); g < groups;
       g += (long long)gridDim.x * (kSetupThreads / 32)) {
    s_near[threadIdx.x] = 0;
    s_far[threadIdx.x] = 0;
    __syncwarp();
    for_group_edges(col_ptr, n, g << 5, [&](int lo, long long col, long long e, long long b0) {
      const int row = row_idx[e];
      if (is_near(row, col, keep)) rows_out[b0 + atomicAdd(&s_near[w0 + lo], 1)] = row;
      else rows_out[b0 + nloc[col] + atomicAdd(&s_far[w0 + lo], 1)] = row;
    });
    __syncwarp();
  }
}

// ---------------------------------------------------------------- the flush --
// Groups of 32 consecutive columns (ascending, grid-strided): lane = column i with
// far edges and H_i != H_old_i pushes w = (H_i - H_old_i) d / #out_i along
// [b0 + nloc_i, b1) through the scatter's push_group (edge-balanced lanes, the
// shared-memory hot window flushed once per CTA), then H_old_i := H_i.
__global__ void __launch_bounds__(kScatterThreads, kScatterMinBlocks)
k_far_flush(Graph g, double *__restrict__ F, const double *__restrict__ H, double *__restrict__ H_old,
            Ctl *ctl) {
  if (ctl->done || !ctl->flush_now) return;
  __shared__ double s_hot[kHot];
  for (int t = threadIdx.x; t < kHot; t += blockDim.x) s_hot[t] = 0.0;
  __syncthreads();
  const Sink s{F, s_hot, g.hot_lo, g.lo, g.n, nullptr, nullptr};
  Stage sg{nullptr, nullptr, 0};
  const long long groups = (g.n + 31) >> 5;
  const unsigned lane = lane_id();
  for (long long q = (long long)blockIdx.x * (kScatterThreads / 32) + (threadIdx.x >> 5); q < groups;
       q += (long long)gridDim.x * (kScatterThreads / 32)) {
    const long long i = (q << 5) + lane;
    long long b0 = 0;
    int nfar = 0;
    double w = 0.0;
    if (i < g.n) {
      const long long c0 = __ldcs(g.col_ptr + i), c1 = __ldcs(g.col_ptr + i + 1);
      const long long nl = __ldcs(g.nloc + i);
      if (c1 - c0 > nl) {
        const double h = __ldcs(H + i), ho = H_old[i];
        const double dh = h - ho;
        if (dh != 0.0) {
          w = dh * (g.d / (double)(c1 - c0));
          b0 = c0 + nl;
          nfar = (int)(c1 - c0 - nl);
          H_old[i] = h;
        }
      }
    }
    if (__any_sync(0xffffffffu, nfar > 0)) push_group<false, false>(g, s, ctl, nullptr, b0, nfar, w, 0, 0, sg);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < kHot; t += blockDim.x) {
    const double v = s_hot[t];
    if (v != 0.0) red_add(F + (g.hot_lo - g.lo) + t, v);
  }
}

// After the flush: nothing is pending; stop if the bound had met the target.
__global__ void k_flush_end(Ctl *ctl) {
  if (!ctl->flush_now) return;
  ctl->pending = 0.0;
  ctl->flush_now = 0;
  ctl->flushes += 1;
  if (ctl->stop_after_flush) {
    ctl->done = ctl->stop_after_flush;
    ctl->stop_after_flush = 0;
  }
}

// Host-driven flush (a di_run that ends with mass pending, e.g. from a
// max_passes stop inside a graph's tail): raise flush_now first.
__global__ void k_flush_force(Ctl *ctl) {
  if (ctl->pending > 0.0) ctl->flush_now = 1;
  ctl->done = 0;
}
__global__ void k_flush_restore(Ctl *ctl, int done) { ctl->done = done; }

}  // namespace
}  // namespace diter

using namespace diter;

// ------------------------------------------------------------------ host --
di_status diter_setup_defer(di_ctx *ctx) {
  const int opt = ctx->opt.far_defer;
  const long long n = ctx->n_local, nnz = ctx->nnz_local;
  ctx->defer_m = 0;
  // off by default: on C4 every cadence measured slower (far-edge deferral)
  if (opt <= 0 || ctx->dist || ctx->fused || ctx->vals || nnz == 0) return DI_OK;
  const int blocks = ctx->num_sms * 8;
  int *nloc = nullptr;
  unsigned long long *d_tot = nullptr;
  TRY(diter_alloc(ctx, (void **)&nloc, sizeof(int) * (size_t)n));
  TRY(diter_alloc(ctx, (void **)&d_tot, sizeof(unsigned long long)));
  CK(cudaMemsetAsync(d_tot, 0, sizeof(unsigned long long), ctx->stream));
  // rows kept on the immediate path: the L2 persisting window (global ids), if any,
  // else the shared-memory hot window
  Keep keep{ctx->hot_lo, (long long)ctx->hot_lo + kHot};
  if (ctx->l2_bytes > 0) keep = Keep{ctx->lo + ctx->l2_lo, ctx->lo + ctx->l2_lo + ctx->l2_bytes / (long long)sizeof(double)};
  k_near_count<<<blocks, kSetupThreads, 0, ctx->stream>>>(ctx->col_ptr, ctx->row_idx, n, nloc, d_tot, keep);
  unsigned long long near_tot = 0;
  CK(cudaMemcpyAsync(&near_tot, d_tot, sizeof(near_tot), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  diter_free(ctx, d_tot);
  const long long far = nnz - (long long)near_tot;
  if (far == 0) {
    diter_free(ctx, nloc);
    CK(cudaStreamSynchronize(ctx->stream));
    return DI_OK;
  }
  int *rows2 = nullptr;
  TRY(diter_alloc(ctx, (void **)&rows2, sizeof(int) * (size_t)nnz));
  k_near_split<<<blocks, kSetupThreads, 0, ctx->stream>>>(ctx->col_ptr, ctx->row_idx, n, nloc, rows2, keep);
  diter_free(ctx, ctx->row_idx);
  ctx->row_idx = rows2;
  TRY(diter_alloc(ctx, (void **)&ctx->H_old, sizeof(double) * (size_t)n));
  CK(cudaMemsetAsync(ctx->H_old, 0, sizeof(double) * (size_t)n, ctx->stream));
  ctx->nloc = nloc;
  ctx->defer_m = opt;
  ctx->far_edges = far;
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaGetLastError());
  return DI_OK;
}

// The flush pair of a captured pass (returns at once unless k_finalize asked for it).
void diter_defer_launch(di_ctx *ctx) {
  if (!ctx->defer_m) return;
  k_far_flush<<<ctx->grid_scatter, kScatterThreads, 0, ctx->stream>>>(diter_graph(ctx), ctx->F, ctx->H, ctx->H_old,
                                                                      ctx->ctl);
  k_flush_end<<<1, 1, 0, ctx->stream>>>(ctx->ctl);
}

// Deliver whatever is pending now (host side, between graph launches); keeps `done`.
di_status diter_defer_flush_now(di_ctx *ctx, int done) {
  if (!ctx->defer_m) return DI_OK;
  k_flush_force<<<1, 1, 0, ctx->stream>>>(ctx->ctl);
  diter_defer_launch(ctx);
  k_flush_restore<<<1, 1, 0, ctx->stream>>>(ctx->ctl, done);
  ctx->kernel_launches += 4;
  CK(cudaGetLastError());
  return DI_OK;
}
