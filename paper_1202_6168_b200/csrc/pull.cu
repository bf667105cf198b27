// pull.cu -- near-edge pull: the +-kPullW-local edges of a dense pass added row by
// row instead of one fp64 RED per edge (one GPU, PageRank contexts).
//
// Why ("near-edge pull"): a pass pushes F_j += p_ji s_i along every
// edge of every taken node (eq. defF); on this B200 a spread fp64
// RED retires at ~187-229 G lanes/s whatever the address pattern
// (profiles/r01_red_microbench.txt), so the scatter is bound by RED issue, not
// by HBM.  On the web-like configs 70 % of the edges join nodes less than 1000 ids
// apart (BASELINE.json configs[1], [3]: "70% local").  A dense pass touches most
// of them, and for those rows the same sum  sum_{i in S_p} p_ji s_i  can be formed
// by the row's owner thread from a table of its near in-edges, with no atomic:
//   * the select marks the taken nodes (Frontier::sel_bits);
//   * the scatter writes sw_i = s_i d / #out_i for each taken node and pushes only
//     the column's other edges (the near ones are stored last, nn_i of them);
//   * k_pull, per tile of kPullR rows, stages sw over the tile +- kPullW in shared
//     memory (zero where not taken) and adds, for each row j, the sw of its near
//     in-edges into F_j -- a plain read-modify-write, coalesced, after the scatter
//     has finished (same stream), so nothing else writes F meanwhile.
// The pass is the same block pass (snapshot semantics): every edge of every taken
// node is added exactly once; only the summation order differs (reading R8).  The
// scatter decides per pass (pull when the select's E_p estimate reaches
// options.pull_permille / 1000 of the edges): a sparse pass pushes everything.
//
// Near in-edge table ("sliced ELL"): per tile the rows are sorted by near
// in-degree (descending, perm[]), 32 consecutive sorted rows form a slice, and a
// slice stores its rows' source offsets (src - row, int16) as max-degree x 32
// column-major pairs: lane l of a warp reads word u*32 + l (two offsets) for u in
// the slice's pair range -- 128 coalesced bytes per warp load.  Short rows are
// padded with an offset that points at the window's zero slot.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "../../include/diter.h"
#include "common.cuh"
#include "ctx.cuh"
#include "types.cuh"

using namespace diter;

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

namespace {

// DITER_TRACE=1: stream-synchronised phase times of the pull setup on stderr
struct SetupTimer {
  const char *tag;
  bool on = std::getenv("DITER_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  explicit SetupTimer(const char *g) : tag(g) {}
  void mark(cudaStream_t s, const char *what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[diter setup] %s %-14s %8.2f ms\n", tag, what,
                 std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

constexpr int kNearMaxDeg = 65535;      // columns with more edges keep every edge on the push path
constexpr int kTileSlices = kPullR / 32;

__device__ __forceinline__ bool is_near(int row, long long src) {
  const long long dd = (long long)row - src;
  return dd >= -kPullW && dd <= kPullW;
}

// ------------------------------------------------------------------- k_pull --
// One pass's near-edge sums.  Persistent CTAs over tiles in ascending order, so the
// halo of a tile's window (its neighbours' sw) is read while the neighbour CTAs have
// it in L2.  Dynamic shared memory: win[kPullZero + 1] (sw over [a - W, a + R + W)
// and the zero slot) + sum[kPullR].
__global__ void __launch_bounds__(kPullThreads, 4)
k_pull(double *__restrict__ F, const double *__restrict__ sw, const unsigned *__restrict__ sel_bits,
       const unsigned short *__restrict__ perm, const unsigned *__restrict__ sptr,
       const unsigned *__restrict__ off, long long n, long long n_tiles, const Ctl *ctl) {
  if (ctl->done || !ctl->pull_pass) return;
  extern __shared__ double smem[];
  double *win = smem;
  double *sum = smem + (kPullZero + 1);
  const unsigned lane = lane_id();
  const int warp = threadIdx.x >> 5;
  for (long long t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const long long a = t * kPullR;
    for (int x = threadIdx.x; x <= kPullZero; x += kPullThreads) {
      const long long src = a - kPullW + x;
      double v = 0.0;
      if (x < kPullZero && src >= 0 && src < n) {
        const unsigned bits = sel_bits[src >> 5];
        if ((bits >> (src & 31)) & 1u) v = sw[src];
      }
      win[x] = v;
    }
    __syncthreads();
    for (int sl = warp; sl < kTileSlices; sl += kPullThreads / 32) {
      const long long gs = t * kTileSlices + sl;
      const unsigned u0 = __ldg(sptr + gs), u1 = __ldg(sptr + gs + 1);
      const int rl = __ldg(perm + t * kPullR + sl * 32 + lane);
      const double *wb = win + rl + kPullW;
      const unsigned *op = off + (size_t)u0 * 32 + lane;
      const int np = (int)(u1 - u0);
      double acc = 0.0;
      int u = 0;
      for (; u + 4 <= np; u += 4) {
        unsigned q[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) q[k] = __ldcs(op + (size_t)(u + k) * 32);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          acc += wb[(short)(q[k] & 0xffffu)];
          acc += wb[(short)(q[k] >> 16)];
        }
      }
      for (; u < np; ++u) {
        const unsigned q = __ldcs(op + (size_t)u * 32);
        acc += wb[(short)(q & 0xffffu)];
        acc += wb[(short)(q >> 16)];
      }
      sum[rl] = acc;
    }
    __syncthreads();
    const int rows = (int)min((long long)kPullR, n - a);
    for (int x = threadIdx.x; x < rows; x += kPullThreads) F[a + x] += sum[x];
    __syncthreads();
  }
}

// ------------------------------------------------------------ setup kernels --
// Warp-cooperative walk over the edges of 32 consecutive columns (lane = column):
// lanes take edges l, l+32, ... of the group's concatenated edge list; the owner
// column of an edge is found by a shuffle binary search over the degree prefix.
template <typename F>
__device__ __forceinline__ void for_group_edges(const long long *col_ptr, long long n, long long c0, F &&f) {
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
    const long long od = __shfl_sync(0xffffffffu, deg, lo);
    if (e < total) f(lo, c0 + lo, ob + (e - oe), od, ob);
  }
}

constexpr int kSetupThreads = 256;

// nn[i] = near edges of column i (0 when #out_i > kNearMaxDeg); cnt[i] the same as int64
__global__ void __launch_bounds__(kSetupThreads)
k_near_count(const long long *__restrict__ col_ptr, const int *__restrict__ row_idx, long long n,
             unsigned short *__restrict__ nn, long long *__restrict__ cnt) {
  __shared__ int s_c[kSetupThreads];
  const int w0 = threadIdx.x & ~31;
  const long long groups = (n + 31) >> 5;
  for (long long g = (long long)blockIdx.x * (kSetupThreads / 32) + (threadIdx.x >> 5); g < groups;
       g += (long long)gridDim.x * (kSetupThreads / 32)) {
    s_c[threadIdx.x] = 0;
    __syncwarp();
    for_group_edges(col_ptr, n, g << 5, [&](int lo, long long col, long long e, long long deg, long long) {
      if (deg <= kNearMaxDeg && is_near(row_idx[e], col)) atomicAdd(&s_c[w0 + lo], 1);
    });
    __syncwarp();
    const long long c = (g << 5) + lane_id();
    if (c < n) {
      nn[c] = (unsigned short)s_c[threadIdx.x];
      cnt[c] = s_c[threadIdx.x];
    }
    __syncwarp();
  }
}

// Column edges re-ordered (other edges first, near edges last) into rows_out, and
// each near edge emitted as (row, src - row) at near_off[i] + k.
__global__ void __launch_bounds__(kSetupThreads)
k_near_split(const long long *__restrict__ col_ptr, const int *__restrict__ row_idx, long long n,
             const unsigned short *__restrict__ nn, const long long *__restrict__ near_off,
             int *__restrict__ rows_out, int *__restrict__ keys, short *__restrict__ vals) {
  __shared__ int s_near[kSetupThreads], s_far[kSetupThreads];
  const int w0 = threadIdx.x & ~31;
  const long long groups = (n + 31) >> 5;
  for (long long g = (long long)blockIdx.x * (kSetupThreads / 32) + (threadIdx.x >> 5); g < groups;
       g += (long long)gridDim.x * (kSetupThreads / 32)) {
    s_near[threadIdx.x] = 0;
    s_far[threadIdx.x] = 0;
    __syncwarp();
    for_group_edges(col_ptr, n, g << 5, [&](int lo, long long col, long long e, long long deg, long long b0) {
      const int row = row_idx[e];
      const int k_near = nn[col];
      if (deg <= kNearMaxDeg && is_near(row, col)) {
        const int k = atomicAdd(&s_near[w0 + lo], 1);
        rows_out[b0 + (deg - k_near) + k] = row;
        keys[near_off[col] + k] = row;
        vals[near_off[col] + k] = (short)(col - row);
      } else {
        const int k = atomicAdd(&s_far[w0 + lo], 1);
        rows_out[b0 + k] = row;
      }
    });
    __syncwarp();
  }
}

// rowptr[j] = first sorted near edge of row j (j in [0, n]); keys sorted ascending.
__global__ void k_row_bounds(const int *__restrict__ keys, long long m, long long n, long long *__restrict__ rowptr) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    const long long k = keys[e];
    const long long prev = e == 0 ? -1 : keys[e - 1];
    for (long long r = prev + 1; r <= k; ++r) rowptr[r] = e;
    if (e == m - 1)
      for (long long r = k + 1; r <= n; ++r) rowptr[r] = m;
  }
}

__global__ void k_narrow(const unsigned long long *__restrict__ in, unsigned *__restrict__ out, long long count) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += stride) out[e] = (unsigned)in[e];
}

// One CTA per tile: rows sorted by near in-degree (descending) -> perm; slice
// lengths in pairs of offsets (the slice's largest degree, rounded up to even).
constexpr int kSortItems = kPullR / kSetupThreads;
__global__ void __launch_bounds__(kSetupThreads)
k_tile_sort(const long long *__restrict__ rowptr, long long n, unsigned short *__restrict__ perm,
            unsigned long long *__restrict__ slice_pairs) {
  using Sort = cub::BlockRadixSort<unsigned, kSetupThreads, kSortItems, unsigned short>;
  __shared__ typename Sort::TempStorage tmp;
  __shared__ unsigned s_deg[kPullR];
  const long long t = blockIdx.x;
  const long long a = t * kPullR;
  unsigned key[kSortItems];
  unsigned short val[kSortItems];
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const int rl = threadIdx.x * kSortItems + k;
    const long long r = a + rl;
    const long long d = r < n ? rowptr[r + 1] - rowptr[r] : 0;
    key[k] = (unsigned)min(d, (long long)0xffffffffu);
    val[k] = (unsigned short)rl;
  }
  Sort(tmp).SortDescendingBlockedToStriped(key, val);
  // striped: item k of thread x is sorted position k * threads + x
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const int pos = k * kSetupThreads + threadIdx.x;
    perm[a + pos] = val[k];
    s_deg[pos] = key[k];
  }
  __syncthreads();
  for (int s = threadIdx.x; s < kTileSlices; s += kSetupThreads)
    slice_pairs[t * kTileSlices + s] = ((unsigned long long)s_deg[s * 32] + 1ull) >> 1;   // slice max = its first row
}

// Thread per tile slot: the slot's row writes its near offsets (and the pads) into
// the slice's column-major pair words.
__global__ void k_fill_slices(const long long *__restrict__ rowptr, const short *__restrict__ vals, long long n,
                              long long n_tiles, const unsigned short *__restrict__ perm,
                              const unsigned *__restrict__ sptr, unsigned *__restrict__ off) {
  const long long slots = n_tiles * kPullR;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < slots; x += stride) {
    const long long t = x / kPullR;
    const int pos = (int)(x - t * kPullR);
    const int rl = perm[x];
    const long long r = t * kPullR + rl;
    const long long gs = t * kTileSlices + (pos >> 5);
    const int lane = pos & 31;
    const unsigned u0 = sptr[gs], u1 = sptr[gs + 1];
    const long long e0 = r < n ? rowptr[r] : 0;
    const long long deg = r < n ? rowptr[r + 1] - e0 : 0;
    const unsigned short pad = (unsigned short)(short)(kPullR + kPullW - rl);   // -> win[kPullZero]
    for (unsigned u = u0; u < u1; ++u) {
      const long long k = 2LL * (u - u0);
      const unsigned short lo16 = k < deg ? (unsigned short)vals[e0 + k] : pad;
      const unsigned short hi16 = k + 1 < deg ? (unsigned short)vals[e0 + k + 1] : pad;
      off[(size_t)u * 32 + lane] = (unsigned)lo16 | ((unsigned)hi16 << 16);
    }
  }
}

}  // namespace

// ------------------------------------------------------------------ host --
// Build the near-edge structures of a one-GPU PageRank context (options.near_pull):
// column re-order (near edges last), nn, the sliced near in-edge table, sw and the
// selection bitmap.  Auto (0) keeps it when near edges are >= 25 % of the edges.
di_status diter_setup_pull(di_ctx *ctx) {
  const int mode = ctx->opt.near_pull;
  const long long n = ctx->n_local, nnz = ctx->nnz_local;
  ctx->pull_on = 0;
  if (mode < 0 || ctx->dist || ctx->fused || ctx->vals || nnz == 0) return DI_OK;
  if (mode == 0 && n < 8LL * kPullR) return DI_OK;
  SetupTimer tr("pull");
  const int blocks = ctx->num_sms * 8;
  unsigned short *nn = nullptr;
  long long *cnt = nullptr, *near_off = nullptr;
  TRY(diter_alloc(ctx, (void **)&nn, sizeof(unsigned short) * (size_t)n));
  TRY(diter_alloc(ctx, (void **)&cnt, sizeof(long long) * (size_t)(n + 1)));
  TRY(diter_alloc(ctx, (void **)&near_off, sizeof(long long) * (size_t)(n + 1)));
  k_near_count<<<blocks, kSetupThreads, 0, ctx->stream>>>(ctx->col_ptr, ctx->row_idx, n, nn, cnt);
  CK(cudaMemsetAsync(cnt + n, 0, sizeof(long long), ctx->stream));
  size_t tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, near_off, (int64_t)(n + 1), ctx->stream));
  void *tmp = nullptr;
  TRY(diter_alloc(ctx, &tmp, tb));
  CK(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, near_off, (int64_t)(n + 1), ctx->stream));
  diter_free(ctx, tmp);
  diter_free(ctx, cnt);
  long long m = 0;
  CK(cudaMemcpyAsync(&m, near_off + n, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  tr.mark(ctx->stream, "near count");
  if (m == 0 || (mode == 0 && 4 * m < nnz)) {
    diter_free(ctx, nn);
    diter_free(ctx, near_off);
    return DI_OK;
  }
  // split the columns and emit the near edges
  int *rows2 = nullptr, *keys = nullptr, *keys2 = nullptr;
  short *vals = nullptr, *vals2 = nullptr;
  TRY(diter_alloc(ctx, (void **)&rows2, sizeof(int) * (size_t)nnz));
  TRY(diter_alloc(ctx, (void **)&keys, sizeof(int) * (size_t)m));
  TRY(diter_alloc(ctx, (void **)&vals, sizeof(short) * (size_t)m));
  k_near_split<<<blocks, kSetupThreads, 0, ctx->stream>>>(ctx->col_ptr, ctx->row_idx, n, nn, near_off, rows2, keys,
                                                          vals);
  diter_free(ctx, ctx->row_idx);
  ctx->row_idx = rows2;
  diter_free(ctx, near_off);
  tr.mark(ctx->stream, "split");
  // sort the near edges by row
  TRY(diter_alloc(ctx, (void **)&keys2, sizeof(int) * (size_t)m));
  TRY(diter_alloc(ctx, (void **)&vals2, sizeof(short) * (size_t)m));
  int end_bit = 1;
  while (end_bit < 31 && ((n - 1) >> end_bit) != 0) ++end_bit;
  tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, vals, vals2, (int64_t)m, 0, end_bit, ctx->stream));
  TRY(diter_alloc(ctx, &tmp, tb));
  CK(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, vals, vals2, (int64_t)m, 0, end_bit, ctx->stream));
  diter_free(ctx, tmp);
  diter_free(ctx, keys);
  diter_free(ctx, vals);
  tr.mark(ctx->stream, "sort");
  long long *rowptr = nullptr;
  TRY(diter_alloc(ctx, (void **)&rowptr, sizeof(long long) * (size_t)(n + 1)));
  k_row_bounds<<<blocks, 256, 0, ctx->stream>>>(keys2, m, n, rowptr);
  diter_free(ctx, keys2);
  // tiles: perm + slice lengths, scan, fill
  const long long n_tiles = (n + kPullR - 1) / kPullR;
  const long long n_slices = n_tiles * kTileSlices;
  unsigned short *perm = nullptr;
  unsigned *sptr = nullptr, *off = nullptr;
  unsigned long long *slen = nullptr, *sptr64 = nullptr;
  TRY(diter_alloc(ctx, (void **)&perm, sizeof(unsigned short) * (size_t)(n_tiles * kPullR)));
  TRY(diter_alloc(ctx, (void **)&slen, sizeof(unsigned long long) * (size_t)(n_slices + 1)));
  TRY(diter_alloc(ctx, (void **)&sptr64, sizeof(unsigned long long) * (size_t)(n_slices + 1)));
  k_tile_sort<<<(unsigned)n_tiles, kSetupThreads, 0, ctx->stream>>>(rowptr, n, perm, slen);
  CK(cudaMemsetAsync(slen + n_slices, 0, sizeof(unsigned long long), ctx->stream));
  tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, slen, sptr64, (int64_t)(n_slices + 1), ctx->stream));
  TRY(diter_alloc(ctx, &tmp, tb));
  CK(cub::DeviceScan::ExclusiveSum(tmp, tb, slen, sptr64, (int64_t)(n_slices + 1), ctx->stream));
  diter_free(ctx, tmp);
  diter_free(ctx, slen);
  unsigned long long pairs = 0;
  CK(cudaMemcpyAsync(&pairs, sptr64 + n_slices, sizeof(pairs), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (pairs >= (1ull << 32)) {     // pathological duplicate-heavy rows: keep the push path
    diter_free(ctx, sptr64); diter_free(ctx, perm); diter_free(ctx, rowptr); diter_free(ctx, vals2); diter_free(ctx, nn);
    CK(cudaStreamSynchronize(ctx->stream));
    return DI_OK;
  }
  TRY(diter_alloc(ctx, (void **)&sptr, sizeof(unsigned) * (size_t)(n_slices + 1)));
  k_narrow<<<blocks, 256, 0, ctx->stream>>>(sptr64, sptr, n_slices + 1);
  diter_free(ctx, sptr64);
  tr.mark(ctx->stream, "tiles");
  TRY(diter_alloc(ctx, (void **)&off, sizeof(unsigned) * 32 * (size_t)std::max(1ull, pairs)));
  k_fill_slices<<<blocks, 256, 0, ctx->stream>>>(rowptr, vals2, n, n_tiles, perm, sptr, off);
  diter_free(ctx, rowptr);
  diter_free(ctx, vals2);
  // per-pass buffers
  TRY(diter_alloc(ctx, (void **)&ctx->pull_sw, sizeof(double) * (size_t)n));
  TRY(diter_alloc(ctx, (void **)&ctx->pull_bits, sizeof(unsigned) * (size_t)(((n + 31) >> 5) + kSelectItems)));
  CK(cudaMemsetAsync(ctx->pull_bits, 0, sizeof(unsigned) * (size_t)(((n + 31) >> 5) + kSelectItems), ctx->stream));
  CK(cudaFuncSetAttribute(k_pull, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)(sizeof(double) * (kPullZero + 1 + kPullR))));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_pull, kPullThreads,
                                                    sizeof(double) * (kPullZero + 1 + kPullR)));
  ctx->grid_pull = (int)std::max(1LL, std::min<long long>(n_tiles, (long long)ctx->num_sms * std::max(1, occ)));
  ctx->pull_nn = nn;
  ctx->pull_perm = perm;
  ctx->pull_sptr = sptr;
  ctx->pull_off = off;
  ctx->pull_tiles = n_tiles;
  ctx->pull_near = m;
  ctx->pull_pairs = (long long)pairs;
  ctx->fr.sel_bits = ctx->pull_bits;
  ctx->pull_on = 1;
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaGetLastError());
  tr.mark(ctx->stream, "fill");
  return DI_OK;
}

void diter_pull_launch(di_ctx *ctx) {
  if (!ctx->pull_on) return;
  k_pull<<<ctx->grid_pull, kPullThreads, sizeof(double) * (kPullZero + 1 + kPullR), ctx->stream>>>(
      ctx->F, ctx->pull_sw, ctx->pull_bits, ctx->pull_perm, ctx->pull_sptr, ctx->pull_off, ctx->n_local,
      ctx->pull_tiles, ctx->ctl);
}

void diter_pull_free(di_ctx *ctx) {
  void *ptrs[] = {ctx->pull_nn, ctx->pull_perm, ctx->pull_sptr, ctx->pull_off, ctx->pull_sw, ctx->pull_bits};
  for (void *p : ptrs) diter_free(ctx, p);
  ctx->pull_nn = nullptr; ctx->pull_perm = nullptr; ctx->pull_sptr = nullptr;
  ctx->pull_off = nullptr; ctx->pull_sw = nullptr; ctx->pull_bits = nullptr;
  ctx->pull_on = 0;
}
