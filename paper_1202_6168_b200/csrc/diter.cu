// diter.cu -- libditer.so: C ABI (include/diter.h) over the sm_100a kernels.
//
// Host side of one context: upload + validation (di_create), the pass loop
// captured as a CUDA graph of `check_interval` passes (di_run), getters.
// No CPU fallback exists: every step of a pass runs in the kernels of
// kernels.cuh; the host only launches graphs and reads the stop flag.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <vector>

#include "../../include/diter.h"
#include "ctx.cuh"
#include "kernels.cuh"

using namespace diter;

static thread_local std::string g_thread_err;

void diter_set_err(di_ctx *ctx, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  g_thread_err = buf;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      diter_set_err(ctx, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),       \
                    __FILE__, __LINE__);                                               \
      return e_ == cudaErrorMemoryAllocation ? DI_ERR_OOM : DI_ERR_CUDA;               \
    }                                                                                  \
  } while (0)

extern "C" size_t di_struct_size(int32_t which) {
  switch (which) {
    case 0: return sizeof(di_options);
    case 1: return sizeof(di_stats);
    case 2: return sizeof(di_pass_log);
    default: return 0;
  }
}

extern "C" void di_default_options(di_options *o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->policy = DI_POLICY_HYBRID;
  o->check_interval = 16;
  o->alpha = 1.5;
  o->hybrid_frac = 0.05;
  o->t0 = 0.0;
  o->max_passes = 1000000;
  o->exchange_mode = DI_EXCHANGE_ASYNC;
  o->device = -1;
  o->scatter_kernel = 0;
  o->profile = 0;
  o->pass_kernel = 0;
  o->receive_rescale = 1;
}

// Device memory of a context comes from one stream-ordered pool per device that
// keeps what contexts free (release threshold = max): the ~11 GB of a C4 context
// is mapped once per process, and create/destroy cycles (bench e2e) no longer pay
// cudaMalloc / cudaFree of multi-GB buffers (measured: usually ~10 ms, sporadically
// 300-400 ms per call).
static cudaMemPool_t device_pool(int dev) {
  static std::mutex mu;
  static std::vector<cudaMemPool_t> pools;
  std::lock_guard<std::mutex> g(mu);
  if ((int)pools.size() <= dev) pools.resize(dev + 1, nullptr);
  if (!pools[dev]) {
    cudaMemPoolProps pr = {};
    pr.allocType = cudaMemAllocationTypePinned;
    pr.location.type = cudaMemLocationTypeDevice;
    pr.location.id = dev;
    cudaMemPool_t mp = nullptr;
    if (cudaMemPoolCreate(&mp, &pr) != cudaSuccess) return nullptr;
    unsigned long long keep = ~0ull;
    cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[dev] = mp;
  }
  return pools[dev];
}

di_status diter_alloc(di_ctx *ctx, void **p, size_t bytes) {
  *p = nullptr;
  cudaMemPool_t mp = device_pool(ctx->device);
  if (!mp) { diter_set_err(ctx, "cudaMemPoolCreate failed on device %d", ctx->device); return DI_ERR_CUDA; }
  CK(cudaMallocFromPoolAsync(p, bytes ? bytes : 1, mp, ctx->stream));
  return DI_OK;
}

// ctx->stream may be null (a context whose stream moved to its rebuilt successor):
// its work is complete, the legacy stream orders the free
void diter_free(di_ctx *ctx, void *p) {
  if (p) cudaFreeAsync(p, ctx->stream);
}

template <typename T>
static di_status dalloc(di_ctx *ctx, T **p, size_t count) {
  return diter_alloc(ctx, (void **)p, (count ? count : 1) * sizeof(T));
}

#define TRY(x)                      \
  do {                              \
    di_status s_ = (x);             \
    if (s_ != DI_OK) return s_;     \
  } while (0)

static void l2_release(di_ctx *ctx);

static void free_ctx(di_ctx *c) {
  if (!c) return;
  const bool tr = std::getenv("DITER_TRACE") != nullptr;
  auto t = std::chrono::steady_clock::now();
  auto mark = [&](const char *what) {
    if (!tr) return;
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[diter destroy] %-16s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  };
  if (c->device >= 0) cudaSetDevice(c->device);
  l2_release(c);
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
  mark("graph exec");
  for (cudaEvent_t e : c->prof_ev)
    if (e) cudaEventDestroy(e);
  void *ptrs[] = {c->col_ptr, c->row_idx, c->vals, c->d_b, c->F, c->H, c->fr.ids, c->fr.S, c->fr.seg_cnt, const_cast<unsigned *>(c->fr.dang_bits), const_cast<unsigned *>(c->fr.cp32),
                  c->fr.hub_w, c->fr.hub_b0, c->fr.hub_deg, c->fr.hub_chunk, c->fr.hub_cslot, c->sel_part, c->sc_part,
                  c->l1_part, c->l1_out, c->ctl, c->log, c->far_off, c->far.rows, c->far.vals, c->far.fill, c->kw, c->nloc, c->H_old};
  if (c->stream) cudaStreamSynchronize(c->stream);
  mark("sync");
  for (void *p : ptrs) diter_free(c, p);
  mark("frees");
  if (c->h_ctl) cudaFreeHost(c->h_ctl);
  mark("free host");
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  diter_dist_free(c);
  cudaStreamSynchronize(c->stream);            // the frees above are stream-ordered
  mark("sync frees");
  if (c->stream) cudaStreamDestroy(c->stream);
  mark("stream");
  delete c;
}

// Launch geometry: persistent kernels sized to the SM count x resident CTAs.
// The select grid fixes the frontier segmentation: n_seg = CTAs x 8 warps, each
// warp owning seg_len consecutive nodes (a multiple of 256); the scatter keeps
// the prefix over segments in (n_seg + 1) ints of dynamic shared memory.
static di_status setup_geometry(di_ctx *ctx) {
  // one attribute query (cudaGetDeviceProperties fills ~100 fields, 3-20 ms)
  CK(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
  const long long n = ctx->n_local;
  constexpr int kWarps = kSelectThreads / 32;
  int occ_sel = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_sel, k_select, kSelectThreads, 0));
  const long long spans = (n + kSelectSpan - 1) / kSelectSpan;             // 256-node warp iterations
  const long long sel_need = (spans + kWarps - 1) / kWarps;
  long long gs = std::min<long long>(sel_need, (long long)ctx->num_sms * std::max(1, std::min(occ_sel, kSelectCtasPerSm)));
  gs = std::max(1LL, std::min<long long>(gs, kMaxSegments / kWarps));
  // fused cooperative pass kernel (small graphs, one GPU): every CTA co-resident, and the
  // select phase runs on the fused grid, so the segmentation follows that grid
  const int pk = ctx->opt.pass_kernel;
  ctx->fused = ctx->dist == nullptr && pk == 2;
  if (ctx->fused) {
    const size_t dyn = sizeof(int) * (size_t)(std::min(ctx->num_sms * 4 * kWarps, kMaxSegments) + 1);
    int occ_f = 0;
    if (ctx->vals) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_f, k_pass_fused<true>, kScatterThreads, dyn));
    else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_f, k_pass_fused<false>, kScatterThreads, dyn));
    ctx->grid_fused = ctx->num_sms * std::max(1, std::min(occ_f, 4));
    // a small graph gets a small grid: the three grid barriers per pass then span few
    // CTAs (1 CTA for configs[0]); one CTA per 4096 nodes
    ctx->grid_fused = (int)std::max(1LL, std::min<long long>(ctx->grid_fused, (n + 4095) / 4096));
    gs = std::min<long long>(ctx->grid_fused, kMaxSegments / kWarps);
  }
  ctx->grid_select = (int)gs;
  ctx->fr.n_seg = (int)gs * kWarps;
  const long long per = (n + ctx->fr.n_seg - 1) / ctx->fr.n_seg;
  ctx->fr.seg_len = std::max<long long>(kSelectSpan, (per + kSelectSpan - 1) / kSelectSpan * kSelectSpan);
  ctx->scatter_smem = sizeof(int) * (size_t)(ctx->fr.n_seg + 1);
  ctx->fr.run = ctx->opt.scatter_run > 0 ? ctx->opt.scatter_run : 2;
  ctx->fr.stripes = (ctx->opt.scatter_stripes > 0 && ctx->opt.scatter_stripes <= kStripes) ? ctx->opt.scatter_stripes : 8;
  int occ_sc = 0;
  if (ctx->vals) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_sc, k_scatter<true>, kScatterThreads, ctx->scatter_smem));
  else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_sc, k_scatter<false>, kScatterThreads, ctx->scatter_smem));
  ctx->grid_scatter = ctx->fused ? ctx->grid_fused : ctx->num_sms * std::max(1, occ_sc);
  // a frontier holds at most n / 32 groups: more than one CTA (8 warps) per 256 nodes
  // would only zero and flush hot windows (C1: 4 CTAs instead of 444)
  if (!ctx->fused) ctx->grid_scatter = (int)std::max(1LL, std::min<long long>(ctx->grid_scatter, (n + 255) / 256));
  ctx->grid_l1 = (int)std::min<long long>(ctx->num_sms * 8LL, std::max(1LL, (n + 255) / 256));
  // hub chunks: k_scatter_hubs holds 8-16 edges in flight per thread at 32-48 registers,
  // so its grid fills every resident CTA slot (DITER_HUB_CTAS_PER_SM caps it; 0 = occupancy)
  int occ_hub = 0;
  if (ctx->vals) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_hub, k_scatter_hubs<true>, kScatterThreads, 0));
  else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_hub, k_scatter_hubs<false>, kScatterThreads, 0));
  if (DITER_HUB_CTAS_PER_SM > 0) occ_hub = std::min(occ_hub, DITER_HUB_CTAS_PER_SM);
  ctx->grid_hubs = ctx->num_sms * std::max(1, occ_hub);
  return DI_OK;
}

// The shared-memory hot window of the scatter: the 2048 consecutive rows (aligned
// to 1024) whose sampled in-degree is largest.  Rows are global ids; on a
// distributed context only rows of the local range are candidates.
static di_status choose_hot_window(di_ctx *ctx) {
  const long long n = ctx->n_rows;
  ctx->hot_lo = (int)ctx->lo;
  if (ctx->opt.hot_window < 0) {           // disabled: no row matches INT_MIN
    ctx->hot_lo = -2147483647 - 1;
    return DI_OK;
  }
  if (ctx->n_local < kHot) {
    // one GPU: the window [0, kHot) covers every row; distributed: the window must
    // lie inside the owned range, so it is disabled (no row matches INT_MIN)
    ctx->hot_lo = (ctx->world == 1) ? 0 : (-2147483647 - 1);
    return DI_OK;
  }
  if (ctx->nnz_local == 0) return DI_OK;
  const long long nb = (n >> 10) + 1;
  unsigned *blk = nullptr;
  TRY(dalloc(ctx, &blk, (size_t)nb));
  CK(cudaMemsetAsync(blk, 0, sizeof(unsigned) * nb, ctx->stream));
  const int stride = ctx->nnz_local > (1LL << 24) ? 64 : 1;
  k_hot_sample<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->row_idx, ctx->nnz_local, stride, blk);
  std::vector<unsigned> &h = ctx->blk_hist;
  h.assign(nb, 0u);
  ctx->blk_stride = stride;
  CK(cudaMemcpyAsync(h.data(), blk, sizeof(unsigned) * nb, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  diter_free(ctx, blk);
  long long best = ctx->lo >> 10, best_mass = -1;
  const long long hi = ctx->lo + ctx->n_local;
  for (long long b = 0; b + 1 < nb; ++b) {
    if ((b << 10) < ctx->lo || (b << 10) + kHot > hi) continue;   // owned rows only
    const long long m = (long long)h[b] + h[b + 1];
    if (m > best_mass) { best_mass = m; best = b; }
  }
  ctx->hot_lo = (int)std::max<long long>(ctx->lo, std::min<long long>(best << 10, hi - kHot));
  return DI_OK;
}

// L2 persisting window (options.l2_persist): the set-aside is a device-wide limit,
// taken by the first context that wants a window and released (with the persisting
// lines) when the last one is destroyed.
static std::mutex g_l2_mu;
static std::vector<int> g_l2_users;

static di_status l2_acquire(di_ctx *ctx, size_t bytes) {
  std::lock_guard<std::mutex> g(g_l2_mu);
  if ((int)g_l2_users.size() <= ctx->device) g_l2_users.resize(ctx->device + 1, 0);
  int maxp = 0;
  CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, ctx->device));
  size_t cur = 0;
  CK(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
  const size_t want = std::min(bytes, (size_t)maxp);
  if (want > cur) CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
  ++g_l2_users[ctx->device];
  return DI_OK;
}

static void l2_release(di_ctx *ctx) {
  if (ctx->l2_bytes == 0) return;
  std::lock_guard<std::mutex> g(g_l2_mu);
  if (ctx->device < (int)g_l2_users.size() && --g_l2_users[ctx->device] == 0) {
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
  }
  ctx->l2_bytes = 0;
}

// Window rows: the 1024-row-aligned range of the window size with the most sampled
// pushes among the owned rows.  Auto: off while F fits in 64 MB (it stays L2-resident
// anyway); else 28 MB when F is at most 2x the L2 and 20 MB above that.  Measured on
// this B200 (126 MB L2): C3 (F 134 MB, permuted R-MAT -- no hot rows, the window just
// keeps part of an oversized working set from thrashing) 219 -> 184 ms at 28-30 MB;
// C4 (F 800 MB, the Zipf-over-id head: 26 % of the pushes in the first 20 MB) 265 ->
// 250 ms at 20 MB.  Larger set-asides slow the select's streaming (C4 24 MB: +6 ms,
// C3 >= 32 MB: +5 ms) and 79 MB (the maximum) loses outright.
static di_status choose_l2_window(di_ctx *ctx) {
  ctx->l2_lo = 0;
  ctx->l2_bytes = 0;
  const int opt = ctx->opt.l2_persist;
  const long long n = ctx->n_local;
  if (opt < 0 || n == 0 || (opt == 0 && ctx->blk_hist.empty())) return DI_OK;
  const long long f_bytes = n * (long long)sizeof(double);
  if (opt == 0 && f_bytes <= (64LL << 20)) return DI_OK;
  int l2 = 0;
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device));
  // asynchronous sweeps have no separate streaming select for the set-aside to slow
  // down, so they take larger windows: C4 182.4 -> 178.8 ms at 28 MB, C3 135.6 -> 130.7
  // ms at 36 MB (profiles/r02s_l2_window.txt)
  const bool sweeps = ctx->opt.sweep == 1 && !ctx->fused &&
                      (!ctx->dist || ctx->opt.exchange_mode != DI_EXCHANGE_SYNC);
  const long long auto_mb = f_bytes <= 2LL * l2 ? (sweeps ? 36 : 28) : (sweeps ? 28 : 20);
  const long long want_rows = ((opt > 0 ? (long long)opt : auto_mb) << 20) / (long long)sizeof(double);
  // no in-degree sample (hot window off): a forced window starts at the owned range
  const std::vector<unsigned> h = ctx->blk_hist.empty() ? std::vector<unsigned>((size_t)((ctx->lo + n + 1023) >> 10), 0u)
                                                        : ctx->blk_hist;
  const long long b_lo = ctx->lo >> 10, b_hi = std::min<long long>((long long)h.size(), (ctx->lo + n + 1023) >> 10);
  const long long wb = std::max(1LL, std::min(want_rows >> 10, b_hi - b_lo));
  long long tot = 0, win = 0, best = -1, best_b = b_lo;
  for (long long b = b_lo; b < b_hi; ++b) tot += h[b];
  for (long long b = b_lo; b < b_hi; ++b) {
    win += h[b];
    if (b - b_lo >= wb) win -= h[b - wb];
    if (b - b_lo + 1 >= wb && win > best) { best = win; best_b = b - wb + 1; }
  }
  const long long row0 = std::max(ctx->lo, best_b << 10) - ctx->lo;             // local row
  const long long rows = std::min(wb << 10, n - row0);
  if (rows <= 0) return DI_OK;
  int max_win = 0;
  CK(cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device));
  const size_t bytes = std::min((size_t)rows * sizeof(double), (size_t)max_win);
  TRY(l2_acquire(ctx, bytes));
  ctx->l2_lo = row0;
  ctx->l2_bytes = (long long)bytes;
  if (std::getenv("DITER_TRACE"))
    std::fprintf(stderr, "[diter setup] L2 window rows [%lld, %lld) %.1f MB, %.1f%% of sampled pushes\n", ctx->lo + row0,
                 ctx->lo + row0 + rows, bytes / 1048576.0, tot ? 100.0 * (double)best / (double)tot : 0.0);
  return diter_set_l2_window(ctx);
}

// The window as the stream's access policy (kernels launched or captured on it
// afterwards carry it); cleared when the context has none.
di_status diter_set_l2_window(di_ctx *ctx) {
  if (!ctx->stream) return DI_OK;
  cudaStreamAttrValue av = {};
  if (ctx->l2_bytes > 0) {
    av.accessPolicyWindow.base_ptr = ctx->F + ctx->l2_lo;
    av.accessPolicyWindow.num_bytes = (size_t)ctx->l2_bytes;
    av.accessPolicyWindow.hitRatio = 1.0f;
    av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  }
  CK(cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &av));
  return DI_OK;
}

// Far-push bins (propagation blocking, Far in types.cuh): one GPU, F too large to
// stay L2-resident.  The warm range is the 2^far_warm_log2 consecutive rows of
// largest sampled in-degree (kept on direct L2 REDs); bins of 2^shift rows, at
// most kMaxBins, sized by an exact census of the edges that can be far.
static di_status setup_far(di_ctx *ctx) {
  ctx->far = Far{};
  ctx->far.warm_len = 0u;
  const int mode = ctx->opt.far_push;
  const long long n = ctx->n_rows;
  const bool want = mode > 0;   // auto = off: on C4 the emission costs more than the tail REDs it saves
  if (!want || mode < 0 || ctx->dist || ctx->fused || ctx->nnz_local == 0 || ctx->blk_hist.empty()) return DI_OK;
  int shift = 20;
  while (((n - 1) >> shift) + 1 > kMaxBins) ++shift;
  const int n_bins = (int)(((n - 1) >> shift) + 1);
  const int wl = ctx->opt.far_warm_log2 > 0 ? std::min(ctx->opt.far_warm_log2, 30) : 21;
  const long long W = std::min<long long>(1LL << wl, n);
  // warm window: W rows (W/1024 blocks) with the largest sampled in-degree mass
  const std::vector<unsigned> &h = ctx->blk_hist;
  const long long nbk = (long long)h.size(), wb = std::max<long long>(1, W >> 10);
  long long best = 0, cur = 0, best_sum = -1;
  for (long long b = 0; b < nbk; ++b) {
    cur += h[b];
    if (b >= wb) cur -= h[b - wb];
    if (b + 1 >= wb && cur > best_sum) { best_sum = cur; best = b + 1 - wb; }
  }
  long long warm_lo = std::min<long long>(best << 10, std::max<long long>(0, n - W));
  ctx->far.warm_lo = (int)warm_lo;
  ctx->far.warm_len = (unsigned)W;
  ctx->far.shift = shift;
  ctx->far.n_bins = n_bins;
  {
    // the far scatter stages records in 24 KB more shared memory per CTA: static +
    // dynamic then exceed the default 48 KB, which needs the opt-in.  The attribute is
    // per function, process-wide: every context sets the same value (the largest
    // prefix), so contexts of different sizes on concurrent threads never shrink the
    // limit under one another's launches.
    const int dyn = (int)(sizeof(int) * (size_t)(kMaxSegments + 1));
    CK(cudaFuncSetAttribute(k_scatter<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    CK(cudaFuncSetAttribute(k_scatter<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    int occ = 0;
    if (ctx->vals) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scatter<true, false, true>, kScatterThreads, ctx->scatter_smem));
    else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scatter<false, false, true>, kScatterThreads, ctx->scatter_smem));
    ctx->grid_scatter = std::min(ctx->grid_scatter, ctx->num_sms * std::max(1, occ));
  }
  unsigned long long *d_cap = nullptr;
  TRY(dalloc(ctx, &d_cap, (size_t)kMaxBins));
  CK(cudaMemsetAsync(d_cap, 0, sizeof(unsigned long long) * kMaxBins, ctx->stream));
  k_far_census<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->col_ptr, ctx->n_local, ctx->row_idx, ctx->lo,
                                                          ctx->hot_lo, ctx->far.warm_lo, ctx->far.warm_len, shift, d_cap);
  std::vector<unsigned long long> cap(kMaxBins);
  CK(cudaMemcpyAsync(cap.data(), d_cap, sizeof(unsigned long long) * kMaxBins, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  diter_free(ctx, d_cap);
  // chunks per bin: every chunk closed before the end of a pass holds > kFarChunk - 32
  // records, and each scatter warp leaves at most one partial chunk per bin
  const long long warps = (long long)ctx->grid_scatter * (kScatterThreads / 32);
  std::vector<long long> coff(n_bins + 1, 0);
  long long recs = 0;
  for (int b = 0; b < n_bins; ++b) {
    recs += (long long)cap[b];
    const long long nch = cap[b] ? (long long)(cap[b] + (kFarChunk - 32) - 1) / (kFarChunk - 32) + warps : 0;
    coff[b + 1] = coff[b] + nch;
  }
  ctx->far_cap = coff[n_bins];
  if (recs == 0) { ctx->far = Far{}; return DI_OK; }
  TRY(dalloc(ctx, &ctx->far_off, (size_t)n_bins + 1));
  CK(cudaMemcpyAsync(ctx->far_off, coff.data(), sizeof(long long) * (n_bins + 1), cudaMemcpyHostToDevice, ctx->stream));
  TRY(dalloc(ctx, &ctx->far.rows, (size_t)ctx->far_cap * kFarChunk));
  TRY(dalloc(ctx, &ctx->far.vals, (size_t)ctx->far_cap * kFarChunk));
  TRY(dalloc(ctx, &ctx->far.fill, (size_t)ctx->far_cap));
  ctx->far.coff = ctx->far_off;
  ctx->far.on = 1;
  CK(cudaStreamSynchronize(ctx->stream));
  return DI_OK;
}

// Selection-key weights (DI_KEY_*, reading R20).  The paper key needs the global
// in-degree of every owned row: a distributed rank gets it by a reduce-scatter.
static di_status setup_key(di_ctx *ctx) {
  const int key = ctx->opt.select_key;
  if (key == DI_KEY_RAW) return DI_OK;
  if (key != DI_KEY_EDGE && key != DI_KEY_PAPER) {
    diter_set_err(ctx, "select_key must be DI_KEY_RAW, DI_KEY_EDGE or DI_KEY_PAPER");
    return DI_ERR_INVALID_ARG;
  }
  const long long n = ctx->n_local;
  TRY(dalloc(ctx, &ctx->kw, (size_t)n));
  unsigned *indeg = nullptr;
  if (key == DI_KEY_PAPER) {
    TRY(dalloc(ctx, &indeg, (size_t)n));
    if (ctx->world > 1) {
      TRY(diter_dist_indegree(ctx, indeg));   // global in-degrees of the owned rows (collective)
    } else {
      CK(cudaMemsetAsync(indeg, 0, sizeof(unsigned) * n, ctx->stream));
      k_in_degree<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->row_idx, ctx->nnz_local, indeg);
    }
  }
  k_key_weights<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->col_ptr, n, indeg, key, ctx->kw);
  CK(cudaStreamSynchronize(ctx->stream));
  if (indeg) diter_free(ctx, indeg);
  CK(cudaGetLastError());
  return DI_OK;
}

Graph diter_graph(const di_ctx *ctx) {
  Graph g{ctx->col_ptr, ctx->row_idx, ctx->vals, ctx->n_local, ctx->d, ctx->hot_lo,
          ctx->lo, ctx->G, ctx->dflags, ctx->far, ctx->nloc,
          ctx->opt.remote_push != DI_REMOTE_PER_DIFFUSION ? 1 : 0};
  g.defer = ctx->defer_m > 0 ? 1 : 0;
  return g;
}

// One sweep (k_sweep, + the hub chunks it listed) on the context's stream.
#ifndef DITER_SWEEP_KEY_DERIVED
#define DITER_SWEEP_KEY_DERIVED 1    // per-edge key from col_ptr in sweeps (no weight stream)
#endif
typedef void (*SweepFn)(Graph, double *, double *, Frontier, Ctl *, SelPartial *, ScPartial *, const float *);

// k_sweep instance: signed / PageRank x key mode (0 raw, 1 kw weights, 2 per-edge key
// derived from col_ptr) x distributed
template <bool SIGNED, bool DIST>
static SweepFn sweep_fn(int key) {
  return key == 0 ? k_sweep<SIGNED, 0, DIST> : key == 1 ? k_sweep<SIGNED, 1, DIST> : k_sweep<SIGNED, 2, DIST>;
}

static int sweep_key_mode(const di_ctx *ctx) {
  if (!ctx->kw) return 0;
  return (DITER_SWEEP_KEY_DERIVED && ctx->opt.select_key == DI_KEY_EDGE) ? 2 : 1;
}

void diter_launch_sweep(di_ctx *ctx) {
  const Graph g = diter_graph(ctx);
  const bool dist = ctx->dist != nullptr;
  const int key = sweep_key_mode(ctx);
  SweepFn sw = dist ? (ctx->vals ? sweep_fn<true, true>(key) : sweep_fn<false, true>(key))
                    : (ctx->vals ? sweep_fn<true, false>(key) : sweep_fn<false, false>(key));
  sw<<<ctx->grid_sweep, kScatterThreads, kSweepDynSmem, ctx->stream>>>(g, ctx->F, ctx->H, ctx->fr, ctx->ctl,
                                                                       ctx->sel_part, ctx->sc_part, ctx->kw);
  if (ctx->cap_hub > 0 && !DITER_SWEEP_HUBS) {
    if (ctx->vals)
      k_scatter_hubs<true><<<ctx->grid_hubs, kScatterThreads, 0, ctx->stream>>>(g, ctx->F, ctx->fr, ctx->ctl);
    else
      k_scatter_hubs<false><<<ctx->grid_hubs, kScatterThreads, 0, ctx->stream>>>(g, ctx->F, ctx->fr, ctx->ctl);
  }
}

// Capture check_interval passes of (select, scatter, finalize) once.
di_status diter_capture_graph(di_ctx *ctx) {
  if (ctx->graph_exec) {
    CK(cudaGraphExecDestroy(ctx->graph_exec));
    ctx->graph_exec = nullptr;
  }
  cudaGraph_t graph;
  CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  Graph g = diter_graph(ctx);
  const bool prof = ctx->opt.profile != 0;
  if (prof && ctx->prof_ev.empty()) {
    ctx->prof_ev.assign(4 * ctx->check_interval, nullptr);
    for (auto &e : ctx->prof_ev) CK(cudaEventCreate(&e));
  }
  for (int k = 0; k < ctx->check_interval; ++k) {
    diter_dist_pass_prologue(ctx);   // DI_EXCHANGE_P2P: merge what has arrived before every pass
    if (prof) CK(cudaEventRecordWithFlags(ctx->prof_ev[4 * k + 0], ctx->stream, cudaEventRecordExternal));
    const bool dist = ctx->dist != nullptr;
    if (ctx->sweep_on) {
      // one-kernel async sweep (select + diffusion; options.sweep): the profile's
      // "select" span is empty, its "scatter" span is the sweep + hub chunks
      if (prof) CK(cudaEventRecordWithFlags(ctx->prof_ev[4 * k + 1], ctx->stream, cudaEventRecordExternal));
      diter_launch_sweep(ctx);
      if (prof) CK(cudaEventRecordWithFlags(ctx->prof_ev[4 * k + 2], ctx->stream, cudaEventRecordExternal));
      k_finalize<<<1, kFinalizeThreads, 0, ctx->stream>>>(ctx->ctl, ctx->sel_part, ctx->grid_sweep, ctx->sc_part,
                                                          ctx->grid_sweep, ctx->log);
      if (ctx->vals) {    // signed P: exact |F|_1 after each sweep (the carried bound is loose)
        k_l1_partial<<<ctx->grid_l1, kSelectThreads, 0, ctx->stream>>>(ctx->F, ctx->n_local, ctx->l1_part);
        k_l1_final<<<1, kFinalizeThreads, 0, ctx->stream>>>(ctx->l1_part, ctx->grid_l1, ctx->l1_out);
        k_sweep_check<<<1, 1, 0, ctx->stream>>>(ctx->ctl, ctx->l1_out);
      }
      if (prof) CK(cudaEventRecordWithFlags(ctx->prof_ev[4 * k + 3], ctx->stream, cudaEventRecordExternal));
      continue;
    }
    k_select<<<ctx->grid_select, kSelectThreads, 0, ctx->stream>>>(ctx->F, ctx->H, ctx->fr, ctx->n_local,
                                                                  ctx->ctl, ctx->sel_part, ctx->kw);
    if (prof) CK(cudaEventRecordWithFlags(ctx->prof_ev[4 * k + 1], ctx->stream, cudaEventRecordExternal));
    // a distributed rank's scatter routes rows outside its range (DIST): its ASYNC / P2P
    // rounds launch this graph for their local passes
    if (ctx->vals)
      (dist ? k_scatter<true, true, false> : ctx->far.on ? k_scatter<true, false, true> : k_scatter<true, false, false>)
          <<<ctx->grid_scatter, kScatterThreads, ctx->scatter_smem, ctx->stream>>>(g, ctx->F, ctx->fr, ctx->ctl, ctx->sc_part);
    else
      (dist ? k_scatter<false, true, false> : ctx->far.on ? k_scatter<false, false, true> : k_scatter<false, false, false>)
          <<<ctx->grid_scatter, kScatterThreads, ctx->scatter_smem, ctx->stream>>>(g, ctx->F, ctx->fr, ctx->ctl, ctx->sc_part);
    if (ctx->cap_hub > 0) {
      if (ctx->vals)
        k_scatter_hubs<true><<<ctx->grid_hubs, kScatterThreads, 0, ctx->stream>>>(g, ctx->F, ctx->fr, ctx->ctl);
      else
        k_scatter_hubs<false><<<ctx->grid_hubs, kScatterThreads, 0, ctx->stream>>>(g, ctx->F, ctx->fr, ctx->ctl);
    }
    if (ctx->far.on)
      k_apply_far<<<ctx->num_sms * 4, kApplyThreads, 0, ctx->stream>>>(ctx->F, ctx->far, ctx->lo, ctx->ctl);
    if (prof) CK(cudaEventRecordWithFlags(ctx->prof_ev[4 * k + 2], ctx->stream, cudaEventRecordExternal));
    k_finalize<<<1, kFinalizeThreads, 0, ctx->stream>>>(ctx->ctl, ctx->sel_part, ctx->grid_select, ctx->sc_part,
                                                        ctx->grid_scatter, ctx->log);
    diter_defer_launch(ctx);    // far-edge increments when k_finalize asked (returns at once otherwise)
    if (prof) CK(cudaEventRecordWithFlags(ctx->prof_ev[4 * k + 3], ctx->stream, cudaEventRecordExternal));
  }
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
  if (e != cudaSuccess) {
    diter_set_err(ctx, "graph capture failed: %s", cudaGetErrorString(e));
    return DI_ERR_CUDA;
  }
  e = cudaGraphInstantiate(&ctx->graph_exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) {
    diter_set_err(ctx, "graph instantiate failed: %s", cudaGetErrorString(e));
    return DI_ERR_CUDA;
  }
  return DI_OK;
}

// T_0 = max |B_i| w_i / alpha (reading R5) unless options.t0 > 0; needs F = B and
// the key weights.  The max is global on a distributed context (collective).
static di_status initial_threshold(di_ctx *ctx, double *T0) {
  if (*T0 > 0.0) return DI_OK;
  const long long n = ctx->n_local;
  double mx = 0.0;
  if (n > 0) {
    k_max_abs<<<ctx->grid_l1, 256, 0, ctx->stream>>>(ctx->F, n, ctx->l1_part, ctx->kw);
    std::vector<double> hp(ctx->grid_l1);
    CK(cudaMemcpyAsync(hp.data(), ctx->l1_part, sizeof(double) * ctx->grid_l1, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (double v : hp) mx = std::max(mx, v);
  }
  TRY(diter_dist_max(ctx, mx, &mx));   // global max over ranks (identity when not distributed)
  *T0 = mx / ctx->opt.alpha;
  return DI_OK;
}

// DITER_TRACE=1: stream-synchronised phase times of the setup on stderr.
struct SetupTrace {
  bool on = std::getenv("DITER_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(cudaStream_t s, const char *what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[diter setup] %-22s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// Shared by di_create and di_create_dist: upload, validate, allocate, init.
di_status diter_setup(di_ctx *ctx, const int64_t *col_ptr, const int32_t *row_idx,
                      const double *values, const double *b, const di_options *opt) {
  NvtxRange nv("diter setup");
  di_options o;
  if (opt) o = *opt; else di_default_options(&o);
  if (!(o.alpha > 1.0) || o.check_interval < 1 || o.check_interval > 4096 || o.max_passes < 1 ||
      (o.policy != DI_POLICY_GEOM && o.policy != DI_POLICY_HYBRID) || !(o.hybrid_frac >= 0.0) ||
      o.key_offset < 0 || o.key_offset > (1 << 20)) {
    diter_set_err(ctx, "invalid options");
    return DI_ERR_INVALID_ARG;
  }
  ctx->opt = o;
  ctx->check_interval = o.check_interval;
  if (o.device >= 0) {
    CK(cudaSetDevice(o.device));
    ctx->device = o.device;
  } else {
    CK(cudaGetDevice(&ctx->device));
  }
  SetupTrace tr;
  CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  CK(cudaEventCreate(&ctx->ev0));
  CK(cudaEventCreate(&ctx->ev1));
  tr.mark(ctx->stream, "stream/events");
  const long long n = ctx->n_local, nnz = ctx->nnz_local;
  TRY(dalloc(ctx, &ctx->col_ptr, (size_t)n + 1));
  TRY(dalloc(ctx, &ctx->row_idx, (size_t)nnz));
  if (values) TRY(dalloc(ctx, &ctx->vals, (size_t)nnz));
  TRY(dalloc(ctx, &ctx->F, (size_t)n));
  TRY(dalloc(ctx, &ctx->H, (size_t)n));
  if (b) TRY(dalloc(ctx, &ctx->d_b, (size_t)n));
  tr.mark(ctx->stream, "malloc graph+F+H");
  // Upload: col_ptr and B on the context stream, row_idx / values on a copy stream.
  // Everything that needs only col_ptr and B (geometry, frontier buffers, dangling
  // bits, edge-key weights, F/H init, T_0) then runs while the row indices are still
  // crossing the host link (~115 ms of a C4 create); the census, which validates
  // both, and whatever reads row_idx wait for the copy stream.
  CK(cudaMemcpyAsync(ctx->col_ptr, col_ptr, sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, ctx->stream));
  if (b) CK(cudaMemcpyAsync(ctx->d_b, b, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  cudaStream_t cs = nullptr;
  cudaEvent_t rows_in = nullptr;
  CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  struct CopyStream {
    cudaStream_t &s; cudaEvent_t &e;
    ~CopyStream() { if (s) { cudaStreamSynchronize(s); cudaStreamDestroy(s); } if (e) cudaEventDestroy(e); }
  } cs_guard{cs, rows_in};
  CK(cudaEventCreateWithFlags(&rows_in, cudaEventDisableTiming));
  CK(cudaEventRecord(ctx->ev1, ctx->stream));    // the pool allocations are ordered on ctx->stream
  CK(cudaStreamWaitEvent(cs, ctx->ev1, 0));
  if (nnz) CK(cudaMemcpyAsync(ctx->row_idx, row_idx, sizeof(int) * nnz, cudaMemcpyHostToDevice, cs));
  if (values && nnz) CK(cudaMemcpyAsync(ctx->vals, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, cs));
  CK(cudaEventRecord(rows_in, cs));
  TRY(setup_geometry(ctx));
  // frontier and per-pass buffers
  const size_t fr_cap = (size_t)ctx->fr.n_seg * (size_t)ctx->fr.seg_len;
  TRY(dalloc(ctx, &ctx->fr.ids, fr_cap));
  TRY(dalloc(ctx, &ctx->fr.S, fr_cap));
  TRY(dalloc(ctx, &ctx->fr.seg_cnt, (size_t)ctx->fr.n_seg));
  {
    unsigned *db = nullptr;
    TRY(dalloc(ctx, &db, (size_t)((n + 31) >> 5) + kSelectItems));   // + a pad word per item of the last span
    CK(cudaMemsetAsync(db, 0, sizeof(unsigned) * (((n + 31) >> 5) + kSelectItems), ctx->stream));
    k_dangling_bits<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->col_ptr, n, db);
    ctx->fr.dang_bits = db;
  }
  TRY(dalloc(ctx, &ctx->sel_part, (size_t)std::max(std::max(ctx->grid_select, ctx->grid_fused), ctx->num_sms * 4)));
  TRY(dalloc(ctx, &ctx->sc_part, (size_t)std::max(ctx->grid_scatter, ctx->num_sms * 4)));
  TRY(dalloc(ctx, &ctx->l1_part, (size_t)ctx->grid_l1));
  TRY(dalloc(ctx, &ctx->l1_out, 1));
  TRY(dalloc(ctx, &ctx->ctl, 1));
  ctx->log_cap = 1 << 18;  // passes logged since create/reset (di_run is resumable)
  TRY(dalloc(ctx, &ctx->log, (size_t)ctx->log_cap));
  CK(cudaHostAlloc((void **)&ctx->h_ctl, sizeof(Ctl), cudaHostAllocDefault));
  // state: F = B, H = 0
  ctx->b_uniform = (1.0 - ctx->d) / (double)ctx->n_rows;
  k_init_state<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->F, ctx->H, ctx->d_b, ctx->b_uniform, n);
  // selection-key weights: the paper key needs in-degrees (row_idx), after the census;
  // T_0 (a max over ranks when distributed) comes last, in diter_setup_finish
  const bool key_early = o.select_key != DI_KEY_PAPER;
  if (key_early) TRY(setup_key(ctx));
  tr.mark(ctx->stream, "col_ptr-only setup");
  // validation + bin census on the device, once the rows are in
  CK(cudaStreamWaitEvent(ctx->stream, rows_in, 0));
  Census *d_c = nullptr;
  TRY(dalloc(ctx, &d_c, 1));
  CK(cudaMemsetAsync(d_c, 0, sizeof(Census), ctx->stream));
  k_census<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->col_ptr, n, ctx->row_idx, nnz, ctx->vals,
                                                      ctx->d, ctx->n_rows, d_c);
  Census hc;
  CK(cudaMemcpyAsync(&hc, d_c, sizeof(Census), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  diter_free(ctx, d_c);
  CK(cudaGetLastError());
  tr.mark(ctx->stream, "H2D rows + census");
  if (hc.bad_ptr) {
    diter_set_err(ctx, "col_ptr is not non-decreasing (%llu columns)", hc.bad_ptr);
    return DI_ERR_INVALID_ARG;
  }
  if (hc.bad_row) {
    diter_set_err(ctx, "%llu row indices out of range [0,%lld)", hc.bad_row, ctx->n_rows);
    return DI_ERR_INVALID_ARG;
  }
  if (hc.bad_contraction) {
    diter_set_err(ctx, "%llu columns have sum |p_ij| > d = %g (not contractive)", hc.bad_contraction, ctx->d);
    return DI_ERR_CONTRACTION;
  }
  TRY(choose_hot_window(ctx));
  TRY(choose_l2_window(ctx));
  tr.mark(ctx->stream, "hot window + L2 window");
  TRY(setup_far(ctx));
  tr.mark(ctx->stream, "far bins");
  ctx->cap_low = hc.n_low;
  ctx->cap_mid = hc.n_mid;
  ctx->cap_hub = hc.n_hub;
  TRY(dalloc(ctx, &ctx->fr.hub_w, hc.n_hub));
  TRY(dalloc(ctx, &ctx->fr.hub_b0, hc.n_hub));
  TRY(dalloc(ctx, &ctx->fr.hub_deg, hc.n_hub));
  TRY(dalloc(ctx, &ctx->fr.hub_chunk, hc.n_hub));
  // sweeps: chunk -> slot table (a pass lists each hub at most once: <= nnz/2048 + n_hub chunks)
  if (hc.n_hub > 0) {
    const size_t nch = (size_t)(ctx->nnz_local / kHubChunk) + (size_t)hc.n_hub;
    TRY(dalloc(ctx, &ctx->fr.hub_cslot, nch));
    CK(cudaMemsetAsync(ctx->fr.hub_cslot, 0, nch * sizeof(unsigned), ctx->stream));
  }
  // one-kernel async sweeps (options.sweep): one GPU, per-phase launches, no far bins
  // distributed ranks: sweeps for the local passes of ASYNC / P2P rounds (SYNC keeps the
  // snapshot pass, which reproduces the one-GPU pass log)
  const bool dist_sweepable = ctx->dist && (o.exchange_mode == DI_EXCHANGE_ASYNC || o.exchange_mode == DI_EXCHANGE_P2P);
  ctx->sweep_on = (o.sweep == 1 && (!ctx->dist || dist_sweepable) && !ctx->fused && !ctx->far.on) ? 1 : 0;
  if (ctx->sweep_on) {
    // per-warp staging in dynamic shared memory (beyond the default 48 KB with the hot window)
    auto attr = [&](const void *fn) { return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepDynSmem); };
    for (int key = 0; key < 3; ++key) {
      CK(attr((const void *)sweep_fn<false, false>(key)));
      CK(attr((const void *)sweep_fn<true, false>(key)));
      CK(attr((const void *)sweep_fn<false, true>(key)));
      CK(attr((const void *)sweep_fn<true, true>(key)));
    }
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep<false, 1>, kScatterThreads, kSweepDynSmem));
    ctx->grid_sweep = (int)std::max(1LL, std::min<long long>((long long)ctx->num_sms * std::max(1, occ),
                                                             (n + kSweepSpan - 1) / kSweepSpan));
  }
  if (ctx->sweep_on && ctx->nnz_local < (1LL << 32)) {
    // the scan's 4-byte col_ptr copy (built last: nothing moves col_ptr after this point)
    unsigned *c32 = nullptr;
    TRY(dalloc(ctx, &c32, (size_t)n + 1));
    k_col_ptr32<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->col_ptr, n, c32);
    ctx->fr.cp32 = c32;
  }
  if (!ctx->sweep_on) TRY(diter_setup_defer(ctx));
  tr.mark(ctx->stream, "far-edge deferral");
  CK(cudaStreamSynchronize(ctx->stream));
  return DI_OK;
}

// The collective tail of a create (distributed: every rank calls it, after all
// ranks agreed that their local setup succeeded): the paper key's in-degrees,
// T_0 = max over ranks, the control block, the captured pass graph.
di_status diter_setup_finish(di_ctx *ctx) {
  NvtxRange nv("diter setup (collective tail)");
  SetupTrace tr;
  const di_options &o = ctx->opt;
  if (o.select_key == DI_KEY_PAPER) TRY(setup_key(ctx));
  double T0 = o.t0;
  TRY(initial_threshold(ctx, &T0));
  tr.mark(ctx->stream, "paper key + T_0");
  Ctl hc0;
  std::memset(&hc0, 0, sizeof(hc0));
  hc0.T = T0;
  hc0.alpha = o.alpha;
  hc0.hybrid_frac = o.hybrid_frac;
  hc0.n_total = (double)ctx->n_rows;
  hc0.policy = o.policy;
  hc0.defer_m = ctx->defer_m;
  hc0.sweep = ctx->sweep_on;
  hc0.key_off = o.key_offset > 0 ? (float)o.key_offset : 1.0f;
  hc0.done = 1;
  hc0.max_pass = o.max_passes;
  hc0.log_cap = ctx->log_cap;
  hc0.r = hc0.r_pred = INFINITY;
  ctx->ctl_init = hc0;
  CK(cudaMemcpyAsync(ctx->ctl, &ctx->ctl_init, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->threshold = T0;
  tr.mark(ctx->stream, "init ctl");
  TRY(diter_capture_graph(ctx));
  tr.mark(ctx->stream, "graph capture");
  return DI_OK;
}

extern "C" di_status di_create(di_ctx **out, int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                               const double *values, const double *b, double d, const di_options *opt) {
  if (!out) { diter_set_err(nullptr, "out is NULL"); return DI_ERR_INVALID_ARG; }
  *out = nullptr;
  if (n < 1 || n > 2147483647LL || !col_ptr || !(d > 0.0 && d < 1.0)) {
    diter_set_err(nullptr, "invalid arguments: need 1 <= n < 2^31, col_ptr, 0 < d < 1");
    return DI_ERR_INVALID_ARG;
  }
  const long long nnz = col_ptr[n];
  if (col_ptr[0] != 0 || nnz < 0 || (nnz > 0 && !row_idx)) {
    diter_set_err(nullptr, "col_ptr[0] must be 0 and col_ptr[n] = nnz >= 0 (row_idx required when nnz > 0)");
    return DI_ERR_INVALID_ARG;
  }
  di_ctx *ctx = new (std::nothrow) di_ctx();
  if (!ctx) { diter_set_err(nullptr, "host OOM"); return DI_ERR_OOM; }
  ctx->n_rows = n;
  ctx->n_local = n;
  ctx->nnz_local = nnz;
  ctx->lo = 0;
  ctx->d = d;
  di_status s = diter_setup(ctx, col_ptr, row_idx, values, b, opt);
  if (s == DI_OK) s = diter_setup_finish(ctx);
  if (s != DI_OK) {
    g_thread_err = ctx->err;
    free_ctx(ctx);
    return s;
  }
  *out = ctx;
  return DI_OK;
}

// Exact |F|_1 of this context's slice into ctx->l1_out (device), deterministic.
di_status diter_l1_launch(di_ctx *ctx) { return diter_l1_launch_of(ctx, ctx->F); }

// Deterministic |v|_1 of a local vector into ctx->l1_out (device).
di_status diter_l1_launch_of(di_ctx *ctx, const double *v) {
  k_l1_partial<<<ctx->grid_l1, kSelectThreads, 0, ctx->stream>>>(v, ctx->n_local, ctx->l1_part);
  k_l1_final<<<1, kFinalizeThreads, 0, ctx->stream>>>(ctx->l1_part, ctx->grid_l1, ctx->l1_out);
  ctx->kernel_launches += 2;
  CK(cudaGetLastError());
  return DI_OK;
}

static di_status read_ctl(di_ctx *ctx) {
  CK(cudaMemcpyAsync(ctx->h_ctl, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return DI_OK;
}

extern "C" di_status di_run(di_ctx *ctx, double target) {
  NvtxRange nv("di_run");
  if (!ctx) { diter_set_err(nullptr, "ctx is NULL"); return DI_ERR_INVALID_ARG; }
  if (!(target >= 0.0)) { diter_set_err(ctx, "target must be >= 0"); return DI_ERR_INVALID_ARG; }
  if (ctx->dist) return diter_dist_run(ctx, target);   // any distributed context, one rank included
  CK(cudaSetDevice(ctx->device));
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  const long long launches0 = ctx->kernel_launches;
  di_status st = DI_OK;
  const long long max_pass_abs = ctx->passes_done + ctx->opt.max_passes;
  for (;;) {
    // exact residual first: the stop test of the previous launch is a prediction
    TRY(diter_l1_launch(ctx));
    k_begin_run<<<1, 1, 0, ctx->stream>>>(ctx->ctl, target, max_pass_abs, ctx->l1_out);
    ctx->kernel_launches += 1;
    TRY(read_ctl(ctx));
    const Ctl *h = reinterpret_cast<const Ctl *>(ctx->h_ctl);
    ctx->residual = h->r_pred;
    if (h->r_pred < target) break;                       // converged (exact |F|_1)
    if (h->pass >= max_pass_abs) { st = DI_ERR_NOT_CONVERGED; break; }
    // fused: one cooperative kernel runs up to 4 x check_interval passes per launch
    if (ctx->fused) {
      Graph g = diter_graph(ctx);
      int has_hubs = ctx->cap_hub > 0 ? 1 : 0, max_p = 4 * ctx->check_interval;
      void *args[] = {&g, &ctx->F, &ctx->H, &ctx->fr, &ctx->ctl, &ctx->sel_part, &ctx->sc_part,
                      &ctx->log, &has_hubs, &max_p, &ctx->kw};
      for (;;) {
        const long long pass_before = h->pass;
        if (ctx->vals)
          CK(cudaLaunchCooperativeKernel((void *)k_pass_fused<true>, ctx->grid_fused, kScatterThreads, args,
                                         ctx->scatter_smem, ctx->stream));
        else
          CK(cudaLaunchCooperativeKernel((void *)k_pass_fused<false>, ctx->grid_fused, kScatterThreads, args,
                                         ctx->scatter_smem, ctx->stream));
        ctx->kernel_launches += 1;
        ctx->graph_launches += 1;
        TRY(read_ctl(ctx));
        ctx->kt_passes += h->pass - pass_before;
        ctx->kt_ms[0] = h->t_sel_us * 1e-3;
        ctx->kt_ms[1] = h->t_sc_us * 1e-3;
        if (h->done) break;
      }
    }
    // graph launches until the device sets done
    for (; !ctx->fused;) {
      const long long pass_before = h->pass;
      CK(cudaGraphLaunch(ctx->graph_exec, ctx->stream));
      ctx->graph_launches += 1;
      ctx->kernel_launches += (ctx->sweep_on ? 2LL + (ctx->cap_hub > 0 && !DITER_SWEEP_HUBS) + (ctx->vals ? 3 : 0)
                                             : 3LL + (ctx->cap_hub > 0) + (ctx->far.on ? 1 : 0) + (ctx->defer_m ? 2 : 0)) *
                              ctx->check_interval;
      TRY(read_ctl(ctx));
      if (ctx->opt.profile) {
        const long long active = std::min<long long>(h->pass - pass_before, ctx->check_interval);
        for (long long k = 0; k < active; ++k) {
          float ms3[3] = {0.f, 0.f, 0.f};
          for (int q = 0; q < 3; ++q) {
            CK(cudaEventElapsedTime(&ms3[q], ctx->prof_ev[4 * k + q], ctx->prof_ev[4 * k + q + 1]));
            ctx->kt_ms[q] += ms3[q];
          }
          ctx->pass_us.push_back({ms3[0] * 1e3, ms3[1] * 1e3});
        }
        ctx->kt_passes += active;
      }
      if (h->done) break;
    }
    if (h->pending > 0.0) {            // guard: a run never ends with far-edge mass undelivered
      TRY(diter_defer_flush_now(ctx, h->done));
      TRY(read_ctl(ctx));
    }
    ctx->passes_done = h->pass;
    if (h->done == 2) {
      TRY(diter_l1_launch(ctx));
      double r;
      CK(cudaMemcpyAsync(&r, ctx->l1_out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      ctx->residual = r;
      st = (r < target) ? DI_OK : DI_ERR_NOT_CONVERGED;
      break;
    }
  }
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  CK(cudaEventSynchronize(ctx->ev1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  ctx->run_ms = ms;
  ctx->run_ms_total += ms;
  const Ctl *h = reinterpret_cast<const Ctl *>(ctx->h_ctl);
  ctx->passes_done = h->pass;
  ctx->edges = h->edges;
  ctx->nodes = h->nodes;
  ctx->dang = h->dang;
  ctx->far_flushes = h->flushes;
  ctx->threshold = h->T;
  ctx->run_kernel_launches = ctx->kernel_launches - launches0;
  if (st == DI_ERR_NOT_CONVERGED) diter_set_err(ctx, "max_passes reached before |F|_1 < %g", target);
  return st;
}

extern "C" di_status di_set_profile(di_ctx *ctx, int32_t on) {
  if (!ctx) { diter_set_err(nullptr, "ctx is NULL"); return DI_ERR_INVALID_ARG; }
  CK(cudaSetDevice(ctx->device));
  if ((ctx->opt.profile != 0) == (on != 0)) return DI_OK;
  ctx->opt.profile = on ? 1 : 0;
  if (on && ctx->prof_ev.empty()) {
    ctx->prof_ev.assign(4 * ctx->check_interval, nullptr);
    for (auto &e : ctx->prof_ev) CK(cudaEventCreate(&e));
  }
  if (ctx->graph_exec) {
    CK(cudaGraphExecDestroy(ctx->graph_exec));
    ctx->graph_exec = nullptr;
  }
  if (!ctx->fused) TRY(diter_capture_graph(ctx));
  return DI_OK;
}

extern "C" di_status di_reset(di_ctx *ctx) {
  if (!ctx) { diter_set_err(nullptr, "ctx is NULL"); return DI_ERR_INVALID_ARG; }
  CK(cudaSetDevice(ctx->device));
  k_init_state<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->F, ctx->H, ctx->d_b, ctx->b_uniform,
                                                          ctx->n_local);
  CK(cudaMemcpyAsync(ctx->ctl, &ctx->ctl_init, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaGetLastError());
  ctx->kernel_launches += 1;
  ctx->passes_done = ctx->edges = ctx->nodes = ctx->dang = ctx->far_flushes = 0;
  if (ctx->defer_m) CK(cudaMemsetAsync(ctx->H_old, 0, sizeof(double) * (size_t)ctx->n_local, ctx->stream));
  ctx->run_kernel_launches = 0;
  ctx->kt_ms[0] = ctx->kt_ms[1] = ctx->kt_ms[2] = 0.0;
  ctx->kt_passes = 0;
  ctx->pass_us.clear();
  ctx->run_ms = ctx->run_ms_total = 0.0;
  ctx->graph_launches = 0;
  ctx->threshold = ctx->ctl_init.T;
  ctx->exchanged_bytes = ctx->exchanges = ctx->alg_bytes_exchange = 0;
  return diter_dist_reset(ctx);
}

extern "C" di_status di_set_state(di_ctx *ctx, const double *f_in, const double *h_in) {
  if (!ctx || !f_in || !h_in) { diter_set_err(ctx, "NULL argument"); return DI_ERR_INVALID_ARG; }
  TRY(di_reset(ctx));
  CK(cudaSetDevice(ctx->device));
  const size_t bytes = sizeof(double) * (size_t)ctx->n_local;
  CK(cudaMemcpyAsync(ctx->F, f_in, bytes, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->H, h_in, bytes, cudaMemcpyHostToDevice, ctx->stream));
  if (ctx->H_old) CK(cudaMemcpyAsync(ctx->H_old, ctx->H, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  double T0 = 0.0;
  TRY(initial_threshold(ctx, &T0));      // synchronises the stream; collective when distributed
  Ctl c = ctx->ctl_init;
  c.T = T0;
  CK(cudaMemcpyAsync(ctx->ctl, &c, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->threshold = T0;
  return DI_OK;
}

static di_status copy_out(const di_ctx *cctx, const double *src, double *dst, cudaMemcpyKind kind) {
  di_ctx *ctx = const_cast<di_ctx *>(cctx);
  if (!ctx || !dst) { diter_set_err(ctx, "NULL argument"); return DI_ERR_INVALID_ARG; }
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(dst, src, sizeof(double) * ctx->n_local, kind, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return DI_OK;
}

extern "C" di_status di_get_history(const di_ctx *ctx, double *h) {
  return copy_out(ctx, ctx ? ctx->H : nullptr, h, cudaMemcpyDeviceToHost);
}
extern "C" di_status di_get_fluid(const di_ctx *ctx, double *f) {
  return copy_out(ctx, ctx ? ctx->F : nullptr, f, cudaMemcpyDeviceToHost);
}
extern "C" di_status di_get_history_device(const di_ctx *ctx, double *h) {
  return copy_out(ctx, ctx ? ctx->H : nullptr, h, cudaMemcpyDeviceToDevice);
}
extern "C" di_status di_get_fluid_device(const di_ctx *ctx, double *f) {
  return copy_out(ctx, ctx ? ctx->F : nullptr, f, cudaMemcpyDeviceToDevice);
}

// Completed PageRank H / |H|_1 (App. A.4), into d_dst (device) or h_dst (host,
// staged in the frontier value buffer, which di_run rewrites every pass).
static di_status pagerank_out(di_ctx *ctx, double *d_dst, double *h_dst) {
  if (!ctx || (!d_dst && !h_dst)) { diter_set_err(ctx, "NULL argument"); return DI_ERR_INVALID_ARG; }
  if (ctx->vals || ctx->d_b) {
    // X / |X|_1 is the completed PageRank only for P = dQ and B = (1-d) V with the
    // completion vector V = 1/N (App. A.4); a signed P or a personalised B has none
    diter_set_err(ctx, "di_get_pagerank: needs a PageRank context with the default B = (1-d)/N");
    return DI_ERR_STATE;
  }
  CK(cudaSetDevice(ctx->device));
  TRY(diter_l1_launch_of(ctx, ctx->H));
  double sh = 0.0;
  CK(cudaMemcpyAsync(&sh, ctx->l1_out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  TRY(diter_dist_sum(ctx, sh, &sh));
  if (!(sh > 0.0)) { diter_set_err(ctx, "|H|_1 = 0: run the solver first"); return DI_ERR_STATE; }
  double *dst = d_dst ? d_dst : ctx->fr.S;
  k_div<<<ctx->grid_l1, 256, 0, ctx->stream>>>(dst, ctx->H, sh, ctx->n_local);
  ctx->kernel_launches += 1;
  if (h_dst) CK(cudaMemcpyAsync(h_dst, dst, sizeof(double) * ctx->n_local, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return DI_OK;
}
extern "C" di_status di_get_pagerank(di_ctx *ctx, double *x) { return pagerank_out(ctx, nullptr, x); }
extern "C" di_status di_get_pagerank_device(di_ctx *ctx, double *d) { return pagerank_out(ctx, d, nullptr); }

extern "C" di_status di_get_residual(di_ctx *ctx, double *r_out) {
  if (!ctx || !r_out) { diter_set_err(ctx, "NULL argument"); return DI_ERR_INVALID_ARG; }
  CK(cudaSetDevice(ctx->device));
  TRY(diter_l1_launch(ctx));
  double r = 0.0;
  CK(cudaMemcpyAsync(&r, ctx->l1_out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  TRY(diter_dist_sum(ctx, r, &r));
  ctx->residual = r;
  *r_out = r;
  return DI_OK;
}

extern "C" di_status di_get_stats(const di_ctx *ctx, di_stats *s) {
  if (!ctx || !s) { diter_set_err(nullptr, "NULL argument"); return DI_ERR_INVALID_ARG; }
  std::memset(s, 0, sizeof(*s));
  s->passes = ctx->passes_done;
  s->edges = ctx->edges;
  s->nodes = ctx->nodes;
  s->residual = ctx->residual;
  s->threshold = ctx->threshold;
  s->run_ms = ctx->run_ms;
  s->run_ms_total = ctx->run_ms_total;
  s->alg_bytes = 8LL * ctx->n_local * ctx->passes_done + 40LL * ctx->nodes +
                 (ctx->vals ? 28LL : 20LL) * ctx->edges + ctx->alg_bytes_exchange;
  s->exchanged_bytes = ctx->exchanged_bytes;
  s->exchanges = ctx->exchanges;
  s->n_local = ctx->n_local;
  s->nnz_local = ctx->nnz_local;
  s->graph_launches = ctx->graph_launches;
  s->kernel_launches = ctx->kernel_launches;
  s->kt_select_ms = ctx->kt_ms[0];
  s->kt_scatter_ms = ctx->kt_ms[1];
  s->kt_finalize_ms = ctx->kt_ms[2];
  s->kt_passes = ctx->kt_passes;
  // the scatter reads the col_ptr pair of every node it diffuses: the selected
  // nodes minus the dangling ones, which the select takes itself
  s->scatter_bytes = (ctx->vals ? 28LL : 20LL) * ctx->edges + 16LL * (ctx->nodes - ctx->dang);
  s->dangling = ctx->dang;
  s->run_kernel_launches = ctx->run_kernel_launches;
  s->remote_pushes = ctx->remote_pushes;
  s->rebalances = ctx->rebalances;
  s->l2_window_bytes = ctx->l2_bytes;
  s->l2_window_row = ctx->l2_bytes > 0 ? ctx->lo + ctx->l2_lo : 0;
  s->far_flushes = ctx->far_flushes;
  s->far_edges = ctx->far_edges;
  diter_dist_stats(ctx, s);
  return DI_OK;
}

extern "C" di_status di_get_pass_log(const di_ctx *cctx, int64_t first, int64_t count, di_pass_log *out,
                                     int64_t *n_copied) {
  di_ctx *ctx = const_cast<di_ctx *>(cctx);
  if (!ctx || (!out && count > 0) || first < 0 || count < 0) {
    diter_set_err(ctx, "invalid arguments");
    return DI_ERR_INVALID_ARG;
  }
  long long avail = std::min<long long>(ctx->passes_done, ctx->log_cap);
  long long k = std::max<long long>(0, std::min<long long>(count, avail - first));
  if (k > 0) {
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemcpyAsync(out, ctx->log + first, sizeof(di_pass_log) * k, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (long long j = 0; j < k; ++j) {
      const long long p = first + j;
      if (p < (long long)ctx->pass_us.size()) {
        out[j].t_select_us = ctx->pass_us[p].first;
        out[j].t_scatter_us = ctx->pass_us[p].second;
      }
    }
  }
  if (n_copied) *n_copied = k;
  return DI_OK;
}

extern "C" const char *di_last_error(const di_ctx *ctx) {
  if (ctx) return ctx->err.c_str();
  return g_thread_err.c_str();
}

extern "C" void di_destroy(di_ctx *ctx) { free_ctx(ctx); }

// ---------------------------------------------------------- partition (K9) --
// bounds[k] = min{ i : C[i] >= ceil(k C[n] / K) } by binary search (C is
// non-decreasing), then forced strictly increasing and leaving >= 1 node per
// later range (reading R10).
extern "C" di_status di_partition_cb(int64_t n, const int64_t *C, int32_t K, int64_t *bounds) {
  if (n < 1 || K < 1 || K > n || !C || !bounds) {
    diter_set_err(nullptr, "di_partition_cb: need 1 <= K <= n and non-NULL arrays");
    return DI_ERR_INVALID_ARG;
  }
  const long long total = C[n];
  bounds[0] = 0;
  for (int k = 1; k < K; ++k) {
    const __int128 num = (__int128)k * total;
    const long long goal = (long long)((num + K - 1) / K);
    long long i = std::lower_bound(C, C + n + 1, (int64_t)goal) - C;
    i = std::max<long long>(i, bounds[k - 1] + 1);
    i = std::min<long long>(i, n - (K - k));
    bounds[k] = i;
  }
  bounds[K] = n;
  return DI_OK;
}
