// kernels.cuh -- the D-iteration hot path on sm_100a.
//
// One pass p:
//   k_select   (K1): r_p = sum |F_i| (warp-shuffle reduction), S_p = {i : |F_i| > T_p},
//                    take (s = F_i, F_i = 0, H_i += s), per-node push value, degree bin.
//   k_scatter  (K2-K4 fused, persistent): F_j += push for every edge of every node of S_p,
//                    hubs CTA-per-chunk, mid-degree warp-per-node, low-degree thread-per-node.
//   k_finalize (K5): deterministic second-level reduction, pass log, T_{p+1}, stop flag.
// Every kernel returns at once when the control block says the run is done, so a
// captured graph of m passes can overrun convergence at the cost of empty launches.
#pragma once
#include "common.cuh"
#include "types.cuh"

namespace diter {

// ---------------------------------------------------------------- K1 select --
// Grid-stride over nodes with a warp-uniform loop; lanes read consecutive F_i
// (coalesced 256 B per warp load).  Selected nodes read col_ptr[i..i+1] to bin
// and to derive p_ji = d/#out_i (PageRank weights are never stored, BASELINE
// north_star) -- push = s * (d / #out_i), the same two roundings as the oracle.
__global__ void __launch_bounds__(kSelectThreads)
k_select(Graph g, double *__restrict__ F, double *__restrict__ H, Bins bins, Ctl *ctl,
         Partial *__restrict__ part) {
  if (ctl->done) return;
  const double T = ctl->T;
  const bool is_signed = (g.vals != nullptr);
  double r = 0.0, loss = 0.0;
  long long edges = 0;
  int cnt = 0, dang = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long warp_base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
  for (long long base = warp_base; base < g.n; base += stride) {
    const long long i = base + lane_id();
    const bool valid = i < g.n;
    double f = valid ? F[i] : 0.0;
    const double af = fabs(f);
    r += af;
    const bool sel = valid && (af > T);
    long long deg = 0;
    double push = 0.0;
    if (sel) {
      F[i] = 0.0;
      H[i] += f;
      const long long b0 = g.col_ptr[i], b1 = g.col_ptr[i + 1];
      deg = b1 - b0;
      push = is_signed ? f : f * (g.d / (double)deg);
      // |F|_1 decreases by at least (1 - sum_j |p_ji|)|s| >= (1-d)|s| (App. A.2);
      // a dangling column pushes nothing, so all of |s| leaves.
      loss += (deg > 0) ? (1.0 - g.d) * af : af;
      edges += deg;
      cnt += 1;
      dang += (deg == 0);
    }
    const bool is_low = sel && deg >= 1 && deg <= kLowMax;
    const bool is_mid = sel && deg > kLowMax && deg <= kMidMax;
    const bool is_hub = sel && deg > kMidMax;
    const unsigned slot_low = warp_append(&ctl->n_low, is_low);
    const unsigned slot_mid = warp_append(&ctl->n_mid, is_mid);
    if (is_low) { bins.low_idx[slot_low] = (int)i; bins.low_w[slot_low] = push; }
    if (is_mid) { bins.mid_idx[slot_mid] = (int)i; bins.mid_w[slot_mid] = push; }
    if (is_hub) {
      // one 64-bit atomic hands out the slot AND the first chunk id, so hub_chunk[]
      // is sorted by slot and the scatter can binary-search it.
      const unsigned long long nch = (unsigned long long)((deg + kHubChunk - 1) / kHubChunk);
      const unsigned long long old = atomicAdd(&ctl->hub_packed, (1ull << 32) | nch);
      const unsigned s = (unsigned)(old >> 32);
      bins.hub_idx[s] = (int)i;
      bins.hub_w[s] = push;
      bins.hub_chunk[s] = (unsigned)(old & 0xffffffffull);
    }
  }
  // block reduction (fixed order -> deterministic given F)
  r = warp_sum(r);
  loss = warp_sum(loss);
  edges = warp_sum(edges);
  cnt = warp_sum(cnt);
  dang = warp_sum(dang);
  __shared__ double s_r[kSelectThreads / 32], s_l[kSelectThreads / 32];
  __shared__ long long s_e[kSelectThreads / 32];
  __shared__ int s_c[kSelectThreads / 32], s_d[kSelectThreads / 32];
  const int w = threadIdx.x >> 5;
  if (lane_id() == 0) { s_r[w] = r; s_l[w] = loss; s_e[w] = edges; s_c[w] = cnt; s_d[w] = dang; }
  __syncthreads();
  if (threadIdx.x == 0) {
    Partial p{0.0, 0.0, 0, 0, 0};
    for (int k = 0; k < kSelectThreads / 32; ++k) {
      p.r += s_r[k]; p.loss += s_l[k]; p.edges += s_e[k]; p.cnt += s_c[k]; p.dang += s_d[k];
    }
    part[blockIdx.x] = p;
  }
}

// ------------------------------------------------------------ K2-K4 scatter --
// Push `w` (x vals[e] in signed mode) along edges [beg, end) with `nt` cooperating
// threads (t = this thread's rank): scalar head up to 16-byte alignment of
// row_idx, int4 body (4 rows per load, coalesced across the group), scalar tail.
template <bool SIGNED>
__device__ __forceinline__ void push_range(const Graph &g, double *__restrict__ F, long long beg,
                                           long long end, double w, int t, int nt) {
  long long a = (beg + 3) & ~3ll;
  if (a > end) a = end;
  for (long long e = beg + t; e < a; e += nt) {
    const int row = ld_stream_i1(g.row_idx + e);
    red_add(F + row, SIGNED ? w * ld_stream_d1(g.vals + e) : w);
  }
  const long long nv = (end - a) >> 2;
  const int4 *r4 = reinterpret_cast<const int4 *>(g.row_idx + a);
  for (long long k = t; k < nv; k += nt) {
    const int4 rr = ld_stream_i4(r4 + k);
    if (SIGNED) {
      const double2 *v2 = reinterpret_cast<const double2 *>(g.vals + a) + 2 * k;
      const double2 va = ld_stream_d2(v2), vb = ld_stream_d2(v2 + 1);
      red_add(F + rr.x, w * va.x);
      red_add(F + rr.y, w * va.y);
      red_add(F + rr.z, w * vb.x);
      red_add(F + rr.w, w * vb.y);
    } else {
      red_add(F + rr.x, w);
      red_add(F + rr.y, w);
      red_add(F + rr.z, w);
      red_add(F + rr.w, w);
    }
  }
  for (long long e = a + nv * 4 + t; e < end; e += nt) {
    const int row = ld_stream_i1(g.row_idx + e);
    red_add(F + row, SIGNED ? w * ld_stream_d1(g.vals + e) : w);
  }
}

// Persistent, one launch per pass: phase A hub chunks (CTA per 2048-edge chunk),
// phase B mid nodes (warp per node), phase C low nodes (thread per node).  The
// phases need no barrier between them: all pushes commute (fp64 RED in L2).
template <bool SIGNED>
__global__ void __launch_bounds__(kScatterThreads)
k_scatter(Graph g, double *__restrict__ F, Bins bins, const Ctl *ctl) {
  if (ctl->done) return;
  // phase A: hubs
  const unsigned long long hp = ctl->hub_packed;
  const unsigned n_hub = (unsigned)(hp >> 32), n_chunks = (unsigned)(hp & 0xffffffffull);
  for (unsigned c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    unsigned lo = 0, hi = n_hub - 1;
    while (lo < hi) {
      const unsigned mid = (lo + hi + 1) >> 1;
      if (bins.hub_chunk[mid] <= c) lo = mid; else hi = mid - 1;
    }
    const int i = bins.hub_idx[lo];
    const double w = bins.hub_w[lo];
    const long long cb = g.col_ptr[i], ce = g.col_ptr[i + 1];
    const long long beg = cb + (long long)(c - bins.hub_chunk[lo]) * kHubChunk;
    const long long end = min(beg + (long long)kHubChunk, ce);
    push_range<SIGNED>(g, F, beg, end, w, threadIdx.x, blockDim.x);
  }
  // phase B: mid-degree, one warp per node
  const unsigned n_mid = ctl->n_mid;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (long long k = gw; k < n_mid; k += warps) {
    const int i = bins.mid_idx[k];
    const double w = bins.mid_w[k];
    push_range<SIGNED>(g, F, g.col_ptr[i], g.col_ptr[i + 1], w, lane_id(), 32);
  }
  // phase C: low-degree, one thread per node
  const unsigned n_low = ctl->n_low;
  const long long threads = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n_low; k += threads) {
    const int i = bins.low_idx[k];
    const double w = bins.low_w[k];
    const long long b0 = g.col_ptr[i], b1 = g.col_ptr[i + 1];
    for (long long e = b0; e < b1; ++e) {
      const int row = ld_stream_i1(g.row_idx + e);
      red_add(F + row, SIGNED ? w * ld_stream_d1(g.vals + e) : w);
    }
  }
}

// -------------------------------------------------------------- K5 finalize --
__global__ void __launch_bounds__(kFinalizeThreads)
k_finalize(Ctl *ctl, const Partial *__restrict__ part, int n_part, di_pass_log *log) {
  if (ctl->done) return;
  double r = 0.0, loss = 0.0;
  long long edges = 0, cnt = 0, dang = 0;
  for (int k = threadIdx.x; k < n_part; k += blockDim.x) {
    const Partial p = part[k];
    r += p.r; loss += p.loss; edges += p.edges; cnt += p.cnt; dang += p.dang;
  }
  r = warp_sum(r); loss = warp_sum(loss); edges = warp_sum(edges);
  cnt = warp_sum(cnt); dang = warp_sum(dang);
  __shared__ double s_r[kFinalizeThreads / 32], s_l[kFinalizeThreads / 32];
  __shared__ long long s_e[kFinalizeThreads / 32], s_c[kFinalizeThreads / 32], s_d[kFinalizeThreads / 32];
  const int w = threadIdx.x >> 5;
  if (lane_id() == 0) { s_r[w] = r; s_l[w] = loss; s_e[w] = edges; s_c[w] = cnt; s_d[w] = dang; }
  __syncthreads();
  if (threadIdx.x != 0) return;
  r = 0.0; loss = 0.0; edges = 0; cnt = 0; dang = 0;
  for (int k = 0; k < kFinalizeThreads / 32; ++k) {
    r += s_r[k]; loss += s_l[k]; edges += s_e[k]; cnt += s_c[k]; dang += s_d[k];
  }
  const long long p = ctl->pass;
  const double T = ctl->T;
  if (p < ctl->log_cap) {
    di_pass_log L;
    L.pass = p; L.T = T; L.r = r; L.frontier = cnt; L.edges = edges; L.dangling = dang;
    L.bin_low = ctl->n_low; L.bin_mid = ctl->n_mid; L.bin_hub = (long long)(ctl->hub_packed >> 32);
    log[p] = L;
  }
  ctl->edges += edges;
  ctl->nodes += cnt;
  ctl->r = r;
  const double pred = r - loss;
  ctl->r_pred = pred;
  // T_{p+1}: GEOM divides every pass; HYBRID only when |S_p| <= f N (readings R4/R6).
  if (ctl->policy == DI_POLICY_GEOM || (double)cnt <= ctl->hybrid_frac * ctl->n_total)
    ctl->T = T / ctl->alpha;
  ctl->pass = p + 1;
  if (r < ctl->target || pred < ctl->target) ctl->done = 1;
  else if (p + 1 >= ctl->max_pass) ctl->done = 2;
  ctl->n_low = 0;
  ctl->n_mid = 0;
  ctl->hub_packed = 0ull;
}

// --------------------------------------------------- exact residual |F|_1 --
__global__ void __launch_bounds__(kSelectThreads)
k_l1_partial(const double *__restrict__ F, long long n, double *__restrict__ part) {
  double r = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    r += fabs(F[i]);
  r = warp_sum(r);
  __shared__ double s[kSelectThreads / 32];
  if (lane_id() == 0) s[threadIdx.x >> 5] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < kSelectThreads / 32; ++k) t += s[k];
    part[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kFinalizeThreads)
k_l1_final(const double *__restrict__ part, int n_part, double *out) {
  double r = 0.0;
  for (int k = threadIdx.x; k < n_part; k += blockDim.x) r += part[k];
  r = warp_sum(r);
  __shared__ double s[kFinalizeThreads / 32];
  if (lane_id() == 0) s[threadIdx.x >> 5] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < kFinalizeThreads / 32; ++k) t += s[k];
    *out = t;
  }
}

// -------------------------------------------------------------- setup kernels --
// F = B (or (1-d)/n), H = 0
__global__ void k_init_state(double *F, double *H, const double *b, double b_uniform, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    F[i] = b ? b[i] : b_uniform;
    H[i] = 0.0;
  }
}

__global__ void k_census(const long long *col_ptr, long long n, const int *row_idx, long long nnz,
                         const double *vals, double d, Census *c) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  unsigned long long bp = 0, lo = 0, mi = 0, hu = 0, da = 0, bc = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long b0 = col_ptr[i], b1 = col_ptr[i + 1];
    const long long deg = b1 - b0;
    if (deg < 0) { ++bp; continue; }
    if (deg == 0) ++da; else if (deg <= kLowMax) ++lo; else if (deg <= kMidMax) ++mi; else ++hu;
    if (vals) {
      double s = 0.0;
      for (long long e = b0; e < b1; ++e) s += fabs(vals[e]);
      if (s > d * (1.0 + 1e-12)) ++bc;
    }
  }
  unsigned long long br = 0;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += stride) {
    const int r = row_idx[e];
    if (r < 0 || (long long)r >= n) ++br;
  }
  if (bp) atomicAdd(&c->bad_ptr, bp);
  if (br) atomicAdd(&c->bad_row, br);
  if (lo) atomicAdd(&c->n_low, lo);
  if (mi) atomicAdd(&c->n_mid, mi);
  if (hu) atomicAdd(&c->n_hub, hu);
  if (da) atomicAdd(&c->n_dang, da);
  if (bc) atomicAdd(&c->bad_contraction, bc);
}

__global__ void k_max_abs(const double *b, long long n, double *part) {
  double m = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    m = fmax(m, fabs(b[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double s[32];
  if (lane_id() == 0) s[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t = fmax(t, s[k]);
    part[blockIdx.x] = t;
  }
}

// Start-of-run control update (no host->device memcpy inside di_run's timed path).
__global__ void k_begin_run(Ctl *ctl, double target, long long max_pass, const double *r_exact) {
  ctl->target = target;
  ctl->max_pass = max_pass;
  ctl->r_pred = *r_exact;
  ctl->done = 0;
  ctl->n_low = 0;
  ctl->n_mid = 0;
  ctl->hub_packed = 0ull;
}

}  // namespace diter
