// dist.cu -- multi-GPU D-iteration.
//
// One process (or thread) per rank; rank k owns the contiguous node range
// Omega_k = [bounds[k], bounds[k+1]) with its F, H and out-columns (PAPER.md:
// 173-176).  Pushes to rows of other ranks accumulate in a remote outbox G
// (global ids) and are shipped as compacted (row, fluid) records:
//
//  SYNC  : every pass ends with an exchange round, so a pass is exactly the
//          single-GPU snapshot pass (same frontier sizes, same T schedule: the
//          pass totals are all-reduced before T_{p+1} is chosen).
//  ASYNC : ranks run check_interval passes on their own (local threshold
//          policy on |Omega_k|, no communication), then meet in an exchange
//          round where rank k ships its outbox only if s_k > r_k / K
//          (eq. send; strict, reading R7) -- otherwise it
//          keeps accumulating.  Received fluid is merged at once ("can be
//          delayed").  Termination: the round all-reduces
//          r_k + s_k (in-flight mass is zero at that point, every record sent
//          in the round has been merged), stop when below the target.
//
// The collectives go through a Fabric: NCCL (one GPU per rank, NVLink /
// NVSwitch), or an in-process loopback that lets K contexts of one process
// (threads) share one GPU for testing -- no kernel ever waits on another rank;
// all waiting is host-side.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/diter.h"
#include "ctx.cuh"
#include "dist.cuh"
#include "kernels.cuh"

#if DITER_WITH_NCCL
#include <nccl.h>
#endif

using namespace diter;

#define CKD(call)                                                                      \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      diter_set_err(ctx, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),       \
                    __FILE__, __LINE__);                                               \
      return e_ == cudaErrorMemoryAllocation ? DI_ERR_OOM : DI_ERR_CUDA;               \
    }                                                                                  \
  } while (0)

#define TRYD(x)                     \
  do {                              \
    di_status s_ = (x);             \
    if (s_ != DI_OK) return s_;     \
  } while (0)

// In-process loopback: K contexts (one host thread each) on one device.
struct LoopGroup {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<double> red;                 // [world * 8]
  std::vector<long long> counts;           // [world * world]
  std::vector<const Rec *> sendp;
  std::vector<std::vector<long long>> soff, scnt;
  std::vector<double> hmax;
  std::vector<unsigned char> gath;         // allgather staging

  explicit LoopGroup(int w) : world(w), red(w * 8), counts(w * w), sendp(w), soff(w), scnt(w), hmax(w) {}

  // false when the group was aborted (a rank failed) or a peer did not arrive in
  // time: the caller reports an error instead of waiting forever
  bool aborted = false;
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) return false;
    const long long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(kLoopTimeoutS), [&] { return generation != gen || aborted; }) ||
        aborted) {
      aborted = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
  static constexpr int kLoopTimeoutS = 600;
};

#define LOOP_BARRIER(ctx)                                                               \
  do {                                                                                 \
    if (!grp->barrier()) {                                                             \
      diter_set_err(ctx, "loopback group aborted (a peer rank failed or timed out)");  \
      return DI_ERR_STATE;                                                             \
    }                                                                                  \
  } while (0)

static std::mutex g_loop_mu;
static std::map<std::string, std::weak_ptr<LoopGroup>> g_loop_groups;

struct LoopFabric : Fabric {
  std::shared_ptr<LoopGroup> grp;
  int rank;
  LoopFabric(std::shared_ptr<LoopGroup> g, int r) : grp(std::move(g)), rank(r) {}
  void abort() override { grp->abort(); }

  di_status allgather(di_ctx *ctx, const void *mine, size_t bytes, void *all) override {
    ++calls;
    {
      std::lock_guard<std::mutex> lk(grp->mu);
      if (grp->gath.size() < bytes * grp->world) grp->gath.resize(bytes * grp->world);
    }
    LOOP_BARRIER(ctx);
    std::memcpy(grp->gath.data() + bytes * rank, mine, bytes);
    LOOP_BARRIER(ctx);
    std::memcpy(all, grp->gath.data(), bytes * grp->world);
    LOOP_BARRIER(ctx);
    return DI_OK;
  }
  di_status allreduce_sum(di_ctx *ctx, double *dev, int count) override {
    ++calls;
    if (count > 8) { diter_set_err(ctx, "host all-reduce of %d > 8 values", count); return DI_ERR_INVALID_ARG; }
    double h[8];
    CKD(cudaMemcpyAsync(h, dev, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
    CKD(cudaStreamSynchronize(ctx->stream));
    std::memcpy(&grp->red[rank * 8], h, sizeof(double) * count);
    LOOP_BARRIER(ctx);
    for (int q = 0; q < count; ++q) {
      double s = 0.0;
      for (int k = 0; k < grp->world; ++k) s += grp->red[k * 8 + q];   // fixed rank order
      h[q] = s;
    }
    LOOP_BARRIER(ctx);
    CKD(cudaMemcpyAsync(dev, h, sizeof(double) * count, cudaMemcpyHostToDevice, ctx->stream));
    CKD(cudaStreamSynchronize(ctx->stream));
    return DI_OK;
  }
  di_status alltoall_counts(di_ctx *ctx, const long long *send, long long *recv) override {
    ++calls;
    const int W = grp->world;
    for (int q = 0; q < W; ++q) grp->counts[rank * W + q] = send[q];
    LOOP_BARRIER(ctx);
    for (int q = 0; q < W; ++q) recv[q] = grp->counts[q * W + rank];
    LOOP_BARRIER(ctx);
    return DI_OK;
  }
  di_status alltoallv(di_ctx *ctx, const Rec *send, const long long *soff, const long long *scnt, Rec *recv,
                      const long long *roff, const long long *rcnt) override {
    ++calls;
    const int W = grp->world;
    CKD(cudaStreamSynchronize(ctx->stream));   // send buffer complete
    grp->sendp[rank] = send;
    grp->soff[rank].assign(soff, soff + W);
    grp->scnt[rank].assign(scnt, scnt + W);
    LOOP_BARRIER(ctx);
    for (int q = 0; q < W; ++q) {
      if (rcnt[q] == 0) continue;
      const Rec *src = grp->sendp[q] + grp->soff[q][rank];
      CKD(cudaMemcpyAsync(recv + roff[q], src, sizeof(Rec) * rcnt[q], cudaMemcpyDeviceToDevice, ctx->stream));
    }
    CKD(cudaStreamSynchronize(ctx->stream));
    LOOP_BARRIER(ctx);                         // peers may now reuse their send buffers
    return DI_OK;
  }
  di_status host_max(di_ctx *ctx, double v, double *out) override {
    ++calls;
    grp->hmax[rank] = v;
    LOOP_BARRIER(ctx);
    double m = grp->hmax[0];
    for (int k = 1; k < grp->world; ++k) m = std::max(m, grp->hmax[k]);
    LOOP_BARRIER(ctx);
    *out = m;
    return DI_OK;
  }
};

// Cross-process loopback over POSIX shared memory: K processes (one GPU or
// several) with host-side collectives only -- what the tests use to run
// DI_EXCHANGE_P2P across processes on one GPU, so that its windows are mapped with
// cudaIpcOpenMemHandle exactly as between the processes of an 8-GPU box (NCCL
// refuses two ranks on one device).  No bulk all-to-all-v (the P2P mode does not use
// one; the paper key's in-degrees, the receiver-computes mode and di_rebalance need
// NCCL or the in-process loopback).
struct ShmGroup {
  std::atomic<int> arrived;
  std::atomic<int> generation;
  std::atomic<int> aborted;
  int world;
  double red[kP2PMaxWorld * 8];
  long long counts[kP2PMaxWorld * kP2PMaxWorld];
  double hmax[kP2PMaxWorld];
  unsigned char gath[kP2PMaxWorld * 256];
};
static_assert(std::atomic<int>::is_always_lock_free, "process-shared atomics need lock-free int");

struct ShmFabric : Fabric {
  ShmGroup *g = nullptr;
  std::string name;
  int rank = 0, world = 1;
  ~ShmFabric() override {
    if (g) munmap(g, sizeof(ShmGroup));
    if (rank == 0 && !name.empty()) shm_unlink(name.c_str());
  }
  bool barrier() {
    const int gen = g->generation.load();
    if (g->arrived.fetch_add(1) + 1 == world) {
      g->arrived.store(0);
      g->generation.fetch_add(1);
      return true;
    }
    const auto t0 = std::chrono::steady_clock::now();
    while (g->generation.load() == gen) {
      if (g->aborted.load()) return false;
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(LoopGroup::kLoopTimeoutS)) {
        g->aborted.store(1);
        return false;
      }
      usleep(20);
    }
    return !g->aborted.load();
  }
  void abort() override { if (g) g->aborted.store(1); }
#define SHM_BARRIER(ctx)                                                                \
  do {                                                                                 \
    if (!barrier()) {                                                                  \
      diter_set_err(ctx, "shared-memory group aborted (a peer failed or timed out)");  \
      return DI_ERR_STATE;                                                             \
    }                                                                                  \
  } while (0)
  di_status allreduce_sum(di_ctx *ctx, double *dev, int count) override {
    ++calls;
    if (count > 8) { diter_set_err(ctx, "host all-reduce of %d > 8 values", count); return DI_ERR_INVALID_ARG; }
    double h[8];
    CKD(cudaMemcpyAsync(h, dev, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
    CKD(cudaStreamSynchronize(ctx->stream));
    std::memcpy(&g->red[rank * 8], h, sizeof(double) * count);
    SHM_BARRIER(ctx);
    for (int q = 0; q < count; ++q) {
      double v = 0.0;
      for (int k = 0; k < world; ++k) v += g->red[k * 8 + q];   // fixed rank order
      h[q] = v;
    }
    SHM_BARRIER(ctx);
    CKD(cudaMemcpyAsync(dev, h, sizeof(double) * count, cudaMemcpyHostToDevice, ctx->stream));
    CKD(cudaStreamSynchronize(ctx->stream));
    return DI_OK;
  }
  di_status alltoall_counts(di_ctx *ctx, const long long *send, long long *recv) override {
    ++calls;
    for (int q = 0; q < world; ++q) g->counts[rank * world + q] = send[q];
    SHM_BARRIER(ctx);
    for (int q = 0; q < world; ++q) recv[q] = g->counts[q * world + rank];
    SHM_BARRIER(ctx);
    return DI_OK;
  }
  di_status alltoallv(di_ctx *ctx, const Rec *, const long long *, const long long *, Rec *, const long long *,
                      const long long *) override {
    diter_set_err(ctx, "the shared-memory fabric has no bulk all-to-all-v (use DI_EXCHANGE_P2P, NCCL or loopback)");
    return DI_ERR_UNSUPPORTED;
  }
  di_status host_max(di_ctx *ctx, double v, double *out) override {
    ++calls;
    g->hmax[rank] = v;
    SHM_BARRIER(ctx);
    double m = g->hmax[0];
    for (int k = 1; k < world; ++k) m = std::max(m, g->hmax[k]);
    SHM_BARRIER(ctx);
    *out = m;
    return DI_OK;
  }
  di_status allgather(di_ctx *ctx, const void *mine, size_t bytes, void *all) override {
    ++calls;
    if (bytes > 256) return DI_ERR_INVALID_ARG;
    std::memcpy(g->gath + 256 * rank, mine, bytes);
    SHM_BARRIER(ctx);
    for (int k = 0; k < world; ++k) std::memcpy(static_cast<unsigned char *>(all) + bytes * k, g->gath + 256 * k, bytes);
    SHM_BARRIER(ctx);
    return DI_OK;
  }
#undef SHM_BARRIER
};

#if DITER_WITH_NCCL
#define CKN(call)                                                                      \
  do {                                                                                 \
    ncclResult_t r_ = (call);                                                          \
    if (r_ != ncclSuccess) {                                                           \
      diter_set_err(ctx, "%s failed: %s", #call, ncclGetErrorString(r_));              \
      return DI_ERR_NCCL;                                                              \
    }                                                                                  \
  } while (0)

struct NcclFabric : Fabric {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  long long *d_cnt = nullptr;   // [2 * world] send/recv counts staging
  double *d_tmp = nullptr;
  ~NcclFabric() override {
    if (d_cnt) cudaFree(d_cnt);
    if (d_tmp) cudaFree(d_tmp);
    if (comm) ncclCommDestroy(comm);
  }
  di_status allreduce_sum(di_ctx *ctx, double *dev, int count) override {
    ++calls;
    CKN(ncclAllReduce(dev, dev, count, ncclDouble, ncclSum, comm, ctx->stream));
    return DI_OK;
  }
  di_status allgather(di_ctx *ctx, const void *mine, size_t bytes, void *all) override {
    ++calls;
    unsigned char *d = nullptr;
    CKD(cudaMalloc(&d, bytes * (world + 1)));
    di_status st = DI_OK;
    if (cudaMemcpyAsync(d + bytes * world, mine, bytes, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
        ncclAllGather(d + bytes * world, d, bytes, ncclChar, comm, ctx->stream) != ncclSuccess ||
        cudaMemcpyAsync(all, d, bytes * world, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
      diter_set_err(ctx, "NCCL allgather failed");
      st = DI_ERR_NCCL;
    }
    cudaFree(d);
    return st;
  }
  di_status alltoall_counts(di_ctx *ctx, const long long *send, long long *recv) override {
    ++calls;
    CKD(cudaMemcpyAsync(d_cnt, send, sizeof(long long) * world, cudaMemcpyHostToDevice, ctx->stream));
    CKN(ncclGroupStart());
    for (int q = 0; q < world; ++q) {
      CKN(ncclSend(d_cnt + q, 1, ncclInt64, q, comm, ctx->stream));
      CKN(ncclRecv(d_cnt + world + q, 1, ncclInt64, q, comm, ctx->stream));
    }
    CKN(ncclGroupEnd());
    CKD(cudaMemcpyAsync(recv, d_cnt + world, sizeof(long long) * world, cudaMemcpyDeviceToHost, ctx->stream));
    CKD(cudaStreamSynchronize(ctx->stream));
    return DI_OK;
  }
  di_status alltoallv(di_ctx *ctx, const Rec *send, const long long *soff, const long long *scnt, Rec *recv,
                      const long long *roff, const long long *rcnt) override {
    ++calls;
    CKN(ncclGroupStart());
    for (int q = 0; q < world; ++q) {
      if (q == rank) continue;
      if (scnt[q] > 0) CKN(ncclSend(send + soff[q], sizeof(Rec) * scnt[q], ncclChar, q, comm, ctx->stream));
      if (rcnt[q] > 0) CKN(ncclRecv(recv + roff[q], sizeof(Rec) * rcnt[q], ncclChar, q, comm, ctx->stream));
    }
    CKN(ncclGroupEnd());
    return DI_OK;
  }
  di_status host_max(di_ctx *ctx, double v, double *out) override {
    ++calls;
    if (!d_tmp) CKD(cudaMalloc(&d_tmp, sizeof(double)));
    CKD(cudaMemcpyAsync(d_tmp, &v, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CKN(ncclAllReduce(d_tmp, d_tmp, 1, ncclDouble, ncclMax, comm, ctx->stream));
    CKD(cudaMemcpyAsync(&v, d_tmp, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CKD(cudaStreamSynchronize(ctx->stream));
    *out = v;
    return DI_OK;
  }
};
#endif

// ----------------------------------------------------------------- kernels --
// Records of the outbox rows owned by peer q, compacted block by block: a warp
// reads 32 dirty flags (1024 rows), then for each dirty 32-row block the lanes
// read G[row] (coalesced), keep the non-zero ones, zero them, and append
// (row - bounds[q], value) with one warp-aggregated atomic per block.
__global__ void k_compact(double *__restrict__ G, unsigned char *__restrict__ dflags, const long long *bounds,
                          int world, int rank, Rec *__restrict__ send, const long long *soff_dev,
                          long long *scnt, int take) {
  const unsigned lane = lane_id();
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (int q = 0; q < world; ++q) {
    if (q == rank) continue;
    const long long a = bounds[q], b = bounds[q + 1];
    const long long blk0 = a >> 5, blk1 = (b + 31) >> 5;
    for (long long sb = blk0 + gw * 32; sb < blk1; sb += warps * 32) {
      const long long myblk = sb + lane;
      const bool dirty = (myblk < blk1) && dflags[myblk];
      unsigned dm = __ballot_sync(0xffffffffu, dirty);
      while (dm) {
        const int j = __ffs(dm) - 1;
        dm &= dm - 1;
        const long long row = ((sb + j) << 5) + lane;
        const bool in = row >= a && row < b;
        double v = in ? G[row] : 0.0;
        const bool keep = in && v != 0.0;
        const unsigned km = __ballot_sync(0xffffffffu, keep);
        if (km == 0u) continue;
        unsigned long long base = 0;
        if (lane == 0) base = (unsigned long long)atomicAdd((unsigned long long *)&scnt[q], (unsigned long long)__popc(km));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) {
          const long long slot = soff_dev[q] + (long long)base + __popc(km & lanemask_lt());
          send[slot] = Rec{row - a, v};
          if (take) G[row] = 0.0;
        }
      }
    }
  }
}

// |G|_1 over dirty blocks of rows this rank does not own (s_k).
__global__ void k_outbox_mass(const double *__restrict__ G, const unsigned char *__restrict__ dflags,
                              long long n_rows, long long lo, long long hi, double *out) {
  double m = 0.0;
  const long long nb = (n_rows + 31) >> 5;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nb * 32; t += stride) {
    const long long blk = t >> 5;
    if (!dflags[blk]) continue;
    if (t < lo || t >= hi) m += (t < n_rows) ? fabs(G[t]) : 0.0;
  }
  m = warp_sum(m);
  if (lane_id() == 0 && m != 0.0) atomicAdd(out, m);
}

// Largest selection key |v| w_row of what a merge added (key_max: a non-negative
// double as its bit pattern, which orders like the value), for the rescale of an
// idle rank's threshold (k_rescale_T).
__device__ __forceinline__ void max_key(double key, double *key_max) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) key = fmax(key, __shfl_xor_sync(0xffffffffu, key, o));
  if (lane_id() == 0 && key > 0.0)
    atomicMax(reinterpret_cast<unsigned long long *>(key_max), (unsigned long long)__double_as_longlong(key));
}

// Merge received records: F[row] += val ("add them to existing
// fluids, node per node").
__global__ void k_merge(double *__restrict__ F, const Rec *__restrict__ recv, long long n, double *recv_mass,
                        const float *__restrict__ kw) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  double m = 0.0, km = 0.0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    const Rec r = recv[k];
    red_add(F + r.row, r.val);
    m += fabs(r.val);
    km = fmax(km, fabs(r.val) * (kw ? (double)kw[r.row] : 1.0));
  }
  m = warp_sum(m);
  if (lane_id() == 0 && m != 0.0) atomicAdd(recv_mass, m);
  max_key(km, recv_mass + 1);
}

// Receive-side threshold rescale ("update the threshold T_k,
// rescaling up by a factor ... proportional to min((r_k + received)/r_k,
// received)"; reading R13): T_k <- T_k (r_k + R) / r_k with R the fluid mass just
// merged and r_k the local residual before the merge.  An idle rank (r_k = 0, the
// ratio unbounded: the min picks the received side) restarts from the received
// fluid as a create starts from B (reading R5): T_k = max key merged / alpha, so
// T never stays at the value it sank to while the rank had nothing to diffuse.
__global__ void k_rescale_T(Ctl *ctl, const double *recv_mass, double r_k) {
  const double R = recv_mass[0], kmax = recv_mass[1];
  if (!(R > 0.0)) return;
  if (r_k > 0.0) ctl->T = ctl->T * ((r_k + R) / r_k);
  else if (kmax > 0.0) ctl->T = kmax / ctl->alpha;
}

// Setup: stable partition of every owned column into local rows (owned by this
// rank), then the remote rows grouped by owning peer in rank order, into new
// arrays; nloc[i] = local edges of column i.  Push order within a column is
// immaterial (sums), so this only reorders storage; the peer grouping lets the
// receiver-computes exchange treat a column's rows of one peer as one range.
__global__ void k_partition_columns(const long long *__restrict__ col_ptr, long long n, const int *__restrict__ ri,
                                    const double *__restrict__ v, const long long *bounds, int world, int rank,
                                    int *__restrict__ ri2, double *__restrict__ v2, int *__restrict__ nloc) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long b = col_ptr[i], e = col_ptr[i + 1];
    long long w = b;
    for (int step = 0; step < world; ++step) {
      const int q = step == 0 ? rank : (step <= rank ? step - 1 : step);   // own rows first, then peers
      const long long a = bounds[q], z = bounds[q + 1];
      for (long long k = b; k < e; ++k) {
        const int r = ri[k];
        if (r >= a && r < z) { ri2[w] = r; if (v) v2[w] = v[k]; ++w; }
      }
      if (step == 0) nloc[i] = (int)(w - b);
    }
  }
}

// DI_REMOTE_INCREMENT: pending remote mass
// s_k = sum_i |H_i - H_old_i| sum_{remote e of i} |p_e| -- the fluid the remote
// edges owe since the last push (p = d/#out, or |vals| signed).
__global__ void k_pending_mass(const long long *__restrict__ col_ptr, const int *__restrict__ nloc,
                               const double *__restrict__ vals, double d, const double *__restrict__ H,
                               const double *__restrict__ H_old, long long n, double *out) {
  double m = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long b = col_ptr[i], e = col_ptr[i + 1];
    const long long nl = nloc[i];
    if (nl == e - b) continue;
    const double dh = H[i] - H_old[i];
    if (dh == 0.0) continue;
    double c = 0.0;
    if (vals) { for (long long k = b + nl; k < e; ++k) c += fabs(vals[k]); }
    else c = d * (double)(e - b - nl) / (double)(e - b);
    m += fabs(dh) * c;
  }
  m = warp_sum(m);
  if (lane_id() == 0 && m != 0.0) atomicAdd(out, m);
}

// DI_REMOTE_INCREMENT push: for every column with H_i != H_old_i, its remote edges
// get (H_i - H_old_i) p_ji in the outbox (dirty-flagged), then H_old_i := H_i.
// One warp per column, lanes over its remote edges.
__global__ void k_push_increment(const long long *__restrict__ col_ptr, const int *__restrict__ nloc,
                                 const int *__restrict__ ri, const double *__restrict__ vals, double d,
                                 const double *__restrict__ H, double *__restrict__ H_old, long long n,
                                 double *__restrict__ G, unsigned char *__restrict__ dflags,
                                 unsigned long long *pushes) {
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const unsigned lane = lane_id();
  long long cnt = 0;
  for (long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    const long long b = col_ptr[i], e = col_ptr[i + 1];
    const long long nl = nloc[i];
    if (nl == e - b) continue;
    const double h = H[i];
    const double dh = h - H_old[i];
    if (dh == 0.0) continue;
    const double w = vals ? dh : dh * (d / (double)(e - b));
    for (long long k = b + nl + lane; k < e; k += 32) {
      const int r = ri[k];
      red_add(G + r, vals ? w * vals[k] : w);
      dflags[r >> 5] = 1;
    }
    if (lane == 0) { H_old[i] = h; cnt += e - b - nl; }
  }
  if (lane == 0 && cnt) atomicAdd(pushes, (unsigned long long)cnt);
}

// ---- DI_REMOTE_RECEIVER (receiver computes, NEXT f3) -------------------------
__device__ __forceinline__ int owner_of(const long long *bounds, int world, long long row) {
  int q = 0;
  while (q + 1 < world && bounds[q + 1] <= row) ++q;
  return q;
}
constexpr int kMaxWorld = 64;   // per-peer shared-memory counters of the setup census

// Setup pass 1: per peer, the (column, peer) pairs and remote edges of the owned
// columns (remote rows are stored after the local ones, ascending, so a column's
// rows of one peer are contiguous).  Block-local counters, then global adds.
__global__ void k_ric_census(const long long *__restrict__ col_ptr, const int *__restrict__ nloc, long long n,
                             const int *__restrict__ ri, const long long *bounds, int world,
                             unsigned long long *pairs, unsigned long long *edges) {
  __shared__ unsigned long long s_p[kMaxWorld], s_e[kMaxWorld];
  for (int q = threadIdx.x; q < kMaxWorld; q += blockDim.x) { s_p[q] = 0; s_e[q] = 0; }
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long e = col_ptr[i + 1];
    long long k = col_ptr[i] + nloc[i];
    while (k < e) {
      const int q = owner_of(bounds, world, ri[k]);
      long long k2 = k;
      while (k2 < e && ri[k2] >= bounds[q] && ri[k2] < bounds[q + 1]) ++k2;
      atomicAdd(&s_p[q], 1ull);
      atomicAdd(&s_e[q], (unsigned long long)(k2 - k));
      k = k2;
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < world; q += blockDim.x) {
    if (s_p[q]) atomicAdd(&pairs[q], s_p[q]);
    if (s_e[q]) atomicAdd(&edges[q], s_e[q]);
  }
}

// Setup pass 2: the column lists per peer and the edge records shipped once to
// each receiver: key = (global source column << 32) | local row at the receiver,
// value = p_ij (d/#out_j, or vals).
__global__ void k_ric_fill(const long long *__restrict__ col_ptr, const int *__restrict__ nloc, long long n,
                           const int *__restrict__ ri, const double *__restrict__ vals, double d, long long lo,
                           const long long *bounds, int world, const long long *pair_off, unsigned long long *pair_cur,
                           int *cols, const long long *edge_off, unsigned long long *edge_cur, Rec *erec) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long b = col_ptr[i], e = col_ptr[i + 1];
    long long k = b + nloc[i];
    const double w = d / (double)(e - b);
    while (k < e) {
      const int q = owner_of(bounds, world, ri[k]);
      long long k2 = k;
      while (k2 < e && ri[k2] >= bounds[q] && ri[k2] < bounds[q + 1]) ++k2;
      const unsigned long long ps = atomicAdd(&pair_cur[q], 1ull);
      cols[pair_off[q] + (long long)ps] = (int)i;
      const unsigned long long es = atomicAdd(&edge_cur[q], (unsigned long long)(k2 - k));
      for (long long t = k; t < k2; ++t) {
        const long long slot = edge_off[q] + (long long)es + (t - k);
        erec[slot] = Rec{(long long)(((unsigned long long)(i + lo) << 32) | (unsigned long long)(ri[t] - bounds[q])),
                         vals ? vals[t] : w};
      }
      k = k2;
    }
  }
}

__global__ void k_unpack_recs(const Rec *__restrict__ r, long long m, unsigned long long *key, double *val) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += stride) {
    key[k] = (unsigned long long)r[k].row;
    val[k] = r[k].val;
  }
}

// Receiver setup: the sorted keys (by source column, then row) become the
// remote-in CSR: unique sources, offsets, rows, weights.
__global__ void k_ric_build(const unsigned long long *__restrict__ key, long long m, const long long *__restrict__ pos,
                            long long *src, long long *off, int *row) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += stride) {
    const unsigned long long kk = key[k];
    row[k] = (int)(kk & 0xffffffffull);
    if (k == 0 || (key[k - 1] >> 32) != (kk >> 32)) {
      src[pos[k]] = (long long)(kk >> 32);
      off[pos[k]] = k;
    }
  }
}
__global__ void k_ric_flags(const unsigned long long *__restrict__ key, long long m, long long *flag) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += stride)
    flag[k] = (k == 0 || (key[k - 1] >> 32) != (key[k] >> 32)) ? 1 : 0;
}

// Round, sender: for every (column j, peer q) pair with H_j != H_old_j, the record
// (global j, H_j - H_old_j) for q.  H_old := H afterwards (a copy).
__global__ void k_send_increments(const int *__restrict__ cols, const long long *__restrict__ pair_off, int world,
                                  int rank, const double *__restrict__ H, const double *__restrict__ H_old,
                                  long long lo, Rec *__restrict__ send, const long long *soff,
                                  long long *scnt) {
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (int q = 0; q < world; ++q) {
    if (q == rank) continue;
    const long long a = pair_off[q], b = pair_off[q + 1];
    for (long long t0 = a + gw * 32; t0 < b; t0 += warps * 32) {
      const long long t = t0 + lane_id();
      double dh = 0.0;
      int j = 0;
      if (t < b) { j = cols[t]; dh = H[j] - H_old[j]; }
      const bool keep = dh != 0.0;
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (!m) continue;
      unsigned long long base = 0;
      if (lane_id() == 0) base = atomicAdd((unsigned long long *)&scnt[q], (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) send[soff[q] + (long long)base + __popc(m & lanemask_lt())] = Rec{(long long)j + lo, dh};
    }
  }
}

// Round, receiver: F_i += dh_j p_ij over the remote in-edges of source j (binary
// search of j in ric_src), warp per record; received mass for the T rescale.
__global__ void k_apply_remote_in(double *__restrict__ F, const Rec *__restrict__ recv, long long n_rec,
                                  const long long *__restrict__ src, const long long *__restrict__ off, long long ric_n,
                                  const int *__restrict__ row, const double *__restrict__ p, double *recv_mass,
                                  unsigned long long *pushes, const float *__restrict__ kw) {
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  double m = 0.0, km = 0.0;
  long long cnt = 0;
  for (long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rec; r += warps) {
    const Rec rc = recv[r];
    long long lo = 0, hi = ric_n - 1;
    while (lo < hi) {
      const long long mid = (lo + hi + 1) >> 1;
      if (src[mid] <= rc.row) lo = mid; else hi = mid - 1;
    }
    if (src[lo] != rc.row) continue;                 // cannot happen: senders ship only listed pairs
    const long long b = off[lo], e = off[lo + 1];
    for (long long k = b + lane_id(); k < e; k += 32) {
      const double v = rc.val * p[k];
      red_add(F + row[k], v);
      m += fabs(v);
      km = fmax(km, fabs(v) * (kw ? (double)kw[row[k]] : 1.0));
    }
    cnt += e - b;
  }
  m = warp_sum(m);
  if (lane_id() == 0) {
    if (m != 0.0) atomicAdd(recv_mass, m);
    if (cnt) atomicAdd(pushes, (unsigned long long)cnt);
  }
  max_key(km, recv_mass + 1);
}

__global__ void k_set_target(Ctl *ctl, double target, long long max_pass, int done) {
  ctl->target = target;
  ctl->max_pass = max_pass;
  ctl->done = done;
  ctl->hub_packed = 0ull;
  reset_tickets(ctl);
}

// ------------------------------------------------------------ host helpers --
void diter_dist_free(di_ctx *ctx) {
  if (!ctx || !ctx->dist) return;
  p2p_free(ctx);
  DistState *ds = ctx->dist;
  void *ptrs[] = {ds->d_bounds, ds->send, ds->recv, ds->d_scnt, ds->d_sums, ds->cols, ds->d_pair_off,
                  ds->ric_src, ds->ric_off, ds->ric_row, ds->ric_p};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  diter_free(ctx, ctx->G);
  diter_free(ctx, ctx->dflags);
  ctx->G = nullptr;
  ctx->dflags = nullptr;
  delete ds;
  ctx->dist = nullptr;
}

__global__ void k_indeg_all(const int *__restrict__ row_idx, long long nnz, unsigned *cnt) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += stride)
    atomicAdd(cnt + row_idx[e], 1u);
}
__global__ void k_indeg_sum(const unsigned *__restrict__ own, const unsigned *__restrict__ recv, int nblk,
                            long long blk_stride, long long n, unsigned *out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    unsigned c = own[i];
    for (int q = 0; q < nblk; ++q) c += recv[q * blk_stride + i];
    out[i] = c;
  }
}

// Global in-degree of the owned rows (DI_KEY_PAPER on a distributed context,
// PAPER.md:210): count this rank's edges into every global row, then a dense
// reduce-scatter through the fabric -- rank k receives every peer's counts for
// Omega_k (blocks padded to 16-byte records) and adds them to its own.  Setup only.
di_status diter_dist_indegree(di_ctx *ctx, unsigned *indeg_local) {
  DistState *ds = ctx->dist;
  const int W = ctx->world, rank = ctx->rank;
  const std::vector<long long> &b = ds->bounds;
  auto pad4 = [](long long x) { return (x + 3) / 4 * 4; };
  std::vector<long long> boff(W + 1, 0), soff(W), scnt(W), roff(W), rcnt(W);
  for (int q = 0; q < W; ++q) boff[q + 1] = boff[q] + pad4(b[q + 1] - b[q]);
  const long long my_blk = pad4(b[rank + 1] - b[rank]);
  unsigned *all = nullptr, *send = nullptr, *recv = nullptr;
  di_status st = DI_OK;
  const long long nr = ctx->n_rows;
  if (cudaMalloc(&all, sizeof(unsigned) * std::max(1LL, nr)) != cudaSuccess ||
      cudaMalloc(&send, sizeof(unsigned) * std::max(4LL, boff[W])) != cudaSuccess ||
      cudaMalloc(&recv, sizeof(unsigned) * std::max(4LL, my_blk * W)) != cudaSuccess) {
    diter_set_err(ctx, "cudaMalloc (in-degree exchange) failed");
    st = DI_ERR_OOM;
  }
  if (st == DI_OK) {
    cudaMemsetAsync(all, 0, sizeof(unsigned) * nr, ctx->stream);
    cudaMemsetAsync(send, 0, sizeof(unsigned) * boff[W], ctx->stream);
    k_indeg_all<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->row_idx, ctx->nnz_local, all);
    for (int q = 0; q < W; ++q)
      cudaMemcpyAsync(send + boff[q], all + b[q], sizeof(unsigned) * (b[q + 1] - b[q]), cudaMemcpyDeviceToDevice,
                      ctx->stream);
    for (int q = 0; q < W; ++q) {
      soff[q] = boff[q] / 4;
      scnt[q] = q == rank ? 0 : pad4(b[q + 1] - b[q]) / 4;
      roff[q] = q * my_blk / 4;
      rcnt[q] = q == rank ? 0 : my_blk / 4;
    }
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) st = DI_ERR_CUDA;
  }
  if (st == DI_OK)
    st = ds->fabric->alltoallv(ctx, reinterpret_cast<const Rec *>(send), soff.data(), scnt.data(),
                               reinterpret_cast<Rec *>(recv), roff.data(), rcnt.data());
  if (st == DI_OK) {
    // own block: my rows' counts from my own edges; peers' blocks in recv (own slot unused)
    cudaMemsetAsync(recv + rank * my_blk, 0, sizeof(unsigned) * my_blk, ctx->stream);
    k_indeg_sum<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(all + b[rank], recv, W, my_blk, b[rank + 1] - b[rank],
                                                            indeg_local);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) st = DI_ERR_CUDA;
  }
  cudaFree(all);
  cudaFree(send);
  cudaFree(recv);
  return st;
}

di_status diter_dist_max(di_ctx *ctx, double v, double *out) {
  *out = v;
  if (!ctx->dist) return DI_OK;
  return ctx->dist->fabric->host_max(ctx, v, out);
}

void diter_dist_pass_prologue(di_ctx *ctx) {
  if (ctx->dist && ctx->dist->p2p.on && ctx->dist->p2p.d_peers) p2p_pass_merge(ctx);
}

void diter_dist_stats(const di_ctx *ctx, di_stats *s) {
  const DistState *ds = ctx->dist;
  if (!ds) return;
  s->collectives = ds->fabric ? ds->fabric->calls : 0;
  s->confirms = ds->p2p.confirms;
  s->sleep_rounds = ds->p2p.sleep_rounds;
  if (ds->p2p.on) {
    s->exchange_bytes_resident = (long long)(ds->p2p.m * (sizeof(double) + sizeof(int)) + ((ds->p2p.m + 31) >> 5) +
                                             ds->p2p.win_bytes);
  } else {
    s->exchange_bytes_resident = (long long)(ctx->n_rows * sizeof(double) + ((ctx->n_rows + 31) >> 5) +
                                             (ds->send_cap + ds->recv_cap) * sizeof(Rec));
  }
}

di_status diter_dist_sum(di_ctx *ctx, double v, double *out) {
  *out = v;
  if (!ctx->dist) return DI_OK;
  DistState *ds = ctx->dist;
  CKD(cudaMemcpyAsync(ds->d_sums, &v, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  TRYD(ds->fabric->allreduce_sum(ctx, ds->d_sums, 1));
  CKD(cudaMemcpyAsync(out, ds->d_sums, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CKD(cudaStreamSynchronize(ctx->stream));
  return DI_OK;
}

di_status diter_dist_reset(di_ctx *ctx) {
  if (!ctx->dist) return DI_OK;
  if (ctx->dist->p2p.on) return p2p_reset(ctx);
  CKD(cudaMemsetAsync(ctx->G, 0, sizeof(double) * ctx->n_rows, ctx->stream));
  CKD(cudaMemsetAsync(ctx->dflags, 0, (size_t)((ctx->n_rows + 31) >> 5), ctx->stream));
  if (ctx->H_old) CKD(cudaMemsetAsync(ctx->H_old, 0, sizeof(double) * ctx->n_local, ctx->stream));
  CKD(cudaStreamSynchronize(ctx->stream));
  ctx->dist->s_k = 0.0;
  return DI_OK;
}

// DI_REMOTE_INCREMENT: push H - H_old along the remote edges into the outbox.
void dist_push_increment(di_ctx *ctx) {
  k_push_increment<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->col_ptr, ctx->nloc, ctx->row_idx, ctx->vals,
                                                              ctx->d, ctx->H, ctx->H_old, ctx->n_local, ctx->G,
                                                              ctx->dflags, &ctx->ctl->remote_pushes);
  ctx->kernel_launches += 1;
}

void dist_pending_mass(di_ctx *ctx, double *out) {
  k_pending_mass<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->col_ptr, ctx->nloc, ctx->vals, ctx->d, ctx->H,
                                                            ctx->H_old, ctx->n_local, out);
  ctx->kernel_launches += 1;
}

void dist_set_target(di_ctx *ctx, double target, long long max_pass) {
  k_set_target<<<1, 1, 0, ctx->stream>>>(ctx->ctl, target, max_pass, 0);
  ctx->kernel_launches += 1;
}

// exact global |F|_1 (+ s_k outbox mass when `with_outbox`)
static di_status global_residual(di_ctx *ctx, double add, double *out) {
  DistState *ds = ctx->dist;
  TRYD(diter_l1_launch(ctx));
  CKD(cudaMemcpyAsync(ds->d_sums, ctx->l1_out, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  double h_add = add;
  CKD(cudaMemcpyAsync(ds->d_sums + 1, &h_add, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  TRYD(ds->fabric->allreduce_sum(ctx, ds->d_sums, 2));
  double h[2];
  CKD(cudaMemcpyAsync(h, ds->d_sums, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CKD(cudaStreamSynchronize(ctx->stream));
  *out = h[0] + h[1];
  return DI_OK;
}

// One exchange round: optional compaction of the whole outbox, record counts,
// all-to-all-v, merge.  Collective.
static di_status exchange(di_ctx *ctx, bool send_now) {
  NvtxRange nv("bulk exchange");
  DistState *ds = ctx->dist;
  const int W = ctx->world;
  CKD(cudaMemsetAsync(ds->d_scnt, 0, sizeof(long long) * W, ctx->stream));
  CKD(cudaMemsetAsync(ds->d_sums + kSums + 1, 0, 2 * sizeof(double), ctx->stream));   // received mass, max key
  if (send_now) {
    long long *d_soff = reinterpret_cast<long long *>(ds->d_sums + kSums + 3);
    CKD(cudaMemcpyAsync(d_soff, ds->soff.data(), sizeof(long long) * W, cudaMemcpyHostToDevice, ctx->stream));
    k_compact<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->G, ctx->dflags, ds->d_bounds, W, ctx->rank,
                                                         ds->send, d_soff, ds->d_scnt, 1);
    CKD(cudaMemsetAsync(ctx->dflags, 0, (size_t)((ctx->n_rows + 31) >> 5), ctx->stream));
    ctx->kernel_launches += 1;
  }
  CKD(cudaMemcpyAsync(ds->scnt.data(), ds->d_scnt, sizeof(long long) * W, cudaMemcpyDeviceToHost, ctx->stream));
  CKD(cudaStreamSynchronize(ctx->stream));
  TRYD(ds->fabric->alltoall_counts(ctx, ds->scnt.data(), ds->rcnt.data()));
  long long tot = 0;
  for (int q = 0; q < W; ++q) {
    ds->roff[q] = tot;
    tot += ds->rcnt[q];
  }
  if (tot > ds->recv_cap) {
    diter_set_err(ctx, "receive overflow (%lld > %lld)", tot, ds->recv_cap);
    return DI_ERR_STATE;
  }
  long long sent = 0;
  for (int q = 0; q < W; ++q) sent += ds->scnt[q];
  TRYD(ds->fabric->alltoallv(ctx, ds->send, ds->soff.data(), ds->scnt.data(), ds->recv, ds->roff.data(),
                             ds->rcnt.data()));
  if (tot > 0) {
    k_merge<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->F, ds->recv, tot, ds->d_sums + kSums + 1, ctx->kw);
    ctx->kernel_launches += 1;
  }
  if (sent > 0) {
    ctx->exchanged_bytes += (long long)sizeof(Rec) * sent;
    ctx->alg_bytes_exchange += 12LL * sent + 20LL * tot;  // 12 B shipped + 20 B merged
    ctx->exchanges += 1;
  }
  if (send_now) ds->s_k = 0.0;
  return DI_OK;
}

// DI_REMOTE_RECEIVER setup (collective): the receivers get, once, the remote
// in-edges of their rows -- (P)_{i in Omega_k, j in Omega} of PAPER.md:268-272 --
// and the senders their per-peer column lists.
#define CKR(call)                                                                      \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      diter_set_err(ctx, "%s failed: %s", #call, cudaGetErrorString(e_));             \
      st = e_ == cudaErrorMemoryAllocation ? DI_ERR_OOM : DI_ERR_CUDA;                 \
      goto done;                                                                       \
    }                                                                                  \
  } while (0)

static di_status setup_receiver(di_ctx *ctx) {
  DistState *ds = ctx->dist;
  const int W = ctx->world;
  di_status st = DI_OK;
  unsigned long long *d_cnt = nullptr;   // [4 W]: pairs, edges, pair cursor, edge cursor
  long long *d_eoff = nullptr, *d_flag = nullptr, *d_pos = nullptr;
  Rec *erec = nullptr, *rrec = nullptr;
  unsigned long long *k1 = nullptr, *k2 = nullptr;
  double *v1 = nullptr;
  void *tmp = nullptr;
  std::vector<unsigned long long> h(2 * W);
  std::vector<long long> eoff(W + 1, 0), ecnt(W), rcnt(W), roff(W + 1, 0);
  long long R = 0;
  const int grid = ctx->num_sms * 8;
  if (W > kMaxWorld) { diter_set_err(ctx, "DI_REMOTE_RECEIVER supports at most %d ranks", kMaxWorld); return DI_ERR_INVALID_ARG; }
  CKR(cudaMalloc(&d_cnt, sizeof(unsigned long long) * 4 * W));
  CKR(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * 4 * W, ctx->stream));
  k_ric_census<<<grid, 256, 0, ctx->stream>>>(ctx->col_ptr, ctx->nloc, ctx->n_local, ctx->row_idx, ds->d_bounds, W,
                                             d_cnt, d_cnt + W);
  CKR(cudaMemcpyAsync(h.data(), d_cnt, sizeof(unsigned long long) * 2 * W, cudaMemcpyDeviceToHost, ctx->stream));
  CKR(cudaStreamSynchronize(ctx->stream));
  ds->pair_off.assign(W + 1, 0);
  for (int q = 0; q < W; ++q) {
    ds->pair_off[q + 1] = ds->pair_off[q] + (long long)h[q];
    ecnt[q] = (long long)h[W + q];
    eoff[q + 1] = eoff[q] + ecnt[q];
  }
  CKR(cudaMalloc(&ds->cols, sizeof(int) * std::max(1LL, ds->pair_off[W])));
  CKR(cudaMalloc(&ds->d_pair_off, sizeof(long long) * (W + 1)));
  CKR(cudaMalloc(&d_eoff, sizeof(long long) * (W + 1)));
  CKR(cudaMalloc(&erec, sizeof(Rec) * std::max(1LL, eoff[W])));
  CKR(cudaMemcpyAsync(ds->d_pair_off, ds->pair_off.data(), sizeof(long long) * (W + 1), cudaMemcpyHostToDevice, ctx->stream));
  CKR(cudaMemcpyAsync(d_eoff, eoff.data(), sizeof(long long) * (W + 1), cudaMemcpyHostToDevice, ctx->stream));
  k_ric_fill<<<grid, 256, 0, ctx->stream>>>(ctx->col_ptr, ctx->nloc, ctx->n_local, ctx->row_idx, ctx->vals, ctx->d,
                                           ctx->lo, ds->d_bounds, W, ds->d_pair_off, d_cnt + 2 * W, ds->cols, d_eoff,
                                           d_cnt + 3 * W, erec);
  CKR(cudaStreamSynchronize(ctx->stream));
  // ship every edge record to its receiver once
  st = ds->fabric->alltoall_counts(ctx, ecnt.data(), rcnt.data());
  if (st != DI_OK) goto done;
  for (int q = 0; q < W; ++q) roff[q + 1] = roff[q] + rcnt[q];
  R = roff[W];
  CKR(cudaMalloc(&rrec, sizeof(Rec) * std::max(1LL, R)));
  st = ds->fabric->alltoallv(ctx, erec, eoff.data(), ecnt.data(), rrec, roff.data(), rcnt.data());
  if (st != DI_OK) goto done;
  ctx->exchanged_bytes += (long long)sizeof(Rec) * eoff[W];
  // sort by (source column, row) and build the remote-in CSR
  ds->ric_e = R;
  CKR(cudaMalloc(&ds->ric_row, sizeof(int) * std::max(1LL, R)));
  CKR(cudaMalloc(&ds->ric_p, sizeof(double) * std::max(1LL, R)));
  if (R > 0) {
    CKR(cudaMalloc(&k1, sizeof(unsigned long long) * R));
    CKR(cudaMalloc(&k2, sizeof(unsigned long long) * R));
    CKR(cudaMalloc(&v1, sizeof(double) * R));
    CKR(cudaMalloc(&d_flag, sizeof(long long) * R));
    CKR(cudaMalloc(&d_pos, sizeof(long long) * R));
    k_unpack_recs<<<grid, 256, 0, ctx->stream>>>(rrec, R, k1, v1);
    size_t t1 = 0, t2 = 0;
    CKR(cub::DeviceRadixSort::SortPairs(nullptr, t1, k1, k2, v1, ds->ric_p, (int64_t)R, 0, 64, ctx->stream));
    CKR(cub::DeviceScan::ExclusiveSum(nullptr, t2, d_flag, d_pos, (int64_t)R, ctx->stream));
    CKR(cudaMalloc(&tmp, std::max(t1, t2)));
    CKR(cub::DeviceRadixSort::SortPairs(tmp, t1, k1, k2, v1, ds->ric_p, (int64_t)R, 0, 64, ctx->stream));
    k_ric_flags<<<grid, 256, 0, ctx->stream>>>(k2, R, d_flag);
    CKR(cub::DeviceScan::ExclusiveSum(tmp, t2, d_flag, d_pos, (int64_t)R, ctx->stream));
    long long last_pos = 0, last_flag = 0;
    CKR(cudaMemcpyAsync(&last_pos, d_pos + R - 1, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
    CKR(cudaMemcpyAsync(&last_flag, d_flag + R - 1, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
    CKR(cudaStreamSynchronize(ctx->stream));
    ds->ric_n = last_pos + last_flag;
  }
  CKR(cudaMalloc(&ds->ric_src, sizeof(long long) * std::max(1LL, ds->ric_n)));
  CKR(cudaMalloc(&ds->ric_off, sizeof(long long) * (ds->ric_n + 1)));
  if (R > 0) {
    k_ric_build<<<grid, 256, 0, ctx->stream>>>(k2, R, d_pos, ds->ric_src, ds->ric_off, ds->ric_row);
    CKR(cudaMemcpyAsync(ds->ric_off + ds->ric_n, &ds->ric_e, sizeof(long long), cudaMemcpyHostToDevice, ctx->stream));
  }
  // round buffers: at most one record per (column, peer) pair out, per source column in
  {
    const long long scap = std::max(1LL, ds->pair_off[W]), rcap = std::max(1LL, ds->ric_n);
    if (scap > ds->send_cap) {
      cudaFree(ds->send);
      ds->send = nullptr;
      CKR(cudaMalloc(&ds->send, sizeof(Rec) * scap));
      ds->send_cap = scap;
    }
    if (rcap > ds->recv_cap) {
      cudaFree(ds->recv);
      ds->recv = nullptr;
      CKR(cudaMalloc(&ds->recv, sizeof(Rec) * rcap));
      ds->recv_cap = rcap;
    }
    for (int q = 0; q < W; ++q) ds->soff[q] = ds->pair_off[q];
  }
  CKR(cudaStreamSynchronize(ctx->stream));
done:
  void *fr_[] = {d_cnt, d_eoff, d_flag, d_pos, erec, rrec, k1, k2, v1, tmp};
  for (void *x : fr_)
    if (x) cudaFree(x);
  return st;
}

// Receiver-computes round (collective): ship (j, H_j - H_old_j) per listed pair,
// H_old := H, exchange, receivers apply their in-edges.
static di_status exchange_receiver(di_ctx *ctx, bool send_now) {
  DistState *ds = ctx->dist;
  const int W = ctx->world;
  CKD(cudaMemsetAsync(ds->d_scnt, 0, sizeof(long long) * W, ctx->stream));
  CKD(cudaMemsetAsync(ds->d_sums + kSums + 1, 0, 2 * sizeof(double), ctx->stream));   // received mass, max key
  if (send_now) {
    long long *d_soff = reinterpret_cast<long long *>(ds->d_sums + kSums + 3);
    CKD(cudaMemcpyAsync(d_soff, ds->soff.data(), sizeof(long long) * W, cudaMemcpyHostToDevice, ctx->stream));
    k_send_increments<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ds->cols, ds->d_pair_off, W, ctx->rank, ctx->H,
                                                                 ctx->H_old, ctx->lo, ds->send, d_soff, ds->d_scnt);
    CKD(cudaMemcpyAsync(ctx->H_old, ctx->H, sizeof(double) * ctx->n_local, cudaMemcpyDeviceToDevice, ctx->stream));
    ctx->kernel_launches += 1;
  }
  CKD(cudaMemcpyAsync(ds->scnt.data(), ds->d_scnt, sizeof(long long) * W, cudaMemcpyDeviceToHost, ctx->stream));
  CKD(cudaStreamSynchronize(ctx->stream));
  TRYD(ds->fabric->alltoall_counts(ctx, ds->scnt.data(), ds->rcnt.data()));
  long long tot = 0, sent = 0;
  for (int q = 0; q < W; ++q) {
    ds->roff[q] = tot;
    tot += ds->rcnt[q];
    sent += ds->scnt[q];
  }
  if (tot > ds->recv_cap) {
    diter_set_err(ctx, "receive overflow (%lld > %lld)", tot, ds->recv_cap);
    return DI_ERR_STATE;
  }
  TRYD(ds->fabric->alltoallv(ctx, ds->send, ds->soff.data(), ds->scnt.data(), ds->recv, ds->roff.data(),
                             ds->rcnt.data()));
  if (tot > 0) {
    k_apply_remote_in<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->F, ds->recv, tot, ds->ric_src, ds->ric_off,
                                                                 ds->ric_n, ds->ric_row, ds->ric_p,
                                                                 ds->d_sums + kSums + 1, &ctx->ctl->remote_pushes, ctx->kw);
    ctx->kernel_launches += 1;
  }
  if (sent > 0) {
    ctx->exchanged_bytes += (long long)sizeof(Rec) * sent;
    ctx->alg_bytes_exchange += 12LL * sent + 20LL * tot;
    ctx->exchanges += 1;
  }
  if (send_now) ds->s_k = 0.0;
  return DI_OK;
}

// One exchange round in the context's remote-push mode (collective).
static di_status round_exchange(di_ctx *ctx, bool send_now) {
  if (ctx->opt.remote_push == DI_REMOTE_RECEIVER) return exchange_receiver(ctx, send_now);
  if (ctx->opt.remote_push == DI_REMOTE_INCREMENT && send_now) dist_push_increment(ctx);
  return exchange(ctx, send_now);
}

// profile=1: events around the select and the scatter of local pass `slot` of a
// round (slot < check_interval), read back after the round's host sync
static void prof_mark(di_ctx *ctx, int slot, int q) {
  if (ctx->opt.profile && !ctx->prof_ev.empty()) cudaEventRecord(ctx->prof_ev[4 * slot + q], ctx->stream);
}

static di_status prof_collect(di_ctx *ctx, int npasses) {
  if (!ctx->opt.profile || ctx->prof_ev.empty()) return DI_OK;
  for (int k = 0; k < npasses; ++k) {
    float a = 0.f, b = 0.f;
    CKD(cudaEventElapsedTime(&a, ctx->prof_ev[4 * k + 0], ctx->prof_ev[4 * k + 1]));
    CKD(cudaEventElapsedTime(&b, ctx->prof_ev[4 * k + 1], ctx->prof_ev[4 * k + 2]));
    ctx->kt_ms[0] += a;
    ctx->kt_ms[1] += b;
    ctx->pass_us.push_back({a * 1e3, b * 1e3});
  }
  ctx->kt_passes += npasses;
  return DI_OK;
}

void dist_launch_pass_kernels(di_ctx *ctx, int slot) {
  Graph g = diter_graph(ctx);
  diter_dist_pass_prologue(ctx);
  prof_mark(ctx, slot, 0);
  if (ctx->sweep_on) {            // ASYNC / P2P local passes as asynchronous sweeps (R26)
    prof_mark(ctx, slot, 1);
    diter_launch_sweep(ctx);
    prof_mark(ctx, slot, 2);
    ctx->kernel_launches += (ctx->cap_hub > 0 && !DITER_SWEEP_HUBS) ? 2 : 1;
    return;
  }
  k_select<<<ctx->grid_select, kSelectThreads, 0, ctx->stream>>>(ctx->F, ctx->H, ctx->fr, ctx->n_local, ctx->ctl,
                                                                ctx->sel_part, ctx->kw);
  prof_mark(ctx, slot, 1);
  if (ctx->vals)
    k_scatter<true, true><<<ctx->grid_scatter, kScatterThreads, ctx->scatter_smem, ctx->stream>>>(
        g, ctx->F, ctx->fr, ctx->ctl, ctx->sc_part);
  else
    k_scatter<false, true><<<ctx->grid_scatter, kScatterThreads, ctx->scatter_smem, ctx->stream>>>(
        g, ctx->F, ctx->fr, ctx->ctl, ctx->sc_part);
  if (ctx->cap_hub > 0) {
    if (ctx->vals)
      k_scatter_hubs<true><<<ctx->grid_hubs, kScatterThreads, 0, ctx->stream>>>(g, ctx->F, ctx->fr, ctx->ctl);
    else
      k_scatter_hubs<false><<<ctx->grid_hubs, kScatterThreads, 0, ctx->stream>>>(g, ctx->F, ctx->fr, ctx->ctl);
  }
  prof_mark(ctx, slot, 2);
  ctx->kernel_launches += ctx->cap_hub > 0 ? 3 : 2;
}

// Partition adaptation rule (reading R22): for each boundary
// omega_k between ranks a = k-1 and b = k, if one side has > 2x the other's
// residual and has done > 1.2x its work (edges) since the last check, 10 % of the
// busier side's nodes move across.  Inputs are gathered from every rank, so all
// ranks compute the same bounds; *nb stays empty when nothing moves.
extern "C" di_status di_rebalance(di_ctx *ctx, const int64_t *nb);
static di_status adapt_bounds(di_ctx *ctx, double r_k, long long work, std::vector<long long> *nb) {
  DistState *ds = ctx->dist;
  const int W = ctx->world;
  std::vector<long long> send(W), rr(W), ww(W);
  long long rbits;
  std::memcpy(&rbits, &r_k, sizeof(double));
  std::fill(send.begin(), send.end(), rbits);
  TRYD(ds->fabric->alltoall_counts(ctx, send.data(), rr.data()));
  std::fill(send.begin(), send.end(), work);
  TRYD(ds->fabric->alltoall_counts(ctx, send.data(), ww.data()));
  std::vector<double> r(W);
  for (int q = 0; q < W; ++q) std::memcpy(&r[q], &rr[q], sizeof(double));
  std::vector<long long> b = ds->bounds;
  bool moved = false;
  for (int k = 1; k < W; ++k) {
    const int a = k - 1, c = k;
    if (r[a] > 2.0 * r[c] && (double)ww[a] > 1.2 * (double)ww[c]) {
      const long long m = std::max(1LL, (b[k] - b[k - 1]) / 10);
      const long long nk = std::max(b[k - 1] + 1, b[k] - m);
      if (nk != b[k]) { b[k] = nk; moved = true; }
    } else if (r[c] > 2.0 * r[a] && (double)ww[c] > 1.2 * (double)ww[a]) {
      const long long m = std::max(1LL, (b[k + 1] - b[k]) / 10);
      const long long nk = std::min(b[k + 1] - 1, b[k] + m);
      if (nk != b[k]) { b[k] = nk; moved = true; }
    }
  }
  if (moved) *nb = b;
  return DI_OK;
}

static di_status dist_run_impl(di_ctx *ctx, double target) {
  if (ctx->dist->p2p.on) return p2p_run(ctx, target);
  DistState *ds = ctx->dist;
  CKD(cudaSetDevice(ctx->device));
  CKD(cudaEventRecord(ctx->ev0, ctx->stream));
  const long long launches0 = ctx->kernel_launches;
  const long long max_pass_abs = ctx->passes_done + ctx->opt.max_passes;
  const bool sync_mode = ctx->opt.exchange_mode == DI_EXCHANGE_SYNC;
  const bool incr = ctx->H_old != nullptr;   // DI_REMOTE_INCREMENT
  Ctl *h = reinterpret_cast<Ctl *>(ctx->h_ctl);
  di_status st = DI_OK;
  double R = 0.0;
  // outbox fluid counts toward the residual (in-flight mass)
  TRYD(global_residual(ctx, ds->s_k, &R));
  ctx->residual = R;
  if (ctx->sweep_on) k_rpred_set<<<1, 1, 0, ctx->stream>>>(ctx->ctl, ctx->l1_out);   // sweeps carry |F|_1
  if (R < target) goto out;
  if (sync_mode) {
    // -------- SYNC: one exchange per pass, pass totals all-reduced ----------
    k_set_target<<<1, 1, 0, ctx->stream>>>(ctx->ctl, target, max_pass_abs, 0);
    for (;;) {
      dist_launch_pass_kernels(ctx, 0);
      k_reduce_partials<<<1, kFinalizeThreads, 0, ctx->stream>>>(ctx->ctl, ctx->sel_part, ctx->grid_select,
                                                                  ctx->sc_part, ctx->grid_scatter, ds->d_sums);
      // the pass totals except the last (the far-edge mass a one-GPU deferral left
      // pending, always 0 on a distributed context): the host fabrics reduce <= 8
      TRYD(ds->fabric->allreduce_sum(ctx, ds->d_sums, kSums - 1));
      TRYD(round_exchange(ctx, true));
      k_apply_pass<<<1, 1, 0, ctx->stream>>>(ctx->ctl, ds->d_sums, ctx->log);
      ctx->kernel_launches += 2;
      CKD(cudaMemcpyAsync(ctx->h_ctl, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
      CKD(cudaStreamSynchronize(ctx->stream));
      TRYD(prof_collect(ctx, 1));
      if (!h->done) continue;
      ctx->passes_done = h->pass;
      TRYD(global_residual(ctx, 0.0, &R));
      ctx->residual = R;
      if (R < target) break;
      if (h->pass >= max_pass_abs) { st = DI_ERR_NOT_CONVERGED; break; }
      k_set_target<<<1, 1, 0, ctx->stream>>>(ctx->ctl, target, max_pass_abs, 0);   // prediction was early
    }
  } else {
    // -------- ASYNC: local passes, exchange rounds every check_interval ------
    long long rounds = 0, edges_mark = h->edges;
    for (;;) {
      // local passes: no target (never "done" locally), local threshold policy
      k_set_target<<<1, 1, 0, ctx->stream>>>(ctx->ctl, 0.0, max_pass_abs, 0);
      if (ctx->graph_exec && !ctx->opt.profile) {
        // the round's local passes as one captured graph (select, scatter, hubs, finalize)
        CKD(cudaGraphLaunch(ctx->graph_exec, ctx->stream));
        ctx->graph_launches += 1;
        ctx->kernel_launches += ((ctx->sweep_on ? 2LL : 3LL) + (ctx->cap_hub > 0 && !(ctx->sweep_on && DITER_SWEEP_HUBS))) * ctx->check_interval;
      } else {
        for (int k = 0; k < ctx->check_interval; ++k) {
          dist_launch_pass_kernels(ctx, k);
          k_finalize<<<1, kFinalizeThreads, 0, ctx->stream>>>(ctx->ctl, ctx->sel_part, diter_n_sel_part(ctx),
                                                              ctx->sc_part, diter_n_sc_part(ctx), ctx->log);
          ctx->kernel_launches += 1;
        }
      }
      // round: s_k (outbox mass, or the pending increment mass) and r_k decide the
      // send (eq. send)
      CKD(cudaMemsetAsync(ds->d_sums, 0, sizeof(double), ctx->stream));
      if (incr)
        k_pending_mass<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->col_ptr, ctx->nloc, ctx->vals, ctx->d, ctx->H,
                                                                  ctx->H_old, ctx->n_local, ds->d_sums);
      else
        k_outbox_mass<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->G, ctx->dflags, ctx->n_rows, ctx->lo,
                                                                 ctx->lo + ctx->n_local, ds->d_sums);
      TRYD(diter_l1_launch(ctx));
      double hs[2];
      CKD(cudaMemcpyAsync(&hs[0], ds->d_sums, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      CKD(cudaMemcpyAsync(&hs[1], ctx->l1_out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      CKD(cudaMemcpyAsync(ctx->h_ctl, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
      CKD(cudaStreamSynchronize(ctx->stream));
      TRYD(prof_collect(ctx, ctx->check_interval));
      ds->s_k = hs[0];
      const double r_k = hs[1];
      const bool send_now = (ds->s_k > r_k / ctx->world) || (r_k == 0.0 && ds->s_k > 0.0);
      TRYD(round_exchange(ctx, send_now));
      if (ctx->opt.receive_rescale) {
        k_rescale_T<<<1, 1, 0, ctx->stream>>>(ctx->ctl, ds->d_sums + kSums + 1, r_k);
        ctx->kernel_launches += 1;
      }
      ctx->passes_done = h->pass;
      TRYD(global_residual(ctx, ds->s_k, &R));
      ctx->residual = R;
      if (ctx->sweep_on) k_rpred_set<<<1, 1, 0, ctx->stream>>>(ctx->ctl, ctx->l1_out);
      const bool stop = R < target, out_of_passes = h->pass >= max_pass_abs;
      if (stop || out_of_passes) {
        // deliver what is left in the outboxes, so that on return F (with H) is
        // the whole state: F = B - (I-P)H on every rank, nothing in flight
        TRYD(round_exchange(ctx, true));
        if (!stop) st = DI_ERR_NOT_CONVERGED;
        break;
      }
      // partition adaptation (NEXT f4, reading R22) every adapt_rounds rounds
      if (ctx->opt.adapt_rounds > 0 && ++rounds % ctx->opt.adapt_rounds == 0) {
        std::vector<long long> nb;
        TRYD(adapt_bounds(ctx, r_k, h->edges - edges_mark, &nb));
        if (!nb.empty()) {
          TRYD(di_rebalance(ctx, reinterpret_cast<const int64_t *>(nb.data())));
          ds = ctx->dist;                              // the context was rebuilt
          h = reinterpret_cast<Ctl *>(ctx->h_ctl);
          CKD(cudaMemcpyAsync(ctx->h_ctl, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
          CKD(cudaStreamSynchronize(ctx->stream));
        }
        edges_mark = h->edges;
      }
    }
  }
out:
  CKD(cudaEventRecord(ctx->ev1, ctx->stream));
  CKD(cudaEventSynchronize(ctx->ev1));
  {
    float ms = 0.f;
    CKD(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    ctx->run_ms = ms;
    ctx->run_ms_total += ms;
  }
  CKD(cudaMemcpyAsync(ctx->h_ctl, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
  CKD(cudaStreamSynchronize(ctx->stream));
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

// A rank that fails inside the collective sequence releases its loopback peers
// (they return DI_ERR_STATE instead of waiting forever).  max_passes is reached by
// every rank in the same round (local pass counts advance together), so it is not
// a failure of one rank.
di_status diter_dist_run(di_ctx *ctx, double target) {
  const di_status st = dist_run_impl(ctx, target);
  if (st != DI_OK && st != DI_ERR_NOT_CONVERGED && ctx->dist && ctx->dist->fabric) ctx->dist->fabric->abort();
  return st;
}

// ----------------------------------------------------------------- create --

static di_status dist_build(di_ctx *ctx, const int64_t *col_ptr_local, const int32_t *row_idx_local,
                            const double *values_local, const double *b_local, const di_options *opt);

// ---------------------------------------------------------- rebalance (f4) --
// PAPER.md:178-184 remark + P:523-543: "an idle PID could take nodes from the
// busiest PID ... we just need to transmit the information F_n and H_n of the
// candidate nodes".  Ranks here hold only their own columns, so the moved
// columns travel too.  Collective: deliver everything in flight, ship each
// node's column (degree, rows, values), F, H and B to its owner under the new
// bounds, rebuild the context on its new range (same fabric, stream, events),
// restore F, H, the control block and the counters.
namespace {
template <typename T>
void put(std::vector<unsigned char> &b, const T *p, size_t n) {
  const size_t o = b.size();
  b.resize(o + sizeof(T) * n);
  if (n) std::memcpy(b.data() + o, p, sizeof(T) * n);
  b.resize((b.size() + 7) & ~size_t(7));
}
template <typename T>
const unsigned char *get(const unsigned char *c, T *p, size_t n) {
  if (n) std::memcpy(p, c, sizeof(T) * n);
  return c + ((sizeof(T) * n + 7) & ~size_t(7));
}
}  // namespace

extern "C" di_status di_rebalance(di_ctx *ctx, const int64_t *nb) {
  NvtxRange nv("di_rebalance");
  if (!ctx || !nb) { diter_set_err(ctx, "NULL argument"); return DI_ERR_INVALID_ARG; }
  if (!ctx->dist || ctx->world < 2) { diter_set_err(ctx, "di_rebalance: distributed contexts only"); return DI_ERR_INVALID_ARG; }
  if (ctx->dist->p2p.on) {
    diter_set_err(ctx, "di_rebalance: not available with DI_EXCHANGE_P2P (its outbox slots are fixed at create)");
    return DI_ERR_UNSUPPORTED;
  }
  const int W = ctx->world, rank = ctx->rank;
  if (nb[0] != 0 || nb[W] != ctx->n_rows) { diter_set_err(ctx, "bounds must start at 0 and end at N"); return DI_ERR_INVALID_ARG; }
  for (int k = 0; k < W; ++k)
    if (nb[k + 1] <= nb[k]) { diter_set_err(ctx, "bounds must be strictly increasing"); return DI_ERR_INVALID_ARG; }
  CKD(cudaSetDevice(ctx->device));
  DistState *ds = ctx->dist;
  TRYD(round_exchange(ctx, true));                 // nothing in flight from here on
  const long long n = ctx->n_local, nnz = ctx->nnz_local, lo = ctx->lo;
  std::vector<long long> cp(n + 1);
  std::vector<int> ri(nnz);
  std::vector<double> vv(ctx->vals ? nnz : 0), F(n), H(n), B(ctx->d_b ? n : 0);
  Ctl c;
  CKD(cudaMemcpyAsync(cp.data(), ctx->col_ptr, sizeof(long long) * (n + 1), cudaMemcpyDeviceToHost, ctx->stream));
  if (nnz) CKD(cudaMemcpyAsync(ri.data(), ctx->row_idx, sizeof(int) * nnz, cudaMemcpyDeviceToHost, ctx->stream));
  if (ctx->vals && nnz) CKD(cudaMemcpyAsync(vv.data(), ctx->vals, sizeof(double) * nnz, cudaMemcpyDeviceToHost, ctx->stream));
  CKD(cudaMemcpyAsync(F.data(), ctx->F, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CKD(cudaMemcpyAsync(H.data(), ctx->H, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  if (ctx->d_b) CKD(cudaMemcpyAsync(B.data(), ctx->d_b, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CKD(cudaMemcpyAsync(&c, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
  CKD(cudaStreamSynchronize(ctx->stream));
  // pack, per new owner q, my nodes [a, z) in its new range
  std::vector<std::vector<unsigned char>> pk(W);
  for (int q = 0; q < W; ++q) {
    const long long a = std::max<long long>(lo, nb[q]), z = std::min<long long>(lo + n, nb[q + 1]);
    if (z <= a) continue;
    const long long m = z - a, e0 = cp[a - lo], e1 = cp[z - lo];
    std::vector<long long> deg(m);
    for (long long i = 0; i < m; ++i) deg[i] = cp[a - lo + i + 1] - cp[a - lo + i];
    const long long hdr[3] = {a, m, e1 - e0};
    put(pk[q], hdr, 3);
    put(pk[q], deg.data(), m);
    put(pk[q], ri.data() + e0, e1 - e0);
    if (ctx->vals) put(pk[q], vv.data() + e0, e1 - e0);
    put(pk[q], F.data() + (a - lo), m);
    put(pk[q], H.data() + (a - lo), m);
    if (ctx->d_b) put(pk[q], B.data() + (a - lo), m);
    pk[q].resize((pk[q].size() + sizeof(Rec) - 1) / sizeof(Rec) * sizeof(Rec));
  }
  std::vector<long long> soff(W, 0), scnt(W, 0), roff(W, 0), rcnt(W, 0);
  long long stot = 0;
  for (int q = 0; q < W; ++q) {
    soff[q] = stot;
    scnt[q] = q == rank ? 0 : (long long)(pk[q].size() / sizeof(Rec));
    stot += scnt[q];
  }
  TRYD(ds->fabric->alltoall_counts(ctx, scnt.data(), rcnt.data()));
  long long rtot = 0;
  for (int q = 0; q < W; ++q) { roff[q] = rtot; rtot += q == rank ? 0 : rcnt[q]; }
  std::vector<unsigned char> hs(std::max<long long>(1, stot) * sizeof(Rec)), hr(std::max<long long>(1, rtot) * sizeof(Rec));
  for (int q = 0; q < W; ++q)
    if (scnt[q]) std::memcpy(hs.data() + soff[q] * sizeof(Rec), pk[q].data(), pk[q].size());
  Rec *dsend = nullptr, *drecv = nullptr;
  CKD(cudaMalloc(&dsend, hs.size()));
  CKD(cudaMalloc(&drecv, hr.size()));
  CKD(cudaMemcpyAsync(dsend, hs.data(), hs.size(), cudaMemcpyHostToDevice, ctx->stream));
  di_status st = ds->fabric->alltoallv(ctx, dsend, soff.data(), scnt.data(), drecv, roff.data(), rcnt.data());
  if (st == DI_OK && cudaMemcpyAsync(hr.data(), drecv, hr.size(), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess)
    st = DI_ERR_CUDA;
  cudaStreamSynchronize(ctx->stream);
  cudaFree(dsend);
  cudaFree(drecv);
  if (st != DI_OK) return st;
  // unpack in source-rank order: the pieces of [nb[rank], nb[rank+1]) ascend
  const long long lo2 = nb[rank], n2 = nb[rank + 1] - nb[rank];
  std::vector<long long> cp2(n2 + 1, 0);
  std::vector<int> ri2;
  std::vector<double> vv2, F2(n2), H2(n2), B2(ctx->d_b ? n2 : 0);
  long long next = lo2;
  for (int q = 0; q < W; ++q) {
    const bool self = q == rank;
    if ((self ? (long long)pk[q].size() : rcnt[q]) == 0) continue;
    const unsigned char *cur = self ? pk[q].data() : hr.data() + roff[q] * sizeof(Rec);
    long long hdr[3];
    cur = get(cur, hdr, 3);
    const long long a = hdr[0], m = hdr[1], e = hdr[2];
    if (a != next || a + m > lo2 + n2) {
      diter_set_err(ctx, "di_rebalance: pieces do not tile the new range (rank %d, piece %lld+%lld)", rank, a, m);
      return DI_ERR_STATE;
    }
    std::vector<long long> deg(m);
    cur = get(cur, deg.data(), m);
    const long long i0 = a - lo2, e_base = (long long)ri2.size();
    for (long long i = 0; i < m; ++i) cp2[i0 + i + 1] = cp2[i0 + i] + deg[i];
    if (cp2[i0 + m] - cp2[i0] != e || cp2[i0] != e_base) { diter_set_err(ctx, "di_rebalance: corrupt piece"); return DI_ERR_STATE; }
    ri2.resize(e_base + e);
    cur = get(cur, ri2.data() + e_base, e);
    if (ctx->vals) { vv2.resize(e_base + e); cur = get(cur, vv2.data() + e_base, e); }
    cur = get(cur, F2.data() + i0, m);
    cur = get(cur, H2.data() + i0, m);
    if (ctx->d_b) cur = get(cur, B2.data() + i0, m);
    next = a + m;
  }
  if (next != lo2 + n2) { diter_set_err(ctx, "di_rebalance: new range not covered"); return DI_ERR_STATE; }
  // rebuild on the new range with the same fabric
  di_ctx *nc = new (std::nothrow) di_ctx();
  if (!nc) { diter_set_err(ctx, "host OOM"); return DI_ERR_OOM; }
  nc->n_rows = ctx->n_rows;
  nc->n_local = n2;
  nc->nnz_local = cp2[n2];
  nc->lo = lo2;
  nc->d = ctx->d;
  nc->rank = rank;
  nc->world = W;
  nc->dist = new DistState();
  nc->dist->fabric = std::move(ds->fabric);
  nc->dist->bounds.assign(nb, nb + W + 1);
  di_options o = ctx->opt;
  o.device = ctx->device;
  st = dist_build(nc, reinterpret_cast<const int64_t *>(cp2.data()), ri2.empty() ? nullptr : ri2.data(), ctx->vals ? vv2.data() : nullptr,
                  ctx->d_b ? B2.data() : nullptr, &o);
  if (st != DI_OK) {
    ds->fabric = std::move(nc->dist->fabric);   // the old context stays usable
    diter_set_err(ctx, "di_rebalance: rebuild failed: %s", nc->err.c_str());
    di_destroy(nc);
    return st;
  }
  // restore the state: F, H (H_old = H: nothing is pending after the flush), the
  // control block (T, pass, counters; per-pass scratch cleared), the pass log
  CKD(cudaMemcpyAsync(nc->F, F2.data(), sizeof(double) * n2, cudaMemcpyHostToDevice, nc->stream));
  CKD(cudaMemcpyAsync(nc->H, H2.data(), sizeof(double) * n2, cudaMemcpyHostToDevice, nc->stream));
  if (nc->H_old) CKD(cudaMemcpyAsync(nc->H_old, H2.data(), sizeof(double) * n2, cudaMemcpyHostToDevice, nc->stream));
  Ctl c2 = c;
  c2.n_total = nc->ctl_init.n_total;
  c2.hub_packed = 0ull;
  std::memset(c2.tickets, 0, sizeof(c2.tickets));
  std::memset(c2.far_cnt, 0, sizeof(c2.far_cnt));
  CKD(cudaMemcpyAsync(nc->ctl, &c2, sizeof(Ctl), cudaMemcpyHostToDevice, nc->stream));
  CKD(cudaMemcpyAsync(nc->log, ctx->log, sizeof(di_pass_log) * std::min(nc->log_cap, ctx->log_cap),
                      cudaMemcpyDeviceToDevice, nc->stream));
  CKD(cudaStreamSynchronize(nc->stream));
  Ctl ci = ctx->ctl_init;                       // di_reset keeps the original T_0
  ci.n_total = nc->ctl_init.n_total;
  nc->ctl_init = ci;
  // the caller's stream and timing events stay with the handle
  cudaEventDestroy(nc->ev0);
  cudaEventDestroy(nc->ev1);
  cudaStreamDestroy(nc->stream);
  nc->stream = ctx->stream;
  nc->ev0 = ctx->ev0;
  nc->ev1 = ctx->ev1;
  ctx->stream = nullptr;
  ctx->ev0 = ctx->ev1 = nullptr;
  (void)diter_set_l2_window(nc);   // a cache hint: the stream now serves the rebuilt context's F
  nc->passes_done = ctx->passes_done;
  nc->edges = ctx->edges;
  nc->nodes = ctx->nodes;
  nc->dang = ctx->dang;
  nc->graph_launches = ctx->graph_launches;
  nc->kernel_launches += ctx->kernel_launches;
  nc->exchanged_bytes = ctx->exchanged_bytes + stot * (long long)sizeof(Rec);
  nc->exchanges = ctx->exchanges;
  nc->alg_bytes_exchange = ctx->alg_bytes_exchange;
  nc->residual = ctx->residual;
  nc->threshold = ctx->threshold;
  nc->run_ms = ctx->run_ms;
  nc->run_ms_total = ctx->run_ms_total;
  nc->kt_passes = ctx->kt_passes;
  for (int k = 0; k < 3; ++k) nc->kt_ms[k] = ctx->kt_ms[k];
  nc->remote_pushes = ctx->remote_pushes;
  nc->rebalances = ctx->rebalances + 1;
  std::swap(*ctx, *nc);
  di_destroy(nc);                               // the old device state (its fabric moved out)
  return DI_OK;
}

extern "C" di_status di_get_bounds(const di_ctx *ctx, int64_t *out) {
  if (!ctx || !out) { diter_set_err(nullptr, "NULL argument"); return DI_ERR_INVALID_ARG; }
  if (ctx->dist) {
    for (int k = 0; k <= ctx->world; ++k) out[k] = ctx->dist->bounds[k];
  } else {
    out[0] = 0;
    out[1] = ctx->n_rows;
  }
  return DI_OK;
}

extern "C" di_status di_get_unique_id(void *comm_id_out) {
  if (!comm_id_out) {
    diter_set_err(nullptr, "NULL argument");
    return DI_ERR_INVALID_ARG;
  }
#if DITER_WITH_NCCL
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    diter_set_err(nullptr, "ncclGetUniqueId failed: %s", ncclGetErrorString(r));
    return DI_ERR_NCCL;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(comm_id_out, &id, 128);
  return DI_OK;
#else
  diter_set_err(nullptr, "built without NCCL");
  return DI_ERR_UNSUPPORTED;
#endif
}

static const char kLoopTag[8] = {'D', 'I', 'L', 'O', 'O', 'P', '0', '1'};
static const char kShmTag[8] = {'D', 'I', 'S', 'H', 'M', '0', '0', '1'};

// Everything of a distributed context after its fabric exists (ds->bounds set,
// ctx->lo / n_local / nnz_local describing this rank's columns): device setup,
// column partition, outbox and exchange buffers, receiver structures.  Shared by
// di_create_dist and di_rebalance.  Collective.
static di_status dist_build_local(di_ctx *ctx, const int64_t *col_ptr_local, const int32_t *row_idx_local,
                                  const double *values_local, const double *b_local, const di_options *opt) {
  DistState *ds = ctx->dist;
  const int world = ctx->world, rank = ctx->rank;
  const long long n_global = ctx->n_rows, nl = ctx->n_local;
  di_status s = diter_setup(ctx, col_ptr_local, row_idx_local, values_local, b_local, opt);
  if (s != DI_OK) return s;
  if (ctx->opt.exchange_mode != DI_EXCHANGE_SYNC && ctx->opt.exchange_mode != DI_EXCHANGE_ASYNC &&
      ctx->opt.exchange_mode != DI_EXCHANGE_P2P) {
    diter_set_err(ctx, "exchange_mode must be DI_EXCHANGE_SYNC, _ASYNC or _P2P");
    return DI_ERR_INVALID_ARG;
  }
  if (ctx->opt.exchange_mode == DI_EXCHANGE_P2P &&
      (ctx->opt.remote_push != DI_REMOTE_INCREMENT || ctx->opt.adapt_rounds != 0 || world > kP2PMaxWorld)) {
    diter_set_err(ctx, "DI_EXCHANGE_P2P needs remote_push = DI_REMOTE_INCREMENT, adapt_rounds = 0 and <= %d ranks",
                  kP2PMaxWorld);
    return DI_ERR_INVALID_ARG;
  }
  // local rows first in every column (nloc), in place via a scratch copy
  {
    const long long n = ctx->n_local, nnz = ctx->nnz_local;
    int *ri2 = nullptr;
    double *v2 = nullptr;
    if (diter_alloc(ctx, (void **)&ctx->nloc, sizeof(int) * std::max(1LL, n)) != DI_OK ||
        cudaMalloc(&ri2, sizeof(int) * std::max(1LL, nnz)) != cudaSuccess ||
        (ctx->vals && cudaMalloc(&v2, sizeof(double) * std::max(1LL, nnz)) != cudaSuccess)) {
      if (ri2) cudaFree(ri2);
      diter_set_err(ctx, "cudaMalloc (column partition) failed");
      return (DI_ERR_OOM);
    }
    long long *d_b = nullptr;
    if (cudaMalloc(&d_b, sizeof(long long) * (world + 1)) != cudaSuccess) {
      cudaFree(ri2);
      if (v2) cudaFree(v2);
      diter_set_err(ctx, "cudaMalloc failed");
      return (DI_ERR_OOM);
    }
    cudaMemcpyAsync(d_b, ds->bounds.data(), sizeof(long long) * (world + 1), cudaMemcpyHostToDevice, ctx->stream);
    k_partition_columns<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->col_ptr, n, ctx->row_idx, ctx->vals, d_b,
                                                                   world, rank, ri2, v2, ctx->nloc);
    cudaMemcpyAsync(ctx->row_idx, ri2, sizeof(int) * nnz, cudaMemcpyDeviceToDevice, ctx->stream);
    if (v2) cudaMemcpyAsync(ctx->vals, v2, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, ctx->stream);
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    cudaFree(ri2);
    cudaFree(d_b);
    if (v2) cudaFree(v2);
    if (e != cudaSuccess) { diter_set_err(ctx, "column partition failed: %s", cudaGetErrorString(e)); return (DI_ERR_CUDA); }
    if (ctx->opt.remote_push == DI_REMOTE_INCREMENT || ctx->opt.remote_push == DI_REMOTE_RECEIVER) {
      if (diter_alloc(ctx, (void **)&ctx->H_old, sizeof(double) * std::max(1LL, n)) != DI_OK) {
        diter_set_err(ctx, "cudaMalloc (H_old) failed");
        return (DI_ERR_OOM);
      }
      cudaMemsetAsync(ctx->H_old, 0, sizeof(double) * std::max(1LL, n), ctx->stream);
    } else if (ctx->opt.remote_push != DI_REMOTE_PER_DIFFUSION) {
      diter_set_err(ctx, "remote_push must be DI_REMOTE_PER_DIFFUSION, DI_REMOTE_INCREMENT or DI_REMOTE_RECEIVER");
      return (DI_ERR_INVALID_ARG);
    }
  }
  // outbox, flags, exchange buffers (P2P: the compact outbox is built by p2p_setup,
  // and no bulk send/receive buffers exist)
  const bool p2p = ctx->opt.exchange_mode == DI_EXCHANGE_P2P;
  if (p2p) {
    ds->p2p.on = true;
    if (cudaMalloc(&ds->d_bounds, sizeof(long long) * (world + 1)) != cudaSuccess ||
        cudaMalloc(&ds->d_sums, sizeof(double) * (kSums + 3) + sizeof(long long) * world) != cudaSuccess) {
      diter_set_err(ctx, "cudaMalloc (exchange buffers) failed");
      return (DI_ERR_OOM);
    }
    cudaMemcpyAsync(ds->d_bounds, ds->bounds.data(), sizeof(long long) * (world + 1), cudaMemcpyHostToDevice, ctx->stream);
    ds->soff.assign(world, 0);
    ds->scnt.assign(world, 0);
    ds->roff.assign(world, 0);
    ds->rcnt.assign(world, 0);
  } else {
    const long long nb = (n_global + 31) >> 5;
    if (diter_alloc(ctx, (void **)&ctx->G, sizeof(double) * n_global) != DI_OK ||
        diter_alloc(ctx, (void **)&ctx->dflags, (size_t)nb) != DI_OK) {
      diter_set_err(ctx, "cudaMalloc (outbox) failed");
      return (DI_ERR_OOM);
    }
    // records to peer q: at most |Omega_q| (one per row); from peers: at most (K-1) |Omega_k|
    ds->soff.assign(world, 0);
    ds->scnt.assign(world, 0);
    ds->roff.assign(world, 0);
    ds->rcnt.assign(world, 0);
    long long cap = 0;
    for (int q = 0; q < world; ++q) {
      ds->soff[q] = cap;
      if (q != rank) cap += ds->bounds[q + 1] - ds->bounds[q];
    }
    ds->send_cap = std::max(1LL, cap);
    ds->recv_cap = std::max(1LL, (long long)(world - 1) * nl);
    if (cudaMalloc(&ds->send, sizeof(Rec) * ds->send_cap) != cudaSuccess ||
        cudaMalloc(&ds->recv, sizeof(Rec) * ds->recv_cap) != cudaSuccess ||
        cudaMalloc(&ds->d_bounds, sizeof(long long) * (world + 1)) != cudaSuccess ||
        cudaMalloc(&ds->d_scnt, sizeof(long long) * world) != cudaSuccess ||
        cudaMalloc(&ds->d_sums, sizeof(double) * (kSums + 3) + sizeof(long long) * world) != cudaSuccess) {
      diter_set_err(ctx, "cudaMalloc (exchange buffers) failed");
      return (DI_ERR_OOM);
    }
    cudaMemcpyAsync(ds->d_bounds, ds->bounds.data(), sizeof(long long) * (world + 1), cudaMemcpyHostToDevice, ctx->stream);
    s = diter_dist_reset(ctx);
    if (s != DI_OK) return (s);
  }
  return DI_OK;
}

// Local setup on every rank, then one agreement (a max over ranks of a failure
// flag) so that a rank whose input fails validation makes every rank fail together
// instead of leaving its peers waiting in a later collective; then the collective
// tail (T_0 = max over ranks |B_i| w_i / alpha, the paper key's in-degrees, the
// receiver structures).  The threshold schedule is global: SYNC applies the HYBRID
// rule to the global |S_p| and N; ASYNC per rank to |S_p^k| and |Omega_k|.
static di_status dist_build(di_ctx *ctx, const int64_t *col_ptr_local, const int32_t *row_idx_local,
                            const double *values_local, const double *b_local, const di_options *opt) {
  di_status s = dist_build_local(ctx, col_ptr_local, row_idx_local, values_local, b_local, opt);
  double any_fail = 0.0;
  const di_status sa = ctx->dist->fabric->host_max(ctx, s != DI_OK ? 1.0 : 0.0, &any_fail);
  if (s != DI_OK) return s;
  if (sa != DI_OK) return sa;
  if (any_fail > 0.0) {
    diter_set_err(ctx, "di_create_dist: a peer rank failed its local setup");
    return DI_ERR_STATE;
  }
  TRYD(diter_setup_finish(ctx));
  if (ctx->opt.remote_push == DI_REMOTE_RECEIVER) TRYD(setup_receiver(ctx));
  if (ctx->dist->p2p.on) TRYD(p2p_setup(ctx));
  if (ctx->opt.exchange_mode != DI_EXCHANGE_SYNC) {
    ctx->ctl_init.n_total = (double)ctx->n_local;
    CKD(cudaMemcpyAsync(ctx->ctl, &ctx->ctl_init, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
    CKD(cudaStreamSynchronize(ctx->stream));
  }
  return DI_OK;
}

extern "C" di_status di_create_dist(di_ctx **out, int32_t rank, int32_t world, const void *comm_id,
                                    const int64_t *bounds, int64_t n_global, const int64_t *col_ptr_local,
                                    const int32_t *row_idx_local, const double *values_local,
                                    const double *b_local, double d, const di_options *opt) {
  if (!out) { diter_set_err(nullptr, "out is NULL"); return DI_ERR_INVALID_ARG; }
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world || !comm_id || !bounds || !col_ptr_local || n_global < 1 ||
      n_global > 2147483647LL || !(d > 0.0 && d < 1.0)) {
    diter_set_err(nullptr, "di_create_dist: invalid arguments");
    return DI_ERR_INVALID_ARG;
  }
  if (bounds[0] != 0 || bounds[world] != n_global) {
    diter_set_err(nullptr, "bounds must start at 0 and end at n_global");
    return DI_ERR_INVALID_ARG;
  }
  for (int k = 0; k < world; ++k)
    if (bounds[k + 1] <= bounds[k]) {
      diter_set_err(nullptr, "bounds must be strictly increasing");
      return DI_ERR_INVALID_ARG;
    }
  const long long lo = bounds[rank], nl = bounds[rank + 1] - bounds[rank];
  const long long nnz = col_ptr_local[nl];
  if (col_ptr_local[0] != 0 || nnz < 0 || (nnz > 0 && !row_idx_local)) {
    diter_set_err(nullptr, "col_ptr_local[0] must be 0 and col_ptr_local[n_local] = nnz >= 0");
    return DI_ERR_INVALID_ARG;
  }
  di_ctx *ctx = new (std::nothrow) di_ctx();
  if (!ctx) { diter_set_err(nullptr, "host OOM"); return DI_ERR_OOM; }
  ctx->n_rows = n_global;
  ctx->n_local = nl;
  ctx->nnz_local = nnz;
  ctx->lo = lo;
  ctx->d = d;
  ctx->rank = rank;
  ctx->world = world;
  auto fail = [&](di_status s) {
    std::string e = ctx->err;
    di_destroy(ctx);
    diter_set_err(nullptr, "%s", e.c_str());
    return s;
  };
  DistState *ds = new DistState();
  ctx->dist = ds;
  ds->bounds.assign(bounds, bounds + world + 1);
  // device of this rank: options.device, else the current device
  {
    int dev = (opt && opt->device >= 0) ? opt->device : -1;
    if (dev < 0) cudaGetDevice(&dev);
    if (cudaSetDevice(dev) != cudaSuccess) { diter_set_err(ctx, "cudaSetDevice failed"); return fail(DI_ERR_CUDA); }
  }
  // fabric
  if (std::memcmp(comm_id, kShmTag, 8) == 0) {
    if (world > kP2PMaxWorld) { diter_set_err(ctx, "shared-memory fabric: at most %d ranks", kP2PMaxWorld); return fail(DI_ERR_INVALID_ARG); }
    const char *raw = static_cast<const char *>(comm_id) + 8;
    std::string nm = "/diter_" + std::string(raw, strnlen(raw, 120));
    const int fd = shm_open(nm.c_str(), O_CREAT | O_RDWR, 0600);
    if (fd < 0 || ftruncate(fd, sizeof(ShmGroup)) != 0) {
      if (fd >= 0) close(fd);
      diter_set_err(ctx, "shm_open/ftruncate %s failed", nm.c_str());
      return fail(DI_ERR_STATE);
    }
    void *p = mmap(nullptr, sizeof(ShmGroup), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) { diter_set_err(ctx, "mmap %s failed", nm.c_str()); return fail(DI_ERR_STATE); }
    ShmFabric *sf = new ShmFabric();
    sf->g = static_cast<ShmGroup *>(p);     // a fresh segment is zero-filled: counters at 0
    sf->name = nm;
    sf->rank = rank;
    sf->world = world;
    sf->g->world = world;
    ds->fabric.reset(sf);
  } else if (std::memcmp(comm_id, kLoopTag, 8) == 0) {
    std::string key(static_cast<const char *>(comm_id), 128);
    std::shared_ptr<LoopGroup> grp;
    {
      std::lock_guard<std::mutex> lk(g_loop_mu);
      auto it = g_loop_groups.find(key);
      if (it != g_loop_groups.end()) grp = it->second.lock();
      if (!grp) {
        grp = std::make_shared<LoopGroup>(world);
        g_loop_groups[key] = grp;
      }
    }
    if (grp->world != world) { diter_set_err(ctx, "loopback group size mismatch"); return fail(DI_ERR_INVALID_ARG); }
    ds->fabric.reset(new LoopFabric(grp, rank));
  } else {
#if DITER_WITH_NCCL
    NcclFabric *nf = new NcclFabric();
    ds->fabric.reset(nf);
    nf->rank = rank;
    nf->world = world;
    ncclUniqueId id;
    std::memcpy(&id, comm_id, 128);
    ncclResult_t r = ncclCommInitRank(&nf->comm, world, id, rank);
    if (r != ncclSuccess) {
      diter_set_err(ctx, "ncclCommInitRank failed: %s", ncclGetErrorString(r));
      return fail(DI_ERR_NCCL);
    }
    if (cudaMalloc(&nf->d_cnt, sizeof(long long) * 2 * world) != cudaSuccess) {
      diter_set_err(ctx, "cudaMalloc failed");
      return fail(DI_ERR_OOM);
    }
#else
    diter_set_err(ctx, "built without NCCL (use a loopback comm id)");
    return fail(DI_ERR_UNSUPPORTED);
#endif
  }
  di_status s = dist_build(ctx, col_ptr_local, row_idx_local, values_local, b_local, opt);
  if (s != DI_OK) {
    ds->fabric->abort();
    return fail(s);
  }
  *out = ctx;
  return DI_OK;
}
