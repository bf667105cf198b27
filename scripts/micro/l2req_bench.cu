// Microbenchmark: what competes with fp64 REDs for the SM's memory pipe on B200?
//   mix A: R REDs (random, L2-resident 8 MB) + S warp shuffles per iteration
//   mix B: REDs + shared-memory fp64 atomic adds (CAS loop) in a given ratio
//   mix C: REDs + coalesced 4-byte loads (the row-index stream)
// Reports G RED lanes/s (and G smem adds/s) for each mix.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL; z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL; return z ^ (z >> 31);
}
constexpr int kR = 8;
template <int S>
__global__ void __launch_bounds__(256, 3) k_red_shfl(double *F, unsigned mask, int iters, int *sink) {
  unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long h = mix(tid);
  int acc = 0;
  for (int k = 0; k < iters; ++k) {
    h = mix(h);
    int v = (int)h;
#pragma unroll
    for (int s = 0; s < S; ++s) v += __shfl_sync(0xffffffffu, v, (v + s) & 31);
    acc += v;
#pragma unroll
    for (int r = 0; r < kR; ++r) atomicAdd(F + ((unsigned)(h >> (4 * r)) & mask), 1.0);
  }
  if (acc == 0x7fffffff) *sink = acc;
}
// per iteration: kR pushes, of which SM go to shared memory and kR - SM to L2
template <int SM>
__global__ void __launch_bounds__(256, 3) k_red_smem(double *F, unsigned mask, int iters, double *out) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0;
  __syncthreads();
  unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long h = mix(tid);
  for (int k = 0; k < iters; ++k) {
    h = mix(h);
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const unsigned a = (unsigned)(h >> (4 * r));
      if (r < SM) atomicAdd(s + (a & 4095u), 1.0);
      else atomicAdd(F + (a & mask), 1.0);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}
// per iteration: kR REDs + L coalesced int loads per lane
template <int L>
__global__ void __launch_bounds__(256, 3) k_red_ldg(double *F, unsigned mask, const int *__restrict__ idx, unsigned imask,
                                                    int iters, int *sink) {
  unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long h = mix(tid);
  int acc = 0;
  unsigned pos = (tid / 32) * 4096u + (tid & 31);
  for (int k = 0; k < iters; ++k) {
    h = mix(h);
#pragma unroll
    for (int l = 0; l < L; ++l) acc += __ldcs(idx + ((pos + 32 * l) & imask));
    pos += 32 * L;
#pragma unroll
    for (int r = 0; r < kR; ++r) atomicAdd(F + ((unsigned)(h >> (4 * r)) & mask), 1.0);
  }
  if (acc == 0x7fffffff) *sink = acc;
}
template <class Fn>
float timeit(Fn fn) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  fn(); cudaDeviceSynchronize();
  cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  const unsigned mask = (1u << 20) - 1;          // 8 MB of doubles: L2 resident
  double *F; double *out; int *sink; int *idx;
  const unsigned ilen = 1u << 28;                // 1 GB of ints: streams from HBM
  cudaMalloc(&F, (size_t)(mask + 1) * 8); cudaMalloc(&out, 1 << 20); cudaMalloc(&sink, 4); cudaMalloc(&idx, (size_t)ilen * 4);
  cudaMemset(F, 0, (size_t)(mask + 1) * 8); cudaMemset(idx, 0, (size_t)ilen * 4);
  const int blocks = 148 * 3, threads = 256, iters = 2048;
  const double pushes = (double)blocks * threads * iters * kR;
#define RUN_A(S) { float ms = timeit([&] { k_red_shfl<S><<<blocks, threads>>>(F, mask, iters, sink); }); \
    printf("A: %d REDs + %2d SHFL per iteration: %.1f G RED lanes/s\n", kR, S, pushes / ms / 1e6); }
  RUN_A(0) RUN_A(8) RUN_A(16) RUN_A(32) RUN_A(64)
#define RUN_B(SM) { float ms = timeit([&] { k_red_smem<SM><<<blocks, threads>>>(F, mask, iters, out); }); \
    printf("B: %d of %d pushes to shared memory: %.1f G pushes/s total (%.1f G RED lanes/s + %.1f G smem adds/s)\n", SM, kR, \
           pushes / ms / 1e6, pushes * (kR - SM) / kR / ms / 1e6, pushes * SM / kR / ms / 1e6); }
  RUN_B(0) RUN_B(1) RUN_B(2) RUN_B(4) RUN_B(6) RUN_B(8)
#define RUN_C(L) { float ms = timeit([&] { k_red_ldg<L><<<blocks, threads>>>(F, mask, idx, ilen - 1, iters, sink); }); \
    printf("C: %d REDs + %d coalesced 4-byte loads per lane per iteration: %.1f G RED lanes/s, %.2f TB/s of loads\n", kR, L, \
           pushes / ms / 1e6, (double)blocks * threads * iters * L * 4 / ms / 1e9); }
  RUN_C(0) RUN_C(1) RUN_C(2) RUN_C(4) RUN_C(8)
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
