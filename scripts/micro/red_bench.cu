// Microbenchmark: fp64 RED / gather throughput on B200 for the scatter roofline.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL; z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL; return z ^ (z >> 31);
}
// mode 0: random over [0,range); mode 1: local window +-1000 around a per-warp moving base
__global__ void k_red(double *F, long long range, long long ops_per_thread, int mode) {
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long h = mix(tid);
  long long base = (tid / 32) * 97 % range;
  for (long long k = 0; k < ops_per_thread; ++k) {
    h = mix(h + k);
    long long a;
    if (mode == 0) a = (long long)(h % (unsigned long long)range);
    else if (mode == 2) { a = (long long)((mix(tid / 32 * 1315423911ull + k) % (unsigned long long)(range / 32)) * 32 + (tid & 31)); }
    else { a = base + (long long)(h % 2001) - 1000; if (a < 0) a += range; if (a >= range) a -= range; base += 7; if (base >= range) base -= range; }
    atomicAdd(F + a, 1.0);
  }
}
__global__ void k_red_f32(float *F, long long range, long long ops_per_thread) {
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long h = mix(tid);
  for (long long k = 0; k < ops_per_thread; ++k) { h = mix(h + k); atomicAdd(F + (h % (unsigned long long)range), 1.0f); }
}
__global__ void k_gather(const double *F, long long range, long long ops_per_thread, double *out) {
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long h = mix(tid);
  double acc = 0;
  for (long long k = 0; k < ops_per_thread; k += 4) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { h = mix(h + k + u); v[u] = __ldg(F + (h % (unsigned long long)range)); }
    acc += v[0] + v[1] + v[2] + v[3];
  }
  if (acc == 12345.0) out[0] = acc;
}
__global__ void k_atoms(double *out, long long ops_per_thread, int words) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0;
  __syncthreads();
  unsigned long long h = mix(blockIdx.x * 1000 + threadIdx.x);
  for (long long k = 0; k < ops_per_thread; ++k) { h = mix(h + k); atomicAdd(s + (h % words), 1.0); }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}
int main() {
  const long long big = 100000000;  // 800 MB
  double *F; float *G; double *out;
  cudaMalloc(&F, big * 8); cudaMalloc(&G, big * 4); cudaMalloc(&out, 1 << 20);
  cudaMemset(F, 0, big * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = 148 * 8, threads = 256; const long long opt = 1024;
  const double ops = (double)blocks * threads * opt;
  long long ranges[] = {1 << 20, 1 << 23, 1 << 26, big};
  for (int mode = 0; mode < 3; ++mode)
    for (long long r : ranges) {
      k_red<<<blocks, threads>>>(F, r, 64, mode);
      cudaEventRecord(a); k_red<<<blocks, threads>>>(F, r, opt, mode); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("RED.F64 mode=%s range=%lld (%.1f MB): %.1f G ops/s\n", mode == 2 ? "warp-contiguous" : (mode ? "local" : "random"), r, r * 8 / 1e6, ops / ms / 1e6);
    }
  for (long long r : ranges) {
    cudaEventRecord(a); k_red_f32<<<blocks, threads>>>(G, r, opt); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("RED.F32 random range=%lld: %.1f G ops/s\n", r, ops / ms / 1e6);
  }
  for (long long r : ranges) {
    cudaEventRecord(a); k_gather<<<blocks, threads>>>(F, r, opt, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("LDG.F64 random gather range=%lld: %.1f G loads/s\n", r, ops / ms / 1e6);
  }
  for (int words : {32, 2048, 4096}) {
    cudaEventRecord(a); k_atoms<<<blocks, threads>>>(out, opt, words); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("ATOMS.F64 (smem) random over %d words: %.1f G ops/s\n", words, ops / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
