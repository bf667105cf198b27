// csc.cu -- K8: COO -> CSC on the GPU (setup path, integer, bit-exact).
//
// p_ij is the weight of edge j -> i, so column j of P holds the
// out-edges of j.  Keys (src << 32 | dst) are radix-sorted (CUB), adjacent
// duplicates dropped (BASELINE.json configs[2] "duplicate edges dropped"),
// the column histogram is scanned into col_ptr.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/diter.h"
#include "ctx.cuh"

namespace {

__global__ void k_make_keys(const int *src, const int *dst, long long m, unsigned long long *keys,
                            int n, unsigned *bad) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    const int s = src[e], t = dst[e];
    if (s < 0 || s >= n || t < 0 || t >= n) atomicAdd(bad, 1u);
    keys[e] = ((unsigned long long)(unsigned)s << 32) | (unsigned)t;
  }
}

// flag[e] = 1 iff key e differs from key e-1 (first of its run)
__global__ void k_unique_flags(const unsigned long long *keys, long long m, int *flag) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride)
    flag[e] = (e == 0 || keys[e] != keys[e - 1]) ? 1 : 0;
}

__global__ void k_scatter_unique(const unsigned long long *keys, const int *flag, const long long *pos,
                                 long long m, int *row_idx, unsigned long long *col_count) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    if (flag[e]) {
      const unsigned long long k = keys[e];
      row_idx[pos[e]] = (int)(unsigned)(k & 0xffffffffull);
      atomicAdd(&col_count[k >> 32], 1ull);
    }
  }
}

}  // namespace

#define CKC(call)                                                                          \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      diter_set_err(nullptr, "%s failed: %s", #call, cudaGetErrorString(e_));             \
      rc = (e_ == cudaErrorMemoryAllocation) ? DI_ERR_OOM : DI_ERR_CUDA;                   \
      goto done;                                                                           \
    }                                                                                      \
  } while (0)

extern "C" di_status di_csc_from_coo(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                                     int64_t *col_ptr, int32_t *row_idx, int64_t *nnz_out) {
  if (n < 1 || n > 2147483647LL || m < 0 || !col_ptr || (m > 0 && (!src || !dst || !row_idx)) || !nnz_out) {
    diter_set_err(nullptr, "di_csc_from_coo: invalid arguments");
    return DI_ERR_INVALID_ARG;
  }
  di_status rc = DI_OK;
  cudaStream_t st = nullptr;
  int *d_src = nullptr, *d_dst = nullptr, *d_flag = nullptr, *d_rows = nullptr;
  unsigned long long *d_keys = nullptr, *d_keys2 = nullptr, *d_cnt = nullptr;
  long long *d_pos = nullptr, *d_ptr = nullptr;
  unsigned *d_bad = nullptr;
  void *d_tmp = nullptr;
  size_t tmp_bytes = 0, t1 = 0, t2 = 0, t3 = 0;
  unsigned bad = 0;
  long long nnz = 0;
  const int blocks = 148 * 8, threads = 256;
  int end_bit = 32;  // keys are (src << 32 | dst): 32 dst bits + bits(n-1) src bits
  while (end_bit < 64 && (((unsigned long long)(n - 1)) >> (end_bit - 32)) != 0ull) ++end_bit;
  CKC(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CKC(cudaMalloc(&d_ptr, sizeof(long long) * (n + 1)));
  CKC(cudaMalloc(&d_cnt, sizeof(unsigned long long) * (n + 1)));
  CKC(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * (n + 1), st));
  if (m > 0) {
    CKC(cudaMalloc(&d_src, sizeof(int) * m));
    CKC(cudaMalloc(&d_dst, sizeof(int) * m));
    CKC(cudaMalloc(&d_keys, sizeof(unsigned long long) * m));
    CKC(cudaMalloc(&d_keys2, sizeof(unsigned long long) * m));
    CKC(cudaMalloc(&d_flag, sizeof(int) * m));
    CKC(cudaMalloc(&d_pos, sizeof(long long) * m));
    CKC(cudaMalloc(&d_bad, sizeof(unsigned)));
    CKC(cudaMemsetAsync(d_bad, 0, sizeof(unsigned), st));
    CKC(cudaMemcpyAsync(d_src, src, sizeof(int) * m, cudaMemcpyHostToDevice, st));
    CKC(cudaMemcpyAsync(d_dst, dst, sizeof(int) * m, cudaMemcpyHostToDevice, st));
    k_make_keys<<<blocks, threads, 0, st>>>(d_src, d_dst, m, d_keys, (int)n, d_bad);
    CKC(cudaMemcpyAsync(&bad, d_bad, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CKC(cudaStreamSynchronize(st));
    if (bad) {
      diter_set_err(nullptr, "di_csc_from_coo: %u endpoints out of range", bad);
      rc = DI_ERR_INVALID_ARG;
      goto done;
    }
    cudaFree(d_src); d_src = nullptr;
    cudaFree(d_dst); d_dst = nullptr;
    // sort keys on the bits that can be non-zero: 32 dst bits + ceil(log2 n) src bits
    CKC(cub::DeviceRadixSort::SortKeys(nullptr, t1, d_keys, d_keys2, (int64_t)m, 0, end_bit, st));
    CKC(cub::DeviceScan::ExclusiveSum(nullptr, t2, d_flag, d_pos, (int64_t)m, st));
    CKC(cub::DeviceScan::InclusiveSum(nullptr, t3, d_cnt, d_ptr + 1, (int64_t)n, st));
    tmp_bytes = t1 > t2 ? t1 : t2;
    if (t3 > tmp_bytes) tmp_bytes = t3;
    CKC(cudaMalloc(&d_tmp, tmp_bytes));
    CKC(cub::DeviceRadixSort::SortKeys(d_tmp, t1, d_keys, d_keys2, (int64_t)m, 0, end_bit, st));
    k_unique_flags<<<blocks, threads, 0, st>>>(d_keys2, m, d_flag);
    CKC(cub::DeviceScan::ExclusiveSum(d_tmp, t2, d_flag, d_pos, (int64_t)m, st));
    CKC(cudaMalloc(&d_rows, sizeof(int) * m));
    k_scatter_unique<<<blocks, threads, 0, st>>>(d_keys2, d_flag, d_pos, m, d_rows, d_cnt);
    CKC(cub::DeviceScan::InclusiveSum(d_tmp, t3, d_cnt, d_ptr + 1, (int64_t)n, st));
  }
  CKC(cudaMemsetAsync(d_ptr, 0, sizeof(long long), st));
  if (m == 0) CKC(cudaMemsetAsync(d_ptr, 0, sizeof(long long) * (n + 1), st));
  CKC(cudaMemcpyAsync(col_ptr, d_ptr, sizeof(long long) * (n + 1), cudaMemcpyDeviceToHost, st));
  CKC(cudaStreamSynchronize(st));
  nnz = col_ptr[n];
  if (nnz > 0) {
    CKC(cudaMemcpyAsync(row_idx, d_rows, sizeof(int) * nnz, cudaMemcpyDeviceToHost, st));
    CKC(cudaStreamSynchronize(st));
  }
  *nnz_out = nnz;
done:
  void *ptrs[] = {d_src, d_dst, d_flag, d_rows, d_keys, d_keys2, d_cnt, d_pos, d_ptr, d_bad, d_tmp};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  if (st) cudaStreamDestroy(st);
  return rc;
}
