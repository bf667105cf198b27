// common.cuh -- device helpers shared by the libditer kernels (sm_100a only).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libditer is built for sm_100a (B200) only"
#endif

namespace diter {

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fire-and-forget fp64 add in L2 (RED.E.ADD.F64.RN): the scatter of the
// diffusion F_j += p_ji * sent.
__device__ __forceinline__ void red_add(double *addr, double v) {
  atomicAdd(addr, v);  // result unused -> RED (no return trip, no ordering with loads)
}

}  // namespace diter
