// Small device helpers: warp/block reductions, lane masks, last-block tickets.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fgbd {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Block-wide sum of NV doubles per thread; result valid in thread 0.
// Fixed shuffle tree + fixed warp order => deterministic.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* s_scratch /*[32*NV]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) s_scratch[warp * NV + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double acc = 0.0;
      for (int w = 0; w < nwarps; ++w) acc += s_scratch[w * NV + k];
      v[k] = acc;
    }
  }
  __syncthreads();
}

// "Last block done": every block calls this after publishing its partial;
// returns true (block-uniform) in exactly one block, after all partials are
// visible.  The caller resets *ticket to 0 when finished.
__device__ __forceinline__ bool last_block(unsigned int* ticket, bool* s_flag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned t = atomicAdd(ticket, 1u);
    *s_flag = (t == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (*s_flag) __threadfence();
  return *s_flag;
}

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

}  // namespace fgbd
