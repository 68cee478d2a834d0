// Cost of a grid-wide barrier for a persistent cooperative grid (148 x 3 x 256):
// cooperative_groups grid.sync() vs a hand-rolled counter/generation barrier.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(256, 3) k_cg(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  int acc = 0;
  for (int i = 0; i < iters; ++i) { acc += i; g.sync(); }
  if (acc == -1) *sink = acc;
}

__device__ __forceinline__ void my_sync(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd((unsigned*)gen, 1u);
    } else {
      while (*gen == g0) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// two-level: blocks arrive on one of 32 group counters; each group's last
// block arrives on the root; release is one generation word.
__device__ __forceinline__ void tree_sync(unsigned* cnt, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g0 = *gen;
    const unsigned groups = 32, grp = blockIdx.x % groups;
    const unsigned members = nblocks / groups + (grp < nblocks % groups ? 1u : 0u);
    __threadfence();
    bool last = false;
    if (atomicAdd(&cnt[64 + grp * 32], 1u) == members - 1) {
      cnt[64 + grp * 32] = 0;
      if (atomicAdd(&cnt[0], 1u) == groups - 1) {
        cnt[0] = 0;
        __threadfence();
        atomicAdd((unsigned*)gen, 1u);
        last = true;
      }
    }
    if (!last) while (*gen == g0) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256, 3) k_tree(int iters, unsigned* bar, int* sink) {
  int acc = 0;
  for (int i = 0; i < iters; ++i) { acc += i; tree_sync(bar, bar + 32, gridDim.x); }
  if (acc == -1) *sink = acc;
}

__global__ void __launch_bounds__(256, 3) k_mine(int iters, unsigned* bar, int* sink) {
  int acc = 0;
  for (int i = 0; i < iters; ++i) { acc += i; my_sync(bar, bar + 32, gridDim.x); }
  if (acc == -1) *sink = acc;
}

int main() {
  int dev = 0, sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cg, 256, 0);
  const int grid = sms * 3;  // the persistent filter kernel's grid
  int* sink; unsigned* bar;
  cudaMalloc(&sink, 4); cudaMalloc(&bar, 8192); cudaMemset(bar, 0, 8192);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 2000;
  for (int rep = 0; rep < 3; ++rep) {
    void* args1[] = {&iters, &sink};
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_cg, grid, 256, args1, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    void* args2[] = {&iters, &bar, &sink};
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_mine, grid, 256, args2, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms2; cudaEventElapsedTime(&ms2, a, b);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_tree, grid, 256, args2, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms3; cudaEventElapsedTime(&ms3, a, b);
    printf("grid=%d  cg::grid.sync %.3f us   counter %.3f us   tree %.3f us  (%s)\n", grid,
           1e3 * ms / iters, 1e3 * ms2 / iters, 1e3 * ms3 / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
