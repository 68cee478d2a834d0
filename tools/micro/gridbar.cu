// Grid-barrier microbenchmark: cost of one barrier across a co-resident
// cooperative grid (148 SMs x B blocks), no work between barriers.
//   (a) cooperative_groups grid.sync()
//   (b) one counter: release atomic per block, relaxed spin, acquire fence
//   (c) two-level: blocks arrive on 16 sub-counters (separate lines), the last
//       arriver of each bumps a top counter, the last top arriver flips a flag
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

__device__ __forceinline__ void bar_flat(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
    unsigned old, cur;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(nb) : "memory");
    do { asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory"); }
    while (((cur ^ old) & 0x80000000u) == 0);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

// sub[k * 32] counters (128-byte apart), top, flag; gen = expected flag value
__device__ __forceinline__ void bar_tree(unsigned* w, unsigned gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int K = 16;
    const int k = blockIdx.x % K;
    const unsigned members = (gridDim.x - k + K - 1) / K;  // blocks with this k
    unsigned* sub = w + k * 32;
    unsigned* top = w + K * 32;
    unsigned* flag = w + K * 32 + 32;
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(sub) : "memory");
    if (old == gen * members + members - 1) {  // last of this group
      unsigned t;
      asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(top) : "memory");
      if (t == gen * K + K - 1)
        asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(flag), "r"(gen + 1) : "memory");
    }
    unsigned cur;
    do { asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(flag) : "memory"); }
    while (cur < gen + 1);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

template <int MODE>
__global__ void k_bar(unsigned* w, int iters, unsigned long long* t) {
  cg::grid_group grid = cg::this_grid();
  unsigned long long t0 = 0, t1;
  if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) grid.sync();
    else if (MODE == 1) bar_flat(w);
    else bar_tree(w, (unsigned)i);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    *t = t1 - t0;
  }
}

int main() {
  unsigned* w;
  unsigned long long* t;
  cudaMalloc(&w, 64 * 1024);
  cudaMalloc(&t, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2000;
  for (int bps : {1, 2, 3}) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(w, 0, 64 * 1024);
        int grid = sms * bps;
        int it = iters;
        void* args[] = {&w, &it, &t};
        void* k = mode == 0 ? (void*)k_bar<0> : mode == 1 ? (void*)k_bar<1> : (void*)k_bar<2>;
        cudaError_t e = cudaLaunchCooperativeKernel(k, grid, 256, args, 0, 0);
        cudaDeviceSynchronize();
        unsigned long long h = 0;
        cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
        if (rep == 1)
          printf("blocks %4d mode %d (%s): %.3f us per barrier %s\n", grid, mode,
                 mode == 0 ? "cg grid.sync" : mode == 1 ? "flat counter" : "two-level",
                 h * 1e-3 / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
