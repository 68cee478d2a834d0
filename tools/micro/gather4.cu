// Microbenchmark: neighbour gathers of 32-byte signal rows by LDG.256 (one
// thread per row, six register-resident gathers -- k_lf_run's scheme) versus
// the TMA gather4 engine (cp.async.bulk.tensor.2d.tile::gather4: one
// instruction fetches four 32-byte rows into shared memory).  Lattice-like
// (+-1, +-k, +-k^2 rows) and random neighbour indices, 1M rows x 6 slots.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 gather4.cu -o gather4 -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>

constexpr int kSlots = 6;

__device__ __forceinline__ double4 ldg256(const double4* p) {
  double4 v;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

__global__ void __launch_bounds__(256, 3) k_ldg(const double4* __restrict__ in, const int* __restrict__ idx,
                                                 double4* __restrict__ out, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double4 g[kSlots];
#pragma unroll
    for (int s = 0; s < kSlots; ++s) g[s] = ldg256(in + idx[s * n + i]);
    double4 o = ldg256(in + i);
#pragma unroll
    for (int s = 0; s < kSlots; ++s) { o.x += g[s].x; o.y += g[s].y; o.z += g[s].z; }
    out[i] = o;
  }
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kWarps = 4;                    // warps per block
constexpr int kStageBytes = 32 * kSlots * 32;  // 32 rows x 6 slots x 32 B

__global__ void __launch_bounds__(kWarps * 32) k_g4(const __grid_constant__ CUtensorMap tmap,
                                                    const double4* __restrict__ in,
                                                    const int* __restrict__ idx,
                                                    double4* __restrict__ out, int n) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[kWarps][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* st0 = smem + warp * 2 * kStageBytes;
  if (lane == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[warp][b])));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
  const int ntiles = (n + 31) / 32;
  auto issue = [&](int tile, int b) {
    if (tile >= ntiles) return;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[warp][b])), "r"(kStageBytes) : "memory");
    __syncwarp();
    // 48 gather4 ops: op k -> slot k / 8, rows 4 (k % 8) .. +3 of the tile
    for (int k = lane; k < 48; k += 32) {
      const int s = k >> 3, q = k & 7;
      int r[4];
      for (int t = 0; t < 4; ++t) {
        const int row = tile * 32 + 4 * q + t;
        r[t] = row < n ? idx[s * n + row] : 0;
      }
      unsigned char* dst = st0 + b * kStageBytes + (s * 32 + 4 * q) * 32;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
          ::"r"(sa(dst)), "l"(&tmap), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(sa(&bar[warp][b]))
          : "memory");
    }
  };
  uint32_t phase[2] = {0, 0};
  int tile = gw, b = 0;
  issue(tile, 0);
  while (tile < ntiles) {
    issue(tile + nw, b ^ 1);
    // wait stage b
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
        ::"r"(sa(&bar[warp][b])), "r"(phase[b]) : "memory");
    phase[b] ^= 1;
    const int i = tile * 32 + lane;
    if (i < n) {
      const double4* S = reinterpret_cast<const double4*>(st0 + b * kStageBytes);
      double4 o = ldg256(in + i);
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        const double4 g = S[s * 32 + lane];
        o.x += g.x; o.y += g.y; o.z += g.z;
      }
      out[i] = o;
    }
    __syncwarp();
    tile += nw;
    b ^= 1;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int n = 1 << 20, k = 100;
  double4* in; double4* out; int* idx;
  cudaMalloc(&in, (size_t)n * 32); cudaMalloc(&out, (size_t)n * 32); cudaMalloc(&idx, (size_t)n * kSlots * 4);
  cudaMemset(in, 0, (size_t)n * 32);
  std::vector<int> h((size_t)n * kSlots);
  const int off[kSlots] = {-k * k, -k, -1, 1, k, k * k};
  std::mt19937 rng(1);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap tmap;
  cuuint64_t gdim[2] = {4, (cuuint64_t)n}, gstride[1] = {32};
  cuuint32_t box[2] = {4, 1}, estr[2] = {1, 1};
  CUresult cr = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, in, gdim, gstride, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("tensor map: %d\n", (int)cr);
  int sm = 0; cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  const int smem = kWarps * 2 * kStageBytes;
  cudaFuncSetAttribute(k_g4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_g4, kWarps * 32, smem);
  printf("gather4 blocks/SM %d (smem %d)\n", per_sm, smem);
  for (int pattern = 0; pattern < 2; ++pattern) {
    for (int i = 0; i < n; ++i)
      for (int s = 0; s < kSlots; ++s) {
        int j = pattern == 0 ? i + off[s] : (int)(rng() % n);
        if (j < 0 || j >= n) j = i;
        h[(size_t)s * n + i] = j;
      }
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float t_ldg = 0, t_g4 = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a); for (int r = 0; r < 20; ++r) k_ldg<<<sm * 3, 256>>>(in, idx, out, n); cudaEventRecord(b);
      cudaEventSynchronize(b); cudaEventElapsedTime(&t_ldg, a, b);
      cudaEventRecord(a); for (int r = 0; r < 20; ++r) k_g4<<<sm * per_sm, kWarps * 32, smem>>>(tmap, in, idx, out, n); cudaEventRecord(b);
      cudaEventSynchronize(b); cudaEventElapsedTime(&t_g4, a, b);
    }
    printf("%s: LDG %.2f us/pass, gather4 %.2f us/pass (err %s)\n", pattern == 0 ? "lattice" : "random",
           1e3 * t_ldg / 20, 1e3 * t_g4 / 20, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
