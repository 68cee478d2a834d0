// Data-model helpers on the device (reference
// cloud.py:89-140): coordinate quantisation and the PSNR error sum.
//
// k_axis_minmax  per-axis min / max of int64 or float64 coordinates (exact:
//                order-preserving integer images of the doubles, atomics)
// k_quantize     rint((c - lo) * scale) -> int64, the reference's operation
//                order (cloud.py:104-107); scale is computed on the host from
//                the exact extrema exactly as numpy does
// k_pairwise     sum of squared colour differences reproducing numpy's
//                pairwise summation (add.reduce over the flattened array):
//                the host plans the recursion's leaves (<= 128 values), one
//                thread sums each leaf with numpy's 8-accumulator pattern,
//                and the host adds the leaf sums back up the same tree -- so
//                psnr() is bit-identical to the reference's np.mean.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "device_util.cuh"
#include "fgbd_internal.cuh"

namespace fgbd {

// monotone map double -> signed 64-bit (total order for non-NaN values)
__device__ __forceinline__ long long ordered(double x) {
  const long long b = __double_as_longlong(x);
  return b >= 0 ? b : (b ^ 0x7fffffffffffffffLL);
}
static double unordered(long long o) {
  const long long b = o >= 0 ? o : (o ^ 0x7fffffffffffffffLL);
  double x;
  std::memcpy(&x, &b, 8);
  return x;
}

// mm[0..2] = min, mm[3..5] = max (int64 values or ordered doubles), mm[6] = NaN seen
__global__ void k_axis_minmax(const int64_t* __restrict__ ci, const double* __restrict__ cf,
                              int64_t n, long long* __restrict__ mm) {
  long long lo[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX};
  long long hi[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
  int nan = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      long long v;
      if (ci) {
        v = ci[3 * i + k];
      } else {
        const double x = cf[3 * i + k];
        nan |= x != x;
        v = ordered(x);
      }
      lo[k] = v < lo[k] ? v : lo[k];
      hi[k] = v > hi[k] ? v : hi[k];
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    for (int o = 16; o; o >>= 1) {
      const long long a = __shfl_xor_sync(0xffffffffu, lo[k], o);
      const long long b = __shfl_xor_sync(0xffffffffu, hi[k], o);
      lo[k] = a < lo[k] ? a : lo[k];
      hi[k] = b > hi[k] ? b : hi[k];
    }
  }
  nan = __any_sync(0xffffffffu, nan);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      atomicMin(&mm[k], lo[k]);
      atomicMax(&mm[3 + k], hi[k]);
    }
    if (nan) atomicOr((unsigned long long*)&mm[6], 1ull);
  }
}

__global__ void k_quantize(const int64_t* __restrict__ ci, const double* __restrict__ cf,
                           int64_t n, double3 lo, double3 scale, int64_t* __restrict__ out) {
  const double l[3] = {lo.x, lo.y, lo.z}, s[3] = {scale.x, scale.y, scale.z};
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < 3 * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e % 3);
    const double c = ci ? (double)ci[e] : cf[e];
    const double q = rint(__dmul_rn(__dsub_rn(c, l[k]), s[k]));
    // numpy float64 -> int64 cast (NaN / out of range: x86 gives INT64_MIN)
    out[e] = (q == q && q >= -9.2233720368547758e18 && q < 9.2233720368547758e18)
                 ? (int64_t)q : INT64_MIN;
  }
}

// one numpy pairwise leaf: n < 8 sequential from 0.0, else 8 accumulators
// strided by 8, combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the rest
__device__ __forceinline__ double sqdiff(const double* a, const double* b, int64_t i) {
  const double d = __dsub_rn(a[i], b[i]);
  return __dmul_rn(d, d);
}

__global__ void k_pairwise(const double* __restrict__ a, const double* __restrict__ b,
                           const int64_t* __restrict__ leaf_off, const int* __restrict__ leaf_len,
                           int nleaves, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nleaves) return;
  const int64_t o = leaf_off[t];
  const int n = leaf_len[t];
  double res;
  if (n < 8) {
    res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, sqdiff(a, b, o + i));
  } else {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = sqdiff(a, b, o + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], sqdiff(a, b, o + i + j));
    res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                    __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, sqdiff(a, b, o + i));
  }
  out[t] = res;
}

// numpy's pairwise recursion (leaves in left-to-right order)
static void plan_leaves(int64_t off, int64_t n, std::vector<int64_t>& lo, std::vector<int>& len) {
  if (n <= 128) {
    lo.push_back(off);
    len.push_back((int)n);
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  plan_leaves(off, n2, lo, len);
  plan_leaves(off + n2, n - n2, lo, len);
}

static double combine(int64_t n, const double* leaf, size_t& k) {
  if (n <= 128) return leaf[k++];
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  const double l = combine(n2, leaf, k);
  const double r = combine(n - n2, leaf, k);
  return l + r;
}

}  // namespace fgbd

using namespace fgbd;

extern "C" {

int32_t fgbd_quantize(fgbd_ctx* ctx, const int64_t* coords_int, const double* coords_float,
                      int64_t n, int32_t bits, int64_t* out, int32_t* passthrough,
                      uint32_t flags) {
  if (!ctx) return set_error(ctx, FGBD_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  if (bits < 1 || bits > 21)
    return set_error(ctx, FGBD_E_CLOUD, "bits must be in [1, 21], got " + std::to_string(bits));
  if (!coords_int == !coords_float) return set_error(ctx, FGBD_E_ARG, "one coordinate array");
  if (passthrough) *passthrough = 0;
  if (n < 1) return FGBD_OK;
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  const size_t bytes = (size_t)n * 24;
  // scratch: input copy | output | min/max words
  const size_t need = ((bytes + 255) & ~size_t(255)) * 2 + 64;
  if (ctx->aux_bytes < need) {
    if (ctx->aux) cudaFree(ctx->aux);
    ctx->aux = nullptr;
    ctx->aux_bytes = 0;
    FGBD_CUDA(ctx, cudaMalloc(&ctx->aux, need));
    ctx->aux_bytes = need;
  }
  ctx->knn_n = -1;  // aux is shared with the kNN graph
  char* a = (char*)ctx->aux;
  void* d_in = a;
  int64_t* d_out = (int64_t*)(a + ((bytes + 255) & ~size_t(255)));
  long long* d_mm = (long long*)(a + 2 * ((bytes + 255) & ~size_t(255)));
  const void* src = coords_int ? (const void*)coords_int : (const void*)coords_float;
  if (dev) {
    d_in = const_cast<void*>(src);
  } else {
    FGBD_CUDA(ctx, cudaMemcpyAsync(d_in, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  }
  const long long init[7] = {LLONG_MAX, LLONG_MAX, LLONG_MAX, LLONG_MIN, LLONG_MIN, LLONG_MIN, 0};
  FGBD_CUDA(ctx, cudaMemcpyAsync(d_mm, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + kBlock - 1) / kBlock,
                                                               ctx->num_sms * 4));
  const int64_t* ci = coords_int ? (const int64_t*)d_in : nullptr;
  const double* cf = coords_int ? nullptr : (const double*)d_in;
  k_axis_minmax<<<grid, kBlock, 0, ctx->stream>>>(ci, cf, n, d_mm);
  FGBD_LAUNCH(ctx);
  long long mm[7];
  FGBD_CUDA(ctx, cudaMemcpyAsync(mm, d_mm, sizeof(mm), cudaMemcpyDeviceToHost, ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    if (coords_int) {
      lo[k] = (double)mm[k];
      hi[k] = (double)mm[3 + k];
    } else {
      lo[k] = mm[6] ? NAN : unordered(mm[k]);
      hi[k] = mm[6] ? NAN : unordered(mm[3 + k]);
    }
  }
  // cloud.py:101-102: integer clouds already on the grid only change bit depth
  if (coords_int) {
    const long long mn = std::min({mm[0], mm[1], mm[2]}), mx = std::max({mm[3], mm[4], mm[5]});
    if (mn >= 0 && mx < (1LL << bits)) {
      if (passthrough) *passthrough = 1;
      return FGBD_OK;
    }
  }
  // cloud.py:103-106, in numpy's operation order
  const double top = (double)((1LL << bits) - 1);
  double sc[3];
  for (int k = 0; k < 3; ++k) {
    const double span = hi[k] - lo[k];
    sc[k] = span > 0 ? top / span : 0.0;
  }
  k_quantize<<<grid, kBlock, 0, ctx->stream>>>(ci, cf, n, make_double3(lo[0], lo[1], lo[2]),
                                               make_double3(sc[0], sc[1], sc[2]),
                                               dev ? out : d_out);
  FGBD_LAUNCH(ctx);
  if (!dev)
    FGBD_CUDA(ctx, cudaMemcpyAsync(out, d_out, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FGBD_OK;
}

int32_t fgbd_sq_error_sum(fgbd_ctx* ctx, const double* a, const double* b, int64_t count,
                          double* sum_out, uint32_t flags) {
  if (!ctx || !sum_out) return set_error(ctx, FGBD_E_ARG, "null argument");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  *sum_out = 0.0;
  if (count < 1) return FGBD_OK;
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  std::vector<int64_t> loff;
  std::vector<int> llen;
  plan_leaves(0, count, loff, llen);
  const int L = (int)loff.size();
  const size_t arr = (((size_t)count * 8) + 255) & ~size_t(255);
  const size_t need = (dev ? 0 : 2 * arr) + (size_t)L * (8 + 4 + 8) + 256;
  if (ctx->aux_bytes < need) {
    if (ctx->aux) cudaFree(ctx->aux);
    ctx->aux = nullptr;
    ctx->aux_bytes = 0;
    FGBD_CUDA(ctx, cudaMalloc(&ctx->aux, need));
    ctx->aux_bytes = need;
  }
  ctx->knn_n = -1;
  char* s = (char*)ctx->aux;
  const double* da = a;
  const double* db = b;
  if (!dev) {
    FGBD_CUDA(ctx, cudaMemcpyAsync(s, a, count * 8, cudaMemcpyHostToDevice, ctx->stream));
    FGBD_CUDA(ctx, cudaMemcpyAsync(s + arr, b, count * 8, cudaMemcpyHostToDevice, ctx->stream));
    da = (const double*)s;
    db = (const double*)(s + arr);
    s += 2 * arr;
  }
  int64_t* d_off = (int64_t*)s;
  double* d_sum = (double*)(s + (size_t)L * 8);
  int* d_len = (int*)(s + (size_t)L * 16);
  FGBD_CUDA(ctx, cudaMemcpyAsync(d_off, loff.data(), (size_t)L * 8, cudaMemcpyHostToDevice,
                                 ctx->stream));
  FGBD_CUDA(ctx, cudaMemcpyAsync(d_len, llen.data(), (size_t)L * 4, cudaMemcpyHostToDevice,
                                 ctx->stream));
  k_pairwise<<<(L + 127) / 128, 128, 0, ctx->stream>>>(da, db, d_off, d_len, L, d_sum);
  FGBD_LAUNCH(ctx);
  std::vector<double> leaf(L);
  FGBD_CUDA(ctx, cudaMemcpyAsync(leaf.data(), d_sum, (size_t)L * 8, cudaMemcpyDeviceToHost,
                                 ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  size_t k = 0;
  *sum_out = 0.0 + combine(count, leaf.data(), k);
  return FGBD_OK;
}

}  // extern "C"
