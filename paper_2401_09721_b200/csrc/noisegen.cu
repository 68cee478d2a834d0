// add_gaussian_noise on the device (reference
// cloud.py:111-123): colours + N(0, sigma^2) clipped to [0, 255], drawing
// exactly numpy's variates -- Generator(Philox(seed)).normal(0, sigma, (N, 3)).
//
// numpy's stream (numpy/random/src/philox/philox.h, distributions.c):
//   draw p = Philox4x64-10(counter0 + 1 + p / 4, key)[p % 4]
//   random_standard_normal, 256-level ziggurat, one attempt at draw p:
//     r = draw p; idx = r & 255; sign = (r >> 8) & 1; rabs = (r >> 9) & (2^52 - 1)
//     x = +-rabs * wi[idx]; accept if rabs < ki[idx]                (1 draw)
//     idx == 0: exponential tail, pairs of uniforms until accepted  (1 + 2k)
//     else wedge: uniform u = draw p+1; accept if
//          (fi[idx-1] - fi[idx]) u + fi[idx] < exp(-x^2 / 2), else retry (2)
//
// An attempt consumes a data-dependent number of draws, so variate k's
// position in the stream depends on every earlier rejection.  Three kernels:
//   k_zig_chunks  the stream is cut into chunks of kZigL attempt positions;
//                 for every possible entry offset s < kZigK (a previous
//                 chunk's last attempt may spill s draws into this one) the
//                 chunk is run and (exit offset, variates emitted) recorded
//   k_zig_scan    one block composes those chunk maps in order from entry 0
//                 (Hillis-Steele over the maps), giving every chunk its true
//                 entry offset and output index
//   k_zig_emit    each chunk re-runs from its true entry and writes
//                 clip(c + (0 + sigma z), 0, 255) for its variates
// An exit offset >= kZigK (a tail loop of >= 8 pairs at a chunk edge) or a
// stream too short for 3N variates is reported; the host then retries with
// the sequential kernel k_zig_serial.
#include <algorithm>
#include <cmath>
#include <string>

#include "device_util.cuh"
#include "fgbd_internal.cuh"
#include "ziggurat_tables.cuh"

namespace fgbd {

constexpr int kZigL = 256;  // attempt positions per chunk
constexpr int kZigK = 16;   // entry offsets tracked per chunk
constexpr int kZigScanThreads = 512;
constexpr double kZigR = 3.6541528853610087963519472518;     // ziggurat_nor_r
constexpr double kZigInvR = 0.27366123732975827203338247596;  // ziggurat_nor_inv_r

struct PhiloxKey {
  unsigned long long k0, k1;
  unsigned long long c0, c1, c2, c3;  // numpy's counter before the first block
};

__device__ __forceinline__ void philox4x64_10(unsigned long long c[4], unsigned long long k0,
                                              unsigned long long k1) {
  const unsigned long long M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    const unsigned long long hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    const unsigned long long hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    const unsigned long long n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

// draws of one Philox stream, read at increasing (mostly consecutive)
// positions; the current 4-draw block is cached
struct Stream {
  PhiloxKey key;
  long long blk = -1;
  unsigned long long v[4];
  __device__ explicit Stream(const PhiloxKey& k) : key(k) {}
  __device__ unsigned long long at(long long p) {
    const long long b = p >> 2;
    if (b != blk) {
      // counter = c + 1 + b, 256-bit
      unsigned long long c[4] = {key.c0, key.c1, key.c2, key.c3};
      const unsigned long long add = (unsigned long long)b + 1ull;
      c[0] += add;
      unsigned long long carry = c[0] < add;
      for (int i = 1; i < 4; ++i) {
        c[i] += carry;
        carry = carry && c[i] == 0;
      }
      philox4x64_10(c, key.k0, key.k1);
      v[0] = c[0];
      v[1] = c[1];
      v[2] = c[2];
      v[3] = c[3];
      blk = b;
    }
    return v[p & 3];
  }
  __device__ double uniform(long long p) { return (double)(at(p) >> 11) * (1.0 / 9007199254740992.0); }
};

// log1p(x) exactly as the host libm numpy calls (glibc 2.39, x86-64): the
// fdlibm algorithm (k / f reduction, s = f / (2 + f), R(z = s^2)) with the
// polynomial evaluated in Estrin form with fused multiply-adds,
//   R = fma(z4, R3, fma(z, Lp1, z2 R2)) + z6 R4 (fused), Rj = fma(z, Lp, Lp'),
// everything else in separately rounded operations.  This operation order
// was identified empirically: it reproduces glibc's log1p(-u) bit for bit on
// 400k random u in [0, 1) (tools/ and tests/test_noisegen.py keep the
// restatement), where CUDA's own log1p differs from glibc in ~7% of cases
// (and is never used here: the tail variate is the log's value itself).
__device__ double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const int hx = (int)(__double_as_longlong(x) >> 32);
  const int ax = hx & 0x7fffffff;
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : NAN;
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      return __dsub_rn(x, __dmul_rn(__dmul_rn(x, x), 0.5));
    }
    if (hx > 0 || hx <= (int)0xbfd2bec3) {
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return __dadd_rn(x, x);
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = __dadd_rn(1.0, x);
      hu = (int)(__double_as_longlong(u) >> 32);
      k = (hu >> 20) - 1023;
      c = k > 0 ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
      c = __ddiv_rn(c, u);
    } else {
      u = x;
      hu = (int)(__double_as_longlong(u) >> 32);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    const long long lo = __double_as_longlong(u) & 0xffffffffLL;
    if (hu < 0x6a09e) {
      u = __longlong_as_double(((long long)(hu | 0x3ff00000) << 32) | lo);
    } else {
      k += 1;
      u = __longlong_as_double(((long long)(hu | 0x3fe00000) << 32) | lo);
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double hfsq = __dmul_rn(__dmul_rn(0.5, f), f);
  const double kd = (double)k;
  if (hu == 0) {  // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = __dadd_rn(c, __dmul_rn(kd, ln2_lo));
      return __dadd_rn(__dmul_rn(kd, ln2_hi), c);
    }
    const double R = __dmul_rn(hfsq, __dsub_rn(1.0, __dmul_rn(0.66666666666666666, f)));
    if (k == 0) return __dsub_rn(f, R);
    return __dsub_rn(__dmul_rn(kd, ln2_hi),
                     __dsub_rn(__dsub_rn(R, __dadd_rn(__dmul_rn(kd, ln2_lo), c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double z = __dmul_rn(s, s);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z4, z2);
  const double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
  double R = __fma_rn(z, Lp1, __dmul_rn(z2, R2));
  R = __fma_rn(z4, R3, R);
  R = __fma_rn(z6, R4, R);
  const double t = __dmul_rn(s, __dadd_rn(hfsq, R));
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, t));
  return __dsub_rn(__dmul_rn(kd, ln2_hi),
                   __dsub_rn(__dsub_rn(hfsq, __dadd_rn(t, __dadd_rn(__dmul_rn(kd, ln2_lo), c))), f));
}

// One ziggurat attempt starting at draw p: returns the next attempt's
// position; *emit / *z are set when the attempt yields a variate.
__device__ __forceinline__ long long zig_attempt(Stream& st, long long p, bool* emit, double* z) {
  unsigned long long r = st.at(p);
  const int idx = (int)(r & 0xff);
  r >>= 8;
  const bool neg = r & 1ull;
  const unsigned long long rabs = (r >> 1) & 0x000fffffffffffffull;
  double x = __dmul_rn((double)rabs, kZigWi[idx]);
  if (neg) x = -x;
  if (rabs < kZigKi[idx]) {
    *emit = true;
    *z = x;
    return p + 1;
  }
  if (idx == 0) {
    long long q = p + 1;
    for (;;) {
      const double xx = __dmul_rn(-kZigInvR, glibc_log1p(-st.uniform(q)));
      const double yy = -glibc_log1p(-st.uniform(q + 1));
      q += 2;
      if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
        *emit = true;
        *z = ((rabs >> 8) & 1ull) ? -__dadd_rn(kZigR, xx) : __dadd_rn(kZigR, xx);
        return q;
      }
    }
  }
  const double u = st.uniform(p + 1);
  const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(kZigFi[idx - 1], kZigFi[idx]), u), kZigFi[idx]);
  *emit = lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x));
  *z = x;
  return p + 2;
}

// map entry [chunk][entry offset]: exit offset (bits 0-7, 255 = overflow) |
// variates (bits 8-31); one thread per (chunk, entry offset)
__global__ void __launch_bounds__(kBlock) k_zig_chunks(PhiloxKey key, int64_t nchunks,
                                                       uint32_t* __restrict__ maps) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nchunks * kZigK) return;
  const int64_t c = g / kZigK;
  const int s = (int)(g % kZigK);
  Stream st(key);
  const long long lo = c * kZigL, hi = lo + kZigL;
  long long p = lo + s;
  uint32_t cnt = 0;
  while (p < hi) {
    bool emit = false;
    double z;
    p = zig_attempt(st, p, &emit, &z);
    cnt += emit;
  }
  const long long ex = p - hi;
  maps[g] = (ex < kZigK ? (uint32_t)ex : 255u) | (cnt << 8);
}

// Compose the chunk maps from entry 0: entry[c] / offset[c] for every chunk.
// ctl[0] = total variates, ctl[1] = 1 if a map overflowed on the true path.
__global__ void __launch_bounds__(kZigScanThreads) k_zig_scan(const uint32_t* __restrict__ maps,
                                                              int64_t nchunks,
                                                              uint8_t* __restrict__ entry,
                                                              int64_t* __restrict__ offset,
                                                              long long* __restrict__ ctl) {
  __shared__ uint8_t s_ex[kZigScanThreads][kZigK];
  __shared__ uint32_t s_ct[kZigScanThreads][kZigK];
  const int t = threadIdx.x;
  const int64_t per = (nchunks + kZigScanThreads - 1) / kZigScanThreads;
  const int64_t c0 = min(nchunks, t * per), c1 = min(nchunks, c0 + per);
  // this thread's chunks composed: state s -> (exit, count); 255 = overflow
  uint8_t ex[kZigK];
  uint32_t ct[kZigK];
  for (int s = 0; s < kZigK; ++s) {
    int e = s;
    uint32_t n = 0;
    for (int64_t c = c0; c < c1 && e != 255; ++c) {
      const uint32_t m = maps[c * kZigK + e];
      n += m >> 8;
      e = (int)(m & 0xff);
    }
    ex[s] = (uint8_t)e;
    ct[s] = n;
  }
  for (int s = 0; s < kZigK; ++s) {
    s_ex[t][s] = ex[s];
    s_ct[t][s] = ct[s];
  }
  __syncthreads();
  // inclusive scan of the maps: M_t <- M_t o M_{t-d} (M_{t-d} applied first)
  for (int d = 1; d < kZigScanThreads; d <<= 1) {
    uint8_t nex[kZigK];
    uint32_t nct[kZigK];
    const bool has = t >= d;
    for (int s = 0; s < kZigK; ++s) {
      if (!has) {
        nex[s] = s_ex[t][s];
        nct[s] = s_ct[t][s];
        continue;
      }
      const int mid = s_ex[t - d][s];
      if (mid == 255) {
        nex[s] = 255;
        nct[s] = 0;
      } else {
        nex[s] = s_ex[t][mid];
        nct[s] = s_ct[t - d][s] + s_ct[t][mid];
      }
    }
    __syncthreads();
    for (int s = 0; s < kZigK; ++s) {
      s_ex[t][s] = nex[s];
      s_ct[t][s] = nct[s];
    }
    __syncthreads();
  }
  // exclusive prefix from entry 0, then walk this thread's chunks
  int e = 0;
  long long off = 0;
  if (t > 0) {
    e = s_ex[t - 1][0];
    off = s_ct[t - 1][0];
  }
  for (int64_t c = c0; c < c1; ++c) {
    if (e == 255) {
      ctl[1] = 1;
      entry[c] = 0;
      offset[c] = -1;
      continue;
    }
    entry[c] = (uint8_t)e;
    offset[c] = off;
    const uint32_t m = maps[c * kZigK + e];
    off += m >> 8;
    e = (int)(m & 0xff);
  }
  if (t == kZigScanThreads - 1) {
    ctl[0] = off;
    if (e == 255) ctl[1] = 1;
  }
}

__device__ __forceinline__ double noisy_value(double c, double sigma, double z) {
  const double v = __dadd_rn(c, __dadd_rn(0.0, __dmul_rn(sigma, z)));  // loc + scale * z
  return fmin(fmax(v, 0.0), 255.0);
}

__global__ void __launch_bounds__(kBlock) k_zig_emit(PhiloxKey key, int64_t nchunks,
                                                     const uint8_t* __restrict__ entry,
                                                     const int64_t* __restrict__ offset,
                                                     const double* __restrict__ in, int64_t count,
                                                     double sigma, double* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  int64_t k = offset[c];
  if (k < 0 || k >= count) return;
  Stream st(key);
  const long long lo = c * kZigL, hi = lo + kZigL;
  long long p = lo + entry[c];
  while (p < hi && k < count) {
    bool emit = false;
    double z;
    p = zig_attempt(st, p, &emit, &z);
    if (emit) {
      out[k] = noisy_value(in[k], sigma, z);
      ++k;
    }
  }
}

// fallback: the whole stream in one thread (never needed in practice)
__global__ void k_zig_serial(PhiloxKey key, const double* __restrict__ in, int64_t count,
                             double sigma, double* __restrict__ out) {
  Stream st(key);
  long long p = 0;
  for (int64_t k = 0; k < count;) {
    bool emit = false;
    double z;
    p = zig_attempt(st, p, &emit, &z);
    if (emit) {
      out[k] = noisy_value(in[k], sigma, z);
      ++k;
    }
  }
}

}  // namespace fgbd

using namespace fgbd;

extern "C" {

int32_t fgbd_gaussian_noise(fgbd_ctx* ctx, const double* colors, int64_t count, double sigma,
                            const uint64_t key[2], const uint64_t counter[4], double* out,
                            uint32_t flags) {
  if (!ctx || !key || !counter || !out) return set_error(ctx, FGBD_E_ARG, "null argument");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  if (!(sigma >= 0.0))
    return set_error(ctx, FGBD_E_CLOUD, "sigma must be >= 0, got " + std::to_string(sigma));
  if (count < 1) return FGBD_OK;
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  PhiloxKey pk{key[0], key[1], counter[0], counter[1], counter[2], counter[3]};
  // stream long enough for `count` variates: ~0.3% of attempts reject
  int64_t positions = count + count / 32 + 4 * kZigL;
  for (int attempt = 0; attempt < 3; ++attempt, positions *= 2) {
    const int64_t nchunks = (positions + kZigL - 1) / kZigL;
    const size_t arr = (((size_t)count * 8) + 255) & ~size_t(255);
    const size_t maps_b = (((size_t)nchunks * kZigK * 4) + 255) & ~size_t(255);
    const size_t off_b = (((size_t)nchunks * 8) + 255) & ~size_t(255);
    const size_t ent_b = ((size_t)nchunks + 255) & ~size_t(255);
    const size_t need = (dev ? 0 : 2 * arr) + maps_b + off_b + ent_b + 256;
    if (ctx->aux_bytes < need) {
      if (ctx->aux) cudaFree(ctx->aux);
      ctx->aux = nullptr;
      ctx->aux_bytes = 0;
      FGBD_CUDA(ctx, cudaMalloc(&ctx->aux, need));
      ctx->aux_bytes = need;
    }
    ctx->knn_n = -1;  // aux is shared with the kNN graph
    char* s = (char*)ctx->aux;
    const double* d_in = colors;
    double* d_out = out;
    if (!dev) {
      FGBD_CUDA(ctx, cudaMemcpyAsync(s, colors, count * 8, cudaMemcpyHostToDevice, ctx->stream));
      d_in = (const double*)s;
      d_out = (double*)(s + arr);
      s += 2 * arr;
    }
    uint32_t* d_maps = (uint32_t*)s;
    int64_t* d_off = (int64_t*)(s + maps_b);
    uint8_t* d_ent = (uint8_t*)(s + maps_b + off_b);
    long long* d_ctl = (long long*)(s + maps_b + off_b + ent_b);
    FGBD_CUDA(ctx, cudaMemsetAsync(d_ctl, 0, 16, ctx->stream));
    const int grid = (int)((nchunks + kBlock - 1) / kBlock);
    k_zig_chunks<<<(int)((nchunks * kZigK + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(
        pk, nchunks, d_maps);
    FGBD_LAUNCH(ctx);
    k_zig_scan<<<1, kZigScanThreads, 0, ctx->stream>>>(d_maps, nchunks, d_ent, d_off, d_ctl);
    FGBD_LAUNCH(ctx);
    long long h[2];
    FGBD_CUDA(ctx, cudaMemcpyAsync(h, d_ctl, 16, cudaMemcpyDeviceToHost, ctx->stream));
    FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    const bool ok = h[1] == 0 && h[0] >= count;
    if (ok) {
      k_zig_emit<<<grid, kBlock, 0, ctx->stream>>>(pk, nchunks, d_ent, d_off, d_in, count, sigma,
                                                   d_out);
      FGBD_LAUNCH(ctx);
    } else if (h[1] != 0 || attempt == 2) {
      k_zig_serial<<<1, 1, 0, ctx->stream>>>(pk, d_in, count, sigma, d_out);
      FGBD_LAUNCH(ctx);
    } else {
      continue;  // stream too short: twice the positions
    }
    if (!dev)
      FGBD_CUDA(ctx, cudaMemcpyAsync(out, d_out, count * 8, cudaMemcpyDeviceToHost, ctx->stream));
    FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return FGBD_OK;
  }
  return FGBD_OK;  // unreachable
}

}  // extern "C"
