// PLY binary little-endian vertex records on the device (
// reference ply.py:134-287).
//
// k_ply_decode   packed records (any stride, x/y/z of any numeric PLY type,
//                red/green/blue uint8) -> coords int64 or float64 (N,3) and
//                colours float64 (N,3) -- ply.py:213-222 / _vertex_columns
// k_ply_encode   colours rounded half-up and clamped (ply.py:234-236) and
//                coordinates as uint32 (quantized) or float32, packed into
//                15-byte records -- byte-identical to ply.py:239-287
// fgbd_denoise_ply  raw body in -> decode into the context's staging ->
//                denoise -> encode -> raw body out: 15 B/pt each way over
//                PCIe instead of 48 + 24.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "device_util.cuh"
#include "fgbd_internal.cuh"

namespace fgbd {

// PLY scalar types (matching ply.py _PLY_DTYPES)
enum PlyType { PT_I1 = 0, PT_U1, PT_I2, PT_U2, PT_I4, PT_U4, PT_F4, PT_F8 };

struct PlyLayout {
  int stride;
  int off[6];   // x y z red green blue
  int type[6];
};

__device__ __forceinline__ double rd_num(const uint8_t* p, int t) {
  switch (t) {
    case PT_I1: return (double)*(const int8_t*)p;
    case PT_U1: return (double)*p;
    case PT_I2: { int16_t v; memcpy(&v, p, 2); return (double)v; }
    case PT_U2: { uint16_t v; memcpy(&v, p, 2); return (double)v; }
    case PT_I4: { int32_t v; memcpy(&v, p, 4); return (double)v; }
    case PT_U4: { uint32_t v; memcpy(&v, p, 4); return (double)v; }
    case PT_F4: { float v; memcpy(&v, p, 4); return (double)v; }
    default: { double v; memcpy(&v, p, 8); return v; }
  }
}

__device__ __forceinline__ long long rd_int(const uint8_t* p, int t) {
  switch (t) {
    case PT_I1: return *(const int8_t*)p;
    case PT_U1: return *p;
    case PT_I2: { int16_t v; memcpy(&v, p, 2); return v; }
    case PT_U2: { uint16_t v; memcpy(&v, p, 2); return v; }
    case PT_I4: { int32_t v; memcpy(&v, p, 4); return v; }
    default: { uint32_t v; memcpy(&v, p, 4); return v; }
  }
}

// int_coords: write int64 coords (all coordinate types integral), else float64
__global__ void __launch_bounds__(kBlock) k_ply_decode(const uint8_t* __restrict__ body, int64_t n,
                                                       PlyLayout L, int int_coords,
                                                       int64_t* __restrict__ ci,
                                                       double* __restrict__ cf,
                                                       double* __restrict__ colors,
                                                       unsigned int* __restrict__ flags) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool neg = false;
  long long mx = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint8_t* rec = body + i * L.stride;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (int_coords) {
        const long long v = rd_int(rec + L.off[k], L.type[k]);
        neg |= v < 0;
        mx = v > mx ? v : mx;
        ci[3 * i + k] = v;
      } else {
        cf[3 * i + k] = rd_num(rec + L.off[k], L.type[k]);
      }
      colors[3 * i + k] = (double)rec[L.off[3 + k]];
    }
  }
  if (neg) atomicOr(flags, 1u);
  // bit length of the largest coordinate (infer_bit_depth, cloud.py:83-86)
  const int bl = mx > 0 ? 64 - __clzll(mx) : 0;
  atomicMax(flags + 1, (unsigned)bl);
}

// 15-byte records: 3 x (uint32 | float32) + 3 x uint8
__global__ void __launch_bounds__(kBlock) k_ply_encode(const int64_t* __restrict__ ci,
                                                       const double* __restrict__ cf,
                                                       const double* __restrict__ colors,
                                                       int64_t n, int quantized,
                                                       uint8_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint8_t* rec = out + i * 15;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (quantized) {
        const uint32_t v = (uint32_t)ci[3 * i + k];
        memcpy(rec + 4 * k, &v, 4);
      } else {
        const float v = (float)cf[3 * i + k];
        memcpy(rec + 4 * k, &v, 4);
      }
      // round half up, clamp (ply.py:234-236)
      const double c = fmin(fmax(floor(colors[3 * i + k] + 0.5), 0.0), 255.0);
      rec[12 + k] = (uint8_t)c;
    }
  }
}

static int grid_of(fgbd_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + kBlock - 1) / kBlock, ctx->num_sms * 8));
}

}  // namespace fgbd

using namespace fgbd;

namespace {

// Context-owned staging for PLY records, grown on demand (never freed per
// call: cudaFree would serialise the device against other contexts' frames).
int ply_stage(fgbd_ctx* ctx, size_t need, uint8_t** out) {
  if (ctx->ply_stage_bytes < need) {
    if (ctx->ply_stage) cudaFree(ctx->ply_stage);
    ctx->ply_stage = nullptr;
    ctx->ply_stage_bytes = 0;
    FGBD_CUDA(ctx, cudaMalloc(&ctx->ply_stage, need));
    ctx->ply_stage_bytes = need;
  }
  *out = (uint8_t*)ctx->ply_stage;
  return FGBD_OK;
}

inline size_t al16(size_t b) { return (b + 15) & ~size_t(15); }

int make_layout(fgbd_ctx* ctx, int32_t stride, const int32_t* offsets, const int32_t* types,
                PlyLayout* L) {
  if (stride <= 0) return set_error(ctx, FGBD_E_ARG, "record stride must be positive");
  L->stride = stride;
  for (int k = 0; k < 6; ++k) {
    if (types[k] < PT_I1 || types[k] > PT_F8) return set_error(ctx, FGBD_E_ARG, "bad type code");
    if (k >= 3 && types[k] != PT_U1)
      return set_error(ctx, FGBD_E_CLOUD, "color properties must be 8-bit");
    static const int sz[8] = {1, 1, 2, 2, 4, 4, 4, 8};
    if (offsets[k] < 0 || offsets[k] + sz[types[k]] > stride)
      return set_error(ctx, FGBD_E_ARG, "property outside the record");
    L->off[k] = offsets[k];
    L->type[k] = types[k];
  }
  return FGBD_OK;
}

}  // namespace

extern "C" {

int32_t fgbd_ply_decode(fgbd_ctx* ctx, const uint8_t* body, int64_t n, int32_t stride,
                        const int32_t* offsets, const int32_t* types, int64_t* coords_int,
                        double* coords_float, double* colors, int32_t* bit_length,
                        uint32_t flags) {
  if (!ctx) return set_error(ctx, FGBD_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  PlyLayout L;
  int rc = make_layout(ctx, stride, offsets, types, &L);
  if (rc) return rc;
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  const int int_coords = coords_int != nullptr;
  if (n == 0) return FGBD_OK;
  const size_t body_bytes = (size_t)n * stride, out_bytes = (size_t)n * 3 * 8;
  uint8_t* d_body;
  if ((rc = ply_stage(ctx, al16(body_bytes) + 2 * out_bytes + 16, &d_body))) return rc;
  double* d_colors = (double*)(d_body + al16(body_bytes));
  void* d_coords = (void*)(d_colors + 3 * n);
  unsigned* d_flags = (unsigned*)((char*)d_coords + out_bytes);
  FGBD_CUDA(ctx, cudaMemsetAsync(d_flags, 0, 8, ctx->stream));
  FGBD_CUDA(ctx, cudaMemcpyAsync(d_body, body, body_bytes,
                                 dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                 ctx->stream));
  k_ply_decode<<<grid_of(ctx, n), kBlock, 0, ctx->stream>>>(
      d_body, n, L, int_coords, (int64_t*)d_coords, (double*)d_coords, d_colors, d_flags);
  FGBD_LAUNCH(ctx);
  const cudaMemcpyKind k = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  FGBD_CUDA(ctx, cudaMemcpyAsync(colors, d_colors, out_bytes, k, ctx->stream));
  FGBD_CUDA(ctx, cudaMemcpyAsync(int_coords ? (void*)coords_int : (void*)coords_float, d_coords,
                                 out_bytes, k, ctx->stream));
  unsigned hf[2] = {0, 0};
  FGBD_CUDA(ctx, cudaMemcpyAsync(hf, d_flags, 8, cudaMemcpyDeviceToHost, ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (hf[0] & 1)
    return set_error(ctx, FGBD_E_CLOUD, "negative integer coordinates are not supported");
  if (bit_length) *bit_length = (int32_t)hf[1];
  return FGBD_OK;
}

int32_t fgbd_ply_encode(fgbd_ctx* ctx, const int64_t* coords_int, const double* coords_float,
                        const double* colors, int64_t n, uint8_t* body_out, uint32_t flags) {
  if (!ctx) return set_error(ctx, FGBD_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  if (n == 0) return FGBD_OK;
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  const size_t in_bytes = (size_t)n * 3 * 8, out_bytes = (size_t)n * 15;
  uint8_t* stage;
  int rc = ply_stage(ctx, 2 * in_bytes + out_bytes + 16, &stage);
  if (rc) return rc;
  double* d_colors = (double*)stage;
  void* d_coords = (void*)(d_colors + 3 * n);
  uint8_t* d_out = (uint8_t*)((char*)d_coords + in_bytes);
  const cudaMemcpyKind k = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  FGBD_CUDA(ctx, cudaMemcpyAsync(d_colors, colors, in_bytes, k, ctx->stream));
  FGBD_CUDA(ctx, cudaMemcpyAsync(d_coords, coords_int ? (const void*)coords_int : (const void*)coords_float,
                                 in_bytes, k, ctx->stream));
  k_ply_encode<<<grid_of(ctx, n), kBlock, 0, ctx->stream>>>(
      (const int64_t*)d_coords, (const double*)d_coords, d_colors, n, coords_int != nullptr, d_out);
  FGBD_LAUNCH(ctx);
  FGBD_CUDA(ctx, cudaMemcpyAsync(body_out, d_out, out_bytes,
                                 dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                 ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FGBD_OK;
}

}  // extern "C"

// Fused PLY-to-PLY denoise: the raw vertex records travel to the device
// once, are decoded straight into the frame's staging buffers, denoised, and
// the result is encoded on the device; only the 15-byte records come back.
extern "C" int32_t fgbd_denoise(fgbd_ctx* ctx, const int64_t* coords, const double* colors,
                                int64_t n, int32_t bits, const fgbd_config* cfg,
                                int32_t cached_q, double cached_sigma, double* out_colors,
                                fgbd_report* rep, uint32_t flags);

extern "C" int32_t fgbd_denoise_ply(fgbd_ctx* ctx, const uint8_t* body, int64_t n, int32_t stride,
                                    const int32_t* offsets, const int32_t* types,
                                    int32_t bit_depth, const fgbd_config* cfg, int32_t cached_q,
                                    double cached_sigma, uint8_t* body_out, fgbd_report* rep,
                                    uint32_t flags) {
  if (!ctx) return set_error(ctx, FGBD_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  PlyLayout L;
  int rc = make_layout(ctx, stride, offsets, types, &L);
  if (rc) return rc;
  for (int k = 0; k < 3; ++k)
    if (types[k] == PT_F4 || types[k] == PT_F8)
      return set_error(ctx, FGBD_E_GRAPH,
                       "graph construction requires integer voxel coordinates; "
                       "run quantize_coordinates first");
  if (n < 1) return FGBD_OK;
  // staging: raw records in, 15-byte records out (grown on demand); the
  // decoded coordinates land in the frame's coords64 buffer and the colours
  // in the (N,3) staging buffer `out`, which the frame consumes (re-laid out
  // into Y) before it writes the result back into the same buffer.
  if ((rc = ensure_capacity(ctx, n, bit_depth > 0 ? 3 * bit_depth > 32 : 1))) return rc;
  const size_t body_bytes = (size_t)n * stride;
  uint8_t* d_body;
  if ((rc = ply_stage(ctx, al16(body_bytes) + al16((size_t)n * 15) + 16, &d_body))) return rc;
  uint8_t* d_rec = d_body + al16(body_bytes);
  unsigned* d_flags = (unsigned*)(d_rec + al16((size_t)n * 15));
  int64_t* d_coords = ctx->coords64;
  double* d_colors = ctx->out;
  double* d_out = ctx->out;
  FGBD_CUDA(ctx, cudaMemsetAsync(d_flags, 0, 8, ctx->stream));
  FGBD_CUDA(ctx, cudaMemcpyAsync(d_body, body, body_bytes, cudaMemcpyHostToDevice, ctx->stream));
  k_ply_decode<<<grid_of(ctx, n), kBlock, 0, ctx->stream>>>(d_body, n, L, 1, d_coords, nullptr,
                                                            d_colors, d_flags);
  FGBD_LAUNCH(ctx);
  unsigned hf[2] = {0, 0};
  FGBD_CUDA(ctx, cudaMemcpyAsync(hf, d_flags, 8, cudaMemcpyDeviceToHost, ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (hf[0] & 1)
    return set_error(ctx, FGBD_E_CLOUD, "negative integer coordinates are not supported");
  const int32_t bits = bit_depth > 0 ? bit_depth : std::max(1, (int)hf[1]);
  if (bits > 21)  // the inferred depth must make a valid cloud (cloud.py:40-49)
    return set_error(ctx, FGBD_E_CLOUD, "bit_depth must be in [1, 21], got " + std::to_string(bits));
  rc = fgbd_denoise(ctx, d_coords, d_colors, n, bits, cfg, cached_q, cached_sigma, d_out, rep,
                    flags | FGBD_FLAG_DEVICE_PTRS);
  if (rc) return rc;
  k_ply_encode<<<grid_of(ctx, n), kBlock, 0, ctx->stream>>>(d_coords, nullptr, d_out, n, 1, d_rec);
  FGBD_LAUNCH(ctx);
  FGBD_CUDA(ctx, cudaMemcpyAsync(body_out, d_rec, (size_t)n * 15, cudaMemcpyDeviceToHost,
                                 ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FGBD_OK;
}
