// Stage entry points that operate on caller-visible intermediates:
// patch materialisation (noise.py:82-119) and Gaussian edge weights on a
// caller-supplied edge list (graph.py:227-245).  Not on the denoise hot
// path (which never materialises patches and weights the ELL in place), but
// kept on the device so the stage API has no host fallback.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "device_util.cuh"
#include "fgbd_internal.cuh"

namespace fgbd {

__global__ void k_elig_flags(const uint32_t* __restrict__ meta, int64_t n, int D,
                             int64_t* __restrict__ flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    flag[i] = ((int)(meta[i] & 7u) >= D - 1) ? 1 : 0;
}

__global__ void k_extract(const uint32_t* __restrict__ meta, const int* __restrict__ ell,
                          const double* __restrict__ colors, int64_t n, int D,
                          const int64_t* __restrict__ pos, int64_t ne,
                          int64_t* __restrict__ pidx, double* __restrict__ vec) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t mt = meta[i];
    if ((int)(mt & 7u) < D - 1) continue;
    const int64_t p = pos[i];
    FGBD_DCHECK(p >= 0 && p < ne);
    if (pidx) pidx[p] = i;
    if (!vec) continue;
    for (int c = 0; c < 3; ++c) vec[((int64_t)c * ne + p) * D] = colors[4 * i + c];
    for (int r = 1; r < D; ++r) {
      const int s = (int)((mt >> (3 + 3 * (r - 1))) & 7u);
      const int64_t j = ell_j(ell[eslot(s, n, i)]);
      for (int c = 0; c < 3; ++c) vec[((int64_t)c * ne + p) * D + r] = colors[4 * j + c];
    }
  }
}

__global__ void __launch_bounds__(kBlock) k_edge_len_sum(const double* __restrict__ sq,
                                                         int64_t e, double* __restrict__ part) {
  __shared__ double s_red[32];
  double v[1] = {0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < e; k += stride)
    v[0] += sqrt(sq[k]);
  block_sum<1>(v, s_red);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

__global__ void __launch_bounds__(kBlock) k_sum_parts(const double* __restrict__ part, int np,
                                                      double* __restrict__ out) {
  __shared__ double s_red[32];
  double v[1] = {0.0};
  for (int k = threadIdx.x; k < np; k += blockDim.x) v[0] += part[k];
  block_sum<1>(v, s_red);
  if (threadIdx.x == 0) *out = v[0];
}

__global__ void k_edge_exp(const double* __restrict__ sq, int64_t e, double sg2,
                           double* __restrict__ w) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < e; k += stride)
    w[k] = exp(__ddiv_rn(-sq[k], sg2));
}

}  // namespace fgbd

using namespace fgbd;

extern "C" {

int32_t fgbd_extract_patches(fgbd_ctx* ctx, const double* colors, int32_t D,
                             int64_t* point_index_out, double* vectors_out, int64_t* ne_out,
                             uint32_t flags) {
  if (!ctx) return set_error(ctx, FGBD_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  if (ctx->g_n < 0) return set_error(ctx, FGBD_E_GRAPH, "no graph held by this context");
  if (int e = require_point_rows(ctx)) return e;
  if (D < 2) return set_error(ctx, FGBD_E_NOISE, "patch_size must be >= 2, got " + std::to_string(D));
  const int64_t n = ctx->g_n;
  int maxdeg = 0;
  if (n >= 2) {
    FGBD_CUDA(ctx, cudaMemcpy(ctx->ctl_host, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    maxdeg = ctx->ctl_host->max_deg;
  }
  if (D > 1 + maxdeg)
    return set_error(ctx, FGBD_E_NOISE, "patch_size " + std::to_string(D) +
                                            " exceeds 1 + max degree (" + std::to_string(1 + maxdeg) +
                                            ") of this graph");
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  const int64_t tiles = (n + 2047) / 2048;
  char* d = nullptr;
  FGBD_CUDA(ctx, cudaMalloc(&d, (size_t)(2 * n + tiles + 1) * 8));
  int64_t* flag = (int64_t*)d;
  int64_t* pos = flag + n;
  int64_t* tmp = pos + n;
  int64_t* total = tmp + tiles;
  int rc = FGBD_OK;
  auto fin = [&](int r) {
    cudaFree(d);
    return r;
  };
  if ((rc = upload_colors(ctx, colors, n, dev))) return fin(rc);
  cudaError_t e;
  const int grid = (int)std::min<int64_t>((n + kBlock - 1) / kBlock, ctx->num_sms * 8);
  k_elig_flags<<<grid, kBlock, 0, ctx->stream>>>(ctx->meta, n, D, flag);
  if ((rc = scan_exclusive(ctx, flag, n, pos, tmp, total))) return fin(rc);
  int64_t ne = 0;
  e = cudaMemcpyAsync(&ne, total, 8, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return fin(cuda_error(ctx, e, "patch count"));
  if (ne_out) *ne_out = ne;
  if ((point_index_out || vectors_out) && ne > 0) {
    int64_t* d_pidx = nullptr;
    double* d_vec = nullptr;
    if (dev) {
      d_pidx = point_index_out;
      d_vec = vectors_out;
    } else {
      if (point_index_out && (e = cudaMalloc(&d_pidx, ne * 8)) != cudaSuccess)
        return fin(cuda_error(ctx, e, "alloc"));
      if (vectors_out && (e = cudaMalloc(&d_vec, 3 * ne * D * 8)) != cudaSuccess) {
        cudaFree(d_pidx);
        return fin(cuda_error(ctx, e, "alloc"));
      }
    }
    k_extract<<<grid, kBlock, 0, ctx->stream>>>(ctx->meta, ctx->nbr, ctx->buf[BUF_Y], n, D, pos,
                                                ne, d_pidx, d_vec);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (!dev) {
      if (e == cudaSuccess && point_index_out)
        e = cudaMemcpy(point_index_out, d_pidx, ne * 8, cudaMemcpyDeviceToHost);
      if (e == cudaSuccess && vectors_out)
        e = cudaMemcpy(vectors_out, d_vec, 3 * ne * D * 8, cudaMemcpyDeviceToHost);
      cudaFree(d_pidx);
      cudaFree(d_vec);
    }
    if (e != cudaSuccess) return fin(cuda_error(ctx, e, "extract"));
  }
  return fin(FGBD_OK);
}

int32_t fgbd_edge_weights(fgbd_ctx* ctx, const double* sqdist, int64_t E, double sigma_g,
                          double* sigma_out, double* weights_out, uint32_t flags) {
  if (!ctx) return set_error(ctx, FGBD_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  const bool need_sigma = std::isnan(sigma_g);
  if (need_sigma && E == 0)
    return set_error(ctx, FGBD_E_GRAPH, "cannot compute a distance scale on an edgeless graph");
  char* d = nullptr;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((E + kBlock - 1) / kBlock, kRedGrid));
  FGBD_CUDA(ctx, cudaMalloc(&d, (size_t)(2 * E + grid + 2) * 8));
  double* d_sq = (double*)d;
  double* d_w = d_sq + E;
  double* d_part = d_w + E;
  double* d_sum = d_part + grid;
  auto fin = [&](int r) {
    cudaFree(d);
    return r;
  };
  cudaError_t e = cudaSuccess;
  if (E) e = cudaMemcpy(d_sq, sqdist, E * 8, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return fin(cuda_error(ctx, e, "upload"));
  double sg = sigma_g;
  if (need_sigma) {
    k_edge_len_sum<<<grid, kBlock, 0, ctx->stream>>>(d_sq, E, d_part);
    k_sum_parts<<<1, kBlock, 0, ctx->stream>>>(d_part, grid, d_sum);
    double s = 0.0;
    e = cudaMemcpyAsync(&s, d_sum, 8, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return fin(cuda_error(ctx, e, "sigma_g"));
    sg = s / (double)E;
  }
  if (sigma_out) *sigma_out = sg;
  if (weights_out) {
    if (!(sg > 0)) {
      char b[96];
      std::snprintf(b, sizeof(b), "sigma_g must be positive, got %.17g", sg);
      return fin(set_error(ctx, FGBD_E_GRAPH, b));
    }
    if (E) {
      const int g2 = (int)std::min<int64_t>((E + kBlock - 1) / kBlock, ctx->num_sms * 8);
      k_edge_exp<<<g2, kBlock, 0, ctx->stream>>>(d_sq, E, sg * sg, d_w);
      e = cudaMemcpyAsync(weights_out, d_w, E * 8,
                          dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
      if (e != cudaSuccess) return fin(cuda_error(ctx, e, "weights"));
    }
  }
  return fin(FGBD_OK);
}

}  // extern "C"
