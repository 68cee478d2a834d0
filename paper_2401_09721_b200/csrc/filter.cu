// FSLR mask, random-walk low-pass filter and the device-resident q scan
// (reference filtering.py:132-256).
//
// k_mask        include_i = !(eligible_i && stat_i > 2 sigma_est), packed to
//               1 bit/point with a warp ballot; sums count and sum_inc y^2;
//               its last block initialises the select_q state (q = 0).
// k_lf_step     one filter step out = (d f + sum_j w_ij f_j) / (2 d) over the
//               ELL graph, exactly the reference's arithmetic order (slot
//               order accumulation from 0.0, no FMA; d = sum_{j>i} w +
//               sum_{j<i} w), fused with the masked sum of out^2.  Its last
//               block evaluates Eq. (6) and runs select_q's bookkeeping
//               (strict improvement, 3-rise early exit, best_crit == 0 stop)
//               and rotates the three signal buffers, so the q loop needs no
//               host round trip: later launches see `stop` and return.
// k_finalize    clip(best, 0, 255) (filtering.py:327).
#include <algorithm>
#include <cmath>
#include <vector>

#include "device_util.cuh"
#include "fgbd_internal.cuh"

namespace fgbd {

__device__ __forceinline__ double criterion(const double sy[3], const double sx[3],
                                            long long count, double sv2, int mode) {
  if (mode == FGBD_CRIT_POOLED) {
    const double ty = (sy[0] + sy[1]) + sy[2];
    const double tx = (sx[0] + sx[1]) + sx[2];
    const double lost = (ty - tx) / ((double)count * 3.0);
    return fabs(sv2 - lost);
  }
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) acc += fabs(sv2 - (sy[c] - sx[c]) / (double)count);
  return acc / 3.0;
}

struct MaskArgs {
  const double* fslr;
  const double* y;
  const uint8_t* inc_bytes;  // explicit mask (stage API) or null
  int64_t n;
  double thr;
  int active;
  uint32_t* mask;
  double* part;  // [7][grid]
  Ctl* ctl;
  int q_max;
  int mode;
  double sv2;
};

__global__ void __launch_bounds__(kBlock) k_mask(MaskArgs a) {
  __shared__ double s_red[32 * 7];
  __shared__ bool s_last;
  double v[7] = {0, 0, 0, 0, 0, 0, 0};  // count, sy_inc[3], sy_all[3]
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < a.n; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    const bool valid = i < a.n;
    bool inc = false;
    if (valid) {
      if (a.inc_bytes) inc = a.inc_bytes[i] != 0;
      else inc = !(a.active && a.fslr[i] > a.thr);
    }
    const unsigned bits = __ballot_sync(kFull, inc);
    if (lane == 0 && i < a.n) a.mask[i >> 5] = bits;
    if (valid) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double y = a.y[3 * i + c];
        const double y2 = y * y;
        v[4 + c] += y2;
        if (inc) v[1 + c] += y2;
      }
      v[0] += inc ? 1.0 : 0.0;
    }
  }
  block_sum<7>(v, s_red);
  if (threadIdx.x == 0)
    for (int k = 0; k < 7; ++k) a.part[k * gridDim.x + blockIdx.x] = v[k];
  if (last_block(&a.ctl->ticket[1], &s_last)) {
    double t[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
#pragma unroll
      for (int k = 0; k < 7; ++k) t[k] += ld_cg(&a.part[k * gridDim.x + b]);
    block_sum<7>(t, s_red);
    if (threadIdx.x == 0) {
      Ctl* c = a.ctl;
      long long cnt = (long long)t[0];
      const bool all_ex = (cnt == 0) && (a.inc_bytes == nullptr) && a.active;
      c->all_excluded = all_ex;
      c->mask_all = all_ex;
      if (all_ex) {
        cnt = a.n;
        for (int k = 0; k < 3; ++k) c->sy[k] = t[4 + k];
      } else {
        for (int k = 0; k < 3; ++k) c->sy[k] = t[1 + k];
      }
      c->included = cnt;
      // select_q initial state: x = y, q = 0 (filtering.py:237-243)
      const double crit0 = cnt > 0 ? criterion(c->sy, c->sy, cnt, a.sv2, a.mode) : 0.0;
      c->q = 0;
      c->best_q = 0;
      c->best_crit = crit0;
      c->prev_crit = crit0;
      c->streak = 0;
      c->steps = 0;
      c->in_buf = BUF_Y;
      c->best_buf = BUF_Y;
      c->out_buf = BUF_A;
      c->stop = (a.q_max <= 0) || (crit0 == 0.0) || (cnt < 1);
      c->trace[0] = crit0;
      c->ticket[1] = 0;
    }
  }
}

struct StepArgs {
  const int2* ell;
  const double* w64;
  double* buf[3];
  const double* in;  // fixed mode
  double* out;       // fixed mode
  const uint32_t* mask;
  int64_t n;
  double* part;  // [3][grid]
  Ctl* ctl;
  int q_max;
  int mode;
  int early_exit;
  double sv2;
};

template <bool W64, bool SELECT>
__global__ void __launch_bounds__(kBlock) k_lf_step(StepArgs a) {
  __shared__ double s_red[32 * 3];
  __shared__ bool s_last;
  Ctl* ctl = a.ctl;
  const double* __restrict__ in;
  double* __restrict__ out;
  bool mask_all = true;
  if (SELECT) {
    if (*(volatile int*)&ctl->stop) return;
    in = a.buf[ctl->in_buf];
    out = a.buf[ctl->out_buf];
    mask_all = ctl->mask_all != 0;
  } else {
    in = a.in;
    out = a.out;
  }
  const int64_t n = a.n;
  double sx[3] = {0.0, 0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    int nb[kSlots];
    double w[kSlots];
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
      const int2 sl = __ldg(&a.ell[s * n + i]);
      nb[s] = sl.x;
      w[s] = W64 ? __ldg(&a.w64[s * n + i]) : (double)__int_as_float(sl.y);
    }
    const double f0 = in[3 * i], f1 = in[3 * i + 1], f2 = in[3 * i + 2];
    double g[kSlots][3];
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
      if (w[s] != 0.0) {
        const double* p = in + 3 * (int64_t)nb[s];
        g[s][0] = p[0];
        g[s][1] = p[1];
        g[s][2] = p[2];
      } else {
        g[s][0] = g[s][1] = g[s][2] = 0.0;
      }
    }
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, lo = 0.0, hi = 0.0;
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
      if (nb[s] < (int)i) lo = __dadd_rn(lo, w[s]);
      else if (nb[s] > (int)i) hi = __dadd_rn(hi, w[s]);
      if (w[s] != 0.0) {
        acc0 = __dadd_rn(acc0, __dmul_rn(w[s], g[s][0]));
        acc1 = __dadd_rn(acc1, __dmul_rn(w[s], g[s][1]));
        acc2 = __dadd_rn(acc2, __dmul_rn(w[s], g[s][2]));
      }
    }
    const double d = __dadd_rn(hi, lo);
    double o0 = f0, o1 = f1, o2 = f2;
    if (d != 0.0) {
      const double d2 = __dmul_rn(2.0, d);
      o0 = __ddiv_rn(__dadd_rn(__dmul_rn(d, f0), acc0), d2);
      o1 = __ddiv_rn(__dadd_rn(__dmul_rn(d, f1), acc1), d2);
      o2 = __ddiv_rn(__dadd_rn(__dmul_rn(d, f2), acc2), d2);
    }
    out[3 * i] = o0;
    out[3 * i + 1] = o1;
    out[3 * i + 2] = o2;
    if (SELECT) {
      const bool inc = mask_all || ((a.mask[i >> 5] >> (i & 31)) & 1u);
      if (inc) {
        sx[0] = fma(o0, o0, sx[0]);
        sx[1] = fma(o1, o1, sx[1]);
        sx[2] = fma(o2, o2, sx[2]);
      }
    }
  }
  if (!SELECT) return;
  block_sum<3>(sx, s_red);
  if (threadIdx.x == 0)
    for (int k = 0; k < 3; ++k) a.part[k * gridDim.x + blockIdx.x] = sx[k];
  if (last_block(&ctl->ticket[2], &s_last)) {
    double t[3] = {0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
#pragma unroll
      for (int k = 0; k < 3; ++k) t[k] += ld_cg(&a.part[k * gridDim.x + b]);
    block_sum<3>(t, s_red);
    if (threadIdx.x == 0) {
      const double crit = criterion(ctl->sy, t, ctl->included, a.sv2, a.mode);
      const int q = ctl->q + 1;
      ctl->q = q;
      ctl->steps = q;
      if (q < FGBD_TRACE_MAX) ctl->trace[q] = crit;
      if (crit < ctl->best_crit) {
        ctl->best_crit = crit;
        ctl->best_q = q;
        ctl->best_buf = ctl->out_buf;
      }
      ctl->streak = crit > ctl->prev_crit ? ctl->streak + 1 : 0;
      ctl->prev_crit = crit;
      ctl->stop = (a.early_exit && ctl->streak >= 3) || (q >= a.q_max) ||
                  (ctl->best_crit == 0.0);
      const int nin = ctl->out_buf;
      int nout = BUF_A;
      const int order[3] = {BUF_A, BUF_B, BUF_Y};
      for (int k = 0; k < 3; ++k)
        if (order[k] != nin && order[k] != ctl->best_buf) {
          nout = order[k];
          break;
        }
      ctl->in_buf = nin;
      ctl->out_buf = nout;
      ctl->ticket[2] = 0;
    }
  }
}

__global__ void __launch_bounds__(kBlock) k_finalize(const double* const* bufs, const Ctl* ctl,
                                                     const double* src, int64_t n3,
                                                     double* __restrict__ dst) {
  const double* s = src ? src : bufs[ctl->best_buf];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n3; k += stride)
    dst[k] = fmin(fmax(s[k], 0.0), 255.0);
}

// CSR step with caller-supplied fp64 slot weights (weight-injection parity).
__global__ void __launch_bounds__(kBlock) k_lf_csr(const int64_t* __restrict__ indptr,
                                                   const int64_t* __restrict__ indices,
                                                   const double* __restrict__ w, int64_t n,
                                                   const double* __restrict__ in,
                                                   double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double acc[3] = {0.0, 0.0, 0.0}, lo = 0.0, hi = 0.0;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
      const int64_t j = indices[k];
      const double wk = w[k];
      if (j < i) lo = __dadd_rn(lo, wk);
      else if (j > i) hi = __dadd_rn(hi, wk);
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(wk, in[3 * j + c]));
    }
    const double d = __dadd_rn(hi, lo);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double f = in[3 * i + c];
      out[3 * i + c] =
          d != 0.0 ? __ddiv_rn(__dadd_rn(__dmul_rn(d, f), acc[c]), __dmul_rn(2.0, d)) : f;
    }
  }
}

// masked sums for selection_criterion: part[8][grid] = count, sy[3], sx[3]
__global__ void __launch_bounds__(kBlock) k_crit_sums(const double* __restrict__ y,
                                                      const double* __restrict__ x,
                                                      const uint8_t* __restrict__ inc,
                                                      int64_t n, double* __restrict__ out7) {
  __shared__ double s_red[32 * 7];
  double v[7] = {0, 0, 0, 0, 0, 0, 0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (inc && !inc[i]) continue;
    v[0] += 1.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      v[1 + c] += y[3 * i + c] * y[3 * i + c];
      v[4 + c] += x[3 * i + c] * x[3 * i + c];
    }
  }
  block_sum<7>(v, s_red);
  if (threadIdx.x == 0)
    for (int k = 0; k < 7; ++k) out7[k * gridDim.x + blockIdx.x] = v[k];
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

static int red_grid(int64_t n) {
  int64_t g = (n + kBlock - 1) / kBlock;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, kRedGrid));
}

int launch_mask(fgbd_ctx* ctx, int64_t n, double sigma_est, int active, int q_max, int mode,
                const uint8_t* d_inc) {
  MaskArgs a;
  a.fslr = ctx->fslr;
  a.y = ctx->buf[BUF_Y];
  a.inc_bytes = d_inc;
  a.n = n;
  a.thr = 2.0 * sigma_est;
  a.active = active;
  a.mask = ctx->mask;
  a.part = ctx->partials;
  a.ctl = ctx->ctl;
  a.q_max = q_max;
  a.mode = mode;
  a.sv2 = sigma_est * sigma_est;
  k_mask<<<red_grid(n), kBlock, 0, ctx->stream>>>(a);
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

int launch_select_steps(fgbd_ctx* ctx, int64_t n, int q_max, int mode, int early_exit,
                        double sigma_est, int w64) {
  StepArgs a{};
  a.ell = ctx->ell;
  a.w64 = ctx->w64;
  for (int k = 0; k < 3; ++k) a.buf[k] = ctx->buf[k];
  a.mask = ctx->mask;
  a.n = n;
  a.part = ctx->partials;
  a.ctl = ctx->ctl;
  a.q_max = q_max;
  a.mode = mode;
  a.early_exit = early_exit;
  a.sv2 = sigma_est * sigma_est;
  const int grid = red_grid(n);
  for (int q = 0; q < q_max; ++q) {
    if (w64) k_lf_step<true, true><<<grid, kBlock, 0, ctx->stream>>>(a);
    else k_lf_step<false, true><<<grid, kBlock, 0, ctx->stream>>>(a);
    FGBD_LAUNCH(ctx);
  }
  return FGBD_OK;
}

int launch_fixed_steps(fgbd_ctx* ctx, int64_t n, int q, int w64, int* final_buf) {
  StepArgs a{};
  a.ell = ctx->ell;
  a.w64 = ctx->w64;
  a.n = n;
  a.ctl = ctx->ctl;
  const int grid = red_grid(n);
  int cur = BUF_Y;
  for (int k = 0; k < q; ++k) {
    const int nxt = (cur == BUF_A) ? BUF_B : BUF_A;
    a.in = ctx->buf[cur];
    a.out = ctx->buf[nxt];
    if (w64) k_lf_step<true, false><<<grid, kBlock, 0, ctx->stream>>>(a);
    else k_lf_step<false, false><<<grid, kBlock, 0, ctx->stream>>>(a);
    FGBD_LAUNCH(ctx);
    cur = nxt;
  }
  *final_buf = cur;
  return FGBD_OK;
}

int launch_finalize(fgbd_ctx* ctx, int64_t n, int src_buf, double* d_out) {
  // src_buf < 0: the buffer select_q marked best (read on the device)
  const double* src = src_buf >= 0 ? ctx->buf[src_buf] : nullptr;
  const int64_t n3 = 3 * n;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n3 + kBlock - 1) / kBlock,
                                                         ctx->num_sms * 8));
  k_finalize<<<grid, kBlock, 0, ctx->stream>>>(ctx->d_bufs, ctx->ctl, src, n3, d_out);
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

int launch_csr_steps(fgbd_ctx* ctx, const int64_t* d_indptr, const int64_t* d_indices,
                     const double* d_w, int64_t n, const double* d_in, double* d_tmp,
                     double* d_out, int q) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + kBlock - 1) / kBlock,
                                                               ctx->num_sms * 8));
  // ping-pong so that the last step lands in d_out
  const double* src = d_in;
  for (int k = 0; k < q; ++k) {
    double* dst = ((q - 1 - k) % 2 == 0) ? d_out : d_tmp;
    k_lf_csr<<<grid, kBlock, 0, ctx->stream>>>(d_indptr, d_indices, d_w, n, src, dst);
    FGBD_LAUNCH(ctx);
    src = dst;
  }
  if (q == 0)
    FGBD_CUDA(ctx, cudaMemcpyAsync(d_out, d_in, 3 * n * sizeof(double), cudaMemcpyDeviceToDevice,
                                   ctx->stream));
  return FGBD_OK;
}

int launch_criterion(fgbd_ctx* ctx, const double* d_y, const double* d_x, const uint8_t* d_inc,
                     int64_t n, double sigma_est, int mode, double* crit_out) {
  const int grid = red_grid(n);
  k_crit_sums<<<grid, kBlock, 0, ctx->stream>>>(d_y, d_x, d_inc, n, ctx->partials);
  FGBD_LAUNCH(ctx);
  std::vector<double> h(7 * grid);
  FGBD_CUDA(ctx, cudaMemcpyAsync(h.data(), ctx->partials, h.size() * sizeof(double),
                                 cudaMemcpyDeviceToHost, ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  double t[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int k = 0; k < 7; ++k)
    for (int b = 0; b < grid; ++b) t[k] += h[k * grid + b];
  const long long cnt = (long long)t[0];
  if (cnt < 1) return set_error(ctx, FGBD_E_FILTER, "criterion needs at least one included point");
  const double sv2 = sigma_est * sigma_est;
  if (mode == FGBD_CRIT_POOLED) {
    const double lost = (((t[1] + t[2]) + t[3]) - ((t[4] + t[5]) + t[6])) / ((double)cnt * 3.0);
    *crit_out = std::fabs(sv2 - lost);
  } else {
    double acc = 0.0;
    for (int c = 0; c < 3; ++c) acc += std::fabs(sv2 - (t[1 + c] - t[4 + c]) / (double)cnt);
    *crit_out = acc / 3.0;
  }
  return FGBD_OK;
}

}  // namespace fgbd
