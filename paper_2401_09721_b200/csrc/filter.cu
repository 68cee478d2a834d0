// FSLR mask, random-walk low-pass filter and the device-resident q scan
// (reference filtering.py:132-256).
//
// Signals live in HBM as (N, 4) fp64 rows (r, g, b, 0): one 32-byte sector
// per point, so every neighbour gather is a single 256-bit load
// (LDG.E.ENL2.256 on sm_100a) instead of three 8-byte loads.
//
// k_mask       include_i = !(eligible_i && stat_i > 2 sigma_est), packed to
//              1 bit/point by warp ballot; sums count and sum_inc y^2; its
//              last block initialises the select_q state (q = 0).
// k_lf_run     the whole q scan in ONE cooperative launch (persistent, 3
//              blocks of 256 per SM): per step every row applies
//              out = (d f + sum_j w_ij f_j) / (2 d) in the reference's exact
//              arithmetic order (slot-order accumulation from 0.0, no FMA,
//              d = sum_{j>i} w + sum_{j<i} w) and adds its masked out^2 to a
//              block partial; the select_q decision for step q-1 (Eq. (6),
//              strict improvement, 3-rise early exit, best_crit == 0 stop)
//              is taken by every block from bulk-copied partials while step
//              q sweeps (lagged by one step), or before it when one more
//              rise would stop the scan (HOLD).  On the denoise path step 1
//              also builds the FSLR mask and select_q's initial totals
//              (k_mask's work, fold).  No host round trip, one launch.
// k_lf_step    one step per launch (variant 0, kept for comparison).
// k_compact    (N,4) -> (N,3), optionally clipped to [0, 255] (filtering.py:327).
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <type_traits>
#include <cmath>
#include <vector>

#ifndef FGBD_LF_DENSE
#define FGBD_LF_DENSE 1
#endif
#ifndef FGBD_ELL_POLICY
#define FGBD_ELL_POLICY 0  // L2 policy of the per-step graph stream: 0 evict_first, 1 evict_last, 2 normal
#endif
#ifndef FGBD_LF_SIGHINT
#define FGBD_LF_SIGHINT 1
#endif
#ifndef FGBD_LF_PF
// prefetch.global.L2 of the graph row FGBD_LF_PFD sweep iterations ahead
// (profiles/r1_summary.md, r1c: -2.4% filter time at distance 2)
#define FGBD_LF_PF 1
#endif
#ifndef FGBD_LF_PFD
#define FGBD_LF_PFD 2
#endif
#ifndef FGBD_LF_RCPDIV
#define FGBD_LF_RCPDIV 1  // the step's three quotients via one reciprocal (div_rcp)
#endif
#ifndef FGBD_LF_SPLITBAR
// split-phase grid barrier: arrive right after a step's rows and partials are
// stored, run the lagged select_q decision, then wait -- the decision no
// longer sits between the slowest block's sweep and the barrier (1: on;
// 0: cooperative_groups grid.sync() after the decision)
#define FGBD_LF_SPLITBAR 0
#endif
// the per-step grid barrier: 1 grid_barrier (relaxed spin, one L1
// invalidation per block), 0 cooperative_groups grid.sync()
#ifndef FGBD_LF_BAR
#define FGBD_LF_BAR 0
#endif
#ifndef FGBD_LF_ELLSMEM
// graph slots of the next FGBD_LF_ELLSMEM rows via cp.async into shared memory (0: registers;
// profiles/r1_summary.md r1c: 1 stage -2.5% filter time, 2 / 3 stages slower -- less L1)
#define FGBD_LF_ELLSMEM 1
#endif
#include "device_util.cuh"
#include "fgbd_internal.cuh"
#include "select_state.cuh"

namespace cg = cooperative_groups;

namespace fgbd {

// ---------------------------------------------------------------------------
// layout conversion
// ---------------------------------------------------------------------------

// row k of the signal holds point rowid[k] (identity when rowid is null)
__global__ void __launch_bounds__(kBlock) k_expand(const double* __restrict__ src, int64_t n,
                                                   double4* __restrict__ dst,
                                                   const uint32_t* __restrict__ rowid) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t p = rowid ? (int64_t)rowid[i] : i;
    FGBD_DCHECK(p >= 0 && p < n);
    st_row(dst + i, make_double4(src[3 * p], src[3 * p + 1], src[3 * p + 2], 0.0));
  }
}

template <bool CLIP>
__global__ void __launch_bounds__(kBlock) k_compact(double* const* bufs, const Ctl* ctl,
                                                    const double4* src, int64_t n,
                                                    double* __restrict__ dst,
                                                    const int* __restrict__ pos) {
  const double4* s = src ? src : reinterpret_cast<const double4*>(bufs[ctl->best_buf]);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    FGBD_DCHECK(!pos || (pos[i] >= 0 && pos[i] < n));
    const double4 v = ld_row(s + (pos ? (int64_t)pos[i] : i));  // point i lives in row pos[i]
    if (CLIP) {
      dst[3 * i] = fmin(fmax(v.x, 0.0), 255.0);
      dst[3 * i + 1] = fmin(fmax(v.y, 0.0), 255.0);
      dst[3 * i + 2] = fmin(fmax(v.z, 0.0), 255.0);
    } else {
      dst[3 * i] = v.x;
      dst[3 * i + 1] = v.y;
      dst[3 * i + 2] = v.z;
    }
  }
}

// ---------------------------------------------------------------------------
// FSLR mask + select_q initialisation
// ---------------------------------------------------------------------------

struct MaskArgs {
  const double* fslr;
  const double4* y;
  const uint8_t* inc_bytes;  // explicit mask (stage API) or null
  int64_t n;
  double thr;
  int active;
  uint32_t* mask;
  double* part;  // [7][grid]
  Ctl* ctl;
  int q_max;
  int mode;
  int early_exit;
  double sv2;
  int defer;        // slab rank: leave the totals in ctl->mask_part (all-gathered later)
  int64_t n_total;  // points of the whole frame (the all-excluded fallback count)
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
      const double4 y = ld_row(a.y + i);
      const double y2[3] = {y.x * y.x, y.y * y.y, y.z * y.z};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        v[4 + c] += y2[c];
        if (inc) v[1 + c] += y2[c];
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
      if (a.defer) {
        for (int k = 0; k < 7; ++k) a.ctl->mask_part[k] = t[k];
      } else {
        mask_finalize(a.ctl, t, a.n, a.inc_bytes != nullptr, a.active, a.q_max, a.mode,
                      a.early_exit, a.sv2);
      }
      a.ctl->ticket[1] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// the filter step
// ---------------------------------------------------------------------------

struct StepArgs {
  EllRef E;
  const double* w64;    // fp64 weights [6][N] (parity mode) or null
  const void* pc;       // packed coordinates (weights recomputed on the fly)
  int bits;
  double4* buf[3];
  const uint32_t* mask;
  int64_t n;
  double* part;  // [2 parities][3][grid]
  Ctl* ctl;
  int fixed_steps;  // cached path: number of steps (Y -> A/B ping-pong)
  int64_t chunk;    // persistent kernels: rows per block (contiguous), 0 = grid-stride
  int halo;         // TMA-staged sweep: window rows either side of a row tile
  const uint32_t* rowid;  // row -> point when rows are in scan-line-1 order (else null)
  unsigned long long* flags;  // P2P: per-block "step published" words (monotone across launches)
  unsigned int* gbar;         // split-phase grid barrier: [0] arrivals, [1] generation
  unsigned long long base;    // P2P: this launch's flag base (published value = base + step)
  // FSLR mask folded into step 1 (fold != 0, select_q from denoise): step 1
  // thresholds fslr[] into the mask and sums the select_q initial totals
  int fold;       // 1: sigma_est etc. below; 2: read from ctl (k_finish_noise)
  const double* fslr;
  double* xpart;  // [10][grid]: count, sum_inc y^2 [3], sum_all y^2 [3], sum_all x1^2 [3]
  int q_max, mode, early_exit;
  double sv2, thr;  // sigma_est^2, 2 sigma_est
  int active;       // FSLR on (filtering.py:285-295)
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Spin until flags[b] >= want for every b in [lo, hi] except `self`.
__device__ __forceinline__ void wait_blocks(const unsigned long long* flags, int lo, int hi,
                                            int self, unsigned long long want) {
  if (lo > hi) return;  // a block without rows depends on nobody
  for (int b = lo + (int)threadIdx.x; b <= hi; b += blockDim.x) {
    if (b == self) continue;
    while (ld_acquire_u64(flags + b) < want) __nanosleep(20);
  }
}

__device__ __forceinline__ uint64_t graph_policy() {
#if FGBD_ELL_POLICY == 1
  return policy_evict_last();
#elif FGBD_ELL_POLICY == 2
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
#else
  return policy_evict_first();
#endif
}

// Where a row's six weights come from.
enum WMode { W_STORED = 0, W_COORDS32 = 1, W_COORDS64 = 2 };

template <typename K>
__device__ __forceinline__ long long sqlen(K a, K b, int bits) {
  const K m = (K(1) << bits) - 1;
  const long long dx = (long long)(a & m) - (long long)(b & m);
  const long long dy = (long long)((a >> bits) & m) - (long long)((b >> bits) & m);
  const long long dz = (long long)(a >> (2 * bits)) - (long long)(b >> (2 * bits));
  return dx * dx + dy * dy + dz * dz;
}

// Load row i's neighbours and weights.  W_STORED reads the fp32 weights the
// weight pass stored; W_COORDS* recompute w = exp(-|g_i - g_j|^2 / sigma_g^2)
// from the 4/8-byte packed coordinates (an L2-resident array), so the
// per-step graph stream is only the 24-byte index row.
template <int WM>
__device__ __forceinline__ void load_row_slots(const StepArgs& a, int64_t i, uint64_t pol,
                                               float neg_inv_sg2, int (&nb)[kSlots],
                                               float (&w)[kSlots]) {
  const int64_t n = a.n;
#pragma unroll
  for (int s = 0; s < kSlots; s += 2) {
    const int4 pr = ld_pair_hint(reinterpret_cast<const int2*>(a.E.nbr + eslot(s, n, i)), pol);
    nb[s] = pr.x;
    nb[s + 1] = pr.z;
    if (WM == W_STORED) {
      w[s] = __int_as_float(pr.y);
      w[s + 1] = __int_as_float(pr.w);
    }
  }
  if (WM != W_STORED) {
    using K = typename std::conditional<WM == W_COORDS32, uint32_t, unsigned long long>::type;
    const K* pc = reinterpret_cast<const K*>(a.pc);
    const K own = pc[a.rowid ? a.rowid[i] : i];
    K pj[kSlots];
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
      const int j = ell_j(nb[s]);
      pj[s] = pc[a.rowid ? a.rowid[j] : j];
    }
#pragma unroll
    for (int s = 0; s < kSlots; ++s)
      w[s] = ell_j(nb[s]) != (int)i ? __expf((float)sqlen(own, pj[s], a.bits) * neg_inv_sg2)
                                    : 0.0f;
  }
}

// out = (d f + sum_s w_s f_s) / (2 d), the reference's order (filtering.py:132-155).

// out = (d f + acc) / (2 d) per channel (filtering.py:148-155); d = 0 keeps f
__device__ __forceinline__ double4 finish_row(double d, const double4& f, double acc0,
                                              double acc1, double acc2) {
  if (d == 0.0) return f;
  const double d2 = __dmul_rn(2.0, d);
#if FGBD_LF_RCPDIV
  // one reciprocal for the three quotients; div_rcp is the correctly
  // rounded a / b (device_util.cuh), so the bits are unchanged
  if (rcp_ok(d2)) {
    const double y = __drcp_rn(d2);
    return make_double4(div_rcp(__dadd_rn(__dmul_rn(d, f.x), acc0), d2, y),
                        div_rcp(__dadd_rn(__dmul_rn(d, f.y), acc1), d2, y),
                        div_rcp(__dadd_rn(__dmul_rn(d, f.z), acc2), d2, y), 0.0);
  }
#endif
  return make_double4(__ddiv_rn(__dadd_rn(__dmul_rn(d, f.x), acc0), d2),
                      __ddiv_rn(__dadd_rn(__dmul_rn(d, f.y), acc1), d2),
                      __ddiv_rn(__dadd_rn(__dmul_rn(d, f.z), acc2), d2), 0.0);
}

template <int FAR = 0>
__device__ __forceinline__ double4 row_from_slots(const int (&nb)[kSlots], const float (&wf)[kSlots],
                                                  const double4* in, int64_t i, uint64_t pol_keep,
                                                  double4* f_out = nullptr) {
  const double4 f = ld_row_hint(in + i, pol_keep);
  if (f_out) *f_out = f;
  double4 g[kSlots];
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, lo = 0.0, hi = 0.0;
#if FGBD_LF_DENSE
  // Every slot is gathered and accumulated: padding slots are (self, 0.0)
  // and zero-weight edges add +0.0 * f_j = +0.0 to a non-negative
  // accumulator, which leaves it bit-identical -- and the row has no
  // per-slot branches.
#pragma unroll
  for (int s = 0; s < kSlots; ++s)
  if (FAR > 0) {
    // far neighbours (scattered gathers on random clouds) bypass L1, so
    // they do not evict the rows the block re-reads (own rows, near ones)
    const int64_t dj = (int64_t)ell_j(nb[s]) - i;
    g[s] = (dj > FAR || dj < -FAR) ? ld_row_cg_hint(in + ell_j(nb[s]), pol_keep)
                                   : ld_row_hint(in + ell_j(nb[s]), pol_keep);
  } else
#if FGBD_LF_SIGHINT
    g[s] = ld_row_hint(in + ell_j(nb[s]), pol_keep);
#else
    g[s] = ld_row(in + ell_j(nb[s]));
#endif

#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    // the ELL word's bit 31 says whether the neighbour's ORIGINAL index is
    // below this row's point; padding (own row, w = 0) adds +0.0 to hi
    const double w = (double)wf[s];
    const bool below = ell_below(nb[s]);
    lo = __dadd_rn(lo, below ? w : 0.0);
    hi = __dadd_rn(hi, below ? 0.0 : w);
    acc0 = __dadd_rn(acc0, __dmul_rn(w, g[s].x));
    acc1 = __dadd_rn(acc1, __dmul_rn(w, g[s].y));
    acc2 = __dadd_rn(acc2, __dmul_rn(w, g[s].z));
  }
#else
#pragma unroll
  for (int s = 0; s < kSlots; ++s)
    g[s] = (wf[s] != 0.0f) ? ld_row_hint(in + ell_j(nb[s]), pol_keep) : make_double4(0, 0, 0, 0);
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    const double w = (double)wf[s];
    if (ell_below(nb[s])) lo = __dadd_rn(lo, w);
    else if (ell_j(nb[s]) != (int)i) hi = __dadd_rn(hi, w);
    if (wf[s] != 0.0f) {
      acc0 = __dadd_rn(acc0, __dmul_rn(w, g[s].x));
      acc1 = __dadd_rn(acc1, __dmul_rn(w, g[s].y));
      acc2 = __dadd_rn(acc2, __dmul_rn(w, g[s].z));
    }
  }
#endif
  return finish_row(__dadd_rn(hi, lo), f, acc0, acc1, acc2);
}

// fp64-weight row for the parity mode (per-step launches only).
__device__ __forceinline__ double4 row_w64(const StepArgs& a, const double4* in, int64_t i) {
  const int64_t n = a.n;
  int nb[kSlots];
  double w[kSlots];
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    nb[s] = __ldg(a.E.nbr + eslot(s, n, i));
    w[s] = __ldg(&a.w64[s * n + i]);
  }
  const double4 f = ld_row(in + i);
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, lo = 0.0, hi = 0.0;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    if (ell_below(nb[s])) lo = __dadd_rn(lo, w[s]);
    else if (ell_j(nb[s]) != (int)i) hi = __dadd_rn(hi, w[s]);
    if (w[s] != 0.0) {
      const double4 g = ld_row(in + ell_j(nb[s]));
      acc0 = __dadd_rn(acc0, __dmul_rn(w[s], g.x));
      acc1 = __dadd_rn(acc1, __dmul_rn(w[s], g.y));
      acc2 = __dadd_rn(acc2, __dmul_rn(w[s], g.z));
    }
  }
  return finish_row(__dadd_rn(hi, lo), f, acc0, acc1, acc2);
}

// select_q bookkeeping after step q (filtering.py:244-255).  Pure function
// of (state, crit): every block evaluates it identically.


__device__ __forceinline__ double4* pick_buf(const StepArgs& a, int b) {
  return b == 0 ? a.buf[0] : (b == 1 ? a.buf[1] : a.buf[2]);
}


// One sweep of this block's rows: out = P in, optionally summing out^2 over
// included rows.  The next row's graph slots are fetched while the current
// row's neighbour gathers are in flight (into registers, or with
// FGBD_LF_ELLSMEM by cp.async into this thread's shared-memory slots, which
// frees 12 registers), and the graph row FGBD_LF_PFD iterations ahead is
// prefetched into L2.
template <int WM, bool SUMS, bool FOLD = false, int FAR = 0>
__device__ __forceinline__ void sweep(const StepArgs& a, const double4* in, double4* out,
                                      bool mask_all, float neg_inv_sg2, double (&sx)[3],
                                      int4* s_ell, double* xs = nullptr /*[10] with FOLD*/,
                                      const double* thr_p = nullptr, const int* active_p = nullptr) {
  const int64_t n = a.n;
  // rows of this block: a contiguous range walked in blockDim strides (the
  // neighbours of raster / scan-ordered clouds then mostly hit this SM's L1),
  // or the grid-stride interleave
  int64_t i, end, stride;
  if (a.chunk > 0) {
    i = (int64_t)blockIdx.x * a.chunk + threadIdx.x;
    end = min(n, (int64_t)(blockIdx.x + 1) * a.chunk);
    stride = blockDim.x;
  } else {
    i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    end = n;
    stride = (int64_t)gridDim.x * blockDim.x;
  }
  const uint64_t pol_stream = graph_policy(), pol_keep = policy_evict_last();
  constexpr bool kSmemEll = FGBD_LF_ELLSMEM && WM == W_STORED;
  int nbc[kSlots], nbn[kSlots];
  float wc[kSlots], wn[kSlots];
  // shared-memory slots [stage][pair][thread]: each thread reads back only
  // what it copied itself, so no block barrier is needed
  constexpr int NS = FGBD_LF_ELLSMEM + 1;  // stages: rows in flight + the one in use
  const int T = blockDim.x;
  int stage = 0;
  auto issue = [&](int64_t r, int st) {
    if (r < end)
#pragma unroll
      for (int s = 0; s < kSlots; s += 2)
        asm volatile(
            "cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(
                smem_u32(s_ell + (st * 3 + (s >> 1)) * T + threadIdx.x)),
            "l"(a.E.nbr + eslot(s, n, r)), "l"(pol_stream)
            : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if constexpr (kSmemEll) {
#pragma unroll
    for (int k = 0; k < NS - 1; ++k) issue(i + k * stride, k);
  } else if (i < end) {
    load_row_slots<WM>(a, i, pol_stream, neg_inv_sg2, nbn, wn);
  }
  while (i < end) {
    const int64_t inext = i + stride;
    if constexpr (kSmemEll) {
      issue(i + (NS - 1) * stride, stage == 0 ? NS - 1 : stage - 1);
      asm volatile("cp.async.wait_group %0;" ::"n"(NS - 1) : "memory");
#pragma unroll
      for (int s = 0; s < kSlots; s += 2) {
        const int4 pr = s_ell[(stage * 3 + (s >> 1)) * T + threadIdx.x];
        nbc[s] = pr.x;
        wc[s] = __int_as_float(pr.y);
        nbc[s + 1] = pr.z;
        wc[s + 1] = __int_as_float(pr.w);
      }
      stage = stage + 1 == NS ? 0 : stage + 1;
    } else {
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        nbc[s] = nbn[s];
        wc[s] = wn[s];
      }
      if (inext < end) load_row_slots<WM>(a, inext, pol_stream, neg_inv_sg2, nbn, wn);
    }
#if FGBD_DEBUG_BOUNDS
#pragma unroll
    for (int s = 0; s < kSlots; ++s) FGBD_DCHECK(ell_j(nbc[s]) < n);
#endif
    if (FGBD_LF_PF && i + FGBD_LF_PFD * stride < end)
#pragma unroll
      for (int s = 0; s < kSlots; s += 2)
        prefetch_l2(a.E.nbr + eslot(s, n, i + FGBD_LF_PFD * stride));
    double4 f;
    const double4 o = row_from_slots<FAR>(nbc, wc, in, i, pol_keep, FOLD ? &f : nullptr);
    st_row_hint(out + i, o, pol_keep);
    if (FOLD) {
      // k_mask's work for this row (filtering.py:175-194, 237-243): the
      // FSLR bit, and the initial totals over included / all rows
      // (the threshold is read from shared memory here, not held in a
      // register across the kernel: that cost the hot loop a spill)
      const bool inc = !(*active_p && a.fslr[i] > *thr_p);
      const unsigned bits = __ballot_sync(__activemask(), inc);
      if ((threadIdx.x & 31) == 0) const_cast<uint32_t*>(a.mask)[i >> 5] = bits;
      const double y2[3] = {f.x * f.x, f.y * f.y, f.z * f.z};
      xs[0] += inc ? 1.0 : 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (inc) xs[1 + c] += y2[c];
        xs[4 + c] += y2[c];
      }
      xs[7] = fma(o.x, o.x, xs[7]);
      xs[8] = fma(o.y, o.y, xs[8]);
      xs[9] = fma(o.z, o.z, xs[9]);
      if (inc) {
        sx[0] = fma(o.x, o.x, sx[0]);
        sx[1] = fma(o.y, o.y, sx[1]);
        sx[2] = fma(o.z, o.z, sx[2]);
      }
    } else if (SUMS && (mask_all || ((a.mask[i >> 5] >> (i & 31)) & 1u))) {
      sx[0] = fma(o.x, o.x, sx[0]);
      sx[1] = fma(o.y, o.y, sx[1]);
      sx[2] = fma(o.z, o.z, sx[2]);
    }
    i = inext;
  }
  if constexpr (kSmemEll) asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---------------------------------------------------------------------------
// TMA-staged sweep (lf_variant 12).  A block walks its contiguous row range in
// tiles of kTile rows, double-buffered through shared memory by the bulk-copy
// engine (cp.async.bulk + mbarrier): per tile, the signal window
// [c0 - halo, c1 + halo) and the tile's three ELL slot-pair planes.  A row's
// own value and every neighbour inside the window come from shared memory;
// only neighbours outside it (for raster-ordered clouds: the scan-line-3
// ones) are gathered from global memory.  The tile after the current one is
// in flight while the current one computes, without costing registers.
// ---------------------------------------------------------------------------
constexpr int kMaxCoopBlocks = 592;  // persistent grids: <= 148 SMs x 4 blocks
constexpr int kTile = 256;
constexpr int kHaloMax = 128;
constexpr int kWinRows = kTile + 2 * kHaloMax;
constexpr int kStageBytes = kWinRows * 32 + 3 * kTile * 16;
constexpr int kTmaSmem = 128 + 2 * kStageBytes;


struct TmaState {
  uint64_t* bar;        // [2]
  unsigned char* stage; // [2][kStageBytes]
  uint32_t uses[2];     // completed phases per stage (uniform over the block)
};

__device__ __forceinline__ void tma_issue(const StepArgs& a, const double4* in, TmaState& t,
                                          int st, int64_t c0, int64_t c1, uint64_t pol_stream,
                                          uint64_t pol_keep) {
  const int64_t n = a.n;
  const int64_t w0 = c0 - a.halo > 0 ? c0 - a.halo : 0;
  const int64_t w1 = c1 + a.halo < n ? c1 + a.halo : n;
  const uint32_t wb = (uint32_t)((w1 - w0) * 32), eb = (uint32_t)((c1 - c0) * 16);
  unsigned char* base = t.stage + st * kStageBytes;
  mbar_expect_tx(&t.bar[st], wb + 3 * eb);
  bulk_g2s(base, in + w0, wb, &t.bar[st], pol_keep);
#pragma unroll
  for (int p = 0; p < 3; ++p)
    bulk_g2s(base + kWinRows * 32 + p * kTile * 16, a.E.nbr + (int64_t)p * 4 * n + 4 * c0, eb,
             &t.bar[st], pol_stream);
}

template <bool SUMS>
__device__ __forceinline__ void sweep_tma(const StepArgs& a, const double4* in, double4* out,
                                          bool mask_all, TmaState& t, double (&sx)[3]) {
  const int64_t n = a.n;
  const int64_t lo = (int64_t)blockIdx.x * a.chunk;
  const int64_t hi = min(n, lo + a.chunk);
  const uint64_t pol_stream = graph_policy(), pol_keep = policy_evict_last();
  const int tiles = hi > lo ? (int)((hi - lo + kTile - 1) / kTile) : 0;
  if (threadIdx.x == 0 && tiles > 0) {
    fence_proxy_async_global();  // last step's generic stores -> this step's bulk reads
    tma_issue(a, in, t, 0, lo, min(hi, lo + kTile), pol_stream, pol_keep);
  }
  // tile k lives in stage (k & 1); stage 0 always takes tile 0 of a step
  uint32_t u0 = t.uses[0], u1 = t.uses[1];
  for (int k = 0; k < tiles; ++k) {
    const int st = k & 1;
    const int64_t c0 = lo + (int64_t)k * kTile, c1 = min(hi, c0 + kTile);
    if (threadIdx.x == 0 && k + 1 < tiles)
      tma_issue(a, in, t, st ^ 1, c1, min(hi, c1 + kTile), pol_stream, pol_keep);
    const uint32_t par = (st ? u1 : u0) & 1;
    mbar_wait(&t.bar[st], par);
    if (st) ++u1; else ++u0;
    const int64_t i = c0 + threadIdx.x;
    if (i < c1) {
      const int64_t w0 = c0 - a.halo > 0 ? c0 - a.halo : 0;
      const int64_t w1 = c1 + a.halo < n ? c1 + a.halo : n;
      const unsigned char* base = t.stage + st * kStageBytes;
      const double4* W = reinterpret_cast<const double4*>(base);
      const int4* E = reinterpret_cast<const int4*>(base + kWinRows * 32);
      int nb[kSlots];
      float wf[kSlots];
      int raw[kSlots];
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const int4 pr = E[p * kTile + threadIdx.x];
        raw[2 * p] = pr.x;
        wf[2 * p] = __int_as_float(pr.y);
        raw[2 * p + 1] = pr.z;
        wf[2 * p + 1] = __int_as_float(pr.w);
      }
#pragma unroll
      for (int s = 0; s < kSlots; ++s) nb[s] = ell_j(raw[s]);
      // far neighbours first (global), then the window (shared)
      double4 g[kSlots];
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        const bool near = nb[s] >= w0 && nb[s] < w1;
        g[s] = (wf[s] != 0.0f && !near) ? ld_row_hint(in + nb[s], pol_keep)
                                        : make_double4(0, 0, 0, 0);
      }
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        const bool near = nb[s] >= w0 && nb[s] < w1;
        if (wf[s] != 0.0f && near) g[s] = W[nb[s] - w0];
      }
      const double4 f = W[i - w0];
      double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, dlo = 0.0, dhi = 0.0;
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        const double w = (double)wf[s];
        if (ell_below(raw[s])) dlo = __dadd_rn(dlo, w);
        else if (nb[s] != (int)i) dhi = __dadd_rn(dhi, w);
        if (wf[s] != 0.0f) {
          acc0 = __dadd_rn(acc0, __dmul_rn(w, g[s].x));
          acc1 = __dadd_rn(acc1, __dmul_rn(w, g[s].y));
          acc2 = __dadd_rn(acc2, __dmul_rn(w, g[s].z));
        }
      }
      const double d = __dadd_rn(dhi, dlo);
      double4 o = f;
      if (d != 0.0) {
        const double d2 = __dmul_rn(2.0, d);
        o = make_double4(__ddiv_rn(__dadd_rn(__dmul_rn(d, f.x), acc0), d2),
                         __ddiv_rn(__dadd_rn(__dmul_rn(d, f.y), acc1), d2),
                         __ddiv_rn(__dadd_rn(__dmul_rn(d, f.z), acc2), d2), 0.0);
      }
      st_row_hint(out + i, o, pol_keep);
      if (SUMS && (mask_all || ((a.mask[i >> 5] >> (i & 31)) & 1u))) {
        sx[0] = fma(o.x, o.x, sx[0]);
        sx[1] = fma(o.y, o.y, sx[1]);
        sx[2] = fma(o.z, o.z, sx[2]);
      }
    }
    __syncthreads();  // stage st is refilled by the issue at k + 1 (tile k + 2)
  }
  t.uses[0] = u0;
  t.uses[1] = u1;
}

// The whole filter-step loop in ONE cooperative launch.
//
// SELECT = false: the cached path (filtering.py:313-326), fixed_steps steps
// ping-ponging Y -> A -> B -> A ...
//
// SELECT = true: select_q with the decision lagged by one step.  At the top
// of iteration c, x_c is complete (buffer in_b) and decisions are known up to
// c-1.  The block sweeps step c+1 into the buffer that is neither x_c's nor
// the best-so-far's (both known without crit_c, so the rotation is safe),
// THEN reduces step c's partials and decides -- the reduction overlaps the
// wait for the slowest block at the next grid barrier.  Every block reduces
// the same partials in the same order, so all reach the same decision.  A
// stop decided at c discards the speculative x_{c+1}; q_max stops never
// compute it.
// P2P = true replaces the grid barrier by neighbourhood waits: a block's
// rows reference (symmetric graph) only rows owned by the blocks in its
// dependency range [dep_lo, dep_hi], computed from its ELL rows at entry.
// Step c+1 may start once those blocks published step c (which also means
// they finished reading the buffer this block is about to overwrite); the
// criterion decision for step c waits for every block's step-c flag, one
// step later, and reads partials from a 4-deep ring (no block is more than
// two steps ahead of any other).
#if FGBD_LF_TLOG
// Timeline instrumentation (experiment builds only, -DFGBD_LF_TLOG=1): per
// step c < kTlogSteps and block, %globaltimer at step start, sweep end and
// barrier entry.  Read back with fgbd_debug_tlog (tools/lf_timeline.py).
constexpr int kTlogSteps = 16;
__device__ unsigned long long g_tlog[kTlogSteps][kMaxCoopBlocks][3];
__device__ unsigned long long g_wlog[kTlogSteps][kMaxCoopBlocks][16];  // per-warp sweep end
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TLOG(c, k)                                                            \
  do {                                                                        \
    if (threadIdx.x == 0 && (c) < kTlogSteps) g_tlog[(c)][blockIdx.x][(k)] = gtimer(); \
  } while (0)
#else
#define TLOG(c, k) \
  do {             \
  } while (0)
#endif

// sum of out^2 over the rows this block sweeps (the all-excluded fallback
// of the folded mask, filtering.py:289-293)
__device__ __forceinline__ void rows_sumsq(const StepArgs& a, const double4* x, double (&u)[3]) {
  int64_t i, end, stride;
  if (a.chunk > 0) {
    i = (int64_t)blockIdx.x * a.chunk + threadIdx.x;
    end = min(a.n, (int64_t)(blockIdx.x + 1) * a.chunk);
    stride = blockDim.x;
  } else {
    i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    end = a.n;
    stride = (int64_t)gridDim.x * blockDim.x;
  }
  for (; i < end; i += stride) {
    const double4 o = ld_row(x + i);
    u[0] = fma(o.x, o.x, u[0]);
    u[1] = fma(o.y, o.y, u[1]);
    u[2] = fma(o.z, o.z, u[2]);
  }
}

// Split-phase grid barrier over the co-resident blocks of a cooperative
// launch: the arrive / wait halves of cooperative_groups' grid.sync() (one
// atomic per block; block 0 adds 2^31 - (blocks - 1), so the word's top bit
// flips exactly when the last block arrives).
__device__ __forceinline__ unsigned int grid_arrive(unsigned int* bar) {
  __syncthreads();  // every thread's stores of this step are issued
  unsigned int old = 0;
  if (threadIdx.x == 0) {
    const unsigned int nb = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
    __threadfence();
    old = atomicAdd(bar, nb);
  }
  return old;  // meaningful in thread 0
}
__device__ __forceinline__ void grid_wait(unsigned int* bar, unsigned int old) {
  if (threadIdx.x == 0) {
    while ((((*(volatile unsigned int*)bar) ^ old) & 0x80000000u) == 0) {
    }
    __threadfence();
  }
  __syncthreads();
}

template <int WM, bool SELECT, int BLK = kBlock, int MINB = 3, bool TMA = false,
          bool P2P = false, int FAR = 0, bool HOLD = false>
__global__ void __launch_bounds__(BLK, MINB) k_lf_run(StepArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  TmaState tma{reinterpret_cast<uint64_t*>(dyn_smem), dyn_smem + 128, {0u, 0u}};
  if (TMA && threadIdx.x == 0) {
    mbar_init(&tma.bar[0], 1);
    mbar_init(&tma.bar[1], 1);
  }
  __shared__ double s_red[32 * 3];
  // graph-slot stages of the sweep (dynamic shared memory, FGBD_LF_ELLSMEM)
  int4* s_ell = reinterpret_cast<int4*>(dyn_smem);
  __shared__ SelState s_st;
  __shared__ double s_sy[3], s_sv2;
  __shared__ long long s_inc;
  __shared__ int s_qmax, s_mode, s_early, s_mask_all;
  __shared__ int s_dep_lo, s_dep_hi;
  __shared__ double s_red10[32 * 10];
  __shared__ int s_fold_stop, s_active;
  __shared__ double s_thr;
  // step c's block partials land here by bulk copy while step c+1 sweeps
  constexpr bool kBulkPart = SELECT && !P2P;
  __shared__ __align__(16) double s_part[kBulkPart ? 3 * kMaxCoopBlocks + 2 : 2];
  __shared__ __align__(8) uint64_t s_pbar;
  uint32_t pbar_uses = 0;
  const int pstride = (3 * gridDim.x + 1) & ~1;  // 16-byte aligned slots
  if (kBulkPart && threadIdx.x == 0) mbar_init(&s_pbar, 1);
  Ctl* ctl = a.ctl;
  const int nb = gridDim.x;
  constexpr int kRing = P2P ? 4 : 2;
  if (P2P) {
    if (threadIdx.x == 0) {
      s_dep_lo = INT_MAX;
      s_dep_hi = -1;
    }
    __syncthreads();
    const int64_t lo = (int64_t)blockIdx.x * a.chunk, hi = min(a.n, lo + a.chunk);
    int mn = INT_MAX, mx = -1;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        const int j = ell_j(__ldg(a.E.nbr + eslot(s, a.n, i)));
        mn = min(mn, j);
        mx = max(mx, j);
      }
    if (mx >= 0) {
      atomicMin(&s_dep_lo, (int)(mn / a.chunk));
      atomicMax(&s_dep_hi, (int)(mx / a.chunk));
    }
  }
  if (threadIdx.x == 0) {
    if (SELECT && a.fold) {
      // the mask and the initial totals come out of step 1 (decided at c = 1);
      // sigma_est comes from k_finish_noise, and a noise error stops at once
      const bool dev_ne = a.fold == 2;
      s_st = SelState{0, 0, 0, a.q_max <= 0 || (dev_ne && ctl->nz_err != 0), BUF_Y, BUF_A, BUF_Y,
                      0.0, 0.0};
      s_sv2 = dev_ne ? ctl->sv2 : a.sv2;
      s_thr = dev_ne ? ctl->fslr_thr : a.thr;
      s_active = dev_ne ? ctl->fslr_active : a.active;
      s_qmax = a.q_max;
      s_mode = a.mode;
      s_early = a.early_exit;
      s_mask_all = 0;
    } else if (SELECT) {
      s_st = SelState{ctl->q, ctl->best_q, ctl->streak, ctl->stop, ctl->in_buf, ctl->out_buf,
                      ctl->best_buf, ctl->best_crit, ctl->prev_crit};
      for (int k = 0; k < 3; ++k) s_sy[k] = ctl->sy[k];
      s_sv2 = ctl->sv2;
      s_inc = ctl->included;
      s_qmax = ctl->q_max;
      s_mode = ctl->mode;
      s_early = ctl->early_exit;
      s_mask_all = ctl->mask_all;
    } else {
      s_st = SelState{0, 0, 0, a.fixed_steps <= 0, BUF_Y, BUF_A, BUF_Y, 0.0, 0.0};
      s_qmax = a.fixed_steps;
      s_mask_all = 1;
    }
  }
  __syncthreads();
  float neg_inv_sg2 = 0.0f;
  if (WM != W_STORED) {
    const double sg = ctl->sigma_g;
    neg_inv_sg2 = (float)(-1.0 / (sg * sg));
  }
  int c = s_st.q;  // x_c complete and decided (c = 0 at entry)
  bool decided = true;
  // thread 0: the criterion of x_c from its totals, and the selection update
  auto decide = [&](const double (&t)[3]) {
    const double crit = criterion(s_sy, t, s_inc, s_sv2, s_mode);
    s_st.out_b = s_st.in_b;  // x_c's buffer becomes the best if crit_c improves
    s_st.q = c - 1;
    select_update(s_st, crit, s_qmax, s_early);
    if (blockIdx.x == 0 && c < FGBD_TRACE_MAX) ctl->trace[c] = crit;
  };
  while (!s_st.stop) {
    if (kBulkPart && !decided && threadIdx.x == 0) {
      const uint32_t bytes = (uint32_t)(pstride * 8);
      fence_proxy_async_global();  // the partials were stored before the barrier
      mbar_expect_tx(&s_pbar, bytes);
      bulk_g2s(s_part, a.part + (c & 1) * pstride, bytes, &s_pbar, policy_evict_last());
    }
    // One more non-improving step would stop the scan (early exit): this
    // pass only decides step c, and the same iteration then sweeps c+1 --
    // a stop no longer costs a discarded step.  (s_st is block-uniform.)
    // (its own instantiation: the check in the loop cost scans that never
    // early-exit ~0.3 us per step)
    const bool hold = HOLD && kBulkPart && !decided && s_early && s_st.streak == 2 &&
                      !(a.fold && c == 1);
    const int ib = s_st.in_b, bb = s_st.best_b;
    int ob = BUF_A;
    if (ob == ib || ob == bb) ob = BUF_B;
    if (ob == ib || ob == bb) ob = BUF_Y;
    TLOG(c, 0);
    if (c < s_qmax && !hold) {
      double sx[3] = {0.0, 0.0, 0.0};
      const bool mask_all = s_mask_all != 0;
      if (TMA) {
        sweep_tma<SELECT>(a, pick_buf(a, ib), pick_buf(a, ob), mask_all, tma, sx);
      } else if (SELECT && !P2P && a.fold && c == 0) {
        // step 1 also does k_mask's work (FSLR bits + the initial totals)
        double xs[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        sweep<WM, SELECT, true, FAR>(a, pick_buf(a, ib), pick_buf(a, ob), mask_all, neg_inv_sg2,
                                     sx, s_ell, xs, &s_thr, &s_active);
        block_sum<10>(xs, s_red10);
        if (threadIdx.x == 0)
          for (int k = 0; k < 10; ++k) a.xpart[k * nb + blockIdx.x] = xs[k];
      } else {
        sweep<WM, SELECT, false, FAR>(a, pick_buf(a, ib), pick_buf(a, ob), mask_all, neg_inv_sg2,
                                      sx, s_ell);
      }
#if FGBD_LF_TLOG
      if ((threadIdx.x & 31) == 0 && c < kTlogSteps && (threadIdx.x >> 5) < 16)
        g_wlog[c][blockIdx.x][threadIdx.x >> 5] = gtimer();
#endif
      if (SELECT) {
        block_sum<3>(sx, s_red);
        TLOG(c, 1);
        if (threadIdx.x == 0)
          for (int k = 0; k < 3; ++k)
            a.part[((c + 1) & (kRing - 1)) * (kBulkPart ? pstride : 3 * nb) + k * nb + blockIdx.x] =
                sx[k];
      }
    }
    if (P2P) {  // publish step c + 1 (rows and partials)
      __syncthreads();
      if (threadIdx.x == 0) st_release_u64(a.flags + blockIdx.x, a.base + c + 1);
    }
    constexpr bool kSplit = FGBD_LF_SPLITBAR && !P2P;
    unsigned int gen0 = 0;
    if (kSplit) gen0 = grid_arrive(a.gbar);  // step c+1 is stored: arrive now, wait below
    if (SELECT && !decided) {
      if (P2P) {
        wait_blocks(a.flags, 0, nb - 1, blockIdx.x, a.base + c);
        __syncthreads();
      }
      const double* part = a.part + (c & (kRing - 1)) * 3 * nb;
      double t[3] = {0.0, 0.0, 0.0};
      if (kBulkPart) {
        mbar_wait(&s_pbar, pbar_uses & 1);
        ++pbar_uses;
        for (int b = threadIdx.x; b < nb; b += blockDim.x)
#pragma unroll
          for (int k = 0; k < 3; ++k) t[k] += s_part[k * nb + b];
      } else {
        for (int b = threadIdx.x; b < nb; b += blockDim.x)
#pragma unroll
          for (int k = 0; k < 3; ++k) t[k] += __ldcg(&part[k * nb + b]);
      }
      block_sum<3>(t, s_red);
      if (SELECT && !P2P && a.fold && c == 1) {
        // the FSLR outcome and select_q's initial state (filtering.py:237-243,
        // 289-293) from step 1's totals -- what k_mask's last block does
        double x[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int b = threadIdx.x; b < nb; b += blockDim.x)
#pragma unroll
          for (int k = 0; k < 10; ++k) x[k] += __ldcg(&a.xpart[k * nb + b]);
        block_sum<10>(x, s_red10);
        if (threadIdx.x == 0) {
          long long cnt = (long long)x[0];
          const bool all_ex = (cnt == 0) && s_active;
          if (all_ex) cnt = a.n;
          for (int k = 0; k < 3; ++k) s_sy[k] = all_ex ? x[4 + k] : x[1 + k];
          s_inc = cnt;
          s_mask_all = all_ex;
          const double crit0 = cnt > 0 ? criterion(s_sy, s_sy, cnt, s_sv2, s_mode) : 0.0;
          s_st.best_crit = crit0;
          s_st.prev = crit0;
          s_fold_stop = (crit0 == 0.0) || (cnt < 1);
          if (all_ex)
            for (int k = 0; k < 3; ++k) t[k] = x[7 + k];  // step 1 over every row
          if (blockIdx.x == 0) {
            ctl->trace[0] = crit0;
            ctl->included = cnt;
            ctl->all_excluded = all_ex;
            ctl->mask_all = all_ex;
            for (int k = 0; k < 3; ++k) ctl->sy[k] = s_sy[k];
            ctl->sv2 = s_sv2;
          }
        }
        __syncthreads();
        if (s_mask_all && c < s_qmax) {
          // step 2 was summed under the (all-zero) mask: sum it over every row
          double u[3] = {0.0, 0.0, 0.0};
          rows_sumsq(a, pick_buf(a, ob), u);
          block_sum<3>(u, s_red);
          if (threadIdx.x == 0)
            for (int k = 0; k < 3; ++k)
              a.part[((c + 1) & (kRing - 1)) * (kBulkPart ? pstride : 3 * nb) + k * nb + blockIdx.x] =
                  u[k];
        }
        if (threadIdx.x == 0) {
          if (s_fold_stop) {  // the reference runs no step (filtering.py:243)
            s_st.q = 0;
            s_st.stop = 1;
          } else {
            decide(t);
          }
        }
      } else if (threadIdx.x == 0) {
        decide(t);
      }
      __syncthreads();
    }
    // (a stop is decided identically by every block, and every block has
    // arrived, so leaving here never strands a waiter)
    if (!SELECT && c >= s_qmax) break;
    if (s_st.stop) break;
    if (hold) {  // step c decided: sweep c+1 now (nothing written, no barrier)
      decided = true;
      continue;
    }
    if (P2P) {
      // x_{c+1} of every block this one reads (and that reads this one) is
      // published; the acquire orders this block's next loads after it
      wait_blocks(a.flags, s_dep_lo, s_dep_hi, blockIdx.x, a.base + c + 1);
    } else if (kSplit) {
      TLOG(c, 2);
      grid_wait(a.gbar, gen0);
    } else {
      TLOG(c, 2);
#if FGBD_LF_BAR
      grid_barrier(a.gbar);
#else
      grid.sync();
#endif
    }
    if (threadIdx.x == 0) {
      s_st.in_b = ob;
      s_st.out_b = ob;
      s_st.q = c + 1;
      if (!SELECT) s_st.best_b = ob;
    }
    __syncthreads();
    c += 1;
    decided = false;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->q = s_st.q;
    ctl->steps = s_st.q;
    ctl->best_q = s_st.best_q;
    ctl->best_crit = s_st.best_crit;
    ctl->best_buf = s_st.best_b;
    ctl->in_buf = s_st.in_b;
    ctl->streak = s_st.streak;
    ctl->prev_crit = s_st.prev;
    ctl->stop = 1;
  }
}

// Variant 0 / parity mode: one step per launch, last-block decision.
template <bool W64, bool SELECT>
__global__ void __launch_bounds__(kBlock) k_lf_step(StepArgs a, int fin, int fout) {
  __shared__ double s_red[32 * 3];
  __shared__ bool s_last;
  Ctl* ctl = a.ctl;
  const double4* in;
  double4* out;
  bool mask_all = true;
  if (SELECT) {
    if (*(volatile int*)&ctl->stop) return;
    in = pick_buf(a, ctl->in_buf);
    out = pick_buf(a, ctl->out_buf);
    mask_all = ctl->mask_all != 0;
  } else {
    in = pick_buf(a, fin);
    out = pick_buf(a, fout);
  }
  const int64_t n = a.n;
  double sx[3] = {0.0, 0.0, 0.0};
  const uint64_t pol_stream = graph_policy(), pol_keep = policy_evict_last();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double4 o;
    if (W64) {
      o = row_w64(a, in, i);
    } else {
      int nbr[kSlots];
      float w[kSlots];
      load_row_slots<W_STORED>(a, i, pol_stream, 0.0f, nbr, w);
      o = row_from_slots(nbr, w, in, i, pol_keep);
    }
    st_row(out + i, o);
    if (SELECT && (mask_all || ((a.mask[i >> 5] >> (i & 31)) & 1u))) {
      sx[0] = fma(o.x, o.x, sx[0]);
      sx[1] = fma(o.y, o.y, sx[1]);
      sx[2] = fma(o.z, o.z, sx[2]);
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
      SelState st{ctl->q, ctl->best_q, ctl->streak, ctl->stop, ctl->in_buf, ctl->out_buf,
                  ctl->best_buf, ctl->best_crit, ctl->prev_crit};
      const double crit = criterion(ctl->sy, t, ctl->included, ctl->sv2, ctl->mode);
      select_update(st, crit, ctl->q_max, ctl->early_exit);
      if (st.q < FGBD_TRACE_MAX) ctl->trace[st.q] = crit;
      ctl->q = st.q;
      ctl->steps = st.q;
      ctl->best_q = st.best_q;
      ctl->best_crit = st.best_crit;
      ctl->best_buf = st.best_b;
      ctl->in_buf = st.in_b;
      ctl->out_buf = st.out_b;
      ctl->streak = st.streak;
      ctl->prev_crit = st.prev;
      ctl->stop = st.stop;
      ctl->ticket[2] = 0;
    }
  }
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

// masked sums for selection_criterion: part[7][grid] = count, sy[3], sx[3]
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

static int fill_grid(fgbd_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + kBlock - 1) / kBlock, ctx->num_sms * 8));
}

int launch_expand(fgbd_ctx* ctx, const double* d_src, int64_t n, int buf, cudaStream_t s) {
  k_expand<<<fill_grid(ctx, n), kBlock, 0, s>>>(d_src, n, (double4*)ctx->buf[buf],
                                                ctx->g_reordered ? ctx->rowid : nullptr);
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

int launch_compact(fgbd_ctx* ctx, int64_t n, int src_buf, double* d_dst, int clip) {
  const double4* src = src_buf >= 0 ? (const double4*)ctx->buf[src_buf] : nullptr;
  const int* pos = ctx->g_reordered ? ctx->pos : nullptr;
  if (clip)
    k_compact<true><<<fill_grid(ctx, n), kBlock, 0, ctx->stream>>>(ctx->d_bufs, ctx->ctl, src, n,
                                                                   d_dst, pos);
  else
    k_compact<false><<<fill_grid(ctx, n), kBlock, 0, ctx->stream>>>(ctx->d_bufs, ctx->ctl, src, n,
                                                                    d_dst, pos);
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

int launch_mask(fgbd_ctx* ctx, int64_t n, double sigma_est, int active, int q_max, int mode,
                int early_exit, const uint8_t* d_inc) {
  MaskArgs a;
  a.fslr = ctx->fslr;
  a.y = (const double4*)ctx->buf[BUF_Y];
  a.inc_bytes = d_inc;
  a.n = n;
  a.thr = 2.0 * sigma_est;
  a.active = active;
  a.mask = ctx->mask;
  a.part = ctx->partials;
  a.ctl = ctx->ctl;
  a.q_max = q_max;
  a.mode = mode;
  a.early_exit = early_exit;
  a.sv2 = sigma_est * sigma_est;
  a.defer = 0;
  a.n_total = n;
  k_mask<<<fill_grid(ctx, n), kBlock, 0, ctx->stream>>>(a);
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

// slab rank: own rows, Y at `y`; totals deferred to ctl->mask_part
int launch_mask_slab(fgbd_ctx* ctx, int64_t n_own, const double4* y, double sigma_est,
                     int active) {
  MaskArgs a{};
  a.fslr = ctx->fslr;
  a.y = y;
  a.inc_bytes = nullptr;
  a.n = n_own;
  a.thr = 2.0 * sigma_est;
  a.active = active;
  a.mask = ctx->mask;
  a.part = ctx->partials;
  a.ctl = ctx->ctl;
  a.sv2 = sigma_est * sigma_est;
  a.defer = 1;
  a.n_total = n_own;
  k_mask<<<fill_grid(ctx, n_own), kBlock, 0, ctx->stream>>>(a);
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

static StepArgs step_args(fgbd_ctx* ctx, int64_t n) {
  StepArgs a{};
  a.E = EllRef{ctx->nbr, ctx->pay};
  a.w64 = ctx->w64;
  a.pc = ctx->pc;
  a.bits = ctx->g_bits;
  for (int k = 0; k < 3; ++k) a.buf[k] = (double4*)ctx->buf[k];
  a.mask = ctx->mask;
  a.n = n;
  a.part = ctx->partials;
  a.ctl = ctx->ctl;
  a.rowid = ctx->g_reordered ? ctx->rowid : nullptr;
  a.gbar = ctx->tickets;
  return a;
}

}  // namespace fgbd

// Rows per block: a contiguous range (the graph streams in long runs, and
// rows a slice apart stay in L2 because the whole signal does) while the
// three signal buffers fit in L2; otherwise grid-stride waves, so a row's
// neighbours one z-slice away (k^2 rows) are read by concurrently running
// blocks and hit L2 (8M lattice: 13.7 -> 9.6 ms for 64 steps).
bool fgbd::lf_contiguous(const fgbd_ctx* ctx, int64_t rows) {
  if (ctx->lf_chunk >= 0) return ctx->lf_chunk != 0;
  return (double)rows * 32.0 * 3.0 <= (double)ctx->l2_bytes;
}

namespace fgbd {

template <int WM, bool SELECT, int BLK, int MINB, bool TMA = false, bool P2P = false,
          int FAR = 0, bool HOLD = false>
static int launch_run_k(fgbd_ctx* ctx, StepArgs& a, int slot) {
  auto kern = k_lf_run<WM, SELECT, BLK, MINB, TMA, P2P, FAR, HOLD>;
  constexpr int kEllSmem = (FGBD_LF_ELLSMEM && WM == W_STORED) ? (FGBD_LF_ELLSMEM + 1) * 3 * BLK * 16 : 0;
  const int smem = TMA ? kTmaSmem : kEllSmem;
  if (ctx->coop_blocks[slot] == 0) {
    if (TMA || kEllSmem > 0) {
      FGBD_CUDA(ctx, cudaFuncSetAttribute((const void*)kern,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      if (TMA)
        FGBD_CUDA(ctx, cudaFuncSetAttribute((const void*)kern,
                                            cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    int per_sm = 0;
    FGBD_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BLK, smem));
    ctx->coop_blocks[slot] = std::max(1, per_sm) * ctx->num_sms;
  }
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>(std::min<int64_t>((a.n + BLK - 1) / BLK, ctx->coop_blocks[slot]),
                           kMaxCoopBlocks));
  a.chunk = (TMA || P2P || lf_contiguous(ctx, a.n)) ? ((a.n + grid - 1) / grid + BLK - 1) / BLK * BLK
                                                     : 0;
  a.halo = std::min(ctx->lf_halo, kHaloMax);
  if (P2P) {
    if (!ctx->p2p_flags) {
      FGBD_CUDA(ctx, cudaMalloc(&ctx->p2p_flags, 8192 * sizeof(unsigned long long)));
      FGBD_CUDA(ctx, cudaMemset(ctx->p2p_flags, 0, 8192 * sizeof(unsigned long long)));
    }
    a.flags = ctx->p2p_flags;
    a.base = ctx->p2p_epoch;
    ctx->p2p_epoch += 1ull << 20;
  }
  void* args[] = {&a};
  FGBD_CUDA(ctx, cudaLaunchCooperativeKernel((void*)kern, grid, BLK, args, smem, ctx->stream));
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

// block shape of the persistent kernel (FGBD_LF_SHAPE): 0 = 256 x 3/SM,
// 1 = 256 x 4/SM (64 registers), 2 = 288 x 3/SM (75 registers), 3 = 256 x 2/SM (128 registers)
template <int WM, bool SELECT>
static int launch_run(fgbd_ctx* ctx, StepArgs& a) {
  const int base = (WM * 2 + (SELECT ? 1 : 0)) * 4 + ctx->lf_shape;
  switch (ctx->lf_shape) {
    case 1: return launch_run_k<WM, SELECT, 256, 4>(ctx, a, base);
    case 2: return launch_run_k<WM, SELECT, 288, 3>(ctx, a, base);
    case 3: return launch_run_k<WM, SELECT, 256, 2>(ctx, a, base);
    default: return launch_run_k<WM, SELECT, 256, 3>(ctx, a, base);
  }
}

// Weight source for the persistent kernels: variant 11 recomputes them from
// the packed coordinates, otherwise the stored fp32 weights are read.
template <bool SELECT>
static int launch_run_any(fgbd_ctx* ctx, StepArgs& a) {
  if (ctx->lf_variant == 11)
    return 3 * ctx->g_bits <= 32 ? launch_run<W_COORDS32, SELECT>(ctx, a)
                                 : launch_run<W_COORDS64, SELECT>(ctx, a);
  if (ctx->lf_variant == 12)  // TMA-staged row tiles (slot 40 + SELECT)
    return launch_run_k<W_STORED, SELECT, kTile, 3, true>(ctx, a, 40 + (SELECT ? 1 : 0));
  if (ctx->lf_variant == 13)  // neighbourhood flags instead of the grid barrier
    return launch_run_k<W_STORED, SELECT, kBlock, 3, false, true>(ctx, a, 42 + (SELECT ? 1 : 0));
  if (ctx->lf_far_now && ctx->lf_shape == 0)  // mostly scattered gathers: far ones skip L1
    return launch_run_k<W_STORED, SELECT, kBlock, 3, false, false, kFarRows>(ctx, a,
                                                                             44 + (SELECT ? 1 : 0));
  return launch_run<W_STORED, SELECT>(ctx, a);
}

int launch_select_steps(fgbd_ctx* ctx, int64_t n, int q_max, int w64) {
  StepArgs a = step_args(ctx, n);
  if (ctx->lf_variant == 0 || w64) {
    const int grid = red_grid(n);
    for (int q = 0; q < q_max; ++q) {
      if (w64) k_lf_step<true, true><<<grid, kBlock, 0, ctx->stream>>>(a, 0, 0);
      else k_lf_step<false, true><<<grid, kBlock, 0, ctx->stream>>>(a, 0, 0);
      FGBD_LAUNCH(ctx);
    }
    return FGBD_OK;
  }
  return launch_run_any<true>(ctx, a);
}

// select_q with k_mask folded into step 1 (default filter kernel only)
bool mask_foldable(const fgbd_ctx* ctx, int q_max, int w64) {
  return ctx->mask_fold && ctx->lf_variant == 10 && !w64 && q_max >= 1;
}

int launch_select_steps_folded(fgbd_ctx* ctx, int64_t n, int q_max, int mode, int early_exit,
                               const double* sigma_est, int active) {
  StepArgs a = step_args(ctx, n);
  // sigma_est given: the host finished NE; null: k_finish_noise left it in ctl
  a.fold = sigma_est ? 1 : 2;
  if (sigma_est) {
    a.sv2 = *sigma_est * *sigma_est;
    a.thr = 2.0 * *sigma_est;
    a.active = active;
  }
  a.fslr = ctx->fslr;
  a.xpart = ctx->partials + (1 << 18);  // 10 x grid, clear of the step partials
  a.q_max = q_max;
  a.mode = mode;
  a.early_exit = early_exit;
  // the early-exit variant when this context's last scan stopped early
  if (ctx->hold_guess && early_exit && ctx->lf_shape == 0)
    return ctx->lf_far_now
               ? launch_run_k<W_STORED, true, kBlock, 3, false, false, kFarRows, true>(ctx, a, 49)
               : launch_run_k<W_STORED, true, kBlock, 3, false, false, 0, true>(ctx, a, 48);
  if (ctx->lf_far_now && ctx->lf_shape == 0)
    return launch_run_k<W_STORED, true, kBlock, 3, false, false, kFarRows>(ctx, a, 45);
  return launch_run<W_STORED, true>(ctx, a);
}

int launch_fixed_steps(fgbd_ctx* ctx, int64_t n, int q, int w64, int* final_buf) {
  *final_buf = q == 0 ? BUF_Y : ((q & 1) ? BUF_A : BUF_B);
  if (q == 0) return FGBD_OK;
  StepArgs a = step_args(ctx, n);
  if (ctx->lf_variant == 0 || w64) {
    const int grid = red_grid(n);
    int cur = BUF_Y;
    for (int k = 0; k < q; ++k) {
      const int nxt = (cur == BUF_A) ? BUF_B : BUF_A;
      if (w64) k_lf_step<true, false><<<grid, kBlock, 0, ctx->stream>>>(a, cur, nxt);
      else k_lf_step<false, false><<<grid, kBlock, 0, ctx->stream>>>(a, cur, nxt);
      FGBD_LAUNCH(ctx);
      cur = nxt;
    }
    return FGBD_OK;
  }
  a.fixed_steps = q;
  return launch_run_any<false>(ctx, a);
}

int launch_csr_steps(fgbd_ctx* ctx, const int64_t* d_indptr, const int64_t* d_indices,
                     const double* d_w, int64_t n, const double* d_in, double* d_tmp,
                     double* d_out, int q) {
  const int grid = fill_grid(ctx, n);
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

#if FGBD_LF_TLOG
extern "C" int fgbd_debug_tlog(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, fgbd::g_tlog, sizeof(fgbd::g_tlog));
}
extern "C" int fgbd_debug_wlog(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, fgbd::g_wlog, sizeof(fgbd::g_wlog));
}
#endif
