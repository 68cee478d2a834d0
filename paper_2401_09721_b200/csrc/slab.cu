// Spatial slab partition of ONE frame over P ranks.
//
// The frame is cut into z-slabs (the z-major scan-line-1 order makes every
// slab a contiguous range of global rows).  Each rank uploads, sorts and
// filters ONLY its own points; everything crosses slab boundaries through
// peer memory (CUDA IPC + NVLink on P GPUs, plain device memory when the P
// ranks are emulated on one GPU):
//
//  1. graph: each rank sorts its points along the 3 scan lines and publishes,
//     per line, its block list (first / last point of every run sharing the
//     line's key above z).  Cross-slab neighbours are the first / last points
//     of (key, rank)-adjacent blocks: every rank derives its own exactly from
//     the peers' lists (wraparounds included), copying the foreign endpoints
//     in as halo records (k_resolve, csrc/graph.cu);
//  2. sigma_g: each rank's exact fixed-point share (csrc/device_util.cuh fx52)
//     -> all-gather -> the same bits as the single-GPU sum;
//  3. NE-GBP: own patches; a foreign patch neighbour's colour is a P2P load
//     from its owner's signal buffer; the 3 x 64 moment sums -> all-gather,
//     summed in rank order, so every rank runs the host Jacobi on the same
//     bits and selects with the same sigma_est;
//  4. FSLR: own mask bits; included count and sum y^2 -> all-gather;
//  5. the q scan (k_lf_slab): one persistent launch per rank; halo signals
//     are P2P loads of the owner's current buffer; the criterion sum goes
//     through per-rank slots + release/acquire flags each step;
//  6. output: own rows -> own points (or pushed into every rank's full frame,
//     followed by one more all-rank tick before anyone reads it).
//
// The all-gathers are k_sync_publish (store this rank's vector into slot r
// of every rank, then a release flag) + k_sync_finalize (acquire all flags,
// reduce in rank order).  Ticks are (frame epoch << 8 | stage), vector slots
// alternate by stage parity, and every stage's reads finish before the rank
// publishes the next stage, so no slot is overwritten while a peer reads it.
// A peer's signal buffers are read only between the block-list tick (its Y
// is complete) and the last step tick of the q scan (every rank has finished
// reading), so the next frame cannot overwrite a buffer a peer still reads.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "device_util.cuh"
#include "fgbd_internal.cuh"
#include "select_state.cuh"

namespace cg = cooperative_groups;

namespace fgbd {

constexpr int kVec = 256;  // doubles per rank per all-gather stage

enum SyncStage { ST_BLOCKS = 1, ST_SIGMA = 2, ST_NOISE = 3, ST_MASK = 4, ST_OUT = 5 };

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// ---------------------------------------------------------------------------
// all-gather of small per-rank vectors
// ---------------------------------------------------------------------------

struct SyncRef {
  int world, rank;
  unsigned long long* flags[kMaxRanks];  // every rank's [P] stage ticks
  double* vec[kMaxRanks];                // every rank's [2][P][kVec] slots
  Ctl* ctl;                              // this rank's control block
};

struct FinArgs {
  int64_t n_total;
  int active, q_max, mode, early_exit;
  double sv2;
};

__device__ __forceinline__ double u64_as_d(unsigned long long v) {
  return __longlong_as_double((long long)v);
}
__device__ __forceinline__ unsigned long long d_as_u64(double v) {
  return (unsigned long long)__double_as_longlong(v);
}

// this rank's share of `stage` -> slot `rank` of every rank, then the tick
__global__ void __launch_bounds__(kBlock) k_sync_publish(SyncRef s, int stage,
                                                        unsigned long long tick) {
  const Ctl* c = s.ctl;
  const int par = (int)(tick & 1ull);
  int nv = 0;
  if (stage == ST_SIGMA) nv = 5;
  else if (stage == ST_NOISE) nv = 3 * 64;
  else if (stage == ST_MASK) nv = 7;
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    double x = 0.0;
    if (stage == ST_SIGMA) {
      const unsigned long long u[5] = {c->sg_fx[0], c->sg_fx[1], c->n_edges,
                                       (unsigned long long)c->max_deg,
                                       (unsigned long long)c->err_flags};
      x = u64_as_d(u[v]);
    } else if (stage == ST_NOISE) {
      x = c->gram[v / 64][v % 64];
    } else {
      x = c->mask_part[v];
    }
    for (int p = 0; p < s.world; ++p) s.vec[p][(par * s.world + s.rank) * kVec + v] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < s.world; ++p) st_release_sys(s.flags[p] + s.rank, tick);
  }
}

// wait for every rank's tick, then reduce the stage's vectors in rank order
__global__ void __launch_bounds__(kBlock) k_sync_finalize(SyncRef s, int stage,
                                                         unsigned long long tick, FinArgs f) {
  Ctl* c = s.ctl;
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    for (int p = 0; p < s.world; ++p)
      while (ld_acquire_sys(s.flags[s.rank] + p) < tick) {
        if (clock64() - t0 > (1ll << 35)) {  // ~17 s: a peer died; report, never hang
          atomicOr(&c->err_flags, 4);
          break;
        }
      }
  }
  __syncthreads();
  const int par = (int)(tick & 1ull);
  const double* v = s.vec[s.rank] + par * s.world * kVec;
  if (stage == ST_SIGMA) {
    if (threadIdx.x == 0) {
      u128 sum = 0;
      unsigned long long cnt = 0, err = 0;
      int maxdeg = 0;
      for (int p = 0; p < s.world; ++p) {
        const double* w = v + p * kVec;
        sum += ((u128)d_as_u64(w[1]) << 64) | d_as_u64(w[0]);
        cnt += d_as_u64(w[2]);
        maxdeg = max(maxdeg, (int)d_as_u64(w[3]));
        err |= d_as_u64(w[4]);
      }
      c->n_edges = cnt;
      c->sigma_g = cnt ? fx52_to_double(sum) / (double)cnt : 0.0;
      c->max_deg = maxdeg;
      c->err_flags |= (int)(err & 1ull);
    }
  } else if (stage == ST_NOISE) {
    for (int k = threadIdx.x; k < 3 * 64; k += blockDim.x) {
      double t = 0.0;
      for (int p = 0; p < s.world; ++p) t += v[p * kVec + k];
      c->gram[k / 64][k % 64] = t;
      if (k == 63) c->eligible = (long long)t;
    }
  } else if (stage == ST_MASK) {
    if (threadIdx.x == 0) {
      double t[7] = {0, 0, 0, 0, 0, 0, 0};
      for (int p = 0; p < s.world; ++p)
        for (int k = 0; k < 7; ++k) t[k] += v[p * kVec + k];
      mask_finalize(c, t, f.n_total, false, f.active, f.q_max, f.mode, f.early_exit, f.sv2);
    }
  }
}

// ---------------------------------------------------------------------------
// the q scan over the slab ranks
// ---------------------------------------------------------------------------

struct SlabGroup {  // one logical rank of this launch
  EllRef E;
  int64_t n_own;
  const uint32_t* mask;
  Ctl* ctl;
};

constexpr int kSlabMaxBlocks = 592;  // cooperative grid cap (148 SMs x 4)

struct SlabArgs {
  int world;   // P
  int rank0;   // global rank of this launch's first group
  int groups;  // logical ranks in this launch
  int bpg;     // blocks per group
  int64_t lo[kMaxRanks + 1];
  double4* bufs[kMaxRanks][3];           // every rank's Y/A/B by GLOBAL row (base - lo[r])
  double* slots[kMaxRanks];              // every rank's [2][P][4] criterion slots
  unsigned long long* flags[kMaxRanks];  // every rank's [P] step ticks
  unsigned long long* release;           // local: "every rank finished step c" for this launch
  double* part;                          // local [2][pstride] block partials (k_lf_run layout)
  SlabGroup grp[kMaxRanks];
  unsigned long long epoch;  // frame epoch: step ticks are epoch << 32 | step
  int fixed_steps;           // cached path when > 0 (no criterion)
  int select;
  int contiguous;            // rows per block: contiguous range (1) or grid-stride waves (0)
  int exchange;              // per-step rank totals + ticks through peer memory (ranks span
                             // GPUs; forced on one GPU to test the protocol)
};

__device__ __forceinline__ int owner_of(const SlabArgs& a, int64_t j) {
  int r = 0;
#pragma unroll 1
  while (r + 1 < a.world && j >= a.lo[r + 1]) ++r;
  return r;
}

// The q scan of the slab ranks (filtering.py:225-256), built like k_lf_run
// (csrc/filter.cu): a cooperative persistent launch, graph rows landed by
// cp.async one sweep iteration ahead, the select_q decision lagged one step
// and taken from block partials bulk-copied into shared memory during the
// next sweep, one grid barrier per step.  Own rows are addressed by global
// row; a foreign neighbour is read from its owner's buffer.
//
// When this launch holds every rank (one GPU; the emulation) the grid
// barrier is the global barrier and the partials of all blocks are the
// global total.  When the ranks span GPUs (`exchange`), after each grid
// barrier the first block of each rank's group reduces the rank's partials,
// stores the total into slot r of every rank, publishes the step tick and
// waits for every rank's tick (so every halo row of the step is written and
// every rank's total has landed), then releases this GPU's blocks; the
// lagged decision then sums the P slots in rank order.
__global__ void __launch_bounds__(kBlock, 3) k_lf_slab(SlabArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) int4 s_ell[];  // [2 stages][3 pairs][kBlock]
  __shared__ double s_red[32 * 3];
  __shared__ __align__(16) double s_part[3 * kSlabMaxBlocks + 2];
  __shared__ __align__(8) uint64_t s_pbar;
  __shared__ SelState s_st;
  __shared__ double s_sy[3], s_sv2;
  __shared__ long long s_inc;
  __shared__ int s_qmax, s_mode, s_early, s_mask_all;
  const int g = blockIdx.x / a.bpg, lb = blockIdx.x % a.bpg;
  const int r = a.rank0 + g;
  const int P = a.world, nb = gridDim.x;
  const bool exchange = a.exchange != 0;
  const bool bulk = a.select && !exchange;  // every rank's blocks are in this launch
  const int pstride = (3 * nb + 1) & ~1;
  uint32_t pbar_uses = 0;
  const SlabGroup G = a.grp[g];
  Ctl* ctl = G.ctl;
  if (threadIdx.x == 0) {
    if (bulk) mbar_init(&s_pbar, 1);
    if (a.select) {
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
  const int64_t lo = a.lo[r], n_own = G.n_own;
  const int64_t chunk = ((n_own + a.bpg - 1) / a.bpg + blockDim.x - 1) / blockDim.x * blockDim.x;
  const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
  int c = s_st.q;  // x_c complete and decided (c = 0 at entry)
  bool decided = true;
  auto decide = [&](const double (&t)[3]) {
    const double crit = criterion(s_sy, t, s_inc, s_sv2, s_mode);
    s_st.out_b = s_st.in_b;  // x_c's buffer becomes the best if crit_c improves
    s_st.q = c - 1;
    select_update(s_st, crit, s_qmax, s_early);
    if (lb == 0 && c < FGBD_TRACE_MAX) ctl->trace[c] = crit;
  };
  while (!s_st.stop) {
    if (bulk && !decided && threadIdx.x == 0) {
      const uint32_t bytes = (uint32_t)(pstride * 8);
      fence_proxy_async_global();  // the partials were stored before the barrier
      mbar_expect_tx(&s_pbar, bytes);
      bulk_g2s(s_part, a.part + (c & 1) * pstride, bytes, &s_pbar, policy_evict_last());
    }
    const int ib = s_st.in_b, bb = s_st.best_b;
    int ob = BUF_A;
    if (ob == ib || ob == bb) ob = BUF_B;
    if (ob == ib || ob == bb) ob = BUF_Y;
    if (c < s_qmax) {
      double sx[3] = {0.0, 0.0, 0.0};
      const double4* own_in = a.bufs[r][ib];
      double4* out = a.bufs[r][ob];
      const bool mask_all = s_mask_all != 0;
      // own (local) rows: a contiguous share, or grid-stride waves over the
      // group when the signals do not fit in L2 (see fgbd::lf_contiguous)
      int64_t i = a.contiguous ? (int64_t)lb * chunk + threadIdx.x
                               : (int64_t)lb * blockDim.x + threadIdx.x;
      const int64_t end = a.contiguous ? min(n_own, (int64_t)(lb + 1) * chunk) : n_own;
      const int64_t rstep = a.contiguous ? (int64_t)blockDim.x : (int64_t)a.bpg * blockDim.x;
      const int T = blockDim.x;
      int stage = 0;
      auto issue = [&](int64_t row, int st) {
        if (row < end)
#pragma unroll
          for (int s = 0; s < kSlots; s += 2)
            asm volatile(
                "cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(
                    smem_u32(s_ell + (st * 3 + (s >> 1)) * T + threadIdx.x)),
                "l"(G.E.nbr + eslot(s, n_own, row)), "l"(pol_stream)
                : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      issue(i, 0);
      while (i < end) {
        const int64_t inext = i + rstep;
        issue(inext, stage ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        int nbs[kSlots];
        float w[kSlots];
#pragma unroll
        for (int s = 0; s < kSlots; s += 2) {
          const int4 pr = s_ell[(stage * 3 + (s >> 1)) * T + threadIdx.x];
          nbs[s] = pr.x;  // GLOBAL row | below-flag (bit 31)
          w[s] = __int_as_float(pr.y);
          nbs[s + 1] = pr.z;
          w[s + 1] = __int_as_float(pr.w);
        }
        stage ^= 1;
        if (i + 2 * rstep < end)
#pragma unroll
          for (int s = 0; s < kSlots; s += 2) prefetch_l2(G.E.nbr + eslot(s, n_own, i + 2 * rstep));
        const int64_t gi = lo + i;
        const double4 f = ld_row_hint(own_in + gi, pol_keep);
        double4 gv[kSlots];
#pragma unroll
        for (int s = 0; s < kSlots; ++s) {
          const int64_t j = ell_j(nbs[s]);
          FGBD_DCHECK(j >= 0 && j < a.lo[P]);
          const double4* src = own_in;
          if (__builtin_expect((uint64_t)(j - lo) >= (uint64_t)n_own, 0))
            src = a.bufs[owner_of(a, j)][ib];  // halo: the owner's buffer (peer memory)
          gv[s] = ld_row_hint(src + j, pol_keep);
        }
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, dlo = 0.0, dhi = 0.0;
#pragma unroll
        for (int s = 0; s < kSlots; ++s) {
          // (sum over original j > i) + (sum over j < i); padding adds +0.0
          const double ws = (double)w[s];
          const bool below = ell_below(nbs[s]);
          dlo = __dadd_rn(dlo, below ? ws : 0.0);
          dhi = __dadd_rn(dhi, below ? 0.0 : ws);
          acc0 = __dadd_rn(acc0, __dmul_rn(ws, gv[s].x));
          acc1 = __dadd_rn(acc1, __dmul_rn(ws, gv[s].y));
          acc2 = __dadd_rn(acc2, __dmul_rn(ws, gv[s].z));
        }
        const double d = __dadd_rn(dhi, dlo);
        double4 o = f;
        if (d != 0.0) {
          const double d2 = __dmul_rn(2.0, d);
          o = make_double4(__ddiv_rn(__dadd_rn(__dmul_rn(d, f.x), acc0), d2),
                           __ddiv_rn(__dadd_rn(__dmul_rn(d, f.y), acc1), d2),
                           __ddiv_rn(__dadd_rn(__dmul_rn(d, f.z), acc2), d2), 0.0);
        }
        st_row_hint(out + gi, o, pol_keep);
        if (a.select && (mask_all || ((G.mask[i >> 5] >> (i & 31)) & 1u))) {
          sx[0] = fma(o.x, o.x, sx[0]);
          sx[1] = fma(o.y, o.y, sx[1]);
          sx[2] = fma(o.z, o.z, sx[2]);
        }
        i = inext;
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      if (a.select) {
        block_sum<3>(sx, s_red);
        if (threadIdx.x == 0)
          for (int k = 0; k < 3; ++k) a.part[((c + 1) & 1) * pstride + k * nb + blockIdx.x] = sx[k];
      }
    }
    if (a.select && !decided) {
      double t[3] = {0.0, 0.0, 0.0};
      if (bulk) {  // every rank's blocks are in this launch: sum them all
        mbar_wait(&s_pbar, pbar_uses & 1);
        ++pbar_uses;
        for (int b = threadIdx.x; b < nb; b += blockDim.x)
#pragma unroll
          for (int k = 0; k < 3; ++k) t[k] += s_part[k * nb + b];
        block_sum<3>(t, s_red);
      } else if (threadIdx.x == 0) {  // the ranks' totals, in rank order
        for (int p = 0; p < P; ++p)
          for (int k = 0; k < 3; ++k) t[k] += ld_cg(a.slots[r] + ((c & 1) * P + p) * 4 + k);
      }
      if (threadIdx.x == 0) decide(t);
      __syncthreads();
    }
    if (!a.select && c >= s_qmax) break;
    if (s_st.stop) break;
    grid.sync();  // this GPU's rows (and partials) of step c+1 are written
    if (exchange) {
      const unsigned long long tick = (a.epoch << 32) | (unsigned long long)(c + 1);
      if (lb == 0) {
        double t[3] = {0.0, 0.0, 0.0};
        if (a.select) {
          for (int b = threadIdx.x; b < a.bpg; b += blockDim.x)
            for (int k = 0; k < 3; ++k)
              t[k] += ld_cg(a.part + ((c + 1) & 1) * pstride + k * nb + g * a.bpg + b);
          block_sum<3>(t, s_red);
        }
        if (threadIdx.x == 0) {
          for (int p = 0; p < P; ++p)
            for (int k = 0; k < 3; ++k) a.slots[p][(((c + 1) & 1) * P + r) * 4 + k] = t[k];
          __threadfence_system();
          for (int p = 0; p < P; ++p) st_release_sys(a.flags[p] + r, tick);
          const long long t0 = clock64();
          for (int p = 0; p < P; ++p)
            while (ld_acquire_sys(a.flags[r] + p) < tick) {
              if (clock64() - t0 > (1ll << 35)) {  // a peer died: report, do not hang
                atomicOr(&ctl->err_flags, 4);
                break;
              }
            }
          st_release_sys(a.release, tick);  // (every group's leader writes the same tick)
        }
      } else if (threadIdx.x == 0) {
        const long long t0 = clock64();
        while (ld_acquire_sys(a.release) < tick) {
          if (clock64() - t0 > (1ll << 35)) {
            atomicOr(&ctl->err_flags, 4);
            break;
          }
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      s_st.in_b = ob;
      s_st.out_b = ob;
      s_st.q = c + 1;
      if (!a.select) s_st.best_b = ob;
    }
    __syncthreads();
    c += 1;
    decided = false;
  }
  if (lb == 0 && threadIdx.x == 0) {
    ctl->q = s_st.q;
    ctl->steps = s_st.q;
    ctl->best_q = s_st.best_q;
    ctl->best_crit = s_st.best_crit;
    ctl->best_buf = s_st.best_b;
    ctl->in_buf = s_st.in_b;
    ctl->stop = 1;
  }
}

// Own rows -> own points (clipped), and with `full` also into every rank's
// full-frame output at the points' global indices (P2P stores).
struct OutArgs {
  const double4* bufs[3];  // this rank's buffers by GLOBAL row
  const Ctl* ctl;
  int64_t lo, n_own;
  const uint32_t* rowid;   // own row -> own point
  const uint32_t* gidx;    // own point -> global index
  double* dst;             // (n_own, 3) own points
  int world;
  double* full[kMaxRanks]; // (n_total, 3) per rank, or null
};

__global__ void __launch_bounds__(kBlock) k_slab_out(OutArgs a) {
  const double4* src = a.bufs[a.ctl->best_buf];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n_own; i += stride) {
    const double4 v = ld_row(src + a.lo + i);
    const double o[3] = {fmin(fmax(v.x, 0.0), 255.0), fmin(fmax(v.y, 0.0), 255.0),
                         fmin(fmax(v.z, 0.0), 255.0)};
    const int64_t p = a.rowid[i];
    for (int c = 0; c < 3; ++c) a.dst[3 * p + c] = o[c];
    if (a.full[0]) {
      const int64_t gp = a.gidx[p];
      for (int q = 0; q < a.world; ++q)
        for (int c = 0; c < 3; ++c) a.full[q][3 * gp + c] = o[c];
    }
  }
}

// (n,3) colours -> (n,4) rows at global row lo + k for own row k (point rowid[k])
__global__ void __launch_bounds__(kBlock) k_slab_expand(const double* __restrict__ src, int64_t n,
                                                        double4* __restrict__ dst_global,
                                                        int64_t lo,
                                                        const uint32_t* __restrict__ rowid) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    const int64_t p = rowid[k];
    st_row(dst_global + lo + k, make_double4(src[3 * p], src[3 * p + 1], src[3 * p + 2], 0.0));
  }
}

}  // namespace fgbd

using namespace fgbd;

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

namespace {

// Region of one rank (peer-visible, identical layout on every rank).
struct Layout {
  size_t bufs[3], lf_slots, lf_flags, sync_flags, vec, hdr, sums[3], full, total;
};

Layout make_layout(int64_t cap_rows, int world, int64_t blk_cap, int64_t n_full) {
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  Layout L{};
  size_t off = 0;
  for (int k = 0; k < 3; ++k) {
    L.bufs[k] = off;
    off += al((size_t)cap_rows * 32);
  }
  L.lf_slots = off;
  off += al((size_t)2 * world * 4 * 8);
  L.lf_flags = off;
  off += al((size_t)world * 8);
  L.sync_flags = off;
  off += al((size_t)world * 8);
  L.vec = off;
  off += al((size_t)2 * world * kVec * 8);
  L.hdr = off;
  off += al(8 * 8);
  for (int l = 0; l < 3; ++l) {
    L.sums[l] = off;
    off += al((size_t)blk_cap * sizeof(SumRec));
  }
  L.full = off;
  off += al((size_t)n_full * 24);
  L.total = off;
  return L;
}

}  // namespace

struct fgbd_slab {
  int world = 1, rank = 0;
  bool emulated = false;
  int full = 0;                 // keep a full-frame output buffer per rank
  int64_t cap_rows = 0, blk_cap = 0, n_total = 0;
  int groups = 1;               // logical ranks run by this process
  Layout L{};
  char* base[kMaxRanks] = {};   // every rank's region (peer-mapped for foreign ranks)
  void* peer_base[kMaxRanks] = {};  // opened IPC mappings
  struct Local {
    fgbd_ctx* ctx = nullptr;    // emulated: a sub-context on the parent's stream
    bool own_ctx = false;
    void* region = nullptr;
    void* ext = nullptr;        // ext_pc | ext_pos | ext_gidx | tile_cnt
    SlabGC g{};
  } loc[kMaxRanks];
  int force_exchange = 0;                 // FGBD_SLAB_EXCHANGE: the P-GPU protocol on one GPU
  unsigned long long* release = nullptr;  // k_lf_slab: "every rank finished the step"
  double* part = nullptr;                 // k_lf_slab block partials [2][3 * blocks]
  int bpg_cap = 0;
  unsigned long long epoch = 1;  // frame counter (incremented at the start of each frame)
  cudaEvent_t rev[kMaxRanks][10] = {};  // per local rank: start/end of its phases
};

namespace {

template <typename T>
T* at(char* base, size_t off) {
  return reinterpret_cast<T*>(base + off);
}

int64_t ext_rows(int64_t cap_rows, int64_t blk_cap) { return cap_rows + 2 * (1 + 2 * blk_cap); }

SyncRef sync_ref(fgbd_slab* s, int r, Ctl* ctl) {
  SyncRef x{};
  x.world = s->world;
  x.rank = r;
  for (int p = 0; p < s->world; ++p) {
    x.flags[p] = at<unsigned long long>(s->base[p], s->L.sync_flags);
    x.vec[p] = at<double>(s->base[p], s->L.vec);
  }
  x.ctl = ctl;
  return x;
}

unsigned long long stage_tick(const fgbd_slab* s, int stage) {
  return (s->epoch << 8) | (unsigned long long)stage;
}

int publish(fgbd_slab* s, int g, int stage) {
  fgbd_ctx* ctx = s->loc[g].ctx;
  k_sync_publish<<<1, kBlock, 0, ctx->stream>>>(sync_ref(s, s->loc[g].g.rank, ctx->ctl), stage,
                                                stage_tick(s, stage));
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

int finalize(fgbd_slab* s, int g, int stage, const FinArgs& f) {
  fgbd_ctx* ctx = s->loc[g].ctx;
  k_sync_finalize<<<1, kBlock, 0, ctx->stream>>>(sync_ref(s, s->loc[g].g.rank, ctx->ctl), stage,
                                                 stage_tick(s, stage), f);
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

// publish `stage` on every local rank, then wait + reduce on every local rank
// (emulated ranks share one stream: all publishes precede all waits)
int all_gather(fgbd_ctx* parent, fgbd_slab* s, int stage, const FinArgs& f) {
  for (int g = 0; g < s->groups; ++g)
    if (publish(s, g, stage)) return set_error(parent, FGBD_E_CUDA, s->loc[g].ctx->err);
  for (int g = 0; g < s->groups; ++g)
    if (finalize(s, g, stage, f)) return set_error(parent, FGBD_E_CUDA, s->loc[g].ctx->err);
  return FGBD_OK;
}

int pull(fgbd_ctx* ctx) {
  FGBD_CUDA(ctx, cudaMemcpyAsync(ctx->ctl_host, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost,
                                 ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FGBD_OK;
}

int alloc_local(fgbd_ctx* parent, fgbd_slab* s, int g) {
  auto& lc = s->loc[g];
  FGBD_CUDA(parent, cudaMalloc(&lc.region, s->L.total));
  FGBD_CUDA(parent, cudaMemset(lc.region, 0, s->L.total));
  const int64_t ext = ext_rows(s->cap_rows, s->blk_cap);
  const int64_t tiles = s->cap_rows / 2048 + 2;
  const size_t bytes = (size_t)ext * (8 + 4 + 4) + (size_t)2 * (tiles + 1) * 4 + 256;
  FGBD_CUDA(parent, cudaMalloc(&lc.ext, bytes));
  char* e = (char*)lc.ext;
  lc.g.ext_pc = e;
  lc.g.ext_pos = reinterpret_cast<int*>(e + (size_t)ext * 8);
  lc.g.ext_gidx = reinterpret_cast<uint32_t*>(e + (size_t)ext * 12);
  lc.g.tile_cnt = reinterpret_cast<unsigned int*>(e + (size_t)ext * 16);
  return FGBD_OK;
}

double ev_sec(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();
    return 0.0;
  }
  return ms * 1e-3;
}

std::mutex& slab_device_mutex(int device) {
  static std::mutex m[64];
  return m[device & 63];
}

// one frame over the slab ranks; the inputs of this process's logical ranks
// are concatenated in rank order (emulated) or are this rank's own points
int slab_frame(fgbd_ctx* parent, fgbd_slab* s, const int64_t* coords, const double* colors,
               const uint32_t* gidx, int64_t gidx_base, const int64_t* counts, int bits,
               const fgbd_config* cfg, int cached_q, double cached_sigma, double* out_colors,
               fgbd_report* rep, uint32_t flags) {
  const int P = s->world;
  int64_t lo[kMaxRanks + 1];
  lo[0] = 0;
  for (int r = 0; r < P; ++r) {
    if (counts[r] < 1)
      return set_error(parent, FGBD_E_ARG, "every slab rank needs at least one point");
    if (counts[r] > s->cap_rows)
      return set_error(parent, FGBD_E_ARG,
                       "slab rank has more points than the slab was created for");
    lo[r + 1] = lo[r] + counts[r];
  }
  if (lo[P] != s->n_total)
    return set_error(parent, FGBD_E_ARG, "slab counts do not sum to n_total");
  const int b = bits;
  if (b > 15) return set_error(parent, FGBD_E_ARG, "slab partition supports bit depths up to 15");
  const bool timing = !(flags & FGBD_FLAG_NO_TIMING);
  cudaEvent_t* ev = parent->ev;
  std::lock_guard<std::mutex> lock(slab_device_mutex(parent->device));
  NvtxRange nv_frame("fgbd.denoise_slab");
  // a fresh epoch per call, taken before anything can fail: a frame that
  // stops early never leaves ticks the next frame could mistake for its own
  // (every rank makes the same calls, so the epochs agree)
  s->epoch += 1;
  if (timing) FGBD_CUDA(parent, cudaEventRecord(ev[0], parent->stream));
  // ---- phase 1: upload own points, sort, block lists, own Y ------------------
  int64_t off = 0;
  for (int g = 0; g < s->groups; ++g) {
    const int r = s->emulated ? g : s->rank;
    auto& lc = s->loc[g];
    fgbd_ctx* ctx = lc.ctx;
    ctx->err.clear();
    ctx->launches = 0;
    const int64_t n_own = counts[r];
    int rc = ensure_capacity(ctx, n_own, 3 * b > 32);
    if (rc) return set_error(parent, rc, ctx->err);
    if (timing) FGBD_CUDA(parent, cudaEventRecord(s->rev[g][0], ctx->stream));
    FGBD_CUDA(parent, cudaMemsetAsync(ctx->ctl, 0, sizeof(Ctl), ctx->stream));
    SlabGC& G = lc.g;
    G.world = P;
    G.rank = r;
    G.b = b;
    G.n_own = n_own;
    G.lo = lo[r];
    G.blk_cap = s->blk_cap;
    for (int l = 0; l < 3; ++l) G.sums[l] = at<SumRec>(s->base[r], s->L.sums[l]);
    G.hdr = at<long long>(s->base[r], s->L.hdr);
    for (int p = 0; p < P; ++p) {
      for (int l = 0; l < 3; ++l) G.peer_sums[p][l] = at<SumRec>(s->base[p], s->L.sums[l]);
      G.peer_hdr[p] = at<long long>(s->base[p], s->L.hdr);
    }
    FGBD_CUDA(parent, cudaMemcpyAsync(ctx->coords64, coords + 3 * off, (size_t)n_own * 24,
                                      cudaMemcpyDefault, ctx->stream));
    FGBD_CUDA(parent, cudaMemcpyAsync(ctx->out, colors + 3 * off, (size_t)n_own * 24,
                                      cudaMemcpyDefault, ctx->stream));
    if (gidx) {
      FGBD_CUDA(parent, cudaMemcpyAsync(G.ext_gidx, gidx + off, (size_t)n_own * 4,
                                        cudaMemcpyDefault, ctx->stream));
    } else if ((rc = launch_iota_u32(ctx, G.ext_gidx, n_own, gidx_base + off))) {
      return set_error(parent, rc, ctx->err);
    }
    ctx->cur_coords = ctx->coords64;
    if (g == s->groups - 1 && timing) FGBD_CUDA(parent, cudaEventRecord(ev[1], parent->stream));
    if ((rc = launch_graph_slab_own(ctx, G))) return set_error(parent, rc, ctx->err);
    double4* ybuf = at<double4>(s->base[r], s->L.bufs[BUF_Y]) - lo[r];
    k_slab_expand<<<ctx->num_sms * 8, kBlock, 0, ctx->stream>>>(ctx->out, n_own, ybuf, lo[r],
                                                                ctx->rowid);
    FGBD_LAUNCH(ctx);
    if (timing) FGBD_CUDA(parent, cudaEventRecord(s->rev[g][1], ctx->stream));
    off += n_own;
  }
  FinArgs fin{};
  fin.n_total = s->n_total;
  if (int rc = all_gather(parent, s, ST_BLOCKS, fin)) return rc;
  // ---- phase 2: cross-slab neighbours, rows, sigma_g -------------------------
  for (int g = 0; g < s->groups; ++g) {
    auto& lc = s->loc[g];
    if (timing) FGBD_CUDA(parent, cudaEventRecord(s->rev[g][2], lc.ctx->stream));
    if (int rc = launch_graph_slab_rows(lc.ctx, lc.g)) return set_error(parent, rc, lc.ctx->err);
    if (timing) FGBD_CUDA(parent, cudaEventRecord(s->rev[g][3], lc.ctx->stream));
  }
  if (int rc = all_gather(parent, s, ST_SIGMA, fin)) return rc;
  for (int g = 0; g < s->groups; ++g)
    if (int rc = pull(s->loc[g].ctx)) return set_error(parent, rc, s->loc[g].ctx->err);
  if (timing) FGBD_CUDA(parent, cudaEventRecord(ev[2], parent->stream));
  {
    const Ctl& h = *s->loc[0].ctx->ctl_host;
    if (h.err_flags & 4)
      return set_error(parent, FGBD_E_NCCL, "slab peer did not reach the barrier (timeout)");
    if (h.err_flags & 1)
      return set_error(parent, FGBD_E_CLOUD,
                       "coordinates out of range for bit_depth=" + std::to_string(bits));
    if (!(h.sigma_g > 0)) {
      char m[96];
      std::snprintf(m, sizeof(m), "sigma_g must be positive, got %.17g", h.sigma_g);
      return set_error(parent, FGBD_E_GRAPH, m);
    }
  }
  const int maxdeg = s->loc[0].ctx->ctl_host->max_deg;
  fgbd_noise nz;
  std::memset(&nz, 0, sizeof(nz));
  // ---- phase 3: NE-GBP + FSLR (or the cached path's weights) -----------------
  auto view_of = [&](int r) {
    SlabView v{};
    v.world = P;
    v.self = r;
    for (int p = 0; p <= P; ++p) v.lo[p] = lo[p];
    for (int p = 0; p < P; ++p) v.y[p] = at<double4>(s->base[p], s->L.bufs[BUF_Y]) - lo[p];
    return v;
  };
  if (cached_q < 0) {
    const int D = cfg->patch_size;
    if (D > 1 + maxdeg)
      return set_error(parent, FGBD_E_NOISE, "patch_size " + std::to_string(D) +
                                                 " exceeds 1 + max degree (" +
                                                 std::to_string(1 + maxdeg) + ") of this graph");
    for (int g = 0; g < s->groups; ++g) {
      auto& lc = s->loc[g];
      if (timing) FGBD_CUDA(parent, cudaEventRecord(s->rev[g][4], lc.ctx->stream));
      if (int rc = launch_noise_slab(lc.ctx, lc.g.n_own, D, view_of(lc.g.rank)))
        return set_error(parent, rc, lc.ctx->err);
      if (timing) FGBD_CUDA(parent, cudaEventRecord(s->rev[g][5], lc.ctx->stream));
    }
    if (int rc = all_gather(parent, s, ST_NOISE, fin)) return rc;
    for (int g = 0; g < s->groups; ++g) {
      fgbd_ctx* ctx = s->loc[g].ctx;
      if (int rc = pull(ctx)) return set_error(parent, rc, ctx->err);
      // identical moment bits on every rank -> identical sigma_est
      if (int rc = finish_noise(ctx, D, cfg->tau_divisor, &nz)) return set_error(parent, rc, ctx->err);
    }
    const double sig = nz.sigma_est;
    const int active = cfg->fslr_enabled && !(sig < cfg->fslr_sigma_floor);
    for (int g = 0; g < s->groups; ++g) {
      auto& lc = s->loc[g];
      const double4* y = at<double4>(s->base[lc.g.rank], s->L.bufs[BUF_Y]);
      if (timing) FGBD_CUDA(parent, cudaEventRecord(s->rev[g][8], lc.ctx->stream));
      if (int rc = launch_mask_slab(lc.ctx, lc.g.n_own, y, sig, active))
        return set_error(parent, rc, lc.ctx->err);
      if (timing) FGBD_CUDA(parent, cudaEventRecord(s->rev[g][9], lc.ctx->stream));
    }
    fin.active = active;
    fin.q_max = cfg->q_max;
    fin.mode = cfg->criterion_mode;
    fin.early_exit = cfg->early_exit;
    fin.sv2 = sig * sig;
    if (int rc = all_gather(parent, s, ST_MASK, fin)) return rc;
  } else {
    for (int g = 0; g < s->groups; ++g) {
      auto& lc = s->loc[g];
      if (int rc = launch_weights_slab(lc.ctx, lc.g)) return set_error(parent, rc, lc.ctx->err);
    }
  }
  if (timing) FGBD_CUDA(parent, cudaEventRecord(ev[3], parent->stream));
  // ---- phase 4: the q scan ---------------------------------------------------
  {
    SlabArgs a{};
    a.world = P;
    a.rank0 = s->emulated ? 0 : s->rank;
    a.groups = s->groups;
    for (int r = 0; r <= P; ++r) a.lo[r] = lo[r];
    for (int r = 0; r < P; ++r) {
      for (int k = 0; k < 3; ++k) a.bufs[r][k] = at<double4>(s->base[r], s->L.bufs[k]) - lo[r];
      a.slots[r] = at<double>(s->base[r], s->L.lf_slots);
      a.flags[r] = at<unsigned long long>(s->base[r], s->L.lf_flags);
    }
    for (int g = 0; g < s->groups; ++g) {
      fgbd_ctx* c = s->loc[g].ctx;
      a.grp[g] = SlabGroup{EllRef{c->nbr, c->pay}, s->loc[g].g.n_own, c->mask, c->ctl};
    }
    a.release = s->release;
    a.part = s->part;
    a.exchange = (s->groups != P || s->force_exchange) ? 1 : 0;
    a.epoch = s->epoch;
    a.select = cached_q < 0;
    a.fixed_steps = cached_q < 0 ? 0 : cached_q;
    const int smem = 2 * 3 * kBlock * (int)sizeof(int4);
    int per_sm = 0;
    FGBD_CUDA(parent,
              cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lf_slab, kBlock, smem));
    const int capacity = std::min(std::max(1, per_sm) * parent->num_sms, s->bpg_cap);
    int64_t max_rows = 1;
    for (int g = 0; g < s->groups; ++g) max_rows = std::max(max_rows, s->loc[g].g.n_own);
    a.bpg = (int)std::max<int64_t>(
        1, std::min<int64_t>(capacity / s->groups, (max_rows + kBlock - 1) / kBlock));
    int64_t rows_here = 0;  // signal rows resident on this GPU
    for (int g = 0; g < s->groups; ++g) rows_here += s->loc[g].g.n_own;
    a.contiguous = lf_contiguous(parent, rows_here) ? 1 : 0;
    void* args[] = {&a};
    FGBD_CUDA(parent, cudaLaunchCooperativeKernel((void*)k_lf_slab, s->groups * a.bpg, kBlock,
                                                  args, smem, parent->stream));
    FGBD_LAUNCH(parent);
  }
  if (timing) FGBD_CUDA(parent, cudaEventRecord(ev[6], parent->stream));
  // ---- phase 5: output -------------------------------------------------------
  off = 0;
  for (int g = 0; g < s->groups; ++g) {
    auto& lc = s->loc[g];
    const int r = lc.g.rank;
    if (timing) FGBD_CUDA(parent, cudaEventRecord(s->rev[g][6], lc.ctx->stream));
    OutArgs o{};
    for (int k = 0; k < 3; ++k) o.bufs[k] = at<double4>(s->base[r], s->L.bufs[k]) - lo[r];
    o.ctl = lc.ctx->ctl;
    o.lo = lo[r];
    o.n_own = lc.g.n_own;
    o.rowid = lc.ctx->rowid;
    o.gidx = lc.g.ext_gidx;
    o.dst = lc.ctx->out;
    o.world = P;
    if (s->full)
      for (int p = 0; p < P; ++p) o.full[p] = at<double>(s->base[p], s->L.full);
    k_slab_out<<<lc.ctx->num_sms * 8, kBlock, 0, lc.ctx->stream>>>(o);
    FGBD_LAUNCH(lc.ctx);
    if (!s->full)
      FGBD_CUDA(parent, cudaMemcpyAsync(out_colors + 3 * off, lc.ctx->out, (size_t)lc.g.n_own * 24,
                                        cudaMemcpyDefault, lc.ctx->stream));
    if (timing) FGBD_CUDA(parent, cudaEventRecord(s->rev[g][7], lc.ctx->stream));
    off += lc.g.n_own;
  }
  if (s->full) {
    // every rank's pushes have landed before anyone reads its full frame
    if (int rc = all_gather(parent, s, ST_OUT, fin)) return rc;
    FGBD_CUDA(parent, cudaMemcpyAsync(out_colors, at<double>(s->base[s->rank], s->L.full),
                                      (size_t)s->n_total * 24, cudaMemcpyDefault, parent->stream));
  }
  if (timing) FGBD_CUDA(parent, cudaEventRecord(ev[4], parent->stream));
  for (int g = 0; g < s->groups; ++g)
    if (int rc = pull(s->loc[g].ctx)) return set_error(parent, rc, s->loc[g].ctx->err);
  if (timing) FGBD_CUDA(parent, cudaEventRecord(ev[5], parent->stream));
  const Ctl& h = *s->loc[0].ctx->ctl_host;
  for (int g = 0; g < s->groups; ++g)
    if (s->loc[g].ctx->ctl_host->err_flags & 4)
      return set_error(parent, FGBD_E_NCCL, "slab peer did not reach the barrier (timeout)");
  rep->n_edges = (int64_t)h.n_edges;
  rep->nnz = 2 * (int64_t)h.n_edges;
  rep->max_degree = h.max_deg;
  rep->sigma_g = h.sigma_g;
  int launches = 0;
  for (int g = 0; g < s->groups; ++g)
    launches += s->loc[g].ctx == parent && g > 0 ? 0 : s->loc[g].ctx->launches;
  rep->gpu_launches = launches;
  if (cached_q >= 0) {
    rep->selected_q = cached_q;
    rep->sigma_est = std::isnan(cached_sigma) ? 0.0 : cached_sigma;
    rep->masked_fraction = 0.0;
    rep->cached = 1;
    rep->steps = cached_q;
  } else {
    rep->selected_q = h.best_q;
    rep->sigma_est = nz.sigma_est;
    rep->masked_fraction = 1.0 - (double)h.included / (double)s->n_total;
    rep->criterion_value = h.best_crit;
    const double eps =
        std::isnan(cfg->epsilon) ? 1e-3 * nz.sigma_est * nz.sigma_est : cfg->epsilon;
    rep->converged = h.best_crit <= eps ? 1 : 0;
    rep->steps = h.steps;
    rep->all_excluded_fallback = h.all_excluded;
    rep->included_count = h.included;
    for (int c = 0; c < 3; ++c) {
      rep->per_channel_sigma[c] = nz.per_channel_sigma[c];
      rep->tail_m[c] = nz.m[c];
      rep->tail_tau[c] = nz.tau[c];
      rep->tail_fallback[c] = nz.fallback[c];
      rep->jacobi_direct_off[c] = nz.jacobi_direct_off[c];
      for (int k = 0; k < FGBD_MAX_PATCH; ++k) rep->eigenvalues[c][k] = nz.eigenvalues[c][k];
    }
    rep->eligible_count = nz.eligible_count;
    rep->n_trace = std::min(h.steps + 1, FGBD_TRACE_MAX);
    for (int k = 0; k < rep->n_trace; ++k) rep->trace[k] = h.trace[k];
  }
  if (timing) {
    rep->t_graph_construction = ev_sec(ev[1], ev[2]);
    rep->t_noise_estimation = cached_q >= 0 ? 0.0 : ev_sec(ev[2], ev[3]);
    rep->t_low_pass_filter = ev_sec(ev[3], ev[4]);
    rep->t_total = ev_sec(ev[0], ev[5]);
    rep->t_lf_steps = ev_sec(ev[3], ev[6]);
    rep->t_h2d = ev_sec(ev[0], ev[1]);
    rep->t_d2h = ev_sec(ev[4], ev[5]);
    for (int g = 0; g < s->groups; ++g) {
      const int r = s->loc[g].g.rank;
      rep->t_slab_rank[r][0] = ev_sec(s->rev[g][0], s->rev[g][1]);
      rep->t_slab_rank[r][1] = ev_sec(s->rev[g][2], s->rev[g][3]);
      rep->t_slab_rank[r][2] = cached_q >= 0 ? 0.0
                                             : ev_sec(s->rev[g][4], s->rev[g][5]) +
                                                   ev_sec(s->rev[g][8], s->rev[g][9]);
      rep->t_slab_rank[r][3] = ev_sec(s->rev[g][6], s->rev[g][7]);
    }
  }
  return FGBD_OK;
}

}  // namespace

extern "C" {

fgbd_slab* fgbd_slab_create(fgbd_ctx* ctx, int32_t world, int32_t rank, int64_t n_total,
                            int64_t max_own, uint32_t flags) {
  const bool emulated = (flags & FGBD_SLAB_EMULATED) != 0;
  if (!ctx || world < 1 || world > kMaxRanks || rank < 0 || rank >= world || n_total < 2 ||
      max_own < 1 || max_own > n_total) {
    set_error(ctx, FGBD_E_ARG, "invalid slab configuration");
    return nullptr;
  }
  cudaSetDevice(ctx->device);
  fgbd_slab* s = new fgbd_slab();
  s->world = world;
  s->rank = emulated ? 0 : rank;
  s->emulated = emulated;
  s->full = (flags & FGBD_SLAB_FULL_OUTPUT) && !emulated;
  s->force_exchange = (flags & FGBD_SLAB_EXCHANGE) != 0;
  s->n_total = n_total;
  s->cap_rows = ((max_own + 65535) / 65536) * 65536;
  s->blk_cap = s->cap_rows + 1;
  s->L = make_layout(s->cap_rows, world, s->blk_cap, s->full ? n_total : 0);
  s->groups = emulated ? world : 1;
  auto fail = [&]() -> fgbd_slab* {
    fgbd_slab_destroy(ctx, s);
    return nullptr;
  };
  for (int g = 0; g < s->groups; ++g) {
    auto& lc = s->loc[g];
    if (emulated && g > 0) {
      lc.ctx = fgbd_ctx_create(ctx->device, s->cap_rows);
      if (!lc.ctx) {
        set_error(ctx, FGBD_E_CUDA, std::string("slab sub-context: ") + fgbd_last_error(nullptr));
        return fail();
      }
      lc.own_ctx = true;
      // one stream for all emulated ranks: their phases run in launch order
      cudaStreamDestroy(lc.ctx->stream);
      cudaStreamDestroy(lc.ctx->side);
      lc.ctx->stream = ctx->stream;
      lc.ctx->side = ctx->side;
    } else {
      lc.ctx = ctx;
    }
    lc.g.rank = emulated ? g : rank;
    if (alloc_local(ctx, s, g) != FGBD_OK) return fail();
    s->base[lc.g.rank] = (char*)lc.region;
  }
  for (int g = 0; g < s->groups; ++g)
    for (auto& e : s->rev[g])
      if (cudaEventCreate(&e) != cudaSuccess) {
        set_error(ctx, FGBD_E_CUDA, "slab event");
        return fail();
      }
  s->bpg_cap = ctx->num_sms * 4;
  if (cudaMalloc(&s->release, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemset(s->release, 0, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&s->part, (size_t)2 * (3 * kSlabMaxBlocks + 2) * sizeof(double)) != cudaSuccess) {
    set_error(ctx, FGBD_E_CUDA, "slab scratch allocation failed");
    return fail();
  }
  return s;
}

void fgbd_slab_destroy(fgbd_ctx* ctx, fgbd_slab* s) {
  if (!s) return;
  if (ctx) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
  }
  for (int r = 0; r < kMaxRanks; ++r)
    if (s->peer_base[r]) cudaIpcCloseMemHandle(s->peer_base[r]);
  for (int g = 0; g < kMaxRanks; ++g) {
    auto& lc = s->loc[g];
    if (lc.region) cudaFree(lc.region);
    if (lc.ext) cudaFree(lc.ext);
    if (lc.own_ctx && lc.ctx) {
      lc.ctx->stream = nullptr;  // the parent's streams
      lc.ctx->side = nullptr;
      fgbd_ctx_destroy(lc.ctx);
    }
  }
  if (s->release) cudaFree(s->release);
  if (s->part) cudaFree(s->part);
  for (auto& row : s->rev)
    for (auto& e : row)
      if (e) cudaEventDestroy(e);
  delete s;
}

int32_t fgbd_slab_export(fgbd_ctx* ctx, fgbd_slab* s, uint8_t* handle_out) {
  if (!ctx || !s || s->emulated) return set_error(ctx, FGBD_E_ARG, "export needs a multi-GPU slab");
  cudaIpcMemHandle_t h;
  FGBD_CUDA(ctx, cudaIpcGetMemHandle(&h, s->loc[0].region));
  std::memcpy(handle_out, &h, sizeof(h));
  return FGBD_OK;
}

int32_t fgbd_slab_import(fgbd_ctx* ctx, fgbd_slab* s, const uint8_t* handles) {
  if (!ctx || !s || s->emulated) return set_error(ctx, FGBD_E_ARG, "import needs a multi-GPU slab");
  cudaSetDevice(ctx->device);
  for (int r = 0; r < s->world; ++r) {
    if (r == s->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + r * sizeof(h), sizeof(h));
    void* p = nullptr;
    FGBD_CUDA(ctx, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    s->peer_base[r] = p;
    s->base[r] = (char*)p;
  }
  return FGBD_OK;
}

int32_t fgbd_slab_handle_size(void) { return (int32_t)sizeof(cudaIpcMemHandle_t); }

int32_t fgbd_denoise_slab(fgbd_ctx* ctx, fgbd_slab* slab, const int64_t* coords,
                          const double* colors, const uint32_t* gidx, int64_t gidx_base,
                          const int64_t* counts, int32_t bits, const fgbd_config* cfg,
                          int32_t cached_q, double cached_sigma, double* out_colors,
                          fgbd_report* rep, uint32_t flags) {
  if (!ctx || !slab || !rep || !counts || !coords || !colors || !out_colors)
    return set_error(ctx, FGBD_E_ARG, "null argument");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  if (!cfg) return set_error(ctx, FGBD_E_ARG, "config must not be NULL");
  if (cfg->q_max < 0)
    return set_error(ctx, FGBD_E_FILTER, "q_max must be >= 0, got " + std::to_string(cfg->q_max));
  if (cfg->patch_size < 2)
    return set_error(ctx, FGBD_E_FILTER,
                     "patch_size must be >= 2, got " + std::to_string(cfg->patch_size));
  if (bits < 1 || bits > 21)
    return set_error(ctx, FGBD_E_GRAPH,
                     "bit depth " + std::to_string(bits) + " exceeds 21 (64-bit code overflow)");
  // step ticks carry the step in their low 32 bits
  if (cfg->q_max > (1 << 30) || cached_q > (1 << 30))
    return set_error(ctx, FGBD_E_FILTER, "q_max above 2^30 is not supported");
  std::memset(rep, 0, sizeof(*rep));
  rep->criterion_value = NAN;
  rep->converged = -1;
  rep->eligible_count = -1;
  return slab_frame(ctx, slab, coords, colors, gidx, gidx_base, counts, bits, cfg, cached_q,
                    cached_sigma, out_colors, rep, flags);
}

}  // extern "C"
