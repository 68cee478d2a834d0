// Spatial slab partition of ONE frame over P ranks.
//
// Every rank holds the full scan-line graph (built redundantly: it is a pure
// function of the coordinates, so every rank builds the same bits) and owns
// the rows [lo_r, hi_r) of the filter.  For raster- or Morton-ordered voxel
// data those ranges are spatial slabs, so only slab-boundary rows have
// foreign neighbours.
//
// k_lf_slab runs the whole q scan per rank in one persistent launch, fusing
// the filter step with its two collectives over peer memory:
//   * halo exchange: a foreign neighbour is read directly from the owner
//     rank's signal buffer (P2P load over NVLink; no pack/unpack, no copy);
//   * criterion all-reduce: the rank's leader block reduces its blocks'
//     partials in block order and stores the rank total into slot r of every
//     rank's slot array (P2P stores), then publishes its step counter into
//     every rank's flag array and waits until all ranks' counters reached the
//     step.  Each rank then sums the P slots in rank order -> the same bits
//     and the same select_q decision on every rank.
// A launch can carry several logical ranks as block groups (`groups`): on a
// single GPU all P ranks run as groups of one cooperative launch (all blocks
// co-resident, so spinning on another group's flags is safe) -- the test
// harness for the multi-GPU protocol.  On P GPUs each rank launches one
// group and the pointer tables hold peer (IPC-mapped) addresses.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "device_util.cuh"
#include "fgbd_internal.cuh"

namespace cg = cooperative_groups;

namespace fgbd {

constexpr int kMaxRanks = 16;

struct SlabArgs {
  EllRef E;
  int64_t n;
  int world;              // P
  int rank0;              // global rank of this launch's first group
  int groups;             // logical ranks in this launch
  int bpg;                // blocks per group
  int64_t lo[kMaxRanks + 1];
  double4* bufs[kMaxRanks][3];      // every rank's Y/A/B (full-size, own rows valid)
  double* slots[kMaxRanks];         // every rank's [2][P][4] rank-total slots
  unsigned long long* flags[kMaxRanks];  // every rank's [P] step counters
  unsigned int* gbar;     // local [groups][2] group-barrier counters
  double* part;           // local [groups][bpg][4] block partials
  const uint32_t* mask;
  Ctl* ctl;               // local control block (state + trace)
  unsigned long long epoch;  // frame epoch: counters are epoch<<32 | step
  int fixed_steps;        // cached path when > 0 (no criterion)
  int select;
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Barrier over the bpg co-resident blocks of one group (sense-reversing).
__device__ __forceinline__ void group_barrier(unsigned int* bar, int nblocks, Ctl* ctl) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = bar + 1;
    const unsigned int g0 = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == (unsigned)nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      const long long t0 = clock64();
      while (*gen == g0) {
        if (clock64() - t0 > (1ll << 35)) {  // ~17 s: never hang the GPU; report it
          atomicOr(&ctl->err_flags, 4);
          break;
        }
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ int owner_of(const SlabArgs& a, int64_t j) {
  int r = 0;
#pragma unroll 1
  while (r + 1 < a.world && j >= a.lo[r + 1]) ++r;
  return r;
}

struct SlabState {
  int q, best_q, streak, stop, in_b, best_b;
  double best_crit, prev;
};

__device__ __forceinline__ double slab_criterion(const double sy[3], const double sx[3],
                                                 long long count, double sv2, int mode) {
  if (mode == FGBD_CRIT_POOLED) {
    const double ty = (sy[0] + sy[1]) + sy[2];
    const double tx = (sx[0] + sx[1]) + sx[2];
    return fabs(sv2 - (ty - tx) / ((double)count * 3.0));
  }
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) acc += fabs(sv2 - (sy[c] - sx[c]) / (double)count);
  return acc / 3.0;
}

__global__ void __launch_bounds__(kBlock, 2) k_lf_slab(SlabArgs a) {
  __shared__ double s_red[32 * 3];
  __shared__ SlabState s_st;
  __shared__ double s_sy[3], s_sv2;
  __shared__ long long s_inc;
  __shared__ int s_qmax, s_mode, s_early, s_mask_all;
  const int g = blockIdx.x / a.bpg, lb = blockIdx.x % a.bpg;
  const int r = a.rank0 + g;
  const int P = a.world;
  Ctl* ctl = a.ctl;
  if (threadIdx.x == 0) {
    if (a.select) {
      s_st = SlabState{ctl->q, ctl->best_q, ctl->streak, ctl->stop, ctl->in_buf, ctl->best_buf,
                       ctl->best_crit, ctl->prev_crit};
      for (int k = 0; k < 3; ++k) s_sy[k] = ctl->sy[k];
      s_sv2 = ctl->sv2;
      s_inc = ctl->included;
      s_qmax = ctl->q_max;
      s_mode = ctl->mode;
      s_early = ctl->early_exit;
      s_mask_all = ctl->mask_all;
    } else {
      s_st = SlabState{0, 0, 0, a.fixed_steps <= 0, BUF_Y, BUF_Y, 0.0, 0.0};
      s_qmax = a.fixed_steps;
      s_mask_all = 1;
    }
  }
  __syncthreads();
  const int64_t lo = a.lo[r], hi = a.lo[r + 1];
  const int64_t chunk = ((hi - lo + a.bpg - 1) / a.bpg + blockDim.x - 1) / blockDim.x * blockDim.x;
  const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
  unsigned int* gbar = a.gbar + 2 * g;
  while (!s_st.stop) {
    const int ib = s_st.in_b, bb = s_st.best_b, q = s_st.q;
    int ob = BUF_A;
    if (ob == ib || ob == bb) ob = BUF_B;
    if (ob == ib || ob == bb) ob = BUF_Y;
    double4* out = a.bufs[r][ob];
    double sx[3] = {0.0, 0.0, 0.0};
    {
      // this block's contiguous share of the rank's rows, next row's slots
      // prefetched; gathers are branch-free (padding = own row, w = 0) and
      // only rows outside [lo, hi) look up their owner's (peer) buffer
      const double4* own_in = a.bufs[r][ib];
      int64_t i = lo + (int64_t)lb * chunk + threadIdx.x;
      const int64_t end = min(hi, lo + (int64_t)(lb + 1) * chunk);
      int nbn[kSlots];
      float wn[kSlots];
      auto load_slots = [&](int64_t row, int (&nb)[kSlots], float (&w)[kSlots]) {
#pragma unroll
        for (int s = 0; s < kSlots; s += 2) {
          const int4 pr =
              ld_pair_hint(reinterpret_cast<const int2*>(a.E.nbr + eslot(s, a.n, row)), pol_stream);
          nb[s] = pr.x;  // row | below-flag (bit 31)
          w[s] = __int_as_float(pr.y);
          nb[s + 1] = pr.z;
          w[s + 1] = __int_as_float(pr.w);
        }
      };
      if (i < end) load_slots(i, nbn, wn);
      while (i < end) {
        int nb[kSlots];
        float w[kSlots];
#pragma unroll
        for (int s = 0; s < kSlots; ++s) {
          nb[s] = nbn[s];
          w[s] = wn[s];
        }
        const int64_t inext = i + blockDim.x;
        if (inext < end) load_slots(inext, nbn, wn);
        const double4 f = ld_row_hint(own_in + i, pol_keep);
        double4 gv[kSlots];
#pragma unroll
        for (int s = 0; s < kSlots; ++s) {
          const int64_t j = ell_j(nb[s]);
          FGBD_DCHECK(j >= 0 && j < a.n);
          const double4* src =
              (j >= lo && j < hi) ? own_in : a.bufs[owner_of(a, j)][ib];  // halo: peer memory
          gv[s] = ld_row_hint(src + j, pol_keep);
        }
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, dlo = 0.0, dhi = 0.0;
#pragma unroll
        for (int s = 0; s < kSlots; ++s) {
          // (sum over original j > i) + (sum over j < i); padding adds +0.0
          const double ws = (double)w[s];
          const bool below = ell_below(nb[s]);
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
        st_row_hint(out + i, o, pol_keep);
        if (a.select && (s_mask_all || ((a.mask[i >> 5] >> (i & 31)) & 1u))) {
          sx[0] = fma(o.x, o.x, sx[0]);
          sx[1] = fma(o.y, o.y, sx[1]);
          sx[2] = fma(o.z, o.z, sx[2]);
        }
        i = inext;
      }
    }
    block_sum<3>(sx, s_red);
    double* part = a.part + ((int64_t)g * a.bpg + lb) * 4;
    if (threadIdx.x == 0)
      for (int k = 0; k < 3; ++k) part[k] = sx[k];
    group_barrier(gbar, a.bpg, ctl);  // this rank's rows of step q+1 are written
    const int par = (q + 1) & 1;
    const unsigned long long tick = (a.epoch << 32) | (unsigned long long)(q + 1);
    if (lb == 0 && threadIdx.x == 0) {
      double t[3] = {0.0, 0.0, 0.0};
      for (int b = 0; b < a.bpg; ++b)
        for (int k = 0; k < 3; ++k) t[k] += ld_cg(a.part + ((int64_t)g * a.bpg + b) * 4 + k);
      for (int p = 0; p < P; ++p)
        for (int k = 0; k < 3; ++k) a.slots[p][(par * P + r) * 4 + k] = t[k];
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
    }
    group_barrier(gbar, a.bpg, ctl);  // every rank's rows and totals of step q+1 are visible
    if (threadIdx.x == 0) {
      if (a.select) {
        double tot[3] = {0.0, 0.0, 0.0};
        for (int p = 0; p < P; ++p)
          for (int k = 0; k < 3; ++k) tot[k] += ld_cg(a.slots[r] + (par * P + p) * 4 + k);
        const double crit = slab_criterion(s_sy, tot, s_inc, s_sv2, s_mode);
        SlabState& s = s_st;
        s.q += 1;
        if (crit < s.best_crit) {
          s.best_crit = crit;
          s.best_q = s.q;
          s.best_b = ob;
        }
        s.streak = crit > s.prev ? s.streak + 1 : 0;
        s.prev = crit;
        s.stop = (s_early && s.streak >= 3) || (s.q >= s_qmax) || (s.best_crit == 0.0);
        s.in_b = ob;
        if (lb == 0 && s.q < FGBD_TRACE_MAX && g == 0) ctl->trace[s.q] = crit;
      } else {
        s_st.q += 1;
        s_st.stop = s_st.q >= s_qmax;
        s_st.in_b = ob;
        s_st.best_b = ob;
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->q = s_st.q;
    ctl->steps = s_st.q;
    ctl->best_q = s_st.best_q;
    ctl->best_crit = s_st.best_crit;
    ctl->best_buf = s_st.best_b;
    ctl->in_buf = s_st.in_b;
    ctl->stop = 1;
  }
}

// Assemble the full (N,3) clipped output from every rank's best buffer
// (peer loads for foreign rows).
__global__ void __launch_bounds__(kBlock) k_slab_gather(SlabArgs a, int best_b,
                                                        double* __restrict__ dst, int clip,
                                                        const int* __restrict__ pos) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    const int64_t r = pos ? (int64_t)pos[i] : i;  // point i lives in row r
    const double4 v = ld_row(a.bufs[owner_of(a, r)][best_b] + r);
    if (clip) {
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

// rank-local copy of the own rows of Y from the frame's full Y
__global__ void k_slab_fill(const double4* __restrict__ y, int64_t lo, int64_t hi,
                            double4* __restrict__ dst) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += stride)
    st_row(dst + i, ld_row(y + i));
}

}  // namespace fgbd

using namespace fgbd;

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

struct fgbd_slab {
  int world = 1, rank = 0;
  int64_t n = 0;
  bool emulated = false;
  // per logical rank (emulation) or only [rank] (multi-GPU) locally owned
  void* region[kMaxRanks] = {};   // local allocations
  size_t region_bytes = 0;
  // pointer tables (peer-mapped in multi-GPU mode)
  double4* bufs[kMaxRanks][3] = {};
  double* slots[kMaxRanks] = {};
  unsigned long long* flags[kMaxRanks] = {};
  void* peer_base[kMaxRanks] = {};  // opened IPC mappings
  unsigned int* gbar = nullptr;
  double* part = nullptr;
  unsigned long long epoch = 1;
  int bpg = 0;
};

namespace {

size_t slab_region_bytes(int64_t n, int world) {
  // 3 signal buffers, slot array [2][P][4], flags [P]; 256-byte aligned pieces
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  return 3 * al((size_t)n * 32) + al((size_t)2 * world * 4 * 8) + al((size_t)world * 8);
}

void carve(fgbd_slab* s, int r, char* base, int64_t n) {
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  size_t off = 0;
  for (int k = 0; k < 3; ++k) {
    s->bufs[r][k] = reinterpret_cast<double4*>(base + off);
    off += al((size_t)n * 32);
  }
  s->slots[r] = reinterpret_cast<double*>(base + off);
  off += al((size_t)2 * s->world * 4 * 8);
  s->flags[r] = reinterpret_cast<unsigned long long*>(base + off);
}

int64_t slab_lo(int64_t n, int world, int r) { return (n * (int64_t)r) / world; }

int slab_args(fgbd_ctx* ctx, fgbd_slab* s, int64_t n, SlabArgs* a) {
  std::memset(a, 0, sizeof(*a));
  a->E = EllRef{ctx->nbr, ctx->pay};
  a->n = n;
  a->world = s->world;
  a->rank0 = s->emulated ? 0 : s->rank;
  a->groups = s->emulated ? s->world : 1;
  for (int r = 0; r <= s->world; ++r) a->lo[r] = slab_lo(n, s->world, r);
  for (int r = 0; r < s->world; ++r) {
    for (int k = 0; k < 3; ++k) a->bufs[r][k] = s->bufs[r][k];
    a->slots[r] = s->slots[r];
    a->flags[r] = s->flags[r];
  }
  a->gbar = s->gbar;
  a->part = s->part;
  a->mask = ctx->mask;
  a->ctl = ctx->ctl;
  a->epoch = s->epoch;
  return FGBD_OK;
}

}  // namespace

namespace fgbd {

// Runs the select (q_max > 0 via ctl) or fixed-step loop across the slab
// ranks and writes the clipped (N,3) result to d_out.
int launch_slab(fgbd_ctx* ctx, fgbd_slab* s, int64_t n, int select, int fixed_steps,
                double* d_out) {
  SlabArgs a;
  slab_args(ctx, s, n, &a);
  a.select = select;
  a.fixed_steps = fixed_steps;
  const int groups = a.groups;
  int per_sm = 0;
  FGBD_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lf_slab, kBlock, 0));
  const int capacity = std::max(1, per_sm) * ctx->num_sms;
  int bpg = capacity / groups;
  const int64_t rows = (n + s->world - 1) / s->world;
  bpg = (int)std::max<int64_t>(1, std::min<int64_t>(bpg, (rows + kBlock - 1) / kBlock));
  a.bpg = bpg;
  // own rows of Y into every local rank's Y buffer
  for (int g = 0; g < groups; ++g) {
    const int r = a.rank0 + g;
    k_slab_fill<<<ctx->num_sms * 4, kBlock, 0, ctx->stream>>>(
        (const double4*)ctx->buf[BUF_Y], a.lo[r], a.lo[r + 1], a.bufs[r][BUF_Y]);
    FGBD_LAUNCH(ctx);
  }
  FGBD_CUDA(ctx, cudaMemsetAsync(s->gbar, 0, 2 * groups * sizeof(unsigned), ctx->stream));
  void* args[] = {&a};
  FGBD_CUDA(ctx, cudaLaunchCooperativeKernel((void*)k_lf_slab, groups * bpg, kBlock, args, 0,
                                             ctx->stream));
  FGBD_LAUNCH(ctx);
  s->epoch += 1;
  // best buffer id is the same on every rank
  FGBD_CUDA(ctx, cudaMemcpyAsync(&ctx->ctl_host->best_buf, &ctx->ctl->best_buf, sizeof(int),
                                 cudaMemcpyDeviceToHost, ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  k_slab_gather<<<ctx->num_sms * 4, kBlock, 0, ctx->stream>>>(
      a, ctx->ctl_host->best_buf, d_out, 1, ctx->g_reordered ? ctx->pos : nullptr);
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

int slab_alloc_local(fgbd_ctx* ctx, fgbd_slab* s, int64_t n, int groups) {
  const size_t bytes = slab_region_bytes(n, s->world);
  for (int g = 0; g < groups; ++g) {
    const int r = s->emulated ? g : s->rank;
    FGBD_CUDA(ctx, cudaMalloc(&s->region[g], bytes));
    FGBD_CUDA(ctx, cudaMemset(s->region[g], 0, bytes));
    carve(s, r, (char*)s->region[g], n);
  }
  s->region_bytes = bytes;
  FGBD_CUDA(ctx, cudaMalloc(&s->gbar, 2 * kMaxRanks * sizeof(unsigned)));
  FGBD_CUDA(ctx, cudaMemset(s->gbar, 0, 2 * kMaxRanks * sizeof(unsigned)));
  FGBD_CUDA(ctx, cudaMalloc(&s->part, (size_t)ctx->num_sms * 16 * 4 * sizeof(double)));
  s->n = n;
  return FGBD_OK;
}

}  // namespace fgbd

extern "C" {

fgbd_slab* fgbd_slab_create(fgbd_ctx* ctx, int32_t world, int32_t rank, int64_t n,
                            int32_t emulated) {
  if (!ctx || world < 1 || world > kMaxRanks || rank < 0 || rank >= world || n < 1) {
    set_error(ctx, FGBD_E_ARG, "invalid slab configuration");
    return nullptr;
  }
  cudaSetDevice(ctx->device);
  fgbd_slab* s = new fgbd_slab();
  s->world = world;
  s->rank = rank;
  s->emulated = emulated != 0;
  if (slab_alloc_local(ctx, s, n, s->emulated ? world : 1) != FGBD_OK) {
    fgbd_slab_destroy(ctx, s);
    return nullptr;
  }
  return s;
}

void fgbd_slab_destroy(fgbd_ctx* ctx, fgbd_slab* s) {
  if (!s) return;
  if (ctx) cudaSetDevice(ctx->device);
  for (int r = 0; r < kMaxRanks; ++r) {
    if (s->peer_base[r]) cudaIpcCloseMemHandle(s->peer_base[r]);
    if (s->region[r]) cudaFree(s->region[r]);
  }
  if (s->gbar) cudaFree(s->gbar);
  if (s->part) cudaFree(s->part);
  delete s;
}

int32_t fgbd_slab_export(fgbd_ctx* ctx, fgbd_slab* s, uint8_t* handle_out) {
  if (!ctx || !s || s->emulated) return set_error(ctx, FGBD_E_ARG, "export needs a multi-GPU slab");
  cudaIpcMemHandle_t h;
  FGBD_CUDA(ctx, cudaIpcGetMemHandle(&h, s->region[0]));
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
    carve(s, r, (char*)p, s->n);
  }
  return FGBD_OK;
}

int32_t fgbd_slab_handle_size(void) { return (int32_t)sizeof(cudaIpcMemHandle_t); }

}  // extern "C"
