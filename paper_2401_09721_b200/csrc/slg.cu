// Scan-line graph front end in ONE cooperative launch (reference
// graph.py:139-224): packed line-1 codes, the three scan-line orders and the
// rank neighbours.
//
//   phase 0   coords int64 -> packed line-1 code pc (coalesced through shared
//             memory), range check, "input already in line-1 order" flag
//   line 1    only when the input is not already in line-1 order: LSD passes
//             over the 3b-bit code, <= 10-bit digits
//   line 2    stable sort of the line-1 order by x alone = the (x, z, y,
//             index) order (one pass for b <= 10)
//   line 3    stable sort of the line-2 order by y = (y, x, z, index)
//   adjacency cand[l][perm_l[k]] = (perm_l[k-1], perm_l[k+1]); pos = line-1 rank
//
// Every pass is a counting sort whose tiles are the grid's warps, in index
// order (block g, warp w owns one contiguous range):
//   A  per-warp digit counts (shared-memory atomics)
//      into shared memory; the block's column goes to a digit-major table
//      cnt[d * G + g]
//   B  grid-wide exclusive scan of that table (block g scans slice g)
//   C  per warp: its digit cursors = the table entry + the earlier warps'
//      counts; re-walk the range and scatter each value to its stable rank
//      (per-bit ballots group the lanes of equal digit)
// with a grid barrier after each phase.  All tiles are resident, so no
// decoupled look-back chain forms: the onesweep passes this replaces spent
// most of their ~30 us (1M keys) waiting down that chain, and the separate
// prep / skipped-pass / neighbour launches cost ~50 us more.


#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "device_util.cuh"
#include "fgbd_internal.cuh"


namespace fgbd {

constexpr int kSlgThreads = 512;
constexpr int kSlgWarps = kSlgThreads / 32;
constexpr int kSlgMaxDigit = 10;
constexpr int kSlgMaxR = 1 << kSlgMaxDigit;
constexpr int kSlgMaxGrid = kSlgThreads;  // phase C scans the G slice totals in one block
constexpr int kFlagUnsortedSlg = 16;      // Ctl::err_flags (as graph.cu's kFlagUnsorted)
constexpr int kFlagReordered = 8;         // Ctl::err_flags: rows differ from points

template <typename K>
struct SlgArgs {
  const int64_t* coords;  // (n, 3) int64
  K* pc;                  // [n] packed line-1 codes (z, y, x)
  int64_t n;
  int b;
  uint32_t* perm[3];      // final orders of lines 1-3
  uint32_t* tmp;          // [n] ping-pong for multi-pass lines
  int2* cand;             // [3][n]
  int* pos;               // [n] point -> row (line-1 rank + row_base), or null
  int64_t row_base;
  Ctl* ctl;
  uint32_t* cnt;          // [kSlgMaxR * G] digit-major counts -> offsets
  uint32_t* tot;          // [G] slice totals
  unsigned int* bar;      // grid barrier word (device_util.cuh grid_barrier)
  int64_t span;           // elements per warp range (multiple of 32)
  unsigned long long* tlog;  // FGBD_SLG_TLOG: %globaltimer of block 0 at each phase, or null
};

constexpr int kSlgTlogMarks = 64;
__device__ __forceinline__ void slg_mark(unsigned long long* tlog, int& k) {
  if (tlog && threadIdx.x == 0) {  // [mark][block] + the mark count
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (k < kSlgTlogMarks - 1) tlog[1 + (size_t)k * 512 + blockIdx.x] = t;
    if (blockIdx.x == 0) tlog[0] = k + 1;
  }
  ++k;
}

// line-1 code of a point (z, y, x) -- graph.py:25
template <typename K>
__device__ __forceinline__ K slg_code(long long x, long long y, long long z, int b) {
  return (K(z) << (2 * b)) | (K(y) << b) | K(x);
}

// the key a line sorts on: line 1 the whole code, lines 2 / 3 (derived) x / y
template <typename K>
__device__ __forceinline__ K slg_key(K code, int line, int b) {
  if (line == 0) return code;
  const K m = (K(1) << b) - 1;
  return line == 1 ? (code & m) : ((code >> b) & m);
}

// block-wide exclusive scan of one value per thread; returns the prefix and
// the block total in *total
__device__ __forceinline__ uint32_t slg_block_scan(uint32_t v, uint32_t* s_w, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  uint32_t wofs = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kSlgWarps; ++w) {
    const uint32_t s = s_w[w];
    wofs += w < warp ? s : 0u;
    all += s;
  }
  __syncthreads();  // s_w is reused by the next call
  *total = all;
  return wofs + inc - v;
}

constexpr int kSlgIPT = 8;                    // elements per lane per batch
constexpr int kSlgBatch = 32 * kSlgIPT;      // elements per warp batch
constexpr int kSlgAdjIPT = 4;                // adjacency positions per thread in flight

// lanes holding the same digit (valid lanes only; d = ~0 marks invalid):
// one ballot per digit bit -- match.any is several times slower here
__device__ __forceinline__ unsigned slg_peers(unsigned d, int width) {
  const bool valid = d != 0xffffffffu;
  unsigned peers = __ballot_sync(kFull, valid);
#pragma unroll 1
  for (int bt = 0; bt < width; ++bt) {
    const bool on = (d >> bt) & 1u;
    const unsigned m = __ballot_sync(kFull, on);
    peers &= on ? m : ~m;
  }
  return peers;
}

// One warp batch of a pass: kSlgIPT rounds of 32 consecutive elements, all
// loads issued before the first round (the rounds are serial per warp; their
// loads are not).
template <typename K>
__device__ __forceinline__ void slg_load(const SlgArgs<K>& a, const uint32_t* __restrict__ src,
                                         uint32_t* id_out, int line, int shift, uint32_t dm,
                                         int64_t b0, int64_t s1, uint32_t (&v)[kSlgIPT],
                                         unsigned (&d)[kSlgIPT]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < kSlgIPT; ++j) {
    const int64_t i = b0 + j * 32 + lane;
    // other blocks wrote src after this block may have cached it: L2 reads
    v[j] = i < s1 ? (src ? __ldcg(&src[i]) : (uint32_t)i) : 0u;
    if (!src && id_out && i < s1) id_out[i] = (uint32_t)i;
  }
#pragma unroll
  for (int j = 0; j < kSlgIPT; ++j) {
    const int64_t i = b0 + j * 32 + lane;
    d[j] = i < s1 ? (unsigned)(slg_key(a.pc[v[j]], line, a.b) >> shift) & dm : 0xffffffffu;
  }
}

// One stable counting-sort pass over `width` bits at `shift` of line
// `line`'s key: dst[rank] = value, values from src (null: the identity; then
// id_out, if given, receives the identity too).
template <typename K>
__device__ __noinline__ int slg_pass(const SlgArgs<K>& a,
                                         const uint32_t* __restrict__ src,
                                         uint32_t* __restrict__ dst, uint32_t* id_out, int line,
                                         int shift, int width, uint32_t* wh, uint32_t* s_tp,
                                         uint32_t* s_w, int mk) {
  // one out-of-line copy for every pass: the passes run once per frame each,
  // and inlined copies (lines 1-3) missed in the instruction cache on every
  // first execution
  const int G = gridDim.x, g = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = 1 << width;
  const uint32_t dm = (uint32_t)R - 1u;
  const int64_t n = a.n;
  const int64_t s0 = ((int64_t)g * kSlgWarps + warp) * a.span;
  const int64_t s1 = min(n, s0 + a.span);
  const bool one = a.span <= kSlgBatch;  // the batch stays in registers across the barriers
  uint32_t* h = wh + warp * R;
  for (int t = tid; t < kSlgWarps * R; t += kSlgThreads) wh[t] = 0;
  __syncthreads();
  // A: per-warp digit counts
  uint32_t v[kSlgIPT];
  unsigned d[kSlgIPT];
  for (int64_t b0 = s0; b0 < s1; b0 += kSlgBatch) {
    slg_load(a, src, id_out, line, shift, dm, b0, s1, v, d);
    // counts only (ranks come in C): one shared-memory atomic per element
#pragma unroll
    for (int j = 0; j < kSlgIPT; ++j)
      if (d[j] != 0xffffffffu) atomicAdd(&h[d[j]], 1u);
  }
  __syncthreads();
  for (int dd = tid; dd < R; dd += kSlgThreads) {
    uint32_t c = 0;
#pragma unroll 4
    for (int w = 0; w < kSlgWarps; ++w) c += wh[w * R + dd];
    a.cnt[(int64_t)dd * G + g] = c;
  }
  slg_mark(a.tlog, mk);
  grid_barrier(a.bar);
  slg_mark(a.tlog, mk);
  // B: exclusive scan of slice g of the digit-major table (R entries, at
  // most 2 per thread)
  {
    const int64_t e0 = (int64_t)g * R + 2 * tid;
    uint32_t c0 = 0, c1 = 0;
    if (2 * tid < R) c0 = __ldcg(&a.cnt[e0]);
    if (2 * tid + 1 < R) c1 = __ldcg(&a.cnt[e0 + 1]);
    uint32_t total;
    const uint32_t ex = slg_block_scan(c0 + c1, s_w, &total);
    if (2 * tid < R) a.cnt[e0] = ex;
    if (2 * tid + 1 < R) a.cnt[e0 + 1] = ex + c0;
    if (tid == 0) a.tot[g] = total;
  }
  grid_barrier(a.bar);
  slg_mark(a.tlog, mk);
  // C: slice prefixes, the warps' digit cursors, then the scatter
  {
    const uint32_t t = tid < G ? __ldcg(&a.tot[tid]) : 0u;
    uint32_t total;
    const uint32_t ex = slg_block_scan(t, s_w, &total);
    if (tid < G) s_tp[tid] = ex;
  }
  __syncthreads();
  for (int dd = tid; dd < R; dd += kSlgThreads) {
    const int64_t e = (int64_t)dd * G + g;
    uint32_t base = __ldcg(&a.cnt[e]) + s_tp[e / R];
#pragma unroll 4
    for (int w = 0; w < kSlgWarps; ++w) {
      const uint32_t c = wh[w * R + dd];
      wh[w * R + dd] = base;
      base += c;
    }
  }
  __syncthreads();
  for (int64_t b0 = s0; b0 < s1; b0 += kSlgBatch) {
    if (!one) slg_load(a, src, nullptr, line, shift, dm, b0, s1, v, d);
#pragma unroll
    for (int j = 0; j < kSlgIPT; ++j) {
      const unsigned peers = slg_peers(d[j], width);
      const int leader = 31 - __clz(peers);
      uint32_t c = 0;
      if (d[j] != 0xffffffffu && lane == leader) {
        c = h[d[j]];
        h[d[j]] = c + __popc(peers);
      }
      c = __shfl_sync(kFull, c, leader);
      if (d[j] != 0xffffffffu) dst[c + __popc(peers & lanemask_lt())] = v[j];
      __syncwarp();
    }
  }
  slg_mark(a.tlog, mk);
  grid_barrier(a.bar);
  slg_mark(a.tlog, mk);
  return mk;
}

// the passes of one line's key (kw bits): balanced digits of <= 10 bits;
// the last pass lands in dst
template <typename K>
__device__ __forceinline__ void slg_line(const SlgArgs<K>& a,
                                         const uint32_t* src, uint32_t* dst, uint32_t* id_out,
                                         int line, int kw, uint32_t* wh, uint32_t* s_tp,
                                         uint32_t* s_w, int& mk) {
  const int passes = (kw + kSlgMaxDigit - 1) / kSlgMaxDigit;
  const int width = (kw + passes - 1) / passes;
  const uint32_t* in = src;
  for (int p = 0; p < passes; ++p) {
    uint32_t* out = ((passes - 1 - p) & 1) ? a.tmp : dst;
    const int w = min(width, kw - p * width);
    mk = slg_pass(a, in, out, p == 0 ? id_out : nullptr, line, p * width, w, wh, s_tp, s_w, mk);
    in = out;
  }
}

constexpr int kSlgStage = 2048;  // points staged per block iteration of phase 0

template <typename K>
__global__ void __launch_bounds__(kSlgThreads, 2) k_slg(const __grid_constant__ SlgArgs<K> a) {
  extern __shared__ __align__(16) uint32_t s_dyn[];
  uint32_t* wh = s_dyn;                          // [kSlgWarps][R]
  uint32_t* s_tp = s_dyn + kSlgWarps * kSlgMaxR; // [G]
  __shared__ uint32_t s_w[kSlgWarps];
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t n = a.n;
  const int b = a.b;
  int mk = 0;
  slg_mark(a.tlog, mk);
  // phase 0: codes, range check, sortedness; coordinates staged through the
  // (not yet used) digit-count memory, 2048 points + the next one
  {
    static_assert((3 * kSlgStage + 3) * 8 <= kSlgWarps * kSlgMaxR * 4, "phase-0 staging");
    long long* s_c = reinterpret_cast<long long*>(wh);
    bool bad = false, unsorted = false;
    const long long lim = 1ll << b;
    for (int64_t i0 = (int64_t)blockIdx.x * kSlgStage; i0 < n;
         i0 += (int64_t)gridDim.x * kSlgStage) {
      const int m = (int)min((int64_t)kSlgStage + 1, n - i0);
      const int64_t* src = a.coords + 3 * i0;
      // asynchronous copies: every load in flight at once, none in registers
      for (int t = tid; t < 3 * m; t += kSlgThreads)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(s_c + t)),
                     "l"(src + t)
                     : "memory");
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
      for (int t = tid; t < min(m, kSlgStage); t += kSlgThreads) {
        const int64_t i = i0 + t;
        const long long x = s_c[3 * t], y = s_c[3 * t + 1], z = s_c[3 * t + 2];
        bad |= (x < 0) | (y < 0) | (z < 0) | (x >= lim) | (y >= lim) | (z >= lim);
        const K code = slg_code<K>(x, y, z, b);
        a.pc[i] = code;
        if (t + 1 < m) {
          const K next = slg_code<K>(s_c[3 * t + 3], s_c[3 * t + 4], s_c[3 * t + 5], b);
          unsorted |= next < code;
        }
      }
      __syncthreads();
    }
    if (bad) atomicOr(&a.ctl->err_flags, 1);
    if (__any_sync(kFull, unsorted) && lane == 0) atomicOr(&a.ctl->err_flags, kFlagUnsortedSlg);
  }
  slg_mark(a.tlog, mk);
  grid_barrier(a.bar);
  slg_mark(a.tlog, mk);
  const bool sorted = !(*(volatile const int*)&a.ctl->err_flags & kFlagUnsortedSlg);
  // line 1 (identity when the input is already in its order)
  if (!sorted) slg_line(a, nullptr, a.perm[0], nullptr, 0, 3 * b, wh, s_tp, s_w, mk);
  // lines 2 and 3, derived; a sorted input's line-1 identity is written by
  // line 2's first pass
  slg_line(a, sorted ? nullptr : a.perm[0], a.perm[1], sorted ? a.perm[0] : nullptr, 1, b,
           wh, s_tp, s_w, mk);
  slg_line(a, a.perm[1], a.perm[2], nullptr, 2, b, wh, s_tp, s_w, mk);
  // adjacency of the three lines: kSlgAdjIPT positions per thread in flight
  bool moved = false;
  const int64_t stride = (int64_t)gridDim.x * kSlgThreads;
  for (int line = 0; line < 3; ++line) {
    const uint32_t* perm = a.perm[line];
    const bool ident = line == 0 && sorted;
    for (int64_t k0 = (int64_t)blockIdx.x * kSlgThreads; k0 < n; k0 += stride * kSlgAdjIPT) {
      int u[kSlgAdjIPT], pv[kSlgAdjIPT], nx[kSlgAdjIPT];
#pragma unroll
      for (int j = 0; j < kSlgAdjIPT; ++j) {
        const int64_t k = k0 + j * stride + tid;  // whole warps stay in (shuffles)
        u[j] = k < n ? (ident ? (int)k : (int)__ldcg(&perm[k])) : -1;
        pv[j] = -1;
        nx[j] = -1;
        if (lane == 0 && k > 0 && k < n) pv[j] = ident ? (int)k - 1 : (int)__ldcg(&perm[k - 1]);
        if (lane == 31 && k + 1 < n) nx[j] = ident ? (int)k + 1 : (int)__ldcg(&perm[k + 1]);
      }
#pragma unroll
      for (int j = 0; j < kSlgAdjIPT; ++j) {
        const int64_t k = k0 + j * stride + tid;
        const int up = __shfl_up_sync(kFull, u[j], 1), dn = __shfl_down_sync(kFull, u[j], 1);
        const int prev = lane == 0 ? pv[j] : up;
        const int next = lane == 31 ? nx[j] : (k + 1 < n ? dn : -1);
        if (k < n) {
          a.cand[line * n + u[j]] = make_int2(prev, next);
          if (line == 0 && a.pos) {
            a.pos[u[j]] = (int)(a.row_base + k);
            moved |= u[j] != (int)k;
          }
        }
      }
    }
  }
  if (__any_sync(kFull, moved) && lane == 0) atomicOr(&a.ctl->err_flags, kFlagReordered);
  slg_mark(a.tlog, mk);
}

template <typename K>
static int slg_grid(fgbd_ctx* ctx, size_t smem) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_slg<K>, kSlgThreads, smem) !=
      cudaSuccess)
    return -1;
  per_sm = std::min(per_sm, 2);
  return std::min(per_sm * ctx->num_sms, kSlgMaxGrid);
}

template <typename K>
static int slg_impl(fgbd_ctx* ctx, int64_t n, int b, int* pos, int64_t row_base) {
  const size_t smem = (size_t)(kSlgWarps * kSlgMaxR + kSlgMaxGrid) * sizeof(uint32_t);
  int& G = ctx->slg_grid[sizeof(K) == 8];
  if (G <= 0) {  // once per context: attribute + co-resident grid
    FGBD_CUDA(ctx, cudaFuncSetAttribute(k_slg<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    G = slg_grid<K>(ctx, smem);
    if (G <= 0) return set_error(ctx, FGBD_E_CUDA, "scan-line kernel cannot be co-resident");
  }
  if (!ctx->slg_cnt) {
    const size_t bytes = ((size_t)kSlgMaxR * kSlgMaxGrid + kSlgMaxGrid + 1) * sizeof(uint32_t);
    FGBD_CUDA(ctx, cudaMalloc((void**)&ctx->slg_cnt, bytes));
    FGBD_CUDA(ctx, cudaMemset(ctx->slg_cnt, 0, bytes));
  }
  SortScratch& S = ctx->sort;
  SlgArgs<K> a{};
  a.coords = ctx->cur_coords;
  a.pc = (K*)ctx->pc;
  a.n = n;
  a.b = b;
  for (int l = 0; l < 3; ++l) a.perm[l] = S.vals[0][l];
  a.tmp = S.vals[1][0];
  a.cand = ctx->cand;
  a.pos = pos;
  a.row_base = row_base;
  a.ctl = ctx->ctl;
  a.cnt = ctx->slg_cnt;
  a.tot = ctx->slg_cnt + (size_t)kSlgMaxR * kSlgMaxGrid;
  a.bar = a.tot + kSlgMaxGrid;
  const int64_t ranges = (int64_t)G * kSlgWarps;
  a.span = std::max<int64_t>(32, ((n + ranges - 1) / ranges + 31) / 32 * 32);
  static unsigned long long* tlog = nullptr;
  static const bool want_tlog = std::getenv("FGBD_SLG_TLOG") != nullptr;
  if (want_tlog && !tlog) cudaMalloc(&tlog, (1 + kSlgTlogMarks * 512) * sizeof(unsigned long long));
  a.tlog = want_tlog ? tlog : nullptr;
  void* args[] = {&a};
  FGBD_CUDA(ctx, cudaLaunchCooperativeKernel((void*)k_slg<K>, G, kSlgThreads, args, smem,
                                             ctx->stream));
  FGBD_LAUNCH(ctx);
  for (int l = 0; l < 3; ++l) ctx->perm[l] = S.vals[0][l];
  if (a.tlog) {  // experiment: per phase, the blocks' durations (min / median / max) and
                 // the spread of their phase ends, in us
    std::vector<unsigned long long> h(1 + kSlgTlogMarks * 512);
    cudaStreamSynchronize(ctx->stream);
    cudaMemcpy(h.data(), a.tlog, h.size() * 8, cudaMemcpyDeviceToHost);
    const int marks = (int)std::min<unsigned long long>(h[0], kSlgTlogMarks - 1);
    auto at = [&](int k, int blk) { return h[1 + (size_t)k * 512 + blk]; };
    unsigned long long t0 = ~0ull;
    for (int g = 0; g < G; ++g) t0 = std::min(t0, at(0, g));
    for (int k = 1; k < marks; ++k) {
      std::vector<double> d(G), e(G);
      for (int g = 0; g < G; ++g) {
        d[g] = (at(k, g) - at(k - 1, g)) * 1e-3;
        e[g] = (at(k, g) - t0) * 1e-3;
      }
      std::sort(d.begin(), d.end());
      std::sort(e.begin(), e.end());
      std::fprintf(stderr, "slg phase %2d: dur %.2f / %.2f / %.2f  end %.2f .. %.2f\n", k, d[0],
                   d[G / 2], d[G - 1], e[0], e[G - 1]);
    }
  }
  return FGBD_OK;
}

int launch_slg(fgbd_ctx* ctx, int64_t n, int b, int* pos, int64_t row_base) {
  return (3 * b <= 32) ? slg_impl<uint32_t>(ctx, n, b, pos, row_base)
                       : slg_impl<unsigned long long>(ctx, n, b, pos, row_base);
}

}  // namespace fgbd
