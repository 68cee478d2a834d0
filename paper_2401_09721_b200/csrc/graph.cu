// Scan-line graph construction on sm_100a (reference graph.py:122-251).
//
// The denoise path builds the three scan-line orders and the rank
// neighbours in one cooperative launch (slg.cu, k_slg) and then runs k_rows
// below.  The kernels before k_rows here (k_prep, k_onesweep, k_neighbors)
// serve the argsort / scan-line stage entry points and FGBD_SLG_COOP=0.
//
//   k_prep       coords int64 -> packed line-1 code (pc) + digit histograms
//                of every radix pass (one read); flags an input that is not
//                already in scan-line-1 order
//   k_onesweep   one stable LSD pass: warp multisplit (per-bit ballots) ->
//                decoupled look-back across tiles -> smem reorder ->
//                coalesced scatter (8-bit digits).  Line 1 takes ceil(3b/8)
//                passes over its code (skipped when the input is already in
//                line-1 order).  Lines 2 and 3 are DERIVED: a stable sort of
//                the line-1 order by x alone is the (x, z, y, index) order of
//                line 2, and a stable sort of that by y is line 3's (y, x, z,
//                index) order -- ceil(b/8) passes each instead of ceil(3b/8).
//   k_neighbors  rank neighbours: cand[l][perm_l[k]] = (perm_l[k-1], perm_l[k+1])
//   k_rows       per point: sort + dedup <= 6 candidates (the reference's
//                np.unique + lexsort, graph.py:188-208), exact squared
//                lengths, patch order by (sqdist, index) (noise.py:112),
//                sigma_g partial sums (graph.py:227-233)
//   k_weights    Eq. (4): w = exp(-sqdist / sigma_g^2) (graph.py:236-245)
//   k_export_*   reference CSR / edge-list conventions for the stage API
#include <algorithm>
#include <cstdio>

#include "device_util.cuh"
#include "fgbd_internal.cuh"

#ifndef FGBD_LOOK_BATCH
#define FGBD_LOOK_BATCH 4
#endif
#ifndef FGBD_SORT_BALLOT
#define FGBD_SORT_BALLOT 1  // warp multisplit by per-bit ballots (1) or match.any (0)
#endif
#ifndef FGBD_SORT_MINB
#define FGBD_SORT_MINB 3
#endif

namespace fgbd {

constexpr int kLookBatch = FGBD_LOOK_BATCH;

// ---------------------------------------------------------------------------
// codes
// ---------------------------------------------------------------------------

// line 0: pc itself (z, y, x); line 1: (x, z, y); line 2: (y, x, z) -- graph.py:25
template <typename K>
__device__ __forceinline__ K line_key(K pc, int line, int b) {
  if (line == 0) return pc;
  const K m = (K(1) << b) - 1;
  const K x = pc & m, y = (pc >> b) & m, z = pc >> (2 * b);
  if (line == 1) return (x << (2 * b)) | (z << b) | y;
  return (y << (2 * b)) | (x << b) | z;
}

template <typename K>
__device__ __forceinline__ void unpack(K pc, int b, long long* x, long long* y, long long* z) {
  const K m = (K(1) << b) - 1;
  *x = (long long)(pc & m);
  *y = (long long)((pc >> b) & m);
  *z = (long long)(pc >> (2 * b));
}

constexpr int kFlagUnsorted = 16;  // Ctl::err_flags: input is not in scan-line-1 order

// sort key of line l's pass p: line 0 its code; lines 1 / 2 (derived) the
// x / y field of the line-1 code
template <typename K>
__device__ __forceinline__ K pass_key(K code, int line, int b, bool derived) {
  if (line == 0) return code;
  if (!derived) return line_key(code, line, b);
  const K m = (K(1) << b) - 1;
  return line == 1 ? (code & m) : ((code >> b) & m);
}

// Histogram of every digit of every pass, warp-aggregated smem atomics.
// hist layout [line][kMaxPasses][256]; line l has passes[l] passes.
template <typename K, bool FROM_COORDS>
__global__ void __launch_bounds__(kBlock) k_prep(const int64_t* __restrict__ coords,
                                                 const K* __restrict__ keys_in, int64_t n,
                                                 int b, int nlines, int passes0, int passes12,
                                                 int derived, K* __restrict__ pc,
                                                 uint32_t* __restrict__ hist,
                                                 Ctl* __restrict__ ctl) {
  // shared histograms packed (line 0's passes, then line 1's, line 2's);
  // hist (global) keeps the [line][kMaxPasses][256] layout
  extern __shared__ uint32_t s_hist[];
  const int nh = (passes0 + (nlines - 1) * passes12) * kRadix;
  for (int t = threadIdx.x; t < nh; t += blockDim.x) s_hist[t] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long lim = (1ll << b);
  bool bad = false, unsorted = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    const bool valid = i < n;
    K code = 0;
    if (valid) {
      if (FROM_COORDS) {
        const long long x = coords[3 * i], y = coords[3 * i + 1], z = coords[3 * i + 2];
        bad |= (x < 0) | (y < 0) | (z < 0) | (x >= lim) | (y >= lim) | (z >= lim);
        code = (K(z) << (2 * b)) | (K(y) << b) | K(x);
        pc[i] = code;
      } else {
        code = keys_in[i];
      }
    }
    if (FROM_COORDS) {
      // an inversion with the next point: the input is not in line-1 order
      K next = __shfl_down_sync(kFull, code, 1);
      if (lane == 31 && i + 1 < n) {
        const long long x = coords[3 * i + 3], y = coords[3 * i + 4], z = coords[3 * i + 5];
        next = (K(z) << (2 * b)) | (K(y) << b) | K(x);
      }
      unsorted |= valid && i + 1 < n && next < code;
    }
    const unsigned vmask = __ballot_sync(kFull, valid);
    for (int l = 0; l < nlines; ++l) {
      const K key = FROM_COORDS ? pass_key(code, l, b, derived != 0) : code;
      const int passes = l == 0 ? passes0 : passes12;
      uint32_t* sh = s_hist + (l == 0 ? 0 : passes0 + (l - 1) * passes12) * kRadix;
      for (int p = 0; p < passes; ++p) {
        const unsigned d = valid ? (unsigned)((key >> (8 * p)) & 0xff) : 0x100u;
        // a digit shared by the whole warp (raster-ordered input, high
        // bytes) costs one atomic; otherwise per-lane atomics, which only
        // contend when equal digits are scattered across the warp
        const unsigned d0 = __shfl_sync(kFull, d, 0);
        if (__all_sync(kFull, d == d0) && d0 < 0x100u) {
          if (lane == 0) atomicAdd(&sh[p * kRadix + d0], (uint32_t)__popc(vmask));
        } else if (valid) {
          atomicAdd(&sh[p * kRadix + d], 1u);
        }
      }
    }
  }
  if (bad) atomicOr(&ctl->err_flags, 1);
  if (__any_sync(kFull, unsorted) && lane == 0) atomicOr(&ctl->err_flags, kFlagUnsorted);
  __syncthreads();
  for (int t = threadIdx.x; t < nh; t += blockDim.x) {
    if (!s_hist[t]) continue;
    const int slot = t / kRadix;  // packed (line, pass) -> [line][kMaxPasses]
    const int l = slot < passes0 ? 0 : 1 + (slot - passes0) / max(passes12, 1);
    const int p = l == 0 ? slot : (slot - passes0) % max(passes12, 1);
    atomicAdd(&hist[(l * kMaxPasses + p) * kRadix + (t % kRadix)], s_hist[t]);
  }
}

// ---------------------------------------------------------------------------
// onesweep pass
// ---------------------------------------------------------------------------

struct SortPass {
  const void* src_keys[3];      // null on pass 0 in SLG mode (keys from pc)
  const void* pc;
  const uint32_t* src_vals[3];  // null on pass 0 (identity); a derived line's pass 0: the
                                // previous line's order
  void* dst_keys[3];
  uint32_t* dst_vals[3];
  const uint32_t* hist;         // [line][kMaxPasses][256] digit counts (k_prep)
  unsigned long long* status;   // [line][tiles][256]
  unsigned int* tile_ctr;       // [line]
  const Ctl* ctl;               // SLG line 0: skip when the input is already sorted
  int64_t n;
  int b, pass, passes, tiles;
  int line0;                    // line of blockIdx.y == 0
  int derived;                  // SLG lines 2/3 sort one field of the previous line's order
  unsigned int epoch;
};

constexpr unsigned long long kFlagAgg = 1ull << 32;
constexpr unsigned long long kFlagPre = 2ull << 32;

#if FGBD_SORT_TLOG
// Timeline instrumentation (experiment builds only, -DFGBD_SORT_TLOG=1):
// %globaltimer per (pass, line, tile) at block start, after the multisplit,
// after the look-back and at the end.  Read back with fgbd_debug_stlog.
constexpr int kStlogTiles = 1024;
__device__ unsigned long long g_stlog[4][3][kStlogTiles][4];
__device__ __forceinline__ unsigned long long sort_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define STLOG(k)                                                                  \
  do {                                                                            \
    if (threadIdx.x == 0 && p.pass < 4 && s_tile < kStlogTiles)                   \
      g_stlog[p.pass][blockIdx.y][s_tile][(k)] = sort_timer();                    \
  } while (0)
#else
#define STLOG(k) \
  do {           \
  } while (0)
#endif

template <typename K, bool FIRST, bool LAST, bool SLG>
__global__ void __launch_bounds__(kSortThreads, FGBD_SORT_MINB) k_onesweep(SortPass p) {
  extern __shared__ __align__(16) unsigned char smem[];
  K* s_keys = reinterpret_cast<K*>(smem);
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + kSortTile);
  uint32_t* s_whist = s_vals + kSortTile;  // [8 warps][256]
  __shared__ uint32_t s_start[kRadix];    // tile-local exclusive digit start
  __shared__ uint32_t s_gofs[kRadix];     // global position - local index
  __shared__ uint32_t s_wsum[8], s_hsum[8];
  __shared__ int s_tile;

  const int line = p.line0 + blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (SLG && line == 0 && !(*(volatile const int*)&p.ctl->err_flags & kFlagUnsorted)) {
    // already in line-1 order: the stable order is the identity
    if (LAST)
      for (int64_t idx = (int64_t)blockIdx.x * kSortTile + tid;
           idx < min(p.n, (int64_t)(blockIdx.x + 1) * kSortTile); idx += kSortThreads)
        p.dst_vals[0][idx] = (uint32_t)idx;
    return;
  }
  if (tid == 0) s_tile = (int)atomicAdd(&p.tile_ctr[line], 1u);
  for (int t = tid; t < 8 * kRadix; t += kSortThreads) s_whist[t] = 0;
  __syncthreads();
  STLOG(0);
  const int tile = s_tile;
  const int64_t base = (int64_t)tile * kSortTile;
  const int shift = 8 * p.pass;

  K key[kSortIPT];
  uint32_t val[kSortIPT];
  uint32_t loc[kSortIPT];
  const K* kin = reinterpret_cast<const K*>(p.src_keys[line]);
  const K* pcp = reinterpret_cast<const K*>(p.pc);
#pragma unroll
  for (int j = 0; j < kSortIPT; ++j) {
    const int64_t idx = base + (int64_t)warp * 32 * kSortIPT + j * 32 + lane;
    if (idx < p.n) {
      if (FIRST && SLG && line > 0 && p.derived) {  // the previous line's order, one field
        val[j] = p.src_vals[line][idx];
        key[j] = pass_key(pcp[val[j]], line, p.b, true);
      } else if (FIRST) {
        key[j] = SLG ? line_key(pcp[idx], line, p.b) : kin[idx];
        val[j] = (uint32_t)idx;
      } else {
        key[j] = kin[idx];
        val[j] = p.src_vals[line][idx];
      }
    } else {
      key[j] = ~K(0);
      val[j] = 0xffffffffu;
    }
  }
  // warp multisplit: stable rank of each key among equal digits of its warp
  uint32_t* wh = s_whist + warp * kRadix;
  // bits above are 0 in every key
  const int kwidth = SLG ? ((line == 0 || !p.derived) ? 3 * p.b : p.b) : (int)(sizeof(K) * 8);
  const int dbits = min(8, max(0, kwidth - shift));
#pragma unroll
  for (int j = 0; j < kSortIPT; ++j) {
    const int64_t idx = base + (int64_t)warp * 32 * kSortIPT + j * 32 + lane;
    const bool valid = idx < p.n;
    const unsigned d = valid ? (unsigned)((key[j] >> shift) & 0xff) : 0x100u;
#if FGBD_SORT_BALLOT
    // lanes with the same 9-bit (valid, digit) value: one ballot per bit
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int bt = 0; bt < 9; ++bt) {
      if (bt < 8 && bt >= dbits) continue;  // digit bits above the key width are 0
      const bool on = (d >> bt) & 1u;
      const unsigned m = __ballot_sync(kFull, on);
      peers &= on ? m : ~m;
    }
#else
    const unsigned peers = __match_any_sync(kFull, d);
#endif
    const int leader = 31 - __clz(peers);
    uint32_t cnt = 0;
    if (valid && lane == leader) {
      cnt = wh[d];
      wh[d] = cnt + __popc(peers);
    }
    cnt = __shfl_sync(kFull, cnt, leader);
    loc[j] = cnt + __popc(peers & lanemask_lt());
    __syncwarp();
  }
  __syncthreads();
  // per digit (thread == digit): warp-exclusive offsets and the tile count
  const int d = tid;
  uint32_t count = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const uint32_t c = s_whist[w * kRadix + d];
    s_whist[w * kRadix + d] = count;
    count += c;
  }
  STLOG(1);
  // this digit's count over the whole pass (its latency hides in the look-back)
  const uint32_t hcount = p.hist[(line * kMaxPasses + p.pass) * kRadix + d];
  // decoupled look-back over preceding tiles of this line
  unsigned long long* st = p.status + ((int64_t)line * p.tiles) * kRadix;
  const unsigned long long ep = (unsigned long long)p.epoch << 34;
  uint32_t excl = 0;
  if (tile == 0) {
    atomicExch(&st[d], ep | kFlagPre | count);
  } else {
    atomicExch(&st[(int64_t)tile * kRadix + d], ep | kFlagAgg | count);
    // look back kLookBatch predecessors per round: their status words are
    // loaded together, then consumed newest-first until an inclusive prefix
    int k = tile - 1;
    bool done = false;
    while (!done) {
      unsigned long long v[kLookBatch];
#pragma unroll
      for (int j = 0; j < kLookBatch; ++j)
        v[j] = k - j >= 0 ? *reinterpret_cast<volatile unsigned long long*>(
                                &st[(int64_t)(k - j) * kRadix + d])
                          : 0ull;
#pragma unroll
      for (int j = 0; j < kLookBatch; ++j) {
        if (done) break;
        if ((v[j] >> 34) != p.epoch || ((v[j] >> 32) & 3ull) == 0) {
          k -= j;  // not published yet: re-read from this tile on
          break;
        }
        excl += (uint32_t)v[j];
        if (((v[j] >> 32) & 3ull) == 2) done = true;
        if (j == kLookBatch - 1) k -= kLookBatch;
      }
    }
    atomicExch(&st[(int64_t)tile * kRadix + d], ep | kFlagPre | (excl + count));
  }
  // tile-local exclusive scan of counts over digits
  // and the pass's global digit base: the same scan over k_prep's histogram
  uint32_t v = count, hv = hcount;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, v, o);
    const uint32_t th = __shfl_up_sync(kFull, hv, o);
    if (lane >= o) {
      v += t;
      hv += th;
    }
  }
  if (lane == 31) {
    s_wsum[warp] = v;
    s_hsum[warp] = hv;
  }
  __syncthreads();
  uint32_t wofs = 0, hofs = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    wofs += (w < warp) ? s_wsum[w] : 0u;
    hofs += (w < warp) ? s_hsum[w] : 0u;
  }
  const uint32_t start = wofs + v - count;
  s_start[d] = start;
  s_gofs[d] = (hofs + hv - hcount) + excl - start;
  __syncthreads();
  STLOG(2);  // every digit's look-back is done
  // reorder the tile in shared memory by digit (stable)
#pragma unroll
  for (int j = 0; j < kSortIPT; ++j) {
    const int64_t idx = base + (int64_t)warp * 32 * kSortIPT + j * 32 + lane;
    if (idx < p.n) {
      const unsigned dd = (unsigned)((key[j] >> shift) & 0xff);
      const uint32_t pos = s_start[dd] + s_whist[warp * kRadix + dd] + loc[j];
      s_keys[pos] = key[j];
      s_vals[pos] = val[j];
    }
  }
  __syncthreads();
  // coalesced write-out: runs of equal digits land contiguously
  const int64_t rem = p.n - base;
  const int tile_n = rem < kSortTile ? (int)rem : kSortTile;
  K* kout = reinterpret_cast<K*>(p.dst_keys[line]);
  uint32_t* vout = p.dst_vals[line];
  for (int i = tid; i < tile_n; i += kSortThreads) {
    const K kk = s_keys[i];
    const unsigned dd = (unsigned)((kk >> shift) & 0xff);
    const uint32_t g = s_gofs[dd] + (uint32_t)i;
    if (!LAST) kout[g] = kk;
    vout[g] = s_vals[i];
  }
#if FGBD_SORT_TLOG
  __syncthreads();
  STLOG(3);
#endif
}

// ---------------------------------------------------------------------------
// adjacency
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kBlock) k_neighbors(const uint32_t* __restrict__ p0,
                                                     const uint32_t* __restrict__ p1,
                                                     const uint32_t* __restrict__ p2,
                                                     int64_t n, int2* __restrict__ cand,
                                                     int* __restrict__ pos, Ctl* __restrict__ ctl,
                                                     int64_t row_base = 0) {
  const int line = blockIdx.y;
  const uint32_t* perm = line == 0 ? p0 : (line == 1 ? p1 : p2);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    const int u = (int)perm[k];
    const int prev = k > 0 ? (int)perm[k - 1] : -1;
    const int next = k + 1 < n ? (int)perm[k + 1] : -1;
    cand[line * n + u] = make_int2(prev, next);
    if (line == 0 && pos) {
      pos[u] = (int)(row_base + k);  // row of point u = its scan-line-1 rank
      // input already in line-1 order (raster scans): rows == points, and
      // k_rows can skip the relabelling work
      if (__any_sync(__activemask(), u != (int)k) && (threadIdx.x & 31) == 0)
        atomicOr(&ctl->err_flags, 8);
    }
  }
}

template <typename T>
__device__ __forceinline__ void cswap(T& a, T& b) {
  const T lo = min(a, b), hi = max(a, b);
  a = lo;
  b = hi;
}

// sort 6 values: a 12-comparator network of depth 5 (checked on all 2^6
// 0/1 inputs)
template <typename T>
__device__ __forceinline__ void sort6(T (&c)[6]) {
  cswap(c[0], c[5]);
  cswap(c[1], c[3]);
  cswap(c[2], c[4]);
  cswap(c[1], c[2]);
  cswap(c[3], c[4]);
  cswap(c[0], c[3]);
  cswap(c[2], c[5]);
  cswap(c[0], c[1]);
  cswap(c[2], c[3]);
  cswap(c[4], c[5]);
  cswap(c[1], c[2]);
  cswap(c[3], c[4]);
}

// Slab rank: rows are the rank's own points in scan-line-1
// order; local ids >= n_own are halo points (foreign neighbours); `pos` maps
// every local id to its GLOBAL row; the reference's index order is the
// global point index gidx[local id], so dedup, "below" flags, sigma_g's
// upper-slot rule and the patch tie-break all compare gidx.
struct RowsSlab {
  const uint32_t* gidx;  // [n_own + halo]
  int64_t lo;            // global row of own row 0
};

#ifndef FGBD_ROWS_MINB
#define FGBD_ROWS_MINB 4  // 64 registers, 4 blocks per SM: k_rows 55 -> 46 us (1M ramp, r2bi)
#endif
template <typename K, bool BIG, bool SLAB = false>
__global__ void __launch_bounds__(kBlock, FGBD_ROWS_MINB) k_rows(const int2* __restrict__ cand,
                                                 const K* __restrict__ pc, int64_t n, int b,
                                                 const int* __restrict__ pos,
                                                 const uint32_t* __restrict__ rowid, EllRef ell,
                                                 uint32_t* __restrict__ meta,
                                                 double* __restrict__ partials,
                                                 Ctl* __restrict__ ctl, RowsSlab sl = RowsSlab{},
                                                 const double* __restrict__ colors = nullptr,
                                                 double4* __restrict__ y_rows = nullptr) {
  __shared__ unsigned long long s_red[32 * 2];
  __shared__ bool s_last;
  u128 sg_sum = 0;  // exact: the same bits for any partition of the edges
  unsigned long long e_cnt = 0, far = 0;
  int maxdeg = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // rows differ from points only when the line-1 order is not the identity
  if (!SLAB && pos && !(*(volatile const int*)&ctl->err_flags & 8)) {
    pos = nullptr;
    rowid = nullptr;
  }
  // walk the ROWS (coalesced ELL / meta writes); row rr holds point i
  for (int64_t rr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; rr < n; rr += stride) {
    const int64_t i = rowid ? (int64_t)rowid[rr] : rr;
    // device-resident colours: k_expand's work for this row rides along
    if (!SLAB && y_rows)
      st_row(y_rows + rr, make_double4(colors[3 * i], colors[3 * i + 1], colors[3 * i + 2], 0.0));
    unsigned c[6];
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const int2 v = cand[l * n + i];
      c[2 * l] = (unsigned)v.x;  // -1 -> 0xffffffff sorts last
      c[2 * l + 1] = (unsigned)v.y;
    }
    unsigned gj[6];  // SLAB: global index of candidate s
    unsigned gi = 0;
    if (SLAB) {
      // order and dedup by the global index (halo copies of one point share it)
      unsigned long long k6[6];
#pragma unroll
      for (int s = 0; s < 6; ++s)
        k6[s] = c[s] == 0xffffffffu ? ~0ull
                                    : ((unsigned long long)sl.gidx[c[s]] << 32) | c[s];
      sort6(k6);
#pragma unroll
      for (int s = 5; s > 0; --s)
        if ((k6[s] >> 32) == (k6[s - 1] >> 32)) k6[s] = ~0ull;
      sort6(k6);
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        c[s] = (unsigned)k6[s];
        gj[s] = (unsigned)(k6[s] >> 32);
      }
      gi = sl.gidx[i];
    } else {
      sort6(c);
#pragma unroll
      for (int s = 5; s > 0; --s)
        if (c[s] == c[s - 1]) c[s] = 0xffffffffu;
      sort6(c);
    }
    int deg = 0;
#pragma unroll
    for (int s = 0; s < 6; ++s) deg += (c[s] != 0xffffffffu);
    long long xi, yi, zi;
    unpack(pc[i], b, &xi, &yi, &zi);
    unsigned long long sq[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      sq[s] = ~0ull;
      if (s < deg) {
        long long xj, yj, zj;
        FGBD_DCHECK(SLAB || (int64_t)c[s] < n);
        unpack(pc[c[s]], b, &xj, &yj, &zj);
        const long long dx = xi - xj, dy = yi - yj, dz = zi - zj;
        sq[s] = (unsigned long long)(dx * dx + dy * dy + dz * dz);
        if (SLAB ? gj[s] > gi : (int64_t)c[s] > i) {
          sg_sum += fx52(sqrt((double)sq[s]));
          e_cnt += 1;
        }
      }
    }
    // patch order: rank by (sqdist, index); rows are index-ascending so
    // the slot number breaks ties exactly like the reference's stable sort
    uint32_t order = 0;
    if (sizeof(K) == 4) {
      // 3b <= 32: sq < 3 * 2^20, so (sq, slot) packs into one 32-bit key
      uint32_t key[6];
#pragma unroll
      for (int s = 0; s < 6; ++s) key[s] = s < deg ? ((uint32_t)sq[s] << 3) | (uint32_t)s : ~0u;
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        int r = 0;
#pragma unroll
        for (int t = 0; t < 6; ++t) r += key[t] < key[s];
        if (s < deg) order |= (uint32_t)s << (3 * r);
      }
    } else {
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        int r = 0;
#pragma unroll
        for (int t = 0; t < 6; ++t)
          r += (t < deg) && (sq[t] < sq[s] || (sq[t] == sq[s] && t < s));
        if (s < deg) order |= (uint32_t)s << (3 * r);
      }
    }
    // the row of point i (its line-1 rank when rows are reordered) and its
    // neighbours' rows
    const int64_t r = rr;
    int word[6];
    unsigned slot_of[6];  // ELL slot that receives candidate slot s
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      int w = (int)(SLAB ? sl.lo + r : r);  // padding: (own row, 0)
      if (s < deg) {
        const int jr = pos ? pos[c[s]] : (int)c[s];
        w = jr | ((SLAB ? gj[s] < gi : (int64_t)c[s] < i) ? kBelowBit : 0);
      }
      word[s] = w;
      slot_of[s] = s;
    }
    if (pos) {
      // reordered rows: store the real slots by ascending neighbour ROW, so
      // the lanes of a warp (consecutive rows) gather slot t from nearby
      // rows -- for point-order rows this is the index order already
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        int rk = 0;
#pragma unroll
        for (int t = 0; t < 6; ++t)
          rk += (t < deg) && (ell_j(word[t]) < ell_j(word[s]) ||
                              (ell_j(word[t]) == ell_j(word[s]) && t < s));
        if (s < deg) slot_of[s] = (unsigned)rk;
      }
      // the patch order names slots: renumber it
      uint32_t o2 = 0;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const unsigned sl = (order >> (3 * k)) & 7u;
        unsigned ns = 0;
#pragma unroll
        for (int s = 0; s < 6; ++s) ns = (sl == (unsigned)s) ? slot_of[s] : ns;
        if (k < deg) o2 |= ns << (3 * k);
      }
      order = o2;
    }
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int t = (int)slot_of[s];
      ell.nbr[eslot(t, n, r)] = word[s];
      ell.pay[eslot(t, n, r)] = (s < deg && !BIG) ? (uint32_t)sq[s] : 0u;
    }
    meta[r] = (uint32_t)deg | (order << 3);
    maxdeg = max(maxdeg, deg);
    const int64_t own = SLAB ? sl.lo + r : r;
#pragma unroll
    for (int s = 0; s < 6; ++s)
      if (s < deg) {
        const int64_t d = (int64_t)ell_j(word[s]) - own;
        far += (d > kFarRows || d < -kFarRows);
      }
  }
  // block reduce (sum, count) and the max degree
  maxdeg = __reduce_max_sync(kFull, maxdeg);
  {
    unsigned long long f = far;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) f += __shfl_xor_sync(kFull, f, o);
    if ((threadIdx.x & 31) == 0 && f) atomicAdd(&ctl->far_slots, f);
  }
  if ((threadIdx.x & 31) == 0 && maxdeg > 0) atomicMax(&ctl->max_deg, maxdeg);
  unsigned long long* up = reinterpret_cast<unsigned long long*>(partials);
  const u128 bs = block_sum_u128(sg_sum, s_red);
  const u128 bc = block_sum_u128((u128)e_cnt, s_red);
  if (threadIdx.x == 0) {
    up[3 * blockIdx.x] = (unsigned long long)bs;
    up[3 * blockIdx.x + 1] = (unsigned long long)(bs >> 64);
    up[3 * blockIdx.x + 2] = (unsigned long long)bc;
  }
  if (last_block(&ctl->ticket[0], &s_last)) {
    u128 a = 0, cnt = 0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) {
      a += ((u128)__ldcg(&up[3 * k + 1]) << 64) | __ldcg(&up[3 * k]);
      cnt += __ldcg(&up[3 * k + 2]);
    }
    a = block_sum_u128(a, s_red);
    cnt = block_sum_u128(cnt, s_red);
    if (threadIdx.x == 0) {
      const unsigned long long e = (unsigned long long)cnt;
      ctl->n_edges = e;
      ctl->sigma_g = e ? fx52_to_double(a) / (double)e : 0.0;
      ctl->sg_fx[0] = (unsigned long long)a;  // a slab rank's share (all-gathered)
      ctl->sg_fx[1] = (unsigned long long)(a >> 64);
      ctl->ticket[0] = 0;
    }
  }
}

// Eq. (4): w = exp(-sqdist / sigma_g^2).  fp64 evaluation, fp32 storage in
// the slot payload (and fp64 copy in parity mode).
template <typename K, bool BIG, bool W64>
__global__ void __launch_bounds__(kBlock) k_weights(EllRef ell,
                                                    double* __restrict__ w64,
                                                    const K* __restrict__ pc, int64_t n,
                                                    int b, const uint32_t* __restrict__ rowid,
                                                    const Ctl* __restrict__ ctl,
                                                    int64_t row_base = 0) {
  const double sg = ctl->sigma_g;
  const double sg2 = sg * sg;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    long long xi = 0, yi = 0, zi = 0;
    if (BIG) unpack(pc[rowid ? rowid[i] : i], b, &xi, &yi, &zi);
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
      int2 sl = make_int2(ell.nbr[eslot(s, n, i)], (int)ell.pay[eslot(s, n, i)]);
      double w = 0.0;
      const int j = ell_j(sl.x);
      if (j != (int)(i + row_base)) {  // padding slots point at the own row
        unsigned long long sq;
        if (BIG) {
          long long xj, yj, zj;
          unpack(pc[rowid ? rowid[j] : j], b, &xj, &yj, &zj);
          const long long dx = xi - xj, dy = yi - yj, dz = zi - zj;
          sq = (unsigned long long)(dx * dx + dy * dy + dz * dz);
        } else {
          sq = (uint32_t)sl.y;
        }
        w = exp(__ddiv_rn(-(double)sq, sg2));
      }
      sl.y = __float_as_int((float)w);
      ell.pay[eslot(s, n, i)] = (uint32_t)sl.y;
      if (W64) w64[s * n + i] = w;
    }
  }
}

// ---------------------------------------------------------------------------
// CSR export (reference conventions)
// ---------------------------------------------------------------------------

__global__ void k_degrees(const uint32_t* __restrict__ meta, const int* __restrict__ ell,
                          int64_t n, int64_t* __restrict__ deg, int64_t* __restrict__ updeg) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int dg = (int)(meta[i] & 7u);
    int up = 0;
    for (int s = 0; s < dg; ++s) up += (ell_j(ell[eslot(s, n, i)]) > (int)i);
    deg[i] = dg;
    updeg[i] = up;
  }
}

// Exclusive scan, 3 phases (only used by the export path).
constexpr int kScanTile = 2048;
__global__ void k_scan_tiles(const int64_t* __restrict__ in, int64_t n,
                             int64_t* __restrict__ tile_sums) {
  __shared__ long long s[kBlock / 32];
  long long acc = 0;
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  for (int t = threadIdx.x; t < kScanTile; t += blockDim.x)
    if (base + t < n) acc += in[base + t];
  acc = warp_sum_ll(acc);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int w = 0; w < kBlock / 32; ++w) tot += s[w];
    tile_sums[blockIdx.x] = tot;
  }
}
__global__ void k_scan_sums(int64_t* tile_sums, int ntiles, int64_t* total) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    long long run = 0;
    for (int t = 0; t < ntiles; ++t) {
      const long long v = tile_sums[t];
      tile_sums[t] = run;
      run += v;
    }
    *total = run;
  }
}
__global__ void k_scan_apply(const int64_t* __restrict__ in, int64_t n,
                             const int64_t* __restrict__ tile_sums, int64_t* __restrict__ out) {
  __shared__ long long s[kScanTile];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  for (int t = threadIdx.x; t < kScanTile; t += blockDim.x)
    s[t] = (base + t < n) ? in[base + t] : 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = tile_sums[blockIdx.x];
    for (int t = 0; t < kScanTile; ++t) {
      const long long v = s[t];
      s[t] = run;
      run += v;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < kScanTile; t += blockDim.x)
    if (base + t < n) out[base + t] = s[t];
}

template <typename K>
__global__ void k_export(const uint32_t* __restrict__ meta, const int* __restrict__ ell,
                         const K* __restrict__ pc, int64_t n, int b,
                         const int64_t* __restrict__ rowoff, const int64_t* __restrict__ eoff,
                         const Ctl* __restrict__ ctl, int64_t* __restrict__ indptr,
                         int64_t* __restrict__ indices, int64_t* __restrict__ csr_edge,
                         int64_t* __restrict__ edge_u, int64_t* __restrict__ edge_v,
                         double* __restrict__ sqd, double* __restrict__ wts,
                         double* __restrict__ wdeg) {
  const double sg = ctl->sigma_g, sg2 = sg * sg;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int dg = (int)(meta[i] & 7u);
    const int64_t r0 = rowoff[i];
    if (indptr) {
      indptr[i] = r0;
      if (i == n - 1) indptr[n] = r0 + dg;
    }
    long long xi, yi, zi;
    unpack(pc[i], b, &xi, &yi, &zi);
    int nlow = 0;
    double lo = 0.0, hi = 0.0;
    for (int s = 0; s < dg; ++s) {
      const int j = ell_j(ell[eslot(s, n, i)]);
      long long xj, yj, zj;
      unpack(pc[j], b, &xj, &yj, &zj);
      const long long dx = xi - xj, dy = yi - yj, dz = zi - zj;
      const double sq = (double)(unsigned long long)(dx * dx + dy * dy + dz * dz);
      const double w = exp(__ddiv_rn(-sq, sg2));
      int64_t eid;
      if (j > (int)i) {
        eid = eoff[i] + (s - nlow);
        if (edge_u) edge_u[eid] = i;
        if (edge_v) edge_v[eid] = j;
        if (sqd) sqd[eid] = sq;
        if (wts) wts[eid] = w;
        hi += w;
      } else {
        ++nlow;
        const int dj = (int)(meta[j] & 7u);
        int cnt = 0;
        for (int t = 0; t < dj; ++t) {
          const int v = ell_j(ell[eslot(t, n, j)]);
          cnt += (v > j) && (v < (int)i);
        }
        eid = eoff[j] + cnt;
        lo += w;
      }
      if (indices) indices[r0 + s] = j;
      if (csr_edge) csr_edge[r0 + s] = eid;
    }
    if (wdeg) wdeg[i] = hi + lo;
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------

static int grid_for(int64_t n, int cap) {
  int64_t g = (n + kBlock - 1) / kBlock;
  if (g < 1) g = 1;
  return (int)std::min<int64_t>(g, cap);
}

template <typename K>
static size_t onesweep_smem() {
  return (size_t)kSortTile * (sizeof(K) + sizeof(uint32_t)) + 8 * kRadix * sizeof(uint32_t);
}

template <typename K, bool FIRST, bool LAST, bool SLG>
static int launch_pass(fgbd_ctx* ctx, SortPass& p, int nlines) {
  const size_t smem = onesweep_smem<K>();
  FGBD_CUDA(ctx, cudaFuncSetAttribute(k_onesweep<K, FIRST, LAST, SLG>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(p.tiles, nlines);
  k_onesweep<K, FIRST, LAST, SLG><<<grid, kSortThreads, smem, ctx->stream>>>(p);
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

// SLG (nlines = 3): line 1 takes `passes` passes over its code, then lines 2
// and 3 ceil(b/8) passes each over one field of the previous line's order.
// Otherwise: `passes` passes over keys_in (one line).  On return
// ctx->perm[l] points at the final permutation of line l.
template <typename K, bool SLG>
static int run_sort(fgbd_ctx* ctx, int64_t n, int b, int nlines, int passes,
                    const K* keys_in) {
  SortScratch& S = ctx->sort;
  const int tiles = (int)((n + kSortTile - 1) / kSortTile);
  const bool derived = SLG && ctx->sort_derived;
  const int passes12 = SLG ? (derived ? (b + 7) / 8 : passes) : 0;
  const int nh = nlines * kMaxPasses * kRadix;
  FGBD_CUDA(ctx, cudaMemsetAsync(S.hist, 0, nh * sizeof(uint32_t), ctx->stream));
  const int nh_used = (passes + (nlines - 1) * passes12) * kRadix;
  FGBD_CUDA(ctx, cudaMemsetAsync(S.tile_ctr, 0, kMaxPasses * 3 * sizeof(unsigned), ctx->stream));
  {
    const size_t smem = nh_used * sizeof(uint32_t);
    const int grid = grid_for(n, ctx->num_sms * ctx->prep_mult);
    if (SLG) {
      k_prep<K, true><<<grid, kBlock, smem, ctx->stream>>>(ctx->cur_coords, nullptr, n, b, nlines,
                                                           passes, passes12, derived ? 1 : 0,
                                                           (K*)ctx->pc, S.hist, ctx->ctl);
    } else {
      k_prep<K, false><<<grid, kBlock, smem, ctx->stream>>>(nullptr, keys_in, n, b, nlines, passes,
                                                            0, 0, nullptr, S.hist, ctx->ctl);
    }
    FGBD_LAUNCH(ctx);
  }
  // derived: one line per launch (each needs the previous line's order);
  // otherwise every line in each launch (blockIdx.y), line 1 skipping when
  // the input is already sorted
  const int groups = derived ? nlines : 1, per_launch = derived ? 1 : nlines;
  for (int lg = 0; lg < groups; ++lg) {
    const int line = lg;
    const int lp = (derived && line > 0) ? passes12 : passes;
    for (int pass = 0; pass < lp; ++pass) {
      SortPass p{};
      for (int l = 0; l < 3; ++l) {
        p.src_keys[l] = pass == 0 ? (const void*)keys_in : S.keys[(pass - 1) & 1][l];
        p.src_vals[l] = pass == 0 ? nullptr : S.vals[(pass - 1) & 1][l];
        p.dst_keys[l] = S.keys[pass & 1][l];
        p.dst_vals[l] = S.vals[pass & 1][l];
      }
      if (derived && line > 0 && pass == 0) p.src_vals[line] = ctx->perm[line - 1];
      p.pc = ctx->pc;
      p.hist = S.hist;
      p.status = S.status;
      p.tile_ctr = S.tile_ctr + pass * 3;
      p.ctl = ctx->ctl;
      p.n = n;
      p.b = b;
      p.pass = pass;
      p.passes = lp;
      p.tiles = tiles;
      p.line0 = line;
      p.derived = derived ? 1 : 0;
      p.epoch = (++S.epoch) & 0x3fffffffu;
      if (p.epoch == 0) p.epoch = S.epoch = 1;
      const bool first = pass == 0, last = pass == lp - 1;
      int rc;
      if (first && last) rc = launch_pass<K, true, true, SLG>(ctx, p, per_launch);
      else if (first) rc = launch_pass<K, true, false, SLG>(ctx, p, per_launch);
      else if (last) rc = launch_pass<K, false, true, SLG>(ctx, p, per_launch);
      else rc = launch_pass<K, false, false, SLG>(ctx, p, per_launch);
      if (rc) return rc;
    }
    for (int l = line; l < line + per_launch; ++l) ctx->perm[l] = S.vals[(lp - 1) & 1][l];
  }
  return FGBD_OK;
}

template <typename K>
static int graph_impl(fgbd_ctx* ctx, int64_t n, int b, bool reorder) {
  // (N,3) device colours to expand into BUF_Y on the way (fgbd_denoise with
  // device-resident colours; taken for this build only)
  const double* colors = ctx->expand_colors;
  ctx->expand_colors = nullptr;
  int* pos = reorder ? ctx->pos : nullptr;
  if (ctx->slg_coop) {
    // codes, the three orders and the rank neighbours in one launch (slg.cu)
    int rc = launch_slg(ctx, n, b, pos, 0);
    if (rc) return rc;
    ctx->rowid = reorder ? ctx->perm[0] : nullptr;
    if (reorder) FGBD_CUDA(ctx, cudaEventRecord(ctx->ev_perm, ctx->stream));
  } else {
    const int passes = (3 * b + 7) / 8;
    int rc = run_sort<K, true>(ctx, n, b, 3, passes, nullptr);
    if (rc) return rc;
    // rows in scan-line-1 order: row k holds the point of line-1 rank k
    ctx->rowid = reorder ? ctx->perm[0] : nullptr;
    if (reorder) FGBD_CUDA(ctx, cudaEventRecord(ctx->ev_perm, ctx->stream));
    dim3 grid(grid_for(n, 1 << 20), 3);
    k_neighbors<<<grid, kBlock, 0, ctx->stream>>>(ctx->perm[0], ctx->perm[1], ctx->perm[2], n,
                                                  ctx->cand, pos, ctx->ctl);
    FGBD_LAUNCH(ctx);
  }
  const int grid = grid_for(n, ctx->rows_grid == 1 ? (1 << 30) : kRowsGrid);
  double4* y_rows = colors ? reinterpret_cast<double4*>(ctx->buf[BUF_Y]) : nullptr;
  if (b > 15) {
    k_rows<K, true><<<grid, kBlock, 0, ctx->stream>>>(ctx->cand, (const K*)ctx->pc, n, b, pos, ctx->rowid,
                                                      EllRef{ctx->nbr, ctx->pay}, ctx->meta, ctx->partials,
                                                      ctx->ctl, RowsSlab{}, colors, y_rows);
  } else {
    k_rows<K, false><<<grid, kBlock, 0, ctx->stream>>>(ctx->cand, (const K*)ctx->pc, n, b, pos, ctx->rowid,
                                                       EllRef{ctx->nbr, ctx->pay}, ctx->meta, ctx->partials,
                                                       ctx->ctl, RowsSlab{}, colors, y_rows);
  }
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

int launch_graph(fgbd_ctx* ctx, int64_t n, int bits, bool reorder) {
  int rc = (3 * bits <= 32) ? graph_impl<uint32_t>(ctx, n, bits, reorder)
                            : graph_impl<unsigned long long>(ctx, n, bits, reorder);
  if (rc) return rc;
  ctx->g_reordered = reorder ? 1 : 0;
  ctx->g_n = n;
  ctx->g_bits = bits;
  ctx->g_have_weights = 0;
  ctx->g_have_noise = 0;
  ctx->held_valid = 0;  // a new graph: the reuse copy no longer describes it
  return FGBD_OK;
}

template <typename K>
static int weights_impl(fgbd_ctx* ctx, int64_t n, int b, int w64) {
  const int grid = grid_for(n, ctx->num_sms * 8);
  const K* pc = (const K*)ctx->pc;
  if (b > 15) {
    if (w64)
      k_weights<K, true, true><<<grid, kBlock, 0, ctx->stream>>>(EllRef{ctx->nbr, ctx->pay}, ctx->w64, pc, n, b, ctx->rowid, ctx->ctl);
    else
      k_weights<K, true, false><<<grid, kBlock, 0, ctx->stream>>>(EllRef{ctx->nbr, ctx->pay}, ctx->w64, pc, n, b, ctx->rowid, ctx->ctl);
  } else {
    if (w64)
      k_weights<K, false, true><<<grid, kBlock, 0, ctx->stream>>>(EllRef{ctx->nbr, ctx->pay}, ctx->w64, pc, n, b, ctx->rowid, ctx->ctl);
    else
      k_weights<K, false, false><<<grid, kBlock, 0, ctx->stream>>>(EllRef{ctx->nbr, ctx->pay}, ctx->w64, pc, n, b, ctx->rowid, ctx->ctl);
  }
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

int launch_weights(fgbd_ctx* ctx, int64_t n, int bits, int w64) {
  if (w64) {
    int rc = ensure_w64(ctx, n);
    if (rc) return rc;
  }
  int rc = (3 * bits <= 32) ? weights_impl<uint32_t>(ctx, n, bits, w64)
                            : weights_impl<unsigned long long>(ctx, n, bits, w64);
  if (rc) return rc;
  ctx->g_have_weights = 1;
  ctx->g_weights64 = w64;
  return FGBD_OK;
}

int launch_argsort64(fgbd_ctx* ctx, const uint64_t* d_keys, int64_t n, int key_bits,
                     uint32_t** d_perm_out) {
  const int passes = (key_bits + 7) / 8;
  int rc = run_sort<unsigned long long, false>(ctx, n, 0, 1, passes,
                                               (const unsigned long long*)d_keys);
  if (rc) return rc;
  *d_perm_out = ctx->perm[0];
  return FGBD_OK;
}

template <typename K>
__global__ void k_codes(const K* __restrict__ pc, int64_t n, int b, int line,
                        uint64_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = (uint64_t)line_key(pc[i], line, b);
}

int launch_scan_line(fgbd_ctx* ctx, int64_t n, int bits, int line, uint64_t* d_codes,
                     uint32_t** d_perm_out) {
  const int passes = (3 * bits + 7) / 8;
  int rc = (3 * bits <= 32) ? run_sort<uint32_t, true>(ctx, n, bits, 3, passes, nullptr)
                            : run_sort<unsigned long long, true>(ctx, n, bits, 3, passes, nullptr);
  if (rc) return rc;
  if (d_codes) {
    const int grid = grid_for(n, ctx->num_sms * 8);
    if (3 * bits <= 32)
      k_codes<uint32_t><<<grid, kBlock, 0, ctx->stream>>>((const uint32_t*)ctx->pc, n, bits,
                                                         line, d_codes);
    else
      k_codes<unsigned long long><<<grid, kBlock, 0, ctx->stream>>>(
          (const unsigned long long*)ctx->pc, n, bits, line, d_codes);
    FGBD_LAUNCH(ctx);
  }
  *d_perm_out = ctx->perm[line];
  return FGBD_OK;
}

int scan_exclusive(fgbd_ctx* ctx, const int64_t* in, int64_t n, int64_t* out,
                          int64_t* tmp, int64_t* d_total) {
  const int tiles = (int)((n + kScanTile - 1) / kScanTile);
  k_scan_tiles<<<tiles, kBlock, 0, ctx->stream>>>(in, n, tmp);
  FGBD_LAUNCH(ctx);
  k_scan_sums<<<1, 32, 0, ctx->stream>>>(tmp, tiles, d_total);
  FGBD_LAUNCH(ctx);
  k_scan_apply<<<tiles, kBlock, 0, ctx->stream>>>(in, n, tmp, out);
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

int launch_export(fgbd_ctx* ctx, int64_t n, int64_t* d_indptr, int64_t* d_indices,
                  int64_t* d_csr_edge, int64_t* d_edge_u, int64_t* d_edge_v, double* d_sqdist,
                  double* d_weights, double* d_wdeg, int64_t* nnz_out, int64_t* e_out) {
  // scratch: deg, updeg, rowoff, eoff (4n) + tile sums + 2 totals
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  const size_t need = (size_t)(4 * n + 2 * tiles + 2) * sizeof(int64_t);
  if (ctx->csr_scratch_bytes < need) {
    if (ctx->csr_scratch) cudaFree(ctx->csr_scratch);
    ctx->csr_scratch = nullptr;
    FGBD_CUDA(ctx, cudaMalloc(&ctx->csr_scratch, need));
    ctx->csr_scratch_bytes = need;
  }
  int64_t* deg = (int64_t*)ctx->csr_scratch;
  int64_t* updeg = deg + n;
  int64_t* rowoff = updeg + n;
  int64_t* eoff = rowoff + n;
  int64_t* t1 = eoff + n;
  int64_t* t2 = t1 + tiles;
  int64_t* totals = t2 + tiles;
  const int grid = grid_for(n, ctx->num_sms * 8);
  k_degrees<<<grid, kBlock, 0, ctx->stream>>>(ctx->meta, ctx->nbr, n, deg, updeg);
  FGBD_LAUNCH(ctx);
  int rc = scan_exclusive(ctx, deg, n, rowoff, t1, totals);
  if (rc) return rc;
  rc = scan_exclusive(ctx, updeg, n, eoff, t2, totals + 1);
  if (rc) return rc;
  if (3 * ctx->g_bits <= 32)
    k_export<uint32_t><<<grid, kBlock, 0, ctx->stream>>>(
        ctx->meta, ctx->nbr, (const uint32_t*)ctx->pc, n, ctx->g_bits, rowoff, eoff, ctx->ctl,
        d_indptr, d_indices, d_csr_edge, d_edge_u, d_edge_v, d_sqdist, d_weights, d_wdeg);
  else
    k_export<unsigned long long><<<grid, kBlock, 0, ctx->stream>>>(
        ctx->meta, ctx->nbr, (const unsigned long long*)ctx->pc, n, ctx->g_bits, rowoff, eoff,
        ctx->ctl, d_indptr, d_indices, d_csr_edge, d_edge_u, d_edge_v, d_sqdist, d_weights,
        d_wdeg);
  FGBD_LAUNCH(ctx);
  int64_t h[2];
  FGBD_CUDA(ctx, cudaMemcpyAsync(h, totals, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  *nnz_out = h[0];
  *e_out = h[1];
  return FGBD_OK;
}

// ---------------------------------------------------------------------------
// slab ranks: block lists, cross-slab neighbours
// ---------------------------------------------------------------------------

// segment key of a scan line: the code bits above z (z is the slab axis)
template <typename K>
__device__ __forceinline__ unsigned long long seg_key(K pc, int line, int b) {
  if (line == 0) return 0ull;
  const K k = line_key(pc, line, b);
  return (unsigned long long)(line == 1 ? (k >> (2 * b)) : (k >> b));
}

constexpr int kBlkIPT = 8;
constexpr int kBlkTile = kBlock * kBlkIPT;

template <typename K>
__device__ __forceinline__ bool blk_start(const uint32_t* perm, const K* pc, int64_t k, int line,
                                          int b) {
  return k == 0 || seg_key(pc[perm[k]], line, b) != seg_key(pc[perm[k - 1]], line, b);
}

// per tile: number of block starts (lines 2 and 3 = blockIdx.y 0 / 1)
template <typename K>
__global__ void __launch_bounds__(kBlock) k_blk_count(const uint32_t* __restrict__ p1,
                                                      const uint32_t* __restrict__ p2,
                                                      const K* __restrict__ pc, int64_t n, int b,
                                                      unsigned int* __restrict__ cnt, int tiles) {
  __shared__ double s_red[32];
  const int line = 1 + blockIdx.y;
  const uint32_t* perm = line == 1 ? p1 : p2;
  const int64_t base = (int64_t)blockIdx.x * kBlkTile;
  double c[1] = {0.0};
  for (int j = 0; j < kBlkIPT; ++j) {
    const int64_t k = base + j * kBlock + threadIdx.x;
    if (k < n && blk_start(perm, pc, k, line, b)) c[0] += 1.0;
  }
  block_sum<1>(c, s_red);
  if (threadIdx.x == 0) cnt[blockIdx.y * (tiles + 1) + blockIdx.x] = (unsigned)c[0];
}

// exclusive tile offsets (in place) and the block counts of the 3 lines
__global__ void k_blk_scan(unsigned int* __restrict__ cnt, int tiles, long long* __restrict__ hdr) {
  if (threadIdx.x < 2) {
    unsigned int* c = cnt + threadIdx.x * (tiles + 1);
    unsigned run = 0;
    for (int t = 0; t < tiles; ++t) {
      const unsigned v = c[t];
      c[t] = run;
      run += v;
    }
    hdr[1 + threadIdx.x] = run;
  }
  if (threadIdx.x == 2) hdr[0] = 1;
}

template <typename K>
__device__ __forceinline__ void put_first(SumRec& r, const K* pc, const uint32_t* gidx,
                                          const int* pos, uint32_t lid, unsigned long long key) {
  r.key = key;
  r.fpc = (unsigned long long)pc[lid];
  r.fgid = (int)gidx[lid];
  r.frow = pos[lid];
  r.flid = (int)lid;
}
template <typename K>
__device__ __forceinline__ void put_last(SumRec& r, const K* pc, const uint32_t* gidx,
                                         const int* pos, uint32_t lid) {
  r.lpc = (unsigned long long)pc[lid];
  r.lgid = (int)gidx[lid];
  r.lrow = pos[lid];
  r.llid = (int)lid;
}

// block records of lines 2 and 3 in sorted order (+ the single line-1 block)
template <typename K>
__global__ void __launch_bounds__(kBlock) k_blk_emit(const uint32_t* __restrict__ p0,
                                                     const uint32_t* __restrict__ p1,
                                                     const uint32_t* __restrict__ p2,
                                                     const K* __restrict__ pc, int64_t n, int b,
                                                     const unsigned int* __restrict__ cnt,
                                                     int tiles, const uint32_t* __restrict__ gidx,
                                                     const int* __restrict__ pos, SumRec* s0,
                                                     SumRec* s1, SumRec* s2) {
  __shared__ unsigned s_w[kBlock / 32];
  const int line = 1 + blockIdx.y;
  const uint32_t* perm = line == 1 ? p1 : p2;
  SumRec* out = line == 1 ? s1 : s2;
  const int64_t base = (int64_t)blockIdx.x * kBlkTile + (int64_t)threadIdx.x * kBlkIPT;
  // this thread's run of kBlkIPT consecutive sorted positions
  bool st[kBlkIPT];
  unsigned mine = 0;
#pragma unroll
  for (int j = 0; j < kBlkIPT; ++j) {
    const int64_t k = base + j;
    st[j] = k < n && blk_start(perm, pc, k, line, b);
    mine += st[j];
  }
  // block-wide exclusive scan of the per-thread counts
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned v = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) s_w[warp] = v;
  __syncthreads();
  unsigned wofs = 0;
  for (int w = 0; w < warp; ++w) wofs += s_w[w];
  unsigned ex = cnt[blockIdx.y * (tiles + 1) + blockIdx.x] + wofs + v - mine;
#pragma unroll
  for (int j = 0; j < kBlkIPT; ++j) {
    const int64_t k = base + j;
    if (k >= n) break;
    const uint32_t lid = perm[k];
    if (st[j]) put_first(out[ex], pc, gidx, pos, lid, seg_key(pc[lid], line, b));
    ex += st[j];
    const bool last = (k == n - 1) || blk_start(perm, pc, k + 1, line, b);
    if (last) put_last(out[ex - 1], pc, gidx, pos, lid);
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    put_first(s0[0], pc, gidx, pos, p0[0], 0ull);
    put_last(s0[0], pc, gidx, pos, p0[n - 1]);
  }
}

// first index in [0, m) with key > k (upper) or >= k (lower)
__device__ __forceinline__ long long bsearch_key(const SumRec* a, long long m,
                                                 unsigned long long k, bool upper) {
  long long lo = 0, hi = m;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    const unsigned long long v = a[mid].key;
    if (upper ? (v <= k) : (v < k)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// For every own block: the (key, rank)-preceding and -following block over
// all ranks.  A foreign neighbour becomes a halo record (local id
// n_own + 2t + side); an own neighbour is already the local sort's.
template <typename K>
__global__ void __launch_bounds__(kBlock) k_resolve(SlabGC g, int2* __restrict__ cand) {
  const long long B1 = g.hdr[1], B2 = g.hdr[2];
  const long long total = 1 + B1 + B2;
  K* epc = reinterpret_cast<K*>(g.ext_pc);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
    const int line = t == 0 ? 0 : (t <= B1 ? 1 : 2);
    const long long bi = t == 0 ? 0 : (line == 1 ? t - 1 : t - 1 - B1);
    const long long nb_own = line == 0 ? 1 : (line == 1 ? B1 : B2);
    const SumRec* own = g.sums[line];
    const SumRec me = own[bi];
    const unsigned long long k = me.key;
    // best predecessor (key', rank') < (k, r) and successor > (k, r)
    int prank = -1, srank = -1;
    long long pidx = -1, sidx = -1;
    unsigned long long pkey = 0, skey = 0;
    auto better_pred = [&](unsigned long long kk, int rr) {
      return prank < 0 || kk > pkey || (kk == pkey && rr > prank);
    };
    auto better_succ = [&](unsigned long long kk, int rr) {
      return srank < 0 || kk < skey || (kk == skey && rr < srank);
    };
    if (bi > 0) {
      prank = g.rank;
      pidx = bi - 1;
      pkey = own[bi - 1].key;
    }
    if (bi + 1 < nb_own) {
      srank = g.rank;
      sidx = bi + 1;
      skey = own[bi + 1].key;
    }
    for (int s = 0; s < g.world; ++s) {
      if (s == g.rank) continue;
      const SumRec* a = g.peer_sums[s][line];
      const long long m = g.peer_hdr[s][line];
      if (m <= 0) continue;
      // pred: s < r -> largest key' <= k; s > r -> largest key' < k
      const long long pp = bsearch_key(a, m, k, s < g.rank) - 1;
      if (pp >= 0) {
        const unsigned long long kk = a[pp].key;
        if (better_pred(kk, s)) {
          prank = s;
          pidx = pp;
          pkey = kk;
        }
      }
      // succ: s > r -> smallest key' >= k; s < r -> smallest key' > k
      const long long ss = bsearch_key(a, m, k, s < g.rank);
      if (ss < m) {
        const unsigned long long kk = a[ss].key;
        if (better_succ(kk, s)) {
          srank = s;
          sidx = ss;
          skey = kk;
        }
      }
    }
    int pred = -1, succ = -1;
    if (prank == g.rank) {
      pred = own[pidx].llid;
    } else if (prank >= 0) {
      const SumRec& o = g.peer_sums[prank][line][pidx];
      const int64_t h = g.n_own + 2 * t;
      epc[h] = (K)o.lpc;
      g.ext_gidx[h] = (uint32_t)o.lgid;
      g.ext_pos[h] = o.lrow;
      pred = (int)h;
    }
    if (srank == g.rank) {
      succ = own[sidx].flid;
    } else if (srank >= 0) {
      const SumRec& o = g.peer_sums[srank][line][sidx];
      const int64_t h = g.n_own + 2 * t + 1;
      epc[h] = (K)o.fpc;
      g.ext_gidx[h] = (uint32_t)o.fgid;
      g.ext_pos[h] = o.frow;
      succ = (int)h;
    }
    cand[(int64_t)line * g.n_own + me.flid].x = pred;
    cand[(int64_t)line * g.n_own + me.llid].y = succ;
  }
}

__global__ void k_iota_u32(uint32_t* __restrict__ out, int64_t n, int64_t base) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = (uint32_t)(base + i);
}

template <typename K>
static int slab_own_impl(fgbd_ctx* ctx, SlabGC& g) {
  const int64_t n = g.n_own;
  const int b = g.b;
  if (ctx->slg_coop) {
    int rc = launch_slg(ctx, n, b, g.ext_pos, g.lo);
    if (rc) return rc;
  } else {
    const int passes = (3 * b + 7) / 8;
    int rc = run_sort<K, true>(ctx, n, b, 3, passes, nullptr);
    if (rc) return rc;
    dim3 grid(grid_for(n, 1 << 20), 3);
    k_neighbors<<<grid, kBlock, 0, ctx->stream>>>(ctx->perm[0], ctx->perm[1], ctx->perm[2], n,
                                                  ctx->cand, g.ext_pos, ctx->ctl, g.lo);
    FGBD_LAUNCH(ctx);
  }
  ctx->rowid = ctx->perm[0];
  // own packed coordinates into the extended array (halo records follow them)
  FGBD_CUDA(ctx, cudaMemcpyAsync(g.ext_pc, ctx->pc, (size_t)n * sizeof(K), cudaMemcpyDeviceToDevice,
                                 ctx->stream));
  const int tiles = (int)((n + kBlkTile - 1) / kBlkTile);
  const K* pc = (const K*)ctx->pc;
  k_blk_count<K><<<dim3(tiles, 2), kBlock, 0, ctx->stream>>>(ctx->perm[1], ctx->perm[2], pc, n, b,
                                                             g.tile_cnt, tiles);
  FGBD_LAUNCH(ctx);
  k_blk_scan<<<1, 32, 0, ctx->stream>>>(g.tile_cnt, tiles, g.hdr);
  FGBD_LAUNCH(ctx);
  k_blk_emit<K><<<dim3(tiles, 2), kBlock, 0, ctx->stream>>>(
      ctx->perm[0], ctx->perm[1], ctx->perm[2], pc, n, b, g.tile_cnt, tiles, g.ext_gidx,
      g.ext_pos, g.sums[0], g.sums[1], g.sums[2]);
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

int launch_graph_slab_own(fgbd_ctx* ctx, SlabGC& g) {
  if (g.n_own < 1) return set_error(ctx, FGBD_E_ARG, "a slab rank needs at least one point");
  int rc = (3 * g.b <= 32) ? slab_own_impl<uint32_t>(ctx, g)
                           : slab_own_impl<unsigned long long>(ctx, g);
  if (rc) return rc;
  ctx->g_reordered = 1;
  ctx->g_n = -1;  // not a stage-API graph
  ctx->g_bits = g.b;
  ctx->g_have_weights = 0;
  ctx->g_have_noise = 0;
  ctx->held_valid = 0;
  return FGBD_OK;
}

template <typename K>
static int slab_rows_impl(fgbd_ctx* ctx, SlabGC& g) {
  const int64_t n = g.n_own;
  const int rgrid = grid_for(1 + 2 * g.blk_cap, ctx->num_sms * 8);
  k_resolve<K><<<rgrid, kBlock, 0, ctx->stream>>>(g, ctx->cand);
  FGBD_LAUNCH(ctx);
  const int grid = grid_for(n, ctx->rows_grid == 1 ? (1 << 30) : kRowsGrid);
  k_rows<K, false, true><<<grid, kBlock, 0, ctx->stream>>>(
      ctx->cand, (const K*)g.ext_pc, n, g.b, g.ext_pos, ctx->rowid, EllRef{ctx->nbr, ctx->pay},
      ctx->meta, ctx->partials, ctx->ctl, RowsSlab{g.ext_gidx, g.lo});
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

int launch_graph_slab_rows(fgbd_ctx* ctx, SlabGC& g) {
  if (g.b > 15)
    return set_error(ctx, FGBD_E_ARG, "slab partition supports bit depths up to 15");
  return (3 * g.b <= 32) ? slab_rows_impl<uint32_t>(ctx, g)
                         : slab_rows_impl<unsigned long long>(ctx, g);
}

int launch_weights_slab(fgbd_ctx* ctx, const SlabGC& g) {
  const int grid = grid_for(g.n_own, ctx->num_sms * 8);
  if (3 * g.b <= 32)
    k_weights<uint32_t, false, false><<<grid, kBlock, 0, ctx->stream>>>(
        EllRef{ctx->nbr, ctx->pay}, nullptr, (const uint32_t*)g.ext_pc, g.n_own, g.b, nullptr,
        ctx->ctl, g.lo);
  else
    k_weights<unsigned long long, false, false><<<grid, kBlock, 0, ctx->stream>>>(
        EllRef{ctx->nbr, ctx->pay}, nullptr, (const unsigned long long*)g.ext_pc, g.n_own, g.b,
        nullptr, ctx->ctl, g.lo);
  FGBD_LAUNCH(ctx);
  ctx->g_have_weights = 1;
  ctx->g_weights64 = 0;
  return FGBD_OK;
}

int launch_iota_u32(fgbd_ctx* ctx, uint32_t* out, int64_t n, int64_t base) {
  k_iota_u32<<<grid_for(n, ctx->num_sms * 8), kBlock, 0, ctx->stream>>>(out, n, base);
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

}  // namespace fgbd

#if FGBD_SORT_TLOG
extern "C" int fgbd_debug_stlog(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, fgbd::g_stlog, sizeof(fgbd::g_stlog));
}
#endif
