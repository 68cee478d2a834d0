// Internal declarations shared by the FGBD B200 translation units.
//
// Device data layout for one frame of N points:
//   pc        packed coordinates = the line-1 scan code z<<2b | y<<b | x,
//             uint32 when 3b <= 32 else uint64 (4 or 8 B/pt)
//   sort      per line: keys/vals ping-pong + onesweep look-back status
//   perm      per line: stable rank order (uint32, the sort's last pass)
//   cand      per line: (prev, next) rank neighbour, int2 (24 B/pt total)
//   ell       6 slots per point, slot-major [s][N], int2 = (neighbour,
//             payload) where payload is the exact squared distance (uint32)
//             until the weight pass replaces it by the fp32 Gaussian weight;
//             padding slots hold (self, 0)
//   meta      per point: degree (3 bits) | patch order (6 x 3 bits)
//   buf[3]    fp64 (N,4) signals (r,g,b,0) -- one 32 B sector per point:
//             Y = noisy input, A, B (select_q rotation)
//   fslr      per point FSLR statistic (fp64, -1 = not eligible)
//   mask      1 bit per point (FSLR include)
//   ctl       device control block (reductions, select_q state)
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <string>

#include "fgbd_b200.h"

namespace fgbd {
struct EllRef;
struct HostStager;
}

namespace fgbd {

constexpr int kBlock = 256;
constexpr int kRedGrid = 148 * 4;      // fixed partition => deterministic sums
constexpr int kRowsGrid = 148 * 8;     // k_rows grid cap (sigma_g is exact: any grid gives its bits)
constexpr int kNeGrid = 148 * 16;      // NE blocks (96 threads: one warp per channel)
constexpr int kSortThreads = 256;
#ifndef FGBD_SORT_IPT
#define FGBD_SORT_IPT 16
#endif
constexpr int kSortIPT = FGBD_SORT_IPT;
constexpr int kSortTile = kSortThreads * kSortIPT;  // keys per onesweep tile
constexpr int kRadix = 256;
constexpr int kMaxPasses = 8;
constexpr int kSlots = 6;              // max SLG degree: 2 neighbours x 3 lines
constexpr int kFarRows = 512;          // a "far" neighbour row (scattered gather) for the filter

enum BufId { BUF_Y = 0, BUF_A = 1, BUF_B = 2 };

// Device control block.  Written by "last block done" reducers, read by the
// next kernel in stream order and mirrored to pinned host memory.
struct Ctl {
  // graph construction
  unsigned long long n_edges;
  double sigma_g;
  int max_deg;
  int err_flags;  // bit0: coordinate out of range, bit3: line-1 order is not the identity
  // noise estimation
  long long eligible;
  double gram[3][64];  // per-channel 8x8 Gram matrix of shifted patch rows
  // FSLR mask
  long long included;
  int mask_all;
  int all_excluded;
  double sy[3];
  // select_q state machine (filtering.py:225-256)
  int q;
  int best_q;
  int stop;
  int streak;
  int steps;
  int in_buf;
  int out_buf;
  int best_buf;
  double best_crit;
  double prev_crit;
  double sv2;       // sigma_est^2
  int q_max;
  int mode;         // FGBD_CRIT_*
  int early_exit;
  double trace[FGBD_TRACE_MAX];
  unsigned int ticket[8];
  // slab ranks: this rank's share before the cross-rank all-gather
  unsigned long long sg_fx[2];  // exact fixed-point sum of edge lengths (k_rows)
  double mask_part[7];          // k_mask totals: count, sum_inc y^2 [3], sum_all y^2 [3]
  // NE-GBP finished on the device (k_finish_noise): noise.py:122-249
  int nz_err;                   // NzErr code (0: ok)
  int nz_err_arg;               // channel / count / degree for the message
  double nz_err_val;            // off-diagonal norm of a non-converged Jacobi
  double nz_sigma, nz_pcs[3], nz_eig[3][8], nz_tau[3];
  int nz_m[3], nz_fb[3], nz_direct[3];
  double fslr_thr;              // 2 sigma_est
  int fslr_active;              // FSLR mask on
  unsigned long long far_slots; // k_rows: edges to rows more than kFarRows away (both ends)
};

enum NzErr {
  NZ_OK = 0, NZ_PATCH = 1, NZ_FEW = 2, NZ_ASYM = 3, NZ_NOCONV = 4, NZ_TAIL_D = 5, NZ_TAIL_SORT = 6
};

constexpr int kMaxRanks = 16;

// One scan-line block of a slab rank: the run of its points that share the
// line's segment key (line 1: everything; line 2: x; line 3: (y, x)) in
// that line's sorted order, with its first and last point.  Because the
// slabs are z-ranges, the global sorted order of a line is the blocks
// ordered by (key, rank): cross-slab scan-line neighbours are exactly the
// last/first points of (key, rank)-adjacent blocks.
struct SumRec {
  unsigned long long key, fpc, lpc;  // segment key; packed coords of first/last point
  int fgid, lgid;                    // global point indices (reference index order)
  int frow, lrow;                    // global rows (global scan-line-1 rank)
  int flid, llid;                    // local ids on the owning rank
};

// Signal rows of every slab rank by GLOBAL row: y[r] + j addresses row j of
// rank r's buffer (y[r] = buffer base - lo[r]; peer-mapped for r != self).
struct SlabView {
  int world, self;
  int64_t lo[kMaxRanks + 1];
  const double4* y[kMaxRanks];
};

// Graph-construction state of one slab rank (csrc/graph.cu, csrc/slab.cu).
struct SlabGC {
  int world, rank, b;
  int64_t n_own, lo;           // own points; global row of own row 0
  int64_t blk_cap;             // per-line capacity of the block lists
  void* ext_pc;                // [n_own + 2 * (1 + 2 blk_cap)] packed coords (own, then halo)
  int* ext_pos;                // same: global row of every local id
  uint32_t* ext_gidx;          // same: global point index of every local id
  unsigned int* tile_cnt;      // scratch [2][tiles + 1]
  SumRec* sums[3];             // own block lists (peer-visible region)
  long long* hdr;              // own block counts [3] (peer-visible region)
  const SumRec* peer_sums[kMaxRanks][3];
  const long long* peer_hdr[kMaxRanks];
};

struct SortScratch {
  void* keys[2][3] = {};        // ping-pong key buffers per line
  uint32_t* vals[2][3] = {};    // ping-pong value buffers per line
  uint32_t* hist = nullptr;     // [3][kMaxPasses][256] counts -> bases
  unsigned long long* status = nullptr;  // [3][tiles][256] look-back words
  unsigned int* tile_ctr = nullptr;      // [kMaxPasses][3]
  int64_t tiles_cap = 0;
  unsigned int epoch = 0;
};

}  // namespace fgbd

struct fgbd_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;   // colour upload, overlapped with graph construction
  cudaEvent_t ev_side = nullptr;
  int64_t cap = 0;        // points the scratch is sized for
  int key64_cap = 0;      // scratch sized for 64-bit keys
  size_t dev_bytes = 0;

  int64_t* coords64 = nullptr;  // (N,3) int64 staging (H2D target)
  const int64_t* cur_coords = nullptr;  // coordinates of the frame being built (device)
  double** d_bufs = nullptr;    // device copy of buf[] (for ctl-selected buffers)
  void* pc = nullptr;           // packed coords (uint32 or uint64)
  fgbd::SortScratch sort;
  uint32_t* perm[3] = {};       // aliases into sort.vals after the last pass
  int2* cand = nullptr;         // [3][N]
  int* nbr = nullptr;           // ELL, interleaved int4 pairs [3][N] (see eslot)
  uint32_t* pay = nullptr;      // = nbr + 1: payload view of the same array
  double* w64 = nullptr;        // [6][N] fp64 weights (parity mode, lazy)
  uint32_t* meta = nullptr;     // [N]
  double* buf[3] = {};          // Y, A, B signals (N,4) fp64
  double* out = nullptr;        // (N,3) fp64 result staging
  double* fslr = nullptr;       // [N]
  uint32_t* mask = nullptr;     // [ceil(N/32)]
  double* partials = nullptr;   // reduction partials (>= 1<<19 doubles)
  unsigned int* tickets = nullptr;  // group tickets for hierarchical reductions
  int lf_variant = 10;          // filter-step kernel (FGBD_LF_VARIANT): 0 per-step, 2+ persistent
  int coop_blocks[64] = {};     // co-resident grid of each persistent instantiation
  int lf_shape = 0;             // persistent kernel block shape (FGBD_LF_SHAPE)
  int lf_halo = 128;            // FGBD_LF_HALO: window rows either side of a TMA tile
  int lf_chunk = -1;            // FGBD_LF_CHUNK: contiguous row range per block (0 = grid-stride,
                                //   -1 = auto: contiguous while 3 signal buffers fit in L2)
  int64_t l2_bytes = 0;         // device L2 capacity
  int reorder_rows = 1;         // FGBD_REORDER: denoise-path rows in scan-line-1 order
  int prep_mult = 8;            // k_prep blocks per SM (FGBD_PREP_MULT)
  int sort_derived = 1;         // FGBD_SORT_DERIVED: lines 2/3 by one field of the previous order
  int mask_fold = 1;             // FGBD_MASK_FOLD: the FSLR mask built by the first filter step
  int lf_far = -1;              // FGBD_LF_FAR: far gathers skip L1 (-1 auto: >= half the slots far)
  int lf_far_now = 0;           // the choice for the frame being filtered
  int held_far = 0;             // far-slot majority of the held (reused) graph
  int slg_coop = 1;             // FGBD_SLG_COOP: scan-line front end in one cooperative launch
  int jacobi_threads = 1;       // FGBD_JACOBI_THREADS: the 3 channels on 3 host threads
  const double* expand_colors = nullptr;  // (N,3) device colours k_rows expands into BUF_Y (one build)
  int rows_expand = 1;          // FGBD_ROWS_EXPAND: device colours expanded by k_rows
  int hold_guess = 0;           // this context's last select-q scan stopped early (early exit)
  int lf_hold = -1;             // FGBD_LF_HOLD: -1 auto (hold_guess), 0 never, 1 always
  int slg_grid[2] = {0, 0};     // its co-resident grid (32- / 64-bit codes)
  uint32_t* slg_cnt = nullptr;  // its digit-count table
  int rows_grid = 0;            // FGBD_ROWS_GRID: k_rows grid, 0 = 8 blocks/SM (grid-stride), 1 = one row per thread
  int l2_persist = 0;           // pin the ELL graph in L2 (FGBD_L2_PERSIST)
  int ne_variant = 1;           // 0: warp per channel, 1: thread per point (FGBD_NE_VARIANT)
  fgbd::Ctl* ctl = nullptr;     // device
  fgbd::Ctl* ctl_host = nullptr;  // pinned mirror
  // scratch for CSR export / injection (lazy)
  int64_t* scan_tmp = nullptr;
  int64_t scan_cap = 0;
  void* csr_scratch = nullptr;
  void* ply_stage = nullptr;     // PLY records in/out (fgbd_denoise_ply)
  size_t ply_stage_bytes = 0;
  unsigned long long* p2p_flags = nullptr;  // persistent-kernel step flags (lf_variant 13)
  unsigned long long p2p_epoch = 1ull << 20;
  void* aux = nullptr;           // off-path scratch (kNN graph), grown on demand
  size_t aux_bytes = 0;
  int64_t knn_n = -1, knn_e = 0;  // kNN graph held in aux
  size_t knn_off[6] = {0, 0, 0, 0, 0, 0};
  size_t csr_scratch_bytes = 0;

  cudaEvent_t ev[8] = {};

  // state of the graph held by the context
  int64_t g_n = -1;
  int g_reordered = 0;            // rows of the held graph are in line-1 order
  const uint32_t* rowid = nullptr;  // row -> point (line-1 perm) when reordered
  int* pos = nullptr;             // point -> row (cap)
  cudaEvent_t ev_perm = nullptr;  // line-1 permutation ready (main stream)
  cudaEvent_t ev_done = nullptr;  // this context's last frame compute finished
  int async_lock = 1;             // FGBD_ASYNC_LOCK: order frames on the GPU, not the host
  // static-geometry reuse (FGBD_FLAG_REUSE_GRAPH): coordinates and header of
  // the held graph
  int64_t* held_coords = nullptr;  // 3 x held_cap int64
  int64_t held_cap = 0;
  int held_valid = 0;
  unsigned long long held_edges = 0;
  double held_sigma_g = 0.0;
  int held_max_deg = 0;
  int g_bits = 0;
  int g_weights64 = 0;
  int g_have_weights = 0;
  int g_have_noise = 0;
  int g_patch = 0;

  int launches = 0;
  std::string err;
  // pageable host inputs: parallel staging through pinned memory (hoststage.cu)
  fgbd::HostStager* stager = nullptr;
  int host_threads = 6;           // FGBD_HOST_THREADS (0: the driver's own pageable copy)
};

namespace fgbd {

// ---- error plumbing ------------------------------------------------------
int set_error(fgbd_ctx* ctx, int code, const std::string& msg);
int cuda_error(fgbd_ctx* ctx, cudaError_t e, const char* where);
#define FGBD_CUDA(ctx, call)                                   \
  do {                                                         \
    cudaError_t e__ = (call);                                  \
    if (e__ != cudaSuccess) return fgbd::cuda_error(ctx, e__, #call); \
  } while (0)
#define FGBD_LAUNCH(ctx)                                       \
  do {                                                         \
    (ctx)->launches++;                                         \
    cudaError_t e__ = cudaGetLastError();                      \
    if (e__ != cudaSuccess) return fgbd::cuda_error(ctx, e__, "kernel launch"); \
  } while (0)

// NVTX range over a host scope (the reference's per-stage timers,
// filtering.py:277-300, as profiler ranges: fgbd.graph / fgbd.noise / ...)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

int ensure_capacity(fgbd_ctx* ctx, int64_t n, int key64);
// host -> device from host memory: pageable sources go through the
// context's pinned staging (region 0 or 1) in parallel chunks, each chunk's
// DMA issued as soon as it has landed; pinned sources copy directly
int host_to_device(fgbd_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t s,
                   int region);
void destroy_stager(fgbd_ctx* ctx);
// src is pageable and large enough for the parallel staging above
bool host_stageable(fgbd_ctx* ctx, const void* src, size_t bytes);
int require_point_rows(fgbd_ctx* ctx);
// (N,3) colours (host or device) -> BUF_Y in the (N,4) layout
int upload_colors(fgbd_ctx* ctx, const double* colors, int64_t n, bool dev);
// same, issued on the side stream; the main stream waits for it at ev_side
int upload_colors_async(fgbd_ctx* ctx, const double* colors, int64_t n, bool dev);
// signal buffer (src_buf < 0: the select_q best) -> (N,3) host/device array
int download_signal(fgbd_ctx* ctx, int src_buf, double* dst, int64_t n, bool dev, int clip);
int ensure_w64(fgbd_ctx* ctx, int64_t n);

// ---- graph construction (graph.cu) --------------------------------------
// Builds pc, sorts the 3 scan lines, writes cand/ell/meta, reduces sigma_g.
// coords64 already on device.  No host sync.
// reorder: store rows in scan-line-1 order (ctx->rowid / ctx->pos) -- the
// denoise path; stage-API graphs keep rows in point order
int launch_graph(fgbd_ctx* ctx, int64_t n, int bits, bool reorder = false);
// slg.cu: codes + scan-line orders + rank neighbours in one cooperative launch
int launch_slg(fgbd_ctx* ctx, int64_t n, int b, int* pos, int64_t row_base);
// Converts the ell payload (squared distances) into Gaussian weights.
int launch_weights(fgbd_ctx* ctx, int64_t n, int bits, int w64);
// Stand-alone stable argsort of 64-bit keys (radix_argsort).
int launch_argsort64(fgbd_ctx* ctx, const uint64_t* d_keys, int64_t n, int key_bits,
                     uint32_t** d_perm_out);
// Codes + perm for one line of the frame (codes written as uint64).
int launch_scan_line(fgbd_ctx* ctx, int64_t n, int bits, int line, uint64_t* d_codes,
                     uint32_t** d_perm_out);
// CSR export helpers (device): writes reference-convention arrays.
int launch_export(fgbd_ctx* ctx, int64_t n, int64_t* d_indptr, int64_t* d_indices,
                  int64_t* d_csr_edge, int64_t* d_edge_u, int64_t* d_edge_v,
                  double* d_sqdist, double* d_weights, double* d_wdeg,
                  int64_t* nnz_out, int64_t* e_out);

// exclusive scan of int64 (3 launches); tmp >= ceil(n/2048), *d_total gets the sum
int scan_exclusive(fgbd_ctx* ctx, const int64_t* in, int64_t n, int64_t* out, int64_t* tmp,
                   int64_t* d_total);

// ---- noise estimation (noise.cu) ----------------------------------------
// NE pass; fuse_weights: also convert the ELL payloads to Gaussian weights
// (only valid before launch_weights ran and when b <= 15)
int launch_noise(fgbd_ctx* ctx, int64_t n, int patch, int fuse_weights);
// slab rank: own rows, neighbour colours by global row through `v`
int launch_noise_slab(fgbd_ctx* ctx, int64_t n_own, int patch, const SlabView& v);
// host side: covariance -> Jacobi -> tail -> sigma (noise.py:122-243)
int finish_noise(fgbd_ctx* ctx, int patch, int divisor, fgbd_noise* out);
// the same on the device, bit for bit (no host round trip): writes the nz_*
// fields, sv2 and the FSLR threshold into ctl
int launch_finish_noise(fgbd_ctx* ctx, int patch, int divisor, int fslr_enabled,
                        double sigma_floor);
// host: the error k_finish_noise recorded (ctl mirror current), as finish_noise would raise it;
// otherwise fills *out from the device results
int collect_noise(fgbd_ctx* ctx, int patch, fgbd_noise* out);
int jacobi_eigenvalues(const double* s, int d, double* out_desc, std::string* err,
                       int* direct_off);
int jacobi_eigenvalues_multi(int nm, const double* const* s, int d, double* const* out_desc,
                             std::string* err, int* rc, int* direct_off);
// wake the Jacobi helper threads (finish_noise follows within ~2 ms)
void jacobi_pool_prepare();
int select_tail_host(const double* lam, int d, int divisor, int* m, double* tau,
                     int* fallback, std::string* err);

// ---- filter (filter.cu) --------------------------------------------------
// (N,3) device colours -> signal buffer `buf` in the (N,4) layout
int launch_expand(fgbd_ctx* ctx, const double* d_src, int64_t n, int buf, cudaStream_t s);
// signal buffer (or the select_q best buffer when src_buf < 0) -> (N,3), optional clip
int launch_compact(fgbd_ctx* ctx, int64_t n, int src_buf, double* d_dst, int clip);
int launch_mask(fgbd_ctx* ctx, int64_t n, double sigma_est, int active, int q_max, int mode,
                int early_exit, const uint8_t* d_include_bytes);
int launch_mask_slab(fgbd_ctx* ctx, int64_t n_own, const double4* y, double sigma_est,
                     int active);
int launch_select_steps(fgbd_ctx* ctx, int64_t n, int q_max, int w64);
// the FSLR mask (k_mask) folded into the first filter step
bool mask_foldable(const fgbd_ctx* ctx, int q_max, int w64);
int launch_select_steps_folded(fgbd_ctx* ctx, int64_t n, int q_max, int mode, int early_exit,
                               const double* sigma_est, int active);
// persistent filter: contiguous row range per block (true) or grid-stride waves
bool lf_contiguous(const fgbd_ctx* ctx, int64_t rows);
int launch_fixed_steps(fgbd_ctx* ctx, int64_t n, int q, int w64, int* final_buf);
int launch_csr_steps(fgbd_ctx* ctx, const int64_t* d_indptr, const int64_t* d_indices,
                     const double* d_w, int64_t n, const double* d_in, double* d_tmp,
                     double* d_out, int q);
int launch_criterion(fgbd_ctx* ctx, const double* d_y, const double* d_x,
                     const uint8_t* d_inc, int64_t n, double sigma_est, int mode,
                     double* crit_out);

}  // namespace fgbd

namespace fgbd {
// ---- slab ranks (graph.cu) -------------------------------------------------
// Phase 1: sort the own points (coords in ctx->cur_coords, gidx in
// g.ext_gidx), rank neighbours, global rows, block lists of the 3 lines.
int launch_graph_slab_own(fgbd_ctx* ctx, SlabGC& g);
// Phase 2 (after every rank published its block lists): cross-slab
// neighbours from the peers' lists, halo records, then the rows (ELL words =
// global rows) and this rank's sigma_g share in ctl->sg_fx / n_edges / max_deg.
int launch_graph_slab_rows(fgbd_ctx* ctx, SlabGC& g);
// Eq. (4) on own rows (cached path; NE fuses it otherwise)
int launch_weights_slab(fgbd_ctx* ctx, const SlabGC& g);
int launch_iota_u32(fgbd_ctx* ctx, uint32_t* out, int64_t n, int64_t base);
}  // namespace fgbd
