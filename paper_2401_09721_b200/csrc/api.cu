// C ABI (include/fgbd_b200.h): context lifetime, the `denoise` drop-in
// (reference filtering.py:259-328) and the stage entry points.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fgbd_internal.cuh"

namespace fgbd {

thread_local std::string g_global_err;

int set_error(fgbd_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  else g_global_err = msg;
  return code;
}

int cuda_error(fgbd_ctx* ctx, cudaError_t e, const char* where) {
  return set_error(ctx, FGBD_E_CUDA,
                   std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e));
}

template <typename T>
static int dalloc(fgbd_ctx* ctx, T** p, size_t count) {
  if (*p) cudaFree(*p);
  *p = nullptr;
  if (count == 0) count = 1;
  const size_t bytes = count * sizeof(T);
  FGBD_CUDA(ctx, cudaMalloc((void**)p, bytes));
  ctx->dev_bytes += bytes;
  return FGBD_OK;
}

static void free_scratch(fgbd_ctx* ctx) {
  auto f = [](void* p) {
    if (p) cudaFree(p);
  };
  f(ctx->coords64);
  f(ctx->pc);
  for (int a = 0; a < 2; ++a)
    for (int l = 0; l < 3; ++l) {
      f(ctx->sort.keys[a][l]);
      f(ctx->sort.vals[a][l]);
      ctx->sort.keys[a][l] = nullptr;
      ctx->sort.vals[a][l] = nullptr;
    }
  f(ctx->sort.status);
  f(ctx->cand);
  f(ctx->nbr);
  f(ctx->w64);
  f(ctx->meta);
  f(ctx->pos);
  for (int k = 0; k < 3; ++k) {
    f(ctx->buf[k]);
    ctx->buf[k] = nullptr;
  }
  f(ctx->out);
  f(ctx->fslr);
  f(ctx->mask);
  ctx->coords64 = nullptr;
  ctx->pc = nullptr;
  ctx->sort.status = nullptr;
  ctx->cand = nullptr;
  ctx->nbr = nullptr;
  ctx->pay = nullptr;
  ctx->w64 = nullptr;
  ctx->meta = nullptr;
  ctx->pos = nullptr;
  ctx->rowid = nullptr;
  ctx->g_reordered = 0;
  ctx->out = nullptr;
  ctx->fslr = nullptr;
  ctx->mask = nullptr;
  ctx->cap = 0;
  ctx->dev_bytes = 0;
  ctx->g_n = -1;
}

int ensure_capacity(fgbd_ctx* ctx, int64_t n, int key64) {
  if (n <= ctx->cap && (!key64 || ctx->key64_cap)) return FGBD_OK;
  ctx->held_valid = 0;
  int64_t cap = std::max<int64_t>(n, ctx->cap);
  cap = ((cap + 65535) / 65536) * 65536;
  const int k64 = key64 || ctx->key64_cap;
  free_scratch(ctx);
  const size_t ksz = k64 ? 8 : 4;
  int rc;
  if ((rc = dalloc(ctx, &ctx->coords64, 3 * cap))) return rc;
  if ((rc = dalloc(ctx, (unsigned long long**)&ctx->pc, cap))) return rc;
  for (int a = 0; a < 2; ++a)
    for (int l = 0; l < 3; ++l) {
      if ((rc = dalloc(ctx, (unsigned char**)&ctx->sort.keys[a][l], cap * ksz))) return rc;
      if ((rc = dalloc(ctx, &ctx->sort.vals[a][l], cap))) return rc;
    }
  const int64_t tiles = (cap + kSortTile - 1) / kSortTile;
  if ((rc = dalloc(ctx, &ctx->sort.status, 3 * tiles * kRadix))) return rc;
  FGBD_CUDA(ctx, cudaMemset(ctx->sort.status, 0, 3 * tiles * kRadix * 8));
  ctx->sort.tiles_cap = tiles;
  if ((rc = dalloc(ctx, &ctx->cand, 3 * cap))) return rc;
  if ((rc = dalloc(ctx, &ctx->nbr, 2 * kSlots * cap))) return rc;
  ctx->pay = reinterpret_cast<uint32_t*>(ctx->nbr + 1);
  if ((rc = dalloc(ctx, &ctx->meta, cap))) return rc;
  if ((rc = dalloc(ctx, &ctx->pos, cap))) return rc;
  for (int k = 0; k < 3; ++k)
    if ((rc = dalloc(ctx, &ctx->buf[k], 4 * cap))) return rc;
  if ((rc = dalloc(ctx, &ctx->out, 3 * cap))) return rc;
  if ((rc = dalloc(ctx, &ctx->fslr, cap))) return rc;
  if ((rc = dalloc(ctx, &ctx->mask, (cap + 31) / 32 + 1))) return rc;
  FGBD_CUDA(ctx, cudaMemcpy(ctx->d_bufs, ctx->buf, sizeof(ctx->buf), cudaMemcpyHostToDevice));
  {
    // reduction partials: one-row-per-thread kernels need 3 per block + group totals
    const int64_t blocks = (cap + kBlock - 1) / kBlock;
    const int64_t need = std::max<int64_t>(1 << 19, 3 * blocks + 3 * (blocks / 64 + 1) + 1024);
    if ((rc = dalloc(ctx, &ctx->partials, need))) return rc;
  }
  ctx->cap = cap;
  ctx->key64_cap = k64;
  return FGBD_OK;
}

int upload_colors(fgbd_ctx* ctx, const double* colors, int64_t n, bool dev) {
  if (n <= 0) return FGBD_OK;
  const double* src = colors;
  if (!dev) {
    FGBD_CUDA(ctx, cudaMemcpyAsync(ctx->out, colors, 3 * n * sizeof(double),
                                   cudaMemcpyHostToDevice, ctx->stream));
    src = ctx->out;
  }
  return launch_expand(ctx, src, n, BUF_Y, ctx->stream);
}

int upload_colors_async(fgbd_ctx* ctx, const double* colors, int64_t n, bool dev) {
  if (n <= 0) return FGBD_OK;
  const double* src = colors;
  if (!dev) {
    FGBD_CUDA(ctx, cudaMemcpyAsync(ctx->out, colors, 3 * n * sizeof(double),
                                   cudaMemcpyHostToDevice, ctx->side));
    src = ctx->out;
  }
  // reordered rows: the expansion gathers through the line-1 permutation
  if (ctx->g_reordered) FGBD_CUDA(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_perm, 0));
  int rc = launch_expand(ctx, src, n, BUF_Y, ctx->side);
  if (rc) return rc;
  FGBD_CUDA(ctx, cudaEventRecord(ctx->ev_side, ctx->side));
  return FGBD_OK;
}

int download_signal(fgbd_ctx* ctx, int src_buf, double* dst, int64_t n, bool dev, int clip) {
  if (n <= 0) return FGBD_OK;
  double* stage = dev ? dst : ctx->out;
  int rc = launch_compact(ctx, n, src_buf, stage, clip);
  if (rc) return rc;
  if (!dev)
    FGBD_CUDA(ctx, cudaMemcpyAsync(dst, ctx->out, 3 * n * sizeof(double), cudaMemcpyDeviceToHost,
                                   ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FGBD_OK;
}

int ensure_w64(fgbd_ctx* ctx, int64_t n) {
  if (ctx->w64) return FGBD_OK;
  return dalloc(ctx, &ctx->w64, kSlots * ctx->cap);
}

}  // namespace fgbd

using namespace fgbd;

namespace {

// Optionally pin the ELL graph in L2 across the filter steps of a frame.
void apply_l2_policy(fgbd_ctx* ctx, int64_t n) {
  if (!ctx->l2_persist) return;
  int max_persist = 0, max_window = 0;
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, ctx->device);
  cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device);
  const size_t bytes = (size_t)2 * kSlots * n * sizeof(int);
  const size_t lim = std::min<size_t>(bytes, (size_t)max_persist);
  const size_t win = std::min<size_t>(bytes, (size_t)max_window);
  if (lim == 0 || win == 0) return;
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim);
  cudaStreamAttrValue v;
  std::memset(&v, 0, sizeof(v));
  v.accessPolicyWindow.base_ptr = ctx->nbr;
  v.accessPolicyWindow.num_bytes = win;
  v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)lim / (float)win);
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &v);
  cudaGetLastError();
}

int check_cfg(fgbd_ctx* ctx, const fgbd_config* c) {
  if (!c) return set_error(ctx, FGBD_E_ARG, "config must not be NULL");
  if (c->q_max < 0)
    return set_error(ctx, FGBD_E_FILTER, "q_max must be >= 0, got " + std::to_string(c->q_max));
  if (c->reestimate_interval < 1)
    return set_error(ctx, FGBD_E_FILTER, "reestimate_interval must be >= 1, got " +
                                             std::to_string(c->reestimate_interval));
  if (c->patch_size < 2)
    return set_error(ctx, FGBD_E_FILTER,
                     "patch_size must be >= 2, got " + std::to_string(c->patch_size));
  if (c->criterion_mode != FGBD_CRIT_POOLED && c->criterion_mode != FGBD_CRIT_PER_CHANNEL)
    return set_error(ctx, FGBD_E_FILTER, "unknown criterion_mode");
  if (c->tau_divisor != FGBD_TAU_COUNT && c->tau_divisor != FGBD_TAU_COUNT_PLUS_ONE)
    return set_error(ctx, FGBD_E_NOISE, "unknown divisor rule");
  return FGBD_OK;
}

int check_graph_input(fgbd_ctx* ctx, int64_t n, int bits) {
  if (bits < 1 || bits > 21)
    return set_error(ctx, FGBD_E_GRAPH, "bit depth " + std::to_string(bits) +
                                            " exceeds 21 (64-bit code overflow)");
  if (n >= (int64_t(1) << 31))
    return set_error(ctx, FGBD_E_GRAPH, "point count exceeds the 2^31 edge-encoding limit");
  if (n > (int64_t)8192 * 64 * kBlock)
    return set_error(ctx, FGBD_E_ARG, "frames above 134M points are not supported by this build");
  return FGBD_OK;
}

int h2d(fgbd_ctx* ctx, void* dst, const void* src, size_t bytes, bool dev) {
  if (bytes == 0) return FGBD_OK;
  FGBD_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes,
                                 dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                 ctx->stream));
  return FGBD_OK;
}

int d2h(fgbd_ctx* ctx, void* dst, const void* src, size_t bytes, bool dev) {
  if (bytes == 0) return FGBD_OK;
  FGBD_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes,
                                 dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                 ctx->stream));
  return FGBD_OK;
}

int pull_ctl(fgbd_ctx* ctx) {
  FGBD_CUDA(ctx, cudaMemcpyAsync(ctx->ctl_host, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost,
                                 ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FGBD_OK;
}

int reset_ctl(fgbd_ctx* ctx) {
  FGBD_CUDA(ctx, cudaMemsetAsync(ctx->ctl, 0, sizeof(Ctl), ctx->stream));
  return FGBD_OK;
}

__global__ void k_differs(const int64_t* __restrict__ a, const int64_t* __restrict__ b, int64_t m,
                          int* __restrict__ flag) {
  int diff = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    diff |= a[e] != b[e];
  if (__syncthreads_or(diff) && threadIdx.x == 0) atomicOr(flag, 1);
}

// *same = 1 when a[0..m) == b[0..m) bit for bit (one pass + a 4-byte D2H)
int coords_equal(fgbd_ctx* ctx, const int64_t* a, const int64_t* b, int64_t m, int* same) {
  int* d_flag = reinterpret_cast<int*>(ctx->partials);
  FGBD_CUDA(ctx, cudaMemsetAsync(d_flag, 0, sizeof(int), ctx->stream));
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((m + kBlock - 1) / kBlock, (int64_t)ctx->num_sms * 8));
  k_differs<<<grid, kBlock, 0, ctx->stream>>>(a, b, m, d_flag);
  FGBD_LAUNCH(ctx);
  int h = 1;
  FGBD_CUDA(ctx, cudaMemcpyAsync(&h, d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  *same = h == 0;
  return FGBD_OK;
}

// keep a copy of the coordinates the held graph is built from
int hold_coords(fgbd_ctx* ctx, const int64_t* src, int64_t n) {
  if (ctx->held_cap < n) {
    if (ctx->held_coords) cudaFree(ctx->held_coords);
    ctx->held_coords = nullptr;
    ctx->held_cap = 0;
    FGBD_CUDA(ctx, cudaMalloc(&ctx->held_coords, (size_t)n * 3 * sizeof(int64_t)));
    ctx->held_cap = n;
  }
  FGBD_CUDA(ctx, cudaMemcpyAsync(ctx->held_coords, src, (size_t)n * 3 * sizeof(int64_t),
                                 cudaMemcpyDeviceToDevice, ctx->stream));
  return FGBD_OK;
}

// graph fields of the control block for a frame that reuses the held graph
int restore_graph_header(fgbd_ctx* ctx) {
  struct {
    unsigned long long n_edges;
    double sigma_g;
    int max_deg, err_flags;
  } hdr{ctx->held_edges, ctx->held_sigma_g, ctx->held_max_deg, 0};
  static_assert(sizeof(hdr) == offsetof(Ctl, eligible), "Ctl graph header layout");
  FGBD_CUDA(ctx, cudaMemcpyAsync(ctx->ctl, &hdr, sizeof(hdr), cudaMemcpyHostToDevice, ctx->stream));
  return FGBD_OK;
}

// Load a frame's coordinates and build the weighted scan-line graph.
int stage_graph(fgbd_ctx* ctx, const int64_t* coords, int64_t n, int bits, bool dev, int w64,
                bool weights = true, bool reorder = false) {
  int rc = ensure_capacity(ctx, n, 3 * bits > 32);
  if (rc) return rc;
  if ((rc = reset_ctl(ctx))) return rc;
  if (dev) {
    ctx->cur_coords = coords;
  } else {
    if ((rc = h2d(ctx, ctx->coords64, coords, 3 * n * sizeof(int64_t), false))) return rc;
    ctx->cur_coords = ctx->coords64;
  }
  if ((rc = launch_graph(ctx, n, bits, reorder))) return rc;
  return weights ? launch_weights(ctx, n, bits, w64) : FGBD_OK;
}



int check_graph_ctl(fgbd_ctx* ctx, int bits) {
  const Ctl& h = *ctx->ctl_host;
  if (h.err_flags & 1)
    return set_error(ctx, FGBD_E_CLOUD,
                     "coordinates out of range for bit_depth=" + std::to_string(bits));
  if (!(h.sigma_g > 0)) {
    char b[96];
    std::snprintf(b, sizeof(b), "sigma_g must be positive, got %.17g", h.sigma_g);
    return set_error(ctx, FGBD_E_GRAPH, b);
  }
  return FGBD_OK;
}

// Contexts on one device run their kernel sections one at a time: the
// persistent filter kernel needs the whole GPU, so interleaving two frames'
// kernels only slows both.  Transfers stay outside the lock, so with several
// host threads frame f+1's upload and frame f-1's download overlap frame f.
std::mutex& device_mutex(int device) {
  static std::mutex m[64];
  return m[device & 63];
}

// The last frame compute enqueued on each device (guarded by device_mutex):
// the next frame's stream waits for it on the GPU, so a frame whose compute
// needs no host round trip can release the lock as soon as it is enqueued.
cudaEvent_t& device_last_compute(int device) {
  static cudaEvent_t ev[64] = {};
  return ev[device & 63];
}

// Far-gather filter variant (k_lf_run FAR): on when at least half of the
// graph's slots point more than kFarRows rows away -- random clouds, whose
// scattered gathers only evict reusable rows from L1 (-8% filter time
// there, +7% on lattices; profiles/r2_summary.md).  FGBD_LF_FAR overrides.
int far_choice(const fgbd_ctx* ctx, const Ctl& h) {
  if (ctx->lf_far >= 0) return ctx->lf_far > 0;
  const unsigned long long nnz = 2 * h.n_edges;
  return nnz > 0 && 2 * h.far_slots >= nnz;
}

double ev_sec(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();
    return 0.0;
  }
  return ms * 1e-3;
}

void fill_noise_report(fgbd_report* r, const fgbd_noise& nz) {
  for (int c = 0; c < 3; ++c) {
    r->per_channel_sigma[c] = nz.per_channel_sigma[c];
    r->tail_m[c] = nz.m[c];
    r->tail_tau[c] = nz.tau[c];
    r->tail_fallback[c] = nz.fallback[c];
    for (int k = 0; k < FGBD_MAX_PATCH; ++k) r->eigenvalues[c][k] = nz.eigenvalues[c][k];
    r->jacobi_direct_off[c] = nz.jacobi_direct_off[c];
  }
  r->eligible_count = nz.eligible_count;
}

}  // namespace

namespace fgbd {
// Stage entry points that exchange per-point arrays other than colours with
// the caller (patches, masks, statistics, the CSR export) work on a graph
// whose rows are in point order -- the one fgbd_build_graph holds.
int require_point_rows(fgbd_ctx* ctx) {
  if (ctx->g_reordered)
    return set_error(ctx, FGBD_E_GRAPH,
                     "the held graph comes from fgbd_denoise (rows in scan-line order); "
                     "call fgbd_build_graph first");
  return FGBD_OK;
}
}  // namespace fgbd

extern "C" {

int32_t fgbd_abi_version(void) { return FGBD_ABI_VERSION; }

const char* fgbd_last_error(const fgbd_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_global_err.c_str();
}

fgbd_ctx* fgbd_ctx_create(int32_t device, int64_t max_points) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    set_error(nullptr, FGBD_E_CUDA, std::string("no CUDA device available: ") +
                                        (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
    return nullptr;
  }
  if (device < 0 || device >= ndev) {
    set_error(nullptr, FGBD_E_ARG, "device index out of range");
    return nullptr;
  }
  fgbd_ctx* ctx = new fgbd_ctx();
  ctx->device = device;
  auto fail = [&](cudaError_t err, const char* w) -> fgbd_ctx* {
    set_error(nullptr, FGBD_E_CUDA, std::string(w) + ": " + cudaGetErrorString(err));
    delete ctx;
    return nullptr;
  };
  if ((e = cudaSetDevice(device)) != cudaSuccess) return fail(e, "cudaSetDevice");
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return fail(e, "props");
  if (prop.major < 10) {
    set_error(nullptr, FGBD_E_CUDA, "device is not sm_100 (Blackwell); this build targets sm_100a");
    delete ctx;
    return nullptr;
  }
  ctx->num_sms = prop.multiProcessorCount;
  ctx->l2_bytes = prop.l2CacheSize;
  if ((e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(e, "stream");
  if ((e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(e, "side stream");
  if ((e = cudaEventCreateWithFlags(&ctx->ev_side, cudaEventDisableTiming)) != cudaSuccess)
    return fail(e, "side event");
  if ((e = cudaEventCreateWithFlags(&ctx->ev_done, cudaEventDisableTiming)) != cudaSuccess)
    return fail(e, "event");
  if ((e = cudaEventCreateWithFlags(&ctx->ev_perm, cudaEventDisableTiming)) != cudaSuccess)
    return fail(e, "perm event");
  for (auto& ev : ctx->ev)
    if ((e = cudaEventCreate(&ev)) != cudaSuccess) return fail(e, "event");
  if ((e = cudaMalloc(&ctx->ctl, sizeof(Ctl))) != cudaSuccess) return fail(e, "ctl");
  if ((e = cudaMemset(ctx->ctl, 0, sizeof(Ctl))) != cudaSuccess) return fail(e, "ctl");
  if ((e = cudaMallocHost(&ctx->ctl_host, sizeof(Ctl))) != cudaSuccess) return fail(e, "ctl host");
  if ((e = cudaMalloc(&ctx->sort.hist, 3 * kMaxPasses * kRadix * sizeof(uint32_t))) != cudaSuccess)
    return fail(e, "hist");
  if ((e = cudaMalloc(&ctx->sort.tile_ctr, 3 * kMaxPasses * sizeof(unsigned))) != cudaSuccess)
    return fail(e, "tile ctr");
  if ((e = cudaMalloc(&ctx->d_bufs, 3 * sizeof(double*))) != cudaSuccess) return fail(e, "bufs");
  if ((e = cudaMalloc(&ctx->tickets, 8192 * sizeof(unsigned))) != cudaSuccess) return fail(e, "tickets");
  if ((e = cudaMemset(ctx->tickets, 0, 8192 * sizeof(unsigned))) != cudaSuccess) return fail(e, "tickets");
  if (const char* v = std::getenv("FGBD_LF_VARIANT")) ctx->lf_variant = std::atoi(v);
  if (const char* v = std::getenv("FGBD_L2_PERSIST")) ctx->l2_persist = std::atoi(v);
  if (const char* v = std::getenv("FGBD_NE_VARIANT")) ctx->ne_variant = std::atoi(v);
  if (const char* v = std::getenv("FGBD_LF_SHAPE")) ctx->lf_shape = std::atoi(v) & 3;
  if (const char* v = std::getenv("FGBD_LF_CHUNK")) ctx->lf_chunk = std::atoi(v);
  if (const char* v = std::getenv("FGBD_ASYNC_LOCK")) ctx->async_lock = std::atoi(v);
  if (const char* v = std::getenv("FGBD_REORDER")) ctx->reorder_rows = std::atoi(v);
  if (const char* v = std::getenv("FGBD_LF_HALO")) ctx->lf_halo = std::max(0, std::atoi(v));
  if (const char* v = std::getenv("FGBD_PREP_MULT")) ctx->prep_mult = std::max(1, std::atoi(v));
  if (const char* v = std::getenv("FGBD_SORT_DERIVED")) ctx->sort_derived = std::atoi(v);
  if (const char* v = std::getenv("FGBD_SLG_COOP")) ctx->slg_coop = std::atoi(v);
  if (const char* v = std::getenv("FGBD_JACOBI_THREADS")) ctx->jacobi_threads = std::atoi(v);
  if (const char* v = std::getenv("FGBD_ROWS_EXPAND")) ctx->rows_expand = std::atoi(v);
  if (const char* v = std::getenv("FGBD_LF_HOLD")) ctx->lf_hold = std::atoi(v);
  if (ctx->lf_hold >= 0) ctx->hold_guess = ctx->lf_hold;
  if (const char* v = std::getenv("FGBD_ROWS_GRID")) ctx->rows_grid = std::atoi(v);
  if (const char* v = std::getenv("FGBD_MASK_FOLD")) ctx->mask_fold = std::atoi(v);
  if (const char* v = std::getenv("FGBD_LF_FAR")) ctx->lf_far = std::atoi(v);
  if (const char* v = std::getenv("FGBD_HOST_THREADS")) ctx->host_threads = std::max(0, std::atoi(v));
  if (ensure_capacity(ctx, max_points > 0 ? max_points : 1, 0) != FGBD_OK) {
    set_error(nullptr, FGBD_E_CUDA, ctx->err);
    fgbd_ctx_destroy(ctx);
    return nullptr;
  }
  return ctx;
}

void fgbd_ctx_destroy(fgbd_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  free_scratch(ctx);
  if (ctx->ctl) cudaFree(ctx->ctl);
  if (ctx->ctl_host) cudaFreeHost(ctx->ctl_host);
  if (ctx->partials) cudaFree(ctx->partials);
  if (ctx->sort.hist) cudaFree(ctx->sort.hist);
  if (ctx->sort.tile_ctr) cudaFree(ctx->sort.tile_ctr);
  if (ctx->slg_cnt) cudaFree(ctx->slg_cnt);
  if (ctx->d_bufs) cudaFree(ctx->d_bufs);
  if (ctx->tickets) cudaFree(ctx->tickets);
  if (ctx->csr_scratch) cudaFree(ctx->csr_scratch);
  if (ctx->ply_stage) cudaFree(ctx->ply_stage);
  if (ctx->aux) cudaFree(ctx->aux);
  if (ctx->p2p_flags) cudaFree(ctx->p2p_flags);
  if (ctx->held_coords) cudaFree(ctx->held_coords);
  destroy_stager(ctx);
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  if (ctx->side) cudaStreamSynchronize(ctx->side);
  if (ctx->ev_side) cudaEventDestroy(ctx->ev_side);
  if (ctx->ev_perm) cudaEventDestroy(ctx->ev_perm);
  if (ctx->ev_done) {
    std::lock_guard<std::mutex> lk(device_mutex(ctx->device));
    if (device_last_compute(ctx->device) == ctx->ev_done) {
      cudaEventSynchronize(ctx->ev_done);
      device_last_compute(ctx->device) = nullptr;
    }
    cudaEventDestroy(ctx->ev_done);
  }
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

void* fgbd_ctx_stream(fgbd_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int64_t fgbd_ctx_device_bytes(const fgbd_ctx* ctx) { return ctx ? (int64_t)ctx->dev_bytes : 0; }

void* fgbd_host_alloc(int64_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, (size_t)bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void fgbd_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

// FGBD_HOST_TLOG=1 (diagnostic): host timestamps of fgbd_denoise's phases
// printed to stderr, microseconds since entry
namespace {
struct HostTlog {
  bool on = false;
  std::chrono::steady_clock::time_point t0;
  char buf[512];
  int len = 0;
  HostTlog() {
    static const bool want = std::getenv("FGBD_HOST_TLOG") != nullptr;
    on = want;
    if (on) t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on || len > 440) return;
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    len += std::snprintf(buf + len, sizeof(buf) - len, " %s=%.1f", what, us);
  }
  ~HostTlog() {
    if (on) std::fprintf(stderr, "host tlog:%s\n", buf);
  }
};
}  // namespace

int32_t fgbd_denoise(fgbd_ctx* ctx, const int64_t* coords, const double* colors, int64_t n,
                     int32_t bits, const fgbd_config* cfg, int32_t cached_q, double cached_sigma,
                     double* out_colors, fgbd_report* rep, uint32_t flags) {
  HostTlog tl;
  if (!ctx || !rep) return set_error(ctx, FGBD_E_ARG, "null context or report");
  NvtxRange nv_frame("fgbd.denoise");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  ctx->launches = 0;
  int rc = check_cfg(ctx, cfg);
  if (rc) return rc;
  std::memset(rep, 0, sizeof(*rep));
  rep->criterion_value = NAN;
  rep->converged = -1;
  rep->eligible_count = -1;
  if (n < 0) return set_error(ctx, FGBD_E_ARG, "n must be >= 0");
  const bool dev = (flags & FGBD_FLAG_DEVICE_PTRS) != 0;
  const bool timing = !(flags & FGBD_FLAG_NO_TIMING);
  const int w64 = (flags & FGBD_FLAG_WEIGHTS_F64) ? 1 : 0;
  if (n < 2) {  // filtering.py:269-275: the input comes back unchanged
    if (n > 0 && out_colors != colors) {
      if (dev) {
        if ((rc = d2h(ctx, out_colors, colors, 3 * n * sizeof(double), true))) return rc;
        FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      } else {
        std::memcpy(out_colors, colors, 3 * n * sizeof(double));
      }
    }
    return FGBD_OK;
  }
  if ((rc = check_graph_input(ctx, n, bits))) return rc;
  cudaEvent_t* ev = ctx->ev;
  if (timing) FGBD_CUDA(ctx, cudaEventRecord(ev[0], ctx->stream));
  tl.mark("ev0");
  if ((rc = ensure_capacity(ctx, n, 3 * bits > 32))) return rc;
  apply_l2_policy(ctx, n);
  const int64_t* frame_coords = dev ? coords : ctx->coords64;
  // static-geometry reuse: the held graph stands if this frame's coordinates
  // are byte-identical to the ones it was built from (exact device compare)
  const bool want_reuse = (flags & (FGBD_FLAG_REUSE_GRAPH | FGBD_FLAG_STATIC_GEOMETRY)) && !w64;
  const bool may_reuse = want_reuse && ctx->held_valid && ctx->g_n == n && ctx->g_bits == bits &&
                         ctx->g_have_weights && !ctx->g_weights64;
  // the caller vouches for the geometry: no coordinate upload, no compare
  const bool trusted = may_reuse && (flags & FGBD_FLAG_STATIC_GEOMETRY);
  // A frame that will probably reuse the graph has no build for the colour
  // upload to hide behind, so its colours travel ahead of the device lock,
  // together with the coordinates.  Both copies go before the compare
  // kernel: copies need only the copy engines, while a kernel may have to
  // wait for another context's persistent filter to release the SMs.
  const double* frame_colors = colors;
  bool colors_dev = dev;
  bool colors_main = dev;  // on the device ahead of the graph build in main-stream order
  if (!dev && !trusted &&
      (rc = host_to_device(ctx, ctx->coords64, coords, 3 * n * sizeof(int64_t), ctx->stream, 0)))
    return rc;
  if (may_reuse && !dev) {
    if ((rc = host_to_device(ctx, ctx->out, colors, 3 * n * sizeof(double), ctx->stream, 1)))
      return rc;
    frame_colors = ctx->out;
    colors_dev = true;
    colors_main = true;
  } else if (!dev && host_stageable(ctx, colors, 3 * n * sizeof(double))) {
    // pageable colours: staged right behind the coordinates, each chunk's
    // DMA (side stream) issued as soon as its copy has landed, so the DMA
    // overlaps the host copies instead of following them (the colour
    // expansion on the side stream then reads them on the device)
    if ((rc = host_to_device(ctx, ctx->out, colors, 3 * n * sizeof(double), ctx->side, 1)))
      return rc;
    frame_colors = ctx->out;
    colors_dev = true;
  }
  bool reuse = false;
  bool expanded = false;  // BUF_Y already written by k_rows
  std::unique_lock<std::mutex> compute_lock(device_mutex(ctx->device), std::defer_lock);
  if (trusted) {
    reuse = true;
  } else if (may_reuse) {
    int same = 0;  // syncs the stream: coordinates (and colours) have landed
    if ((rc = coords_equal(ctx, frame_coords, ctx->held_coords, 3 * n, &same))) return rc;
    reuse = same != 0;
  } else if (!dev) {
    // The coordinates are uploading.  A free device: queue the frame behind
    // them at once (stream order; the host waiting first left the GPU idle
    // ~19 us while it enqueued the graph).  A busy one: let them land before
    // queuing for it, so another context's compute overlaps this upload.
    if (!compute_lock.try_lock()) FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  if (!compute_lock.owns_lock()) compute_lock.lock();
  // the side stream starts after the coordinates have landed (full PCIe
  // bandwidth for them) and after all earlier main-stream work on the
  // staging buffers; it then overlaps the colour upload with the graph build
  FGBD_CUDA(ctx, cudaEventRecord(ctx->ev_side, ctx->stream));
  FGBD_CUDA(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_side, 0));
  // this frame's compute starts after the previous frame's on the device
  // (the colour upload on the side stream need not wait for it)
  if (cudaEvent_t prev = device_last_compute(ctx->device))
    FGBD_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, prev, 0));
  if (timing) FGBD_CUDA(ctx, cudaEventRecord(ev[1], ctx->stream));
  tl.mark("ev1");
  // the NE pass converts the ELL payloads to weights itself when it can
  const bool fuse_w = !reuse && cached_q < 0 && !w64 && bits <= 15 && ctx->ne_variant == 1;
  if (reuse) {
    if ((rc = reset_ctl(ctx))) return rc;
    if ((rc = restore_graph_header(ctx))) return rc;
    ctx->cur_coords = trusted ? ctx->held_coords : frame_coords;
  } else {
    NvtxRange nv("fgbd.graph");
    // device-resident colours: k_rows lays them out as it walks the rows
    // (k_expand after k_rows sat on the way to the NE kernel: k_rows fills
    // the register file, so the two never ran side by side)
    if (colors_main && ctx->rows_expand) ctx->expand_colors = frame_colors;
    if ((rc = stage_graph(ctx, frame_coords, n, bits, true, w64, !fuse_w, ctx->reorder_rows != 0)))
      return rc;
    expanded = colors_main && ctx->rows_expand;
    ctx->expand_colors = nullptr;
    if (want_reuse && (rc = hold_coords(ctx, frame_coords, n))) return rc;
  }
  rep->graph_reused = reuse ? 1 : 0;
  if (timing) FGBD_CUDA(ctx, cudaEventRecord(ev[2], ctx->stream));
  tl.mark("graph");
  // colours travel (and are re-laid out) while the graph is being built
  if (!expanded) {
    if ((rc = upload_colors_async(ctx, frame_colors, n, colors_dev))) return rc;
    FGBD_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_side, 0));
  }

  fgbd_noise nz;
  std::memset(&nz, 0, sizeof(nz));
  bool folded = false;     // the FSLR mask folded into the first filter step
  bool device_ne = false;  // NE finished on the device (FGBD_FLAG_DEVICE_NE)
  // the filter's far-gather variant: known here only for a reused graph
  ctx->lf_far_now = reuse ? ctx->held_far : (ctx->lf_far > 0);
  if (cached_q >= 0) {
    if (timing) FGBD_CUDA(ctx, cudaEventRecord(ev[3], ctx->stream));
    int fin = BUF_Y;
    if ((rc = launch_fixed_steps(ctx, n, cached_q, w64, &fin))) return rc;
    if (timing) FGBD_CUDA(ctx, cudaEventRecord(ev[6], ctx->stream));
    if ((rc = launch_compact(ctx, n, fin, dev ? out_colors : ctx->out, 1))) return rc;
  } else {
    const int D = cfg->patch_size;
    NvtxRange nv("fgbd.noise+filter");
    if ((rc = launch_noise(ctx, n, D, fuse_w ? 1 : 0))) return rc;
    if (fuse_w) {
      ctx->g_have_weights = 1;
      ctx->g_weights64 = 0;
    }
    folded = mask_foldable(ctx, cfg->q_max, w64);
    device_ne = folded && (flags & FGBD_FLAG_DEVICE_NE);
  }
  if (cached_q < 0 && device_ne) {
    // the whole frame without a host round trip: NE finished on the device
    // (bit-identical to finish_noise), the FSLR mask built by step 1
    if ((rc = launch_finish_noise(ctx, cfg->patch_size, cfg->tau_divisor, cfg->fslr_enabled,
                                  cfg->fslr_sigma_floor)))
      return rc;
    if (timing) FGBD_CUDA(ctx, cudaEventRecord(ev[3], ctx->stream));
    if ((rc = launch_select_steps_folded(ctx, n, cfg->q_max, cfg->criterion_mode,
                                         cfg->early_exit, nullptr, 0)))
      return rc;
    if (timing) FGBD_CUDA(ctx, cudaEventRecord(ev[6], ctx->stream));
    if ((rc = launch_compact(ctx, n, -1, dev ? out_colors : ctx->out, 1))) return rc;
  } else if (cached_q < 0) {
    const int D = cfg->patch_size;
    if (ctx->jacobi_threads) jacobi_pool_prepare();  // helpers spin while NE runs
    tl.mark("ne_launched");
    if ((rc = pull_ctl(ctx))) return rc;
    tl.mark("ne_pulled");
    ctx->lf_far_now = far_choice(ctx, *ctx->ctl_host);
    if ((rc = check_graph_ctl(ctx, bits))) return rc;
    const int maxdeg = ctx->ctl_host->max_deg;
    if (D > 1 + maxdeg)
      return set_error(ctx, FGBD_E_NOISE, "patch_size " + std::to_string(D) +
                                              " exceeds 1 + max degree (" +
                                              std::to_string(1 + maxdeg) + ") of this graph");
    if ((rc = finish_noise(ctx, D, cfg->tau_divisor, &nz))) return rc;
    tl.mark("ne_done");
    const double sig = nz.sigma_est;
    const int active = cfg->fslr_enabled && !(sig < cfg->fslr_sigma_floor);
    if (!folded && (rc = launch_mask(ctx, n, sig, active, cfg->q_max, cfg->criterion_mode,
                                     cfg->early_exit, nullptr)))
      return rc;
    if (timing) FGBD_CUDA(ctx, cudaEventRecord(ev[3], ctx->stream));
    tl.mark("ev3");
    if (folded) {
      if ((rc = launch_select_steps_folded(ctx, n, cfg->q_max, cfg->criterion_mode,
                                           cfg->early_exit, &sig, active)))
        return rc;
      tl.mark("lf_launched");
    } else if ((rc = launch_select_steps(ctx, n, cfg->q_max, w64))) {
      return rc;
    }
    if (timing) FGBD_CUDA(ctx, cudaEventRecord(ev[6], ctx->stream));
    if ((rc = launch_compact(ctx, n, -1, dev ? out_colors : ctx->out, 1))) return rc;
  }
  if (timing) FGBD_CUDA(ctx, cudaEventRecord(ev[4], ctx->stream));
  FGBD_CUDA(ctx, cudaEventRecord(ctx->ev_done, ctx->stream));
  device_last_compute(ctx->device) = ctx->ev_done;
  // the frame's control block travels right behind its last kernel, so the
  // one wait below (the lock's or the download's) also covers it -- but
  // after ev_done: the next frame's kernels wait for ev_done, and a copy in
  // front of it queued them behind this frame's output download (r2f3:
  // 300-frame video 721 -> 609 frames/s)
  FGBD_CUDA(ctx, cudaMemcpyAsync(ctx->ctl_host, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost,
                                 ctx->stream));
  // a frame with a host round trip inside keeps the lock until it is done
  const bool held = !ctx->async_lock || (cached_q < 0 && !device_ne);
  // device outputs: nothing follows, so the frame's last event goes in now
  // (recording it after the wait cost a submission round trip, ~10 us);
  // host outputs: the download too, right behind the compute -- enqueued
  // after the wait it started a host wake-up late.  It is outside the
  // compute order (ev_done), so other contexts' frames never wait for it.
  NvtxRange nv_out("fgbd.download");
  if (!dev && (rc = d2h(ctx, out_colors, ctx->out, 3 * n * sizeof(double), false))) return rc;
  if (timing) FGBD_CUDA(ctx, cudaEventRecord(ev[5], ctx->stream));
  tl.mark("enqueued");
  // Each elapsed-time query is a ~3.5 us driver call: a frame that waits
  // here anyway reads the stage times while the filter still runs, so only
  // the last one falls after the frame's end
  bool stages_read = false;
  auto read_stage_times = [&]() {
    rep->t_h2d = ev_sec(ev[0], ev[1]);
    rep->t_graph_construction = ev_sec(ev[1], ev[2]);
    cudaEventSynchronize(ev[3]);
    rep->t_noise_estimation = cached_q >= 0 ? 0.0 : ev_sec(ev[2], ev[3]);
    cudaEventSynchronize(ev[6]);
    rep->t_lf_steps = ev_sec(ev[3], ev[6]);
    cudaEventSynchronize(ev[4]);
    rep->t_low_pass_filter = ev_sec(ev[3], ev[4]);
    stages_read = true;
  };
  if (held && timing) read_stage_times();
  if (held) {
    // device outputs: the wait covers the control block too
    if (dev && timing) FGBD_CUDA(ctx, cudaEventSynchronize(ev[5]));
    else if (dev) FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    else FGBD_CUDA(ctx, cudaEventSynchronize(ctx->ev_done));
  }
  tl.mark("done");
  compute_lock.unlock();
  if (!dev || !held) FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  tl.mark("synced");
  if ((rc = check_graph_ctl(ctx, bits))) return rc;
  if (cached_q < 0 && device_ne && (rc = collect_noise(ctx, cfg->patch_size, &nz))) return rc;
  const Ctl& h = *ctx->ctl_host;
  if (want_reuse && !reuse) {  // the copy now describes a complete graph with weights
    ctx->held_far = far_choice(ctx, h);
    ctx->held_edges = h.n_edges;
    ctx->held_sigma_g = h.sigma_g;
    ctx->held_max_deg = h.max_deg;
    ctx->held_valid = 1;
  }
  rep->n_edges = (int64_t)h.n_edges;
  rep->nnz = 2 * (int64_t)h.n_edges;
  rep->max_degree = h.max_deg;
  rep->sigma_g = h.sigma_g;
  if (cached_q >= 0) {
    rep->selected_q = cached_q;
    rep->sigma_est = std::isnan(cached_sigma) ? 0.0 : cached_sigma;
    rep->masked_fraction = 0.0;
    rep->cached = 1;
    rep->steps = cached_q;
  } else {
    rep->selected_q = h.best_q;
    rep->sigma_est = nz.sigma_est;
    // the next frame's filter variant: decide-before-sweep pays off when the
    // scan ends by early exit rather than at q_max
    ctx->hold_guess = ctx->lf_hold >= 0 ? ctx->lf_hold : (h.steps < cfg->q_max);
    rep->masked_fraction = 1.0 - (double)h.included / (double)n;
    rep->criterion_value = h.best_crit;
    const double eps = std::isnan(cfg->epsilon) ? 1e-3 * nz.sigma_est * nz.sigma_est : cfg->epsilon;
    rep->converged = h.best_crit <= eps ? 1 : 0;
    rep->steps = h.steps;
    rep->all_excluded_fallback = h.all_excluded;
    rep->included_count = h.included;
    fill_noise_report(rep, nz);
    rep->n_trace = std::min(h.steps + 1, FGBD_TRACE_MAX);
    for (int k = 0; k < rep->n_trace; ++k) rep->trace[k] = h.trace[k];
  }
  tl.mark("report");
  if (timing) {
    if (!stages_read) read_stage_times();
    // device outputs have no download (ev4 -> ev5 spans only the control
    // block's copy): no query after the frame at all
    rep->t_d2h = dev ? 0.0 : ev_sec(ev[4], ev[5]);
    // the chain ev0 .. ev5, summed (one driver query fewer)
    rep->t_total = rep->t_h2d + rep->t_graph_construction + rep->t_noise_estimation +
                   rep->t_low_pass_filter + rep->t_d2h;
  }
  rep->gpu_launches = ctx->launches;
  tl.mark("exit");
  return FGBD_OK;
}

int32_t fgbd_radix_argsort(fgbd_ctx* ctx, const uint64_t* keys, int64_t n, int32_t key_bits,
                           int64_t* perm_out, uint32_t flags) {
  if (!ctx) return set_error(ctx, FGBD_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  if (key_bits < 1 || key_bits > 64)
    return set_error(ctx, FGBD_E_ARG, "key_bits must be in [1, 64], got " + std::to_string(key_bits));
  if (n >= (int64_t(1) << 31)) return set_error(ctx, FGBD_E_ARG, "n too large");
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  if (n < 2) {
    const int64_t zero = 0;
    if (n == 1) FGBD_CUDA(ctx, cudaMemcpy(perm_out, &zero, 8, cudaMemcpyDefault));
    return FGBD_OK;
  }
  int rc = ensure_capacity(ctx, n, 1);
  if (rc) return rc;
  if ((rc = h2d(ctx, ctx->coords64, keys, n * sizeof(uint64_t), dev))) return rc;
  uint32_t* d_perm = nullptr;
  if ((rc = launch_argsort64(ctx, (const uint64_t*)ctx->coords64, n, key_bits, &d_perm))) return rc;
  std::vector<uint32_t> h(n);
  FGBD_CUDA(ctx, cudaMemcpyAsync(h.data(), d_perm, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (dev) {
    std::vector<int64_t> w(h.begin(), h.end());
    FGBD_CUDA(ctx, cudaMemcpy(perm_out, w.data(), n * 8, cudaMemcpyHostToDevice));
  } else {
    for (int64_t i = 0; i < n; ++i) perm_out[i] = h[i];
  }
  ctx->g_n = -1;  // sort scratch reused: the held graph is gone
  return FGBD_OK;
}

int32_t fgbd_scan_line(fgbd_ctx* ctx, const int64_t* coords, int64_t n, int32_t bits,
                       int32_t line, uint64_t* codes_out, int64_t* perm_out, uint32_t flags) {
  if (!ctx) return set_error(ctx, FGBD_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  int rc = check_graph_input(ctx, n, bits);
  if (rc) return rc;
  if (line < 1 || line > 3)
    return set_error(ctx, FGBD_E_GRAPH, "line must be 1, 2 or 3, got " + std::to_string(line));
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  if (n < 1) return FGBD_OK;
  if ((rc = ensure_capacity(ctx, n, 3 * bits > 32))) return rc;
  if ((rc = reset_ctl(ctx))) return rc;
  if (dev) ctx->cur_coords = coords;
  else {
    if ((rc = h2d(ctx, ctx->coords64, coords, 3 * n * 8, false))) return rc;
    ctx->cur_coords = ctx->coords64;
  }
  uint32_t* d_perm = nullptr;
  uint64_t* d_codes = (uint64_t*)ctx->out;  // (3n doubles) >= n codes
  if ((rc = launch_scan_line(ctx, n, bits, line - 1, d_codes, &d_perm))) return rc;
  if (codes_out) {
    if ((rc = d2h(ctx, codes_out, d_codes, n * 8, dev))) return rc;
  }
  std::vector<uint32_t> h(n);
  FGBD_CUDA(ctx, cudaMemcpyAsync(h.data(), d_perm, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if ((rc = pull_ctl(ctx))) return rc;
  if (ctx->ctl_host->err_flags & 1)
    return set_error(ctx, FGBD_E_CLOUD, "coordinates out of range for bit_depth=" + std::to_string(bits));
  if (perm_out) {
    if (dev) {
      std::vector<int64_t> w(h.begin(), h.end());
      FGBD_CUDA(ctx, cudaMemcpy(perm_out, w.data(), n * 8, cudaMemcpyHostToDevice));
    } else {
      for (int64_t i = 0; i < n; ++i) perm_out[i] = h[i];
    }
  }
  ctx->g_n = -1;
  return FGBD_OK;
}

int32_t fgbd_build_graph(fgbd_ctx* ctx, const int64_t* coords, int64_t n, int32_t bits,
                         fgbd_graph_info* info, uint32_t flags) {
  if (!ctx || !info) return set_error(ctx, FGBD_E_ARG, "null argument");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  std::memset(info, 0, sizeof(*info));
  info->n = n;
  int rc = check_graph_input(ctx, n, bits);
  if (rc) return rc;
  if (n < 2) {
    ctx->g_n = n;
    ctx->g_bits = bits;
    return FGBD_OK;
  }
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  if ((rc = stage_graph(ctx, coords, n, bits, dev, (flags & FGBD_FLAG_WEIGHTS_F64) ? 1 : 0)))
    return rc;
  if ((rc = pull_ctl(ctx))) return rc;
  const Ctl& h = *ctx->ctl_host;
  if (h.err_flags & 1) {
    ctx->g_n = -1;
    return set_error(ctx, FGBD_E_CLOUD, "coordinates out of range for bit_depth=" + std::to_string(bits));
  }
  info->n_edges = (int64_t)h.n_edges;
  info->nnz = 2 * (int64_t)h.n_edges;
  info->max_degree = h.max_deg;
  info->sigma_g = h.sigma_g;
  return FGBD_OK;
}

int32_t fgbd_graph_export(fgbd_ctx* ctx, int64_t* indptr, int64_t* indices, int64_t* csr_edge,
                          int64_t* edge_u, int64_t* edge_v, double* edge_sqdist,
                          double* edge_weights, double* wdeg) {
  if (!ctx) return set_error(ctx, FGBD_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  if (ctx->g_n < 0) return set_error(ctx, FGBD_E_GRAPH, "no graph held by this context");
  if (int e = require_point_rows(ctx)) return e;
  const int64_t n = ctx->g_n;
  if (n < 2) {
    if (indptr)
      for (int64_t i = 0; i <= n; ++i) indptr[i] = 0;
    if (wdeg)
      for (int64_t i = 0; i < n; ++i) wdeg[i] = 0.0;
    return FGBD_OK;
  }
  if ((int)pull_ctl(ctx)) return FGBD_E_CUDA;
  const int64_t E = (int64_t)ctx->ctl_host->n_edges, nnz = 2 * E;
  // device staging, one allocation
  const size_t bytes = (size_t)(n + 1 + 2 * nnz + 2 * E) * 8 + (size_t)(2 * E + n) * 8;
  char* d = nullptr;
  FGBD_CUDA(ctx, cudaMalloc(&d, bytes));
  int64_t* d_indptr = (int64_t*)d;
  int64_t* d_indices = d_indptr + n + 1;
  int64_t* d_csr = d_indices + nnz;
  int64_t* d_u = d_csr + nnz;
  int64_t* d_v = d_u + E;
  double* d_sq = (double*)(d_v + E);
  double* d_w = d_sq + E;
  double* d_wd = d_w + E;
  int64_t nnz2 = 0, e2 = 0;
  int rc = launch_export(ctx, n, d_indptr, d_indices, d_csr, d_u, d_v, d_sq, d_w, d_wd, &nnz2, &e2);
  if (rc == FGBD_OK && (nnz2 != nnz || e2 != E))
    rc = set_error(ctx, FGBD_E_GRAPH, "internal: edge count mismatch in export");
  auto cp = [&](void* dst, const void* src, size_t b) {
    if (dst && rc == FGBD_OK && b) {
      cudaError_t e = cudaMemcpy(dst, src, b, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) rc = cuda_error(ctx, e, "export copy");
    }
  };
  cp(indptr, d_indptr, (n + 1) * 8);
  cp(indices, d_indices, nnz * 8);
  cp(csr_edge, d_csr, nnz * 8);
  cp(edge_u, d_u, E * 8);
  cp(edge_v, d_v, E * 8);
  cp(edge_sqdist, d_sq, E * 8);
  cp(edge_weights, d_w, E * 8);
  cp(wdeg, d_wd, n * 8);
  cudaFree(d);
  return rc;
}

int32_t fgbd_estimate_noise(fgbd_ctx* ctx, const double* colors, int32_t patch_size,
                            int32_t tau_divisor, fgbd_noise* out, double* fslr_stat_out,
                            uint32_t flags) {
  if (!ctx || !out) return set_error(ctx, FGBD_E_ARG, "null argument");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  std::memset(out, 0, sizeof(*out));
  if (ctx->g_n < 0) return set_error(ctx, FGBD_E_GRAPH, "no graph held by this context");
  if (int e = require_point_rows(ctx)) return e;
  const int64_t n = ctx->g_n;
  const int D = patch_size;
  if (D < 2) return set_error(ctx, FGBD_E_NOISE, "patch_size must be >= 2, got " + std::to_string(D));
  int maxdeg = 0;
  if (n >= 2) {
    if (pull_ctl(ctx)) return FGBD_E_CUDA;
    maxdeg = ctx->ctl_host->max_deg;
  }
  if (D > 1 + maxdeg)
    return set_error(ctx, FGBD_E_NOISE, "patch_size " + std::to_string(D) +
                                            " exceeds 1 + max degree (" + std::to_string(1 + maxdeg) +
                                            ") of this graph");
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  int rc = upload_colors(ctx, colors, n, dev);
  if (rc) return rc;
  if ((rc = launch_noise(ctx, n, D, 0))) return rc;
  if ((rc = pull_ctl(ctx))) return rc;
  if ((rc = finish_noise(ctx, D, tau_divisor, out))) return rc;
  if (fslr_stat_out) {
    if ((rc = d2h(ctx, fslr_stat_out, ctx->fslr, n * sizeof(double), dev))) return rc;
    FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  ctx->g_have_noise = 1;
  ctx->g_patch = D;
  return FGBD_OK;
}

int32_t fgbd_fslr_mask(fgbd_ctx* ctx, double sigma_est, double sigma_floor, uint8_t* include_out,
                       int32_t* all_excluded) {
  if (!ctx || !include_out) return set_error(ctx, FGBD_E_ARG, "null argument");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  if (int e = require_point_rows(ctx)) return e;
  if (all_excluded) *all_excluded = 0;
  if (!ctx->g_have_noise)
    return set_error(ctx, FGBD_E_NOISE, "run fgbd_estimate_noise before fgbd_fslr_mask");
  const int64_t n = ctx->g_n;
  const int active = !(sigma_est < sigma_floor);
  int rc = launch_mask(ctx, n, sigma_est, active, 0, FGBD_CRIT_POOLED, 0, nullptr);
  if (rc) return rc;
  std::vector<uint32_t> bits((n + 31) / 32);
  FGBD_CUDA(ctx, cudaMemcpyAsync(bits.data(), ctx->mask, bits.size() * 4, cudaMemcpyDeviceToHost,
                                 ctx->stream));
  if ((rc = pull_ctl(ctx))) return rc;
  for (int64_t i = 0; i < n; ++i) include_out[i] = (bits[i >> 5] >> (i & 31)) & 1u;
  if (ctx->ctl_host->all_excluded) {
    if (all_excluded) *all_excluded = 1;
    return set_error(ctx, FGBD_E_FILTER,
                     "the variance threshold excluded every point; fall back to unmasked "
                     "selection (disable the mask or raise sigma_floor)");
  }
  return FGBD_OK;
}

int32_t fgbd_filter_steps_csr(fgbd_ctx* ctx, const int64_t* indptr, const int64_t* indices,
                              const double* slot_weights, int64_t n, int64_t nnz,
                              const double* colors_in, int32_t q, double* colors_out,
                              uint32_t flags) {
  if (!ctx) return set_error(ctx, FGBD_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  if (q < 0) return set_error(ctx, FGBD_E_FILTER, "q must be >= 0, got " + std::to_string(q));
  if (n < 1) return FGBD_OK;
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  const size_t bytes = (size_t)(n + 1 + nnz) * 8 + (size_t)nnz * 8 + (size_t)9 * n * 8;
  char* d = nullptr;
  FGBD_CUDA(ctx, cudaMalloc(&d, bytes));
  int64_t* d_ip = (int64_t*)d;
  int64_t* d_ix = d_ip + n + 1;
  double* d_w = (double*)(d_ix + nnz);
  double* d_in = d_w + nnz;
  double* d_tmp = d_in + 3 * n;
  double* d_out = d_tmp + 3 * n;
  int rc = FGBD_OK;
  auto up = [&](void* dst, const void* src, size_t b) {
    if (rc == FGBD_OK && b) {
      cudaError_t e = cudaMemcpy(dst, src, b, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
      if (e != cudaSuccess) rc = cuda_error(ctx, e, "csr upload");
    }
  };
  up(d_ip, indptr, (n + 1) * 8);
  up(d_ix, indices, nnz * 8);
  up(d_w, slot_weights, nnz * 8);
  up(d_in, colors_in, 3 * n * 8);
  if (rc == FGBD_OK) rc = launch_csr_steps(ctx, d_ip, d_ix, d_w, n, d_in, d_tmp, d_out, q);
  if (rc == FGBD_OK) {
    cudaError_t e = cudaMemcpyAsync(colors_out, d_out, 3 * n * 8,
                                    dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                    ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = cuda_error(ctx, e, "csr download");
  }
  cudaFree(d);
  return rc;
}

int32_t fgbd_apply_filter(fgbd_ctx* ctx, const double* colors_in, int32_t q, double* colors_out,
                          uint32_t flags) {
  if (!ctx) return set_error(ctx, FGBD_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  if (q < 0) return set_error(ctx, FGBD_E_FILTER, "q must be >= 0, got " + std::to_string(q));
  if (ctx->g_n < 0) return set_error(ctx, FGBD_E_GRAPH, "no graph held by this context");
  const int64_t n = ctx->g_n;
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  if (n < 2) {
    if (n) FGBD_CUDA(ctx, cudaMemcpy(colors_out, colors_in, 3 * n * 8, cudaMemcpyDefault));
    return FGBD_OK;
  }
  int rc = upload_colors(ctx, colors_in, n, dev);
  if (rc) return rc;
  int fin = BUF_Y;
  if ((rc = launch_fixed_steps(ctx, n, q, ctx->g_weights64, &fin))) return rc;
  return download_signal(ctx, fin, colors_out, n, dev, 0);
}

int32_t fgbd_select_q(fgbd_ctx* ctx, const double* colors, const uint8_t* include,
                      double sigma_est, const fgbd_config* cfg, int32_t* q_out, double* x_out,
                      fgbd_report* rep, uint32_t flags) {
  if (!ctx || !cfg) return set_error(ctx, FGBD_E_ARG, "null argument");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  int rc = check_cfg(ctx, cfg);
  if (rc) return rc;
  if (sigma_est < 0) {
    char b[96];
    std::snprintf(b, sizeof(b), "sigma_est must be >= 0, got %.17g", sigma_est);
    return set_error(ctx, FGBD_E_FILTER, b);
  }
  if (ctx->g_n < 0) return set_error(ctx, FGBD_E_GRAPH, "no graph held by this context");
  if (int e = require_point_rows(ctx)) return e;
  const int64_t n = ctx->g_n;
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  if ((rc = upload_colors(ctx, colors, n, dev))) return rc;
  uint8_t* d_inc = nullptr;
  std::vector<uint8_t> ones;
  if (include) {
    FGBD_CUDA(ctx, cudaMalloc(&d_inc, n));
    cudaError_t e = cudaMemcpy(d_inc, include, n, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaFree(d_inc);
      return cuda_error(ctx, e, "include upload");
    }
  } else {
    ones.assign(n, 1);
    FGBD_CUDA(ctx, cudaMalloc(&d_inc, n));
    FGBD_CUDA(ctx, cudaMemcpy(d_inc, ones.data(), n, cudaMemcpyHostToDevice));
  }
  rc = launch_mask(ctx, n, sigma_est, 0, cfg->q_max, cfg->criterion_mode, cfg->early_exit, d_inc);
  if (rc == FGBD_OK) rc = launch_select_steps(ctx, n, cfg->q_max, ctx->g_weights64);
  if (rc == FGBD_OK) rc = pull_ctl(ctx);
  cudaFree(d_inc);
  if (rc) return rc;
  const Ctl& h = *ctx->ctl_host;
  if (h.included < 1)
    return set_error(ctx, FGBD_E_FILTER, "criterion needs at least one included point");
  if (q_out) *q_out = h.best_q;
  if (x_out && (rc = download_signal(ctx, h.best_buf, x_out, n, dev, 0))) return rc;
  if (rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->selected_q = h.best_q;
    rep->sigma_est = sigma_est;
    rep->criterion_value = h.best_crit;
    rep->steps = h.steps;
    rep->included_count = h.included;
    rep->masked_fraction = 1.0 - (double)h.included / (double)n;
    rep->n_trace = std::min(h.steps + 1, FGBD_TRACE_MAX);
    for (int k = 0; k < rep->n_trace; ++k) rep->trace[k] = h.trace[k];
  }
  return FGBD_OK;
}

int32_t fgbd_selection_criterion(fgbd_ctx* ctx, const double* y, const double* x,
                                 const uint8_t* include, int64_t n, double sigma_est, int32_t mode,
                                 double* crit_out, uint32_t flags) {
  if (!ctx || !crit_out) return set_error(ctx, FGBD_E_ARG, "null argument");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  if (mode != FGBD_CRIT_POOLED && mode != FGBD_CRIT_PER_CHANNEL)
    return set_error(ctx, FGBD_E_FILTER, "unknown criterion mode");
  if (n < 1) return set_error(ctx, FGBD_E_FILTER, "criterion needs at least one included point");
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  char* d = nullptr;
  FGBD_CUDA(ctx, cudaMalloc(&d, 6 * n * 8 + n));
  double* d_y = (double*)d;
  double* d_x = d_y + 3 * n;
  uint8_t* d_inc = include ? (uint8_t*)(d_x + 3 * n) : nullptr;
  const cudaMemcpyKind k = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  cudaError_t e = cudaMemcpy(d_y, y, 3 * n * 8, k);
  if (e == cudaSuccess) e = cudaMemcpy(d_x, x, 3 * n * 8, k);
  if (e == cudaSuccess && include) e = cudaMemcpy(d_inc, include, n, k);
  int rc = e == cudaSuccess ? launch_criterion(ctx, d_y, d_x, d_inc, n, sigma_est, mode, crit_out)
                            : cuda_error(ctx, e, "criterion upload");
  cudaFree(d);
  return rc;
}

int32_t fgbd_symmetric_eigenvalues(const double* s, int32_t d, double* out_desc, char* err,
                                   int32_t err_len) {
  std::string msg;
  if (d < 1) msg = "matrix must be square";
  int rc = d < 1 ? FGBD_E_NOISE : jacobi_eigenvalues(s, d, out_desc, &msg, nullptr);
  if (rc && err && err_len > 0) std::snprintf(err, err_len, "%s", msg.c_str());
  return rc;
}

int32_t fgbd_symmetric_eigenvalues_ex(const double* s, int32_t d, double* out_desc,
                                      int32_t* direct_off, char* err, int32_t err_len) {
  std::string msg;
  int flag = 0;
  if (d < 1) msg = "matrix must be square";
  int rc = d < 1 ? FGBD_E_NOISE : jacobi_eigenvalues(s, d, out_desc, &msg, &flag);
  if (direct_off) *direct_off = flag;
  if (rc && err && err_len > 0) std::snprintf(err, err_len, "%s", msg.c_str());
  return rc;
}

int32_t fgbd_select_tail(const double* lam, int32_t d, int32_t tau_divisor, int32_t* m,
                         double* tau, int32_t* fallback, char* err, int32_t err_len) {
  std::string msg;
  int mm = 0, fb = 0;
  double t = 0;
  int rc = select_tail_host(lam, d, tau_divisor, &mm, &t, &fb, &msg);
  if (rc) {
    if (err && err_len > 0) std::snprintf(err, err_len, "%s", msg.c_str());
    return rc;
  }
  *m = mm;
  *tau = t;
  *fallback = fb;
  return FGBD_OK;
}

}  // extern "C"
