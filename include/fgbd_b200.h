/*
 * fgbd_b200.h -- C ABI of the B200-native FGBD denoise path.
 *
 * The reference (/root/reference/pkg/src/fgbd) is a pure-Python package; it
 * has no FFI.  Its drop-in boundary for this path is the Python function
 *
 *     fgbd.denoise(pc_noisy, cfg=FilterConfig(), cached_q=None,
 *                  cached_sigma_est=None) -> (PointCloud, DenoiseReport)
 *                                               (filtering.py:259-328)
 *
 * and the public stage functions it is built from (__init__.py:18-56).
 * Every entry point below replaces one of those; the reference interface is
 * cited beside it.  The Python package `paper_2401_09721_b200` binds these
 * symbols with ctypes (see INTEGRATION.md for the binding a maintainer
 * would add to the reference).
 *
 * Conventions
 *   - plain pointers + sizes, no torch types;
 *   - coordinates are the reference's (N, 3) int64 row-major array, colours
 *     its (N, 3) float64 row-major array in [0, 255];
 *   - pointers are HOST pointers unless FGBD_FLAG_DEVICE_PTRS is set;
 *     pinned host memory is detected and copied asynchronously;
 *   - every call is stream-ordered on the context's stream and synchronous
 *     at return (Python semantics);
 *   - a context is bound to one device and is NOT thread-safe: use one
 *     context per host thread (the Python layer keeps one per thread);
 *   - functions return FGBD_OK or an error code mapped 1:1 onto the
 *     reference's exception classes; fgbd_last_error() holds the message.
 */
#ifndef FGBD_B200_H
#define FGBD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FGBD_ABI_VERSION 1

/* status codes (errors.py maps them to the reference's ValueError tree) */
enum {
  FGBD_OK = 0,
  FGBD_E_CLOUD = 1,   /* CloudError            cloud.py:13            */
  FGBD_E_GRAPH = 2,   /* GraphError            graph.py:20            */
  FGBD_E_NOISE = 3,   /* NoiseEstimationError  noise.py:26            */
  FGBD_E_FILTER = 4,  /* FilterError           filtering.py:25        */
  FGBD_E_CUDA = 5,    /* device failure (no reference analogue)       */
  FGBD_E_NCCL = 6,    /* collective failure (no reference analogue)   */
  FGBD_E_ARG = 7      /* invalid argument to the ABI itself           */
};

/* flags */
#define FGBD_FLAG_DEVICE_PTRS  0x1u  /* all array arguments are device pointers */
#define FGBD_FLAG_WEIGHTS_F64  0x2u  /* keep edge weights in fp64 (parity mode)  */
#define FGBD_FLAG_NO_TIMING    0x4u  /* skip per-stage CUDA events               */
/* fgbd_denoise / fgbd_denoise_ply: if this context's last graph was built from
 * byte-identical coordinates (same n and bit depth), reuse it instead of
 * rebuilding (the SLG is a pure function of the coordinates; the check is an
 * exact device-side comparison).  For static-geometry frame sequences. */
#define FGBD_FLAG_REUSE_GRAPH  0x8u
/* fgbd_denoise: the CALLER guarantees this frame's coordinates are the ones
 * of the graph this context holds (same n and bit depth): the coordinates are
 * neither uploaded nor compared, so a static-geometry frame moves only its
 * colours over PCIe.  Without a held graph it behaves as REUSE_GRAPH.  A
 * caller that breaks the guarantee gets the held graph's results. */
#define FGBD_FLAG_STATIC_GEOMETRY 0x10u
/* fgbd_denoise: finish NE-GBP (covariance, Jacobi, tail rule) on the device,
 * bit-identical to the host finish (csrc/noise.cu k_finish_noise, glibc's
 * hypot reproduced).  A head frame then needs no host round trip and frees
 * the device for the next frame at enqueue -- a throughput win for
 * concurrent frames, though one frame alone is ~0.1 ms slower (the 7x7 fp64
 * Jacobi runs on one thread per channel). */
#define FGBD_FLAG_DEVICE_NE 0x20u

enum { FGBD_CRIT_POOLED = 0, FGBD_CRIT_PER_CHANNEL = 1 };   /* filtering.py:47 */
enum { FGBD_TAU_COUNT = 0, FGBD_TAU_COUNT_PLUS_ONE = 1 };   /* filtering.py:49 */

/* Mirror of FilterConfig (filtering.py:33-59).  epsilon = NaN means None. */
typedef struct fgbd_config {
  int32_t q_max;               /* 64   */
  double epsilon;              /* NaN  */
  int32_t fslr_enabled;        /* 1    */
  int32_t patch_size;          /* 7    */
  int32_t reestimate_interval; /* 10 (used by the frame-sequence driver) */
  double fslr_sigma_floor;     /* 0.5  */
  int32_t criterion_mode;      /* FGBD_CRIT_POOLED */
  int32_t early_exit;          /* 1    */
  int32_t tau_divisor;         /* FGBD_TAU_COUNT */
} fgbd_config;

#define FGBD_MAX_PATCH 7   /* 1 + max SLG degree (6)                     */
#define FGBD_TRACE_MAX 1025 /* criterion values recorded for q = 0..1024 */

/* Mirror of DenoiseReport (filtering.py:86-116) + device diagnostics. */
typedef struct fgbd_report {
  int32_t selected_q;
  double sigma_est;
  double masked_fraction;
  double criterion_value;      /* NaN when not computed (cached / N<2) */
  int32_t converged;           /* -1 = None, 0/1 otherwise */
  int32_t cached;
  int64_t eligible_count;      /* -1 = None */
  /* stage_timings, seconds (CUDA events) */
  double t_graph_construction;
  double t_noise_estimation;
  double t_low_pass_filter;
  double t_total;
  /* diagnostics */
  int32_t steps;               /* filter steps executed by select_q (S) */
  int32_t all_excluded_fallback; /* FSLR excluded everyone -> warn + unmasked */
  int64_t n_edges;
  int64_t nnz;
  int32_t max_degree;
  double sigma_g;
  int64_t included_count;
  double per_channel_sigma[3];
  double eigenvalues[3][FGBD_MAX_PATCH]; /* descending, first patch_size used */
  int32_t tail_m[3];
  double tail_tau[3];
  int32_t tail_fallback[3];
  int32_t n_trace;             /* entries valid in trace[] */
  double trace[FGBD_TRACE_MAX];/* criterion at q = 0..steps */
  int32_t gpu_launches;        /* kernels launched by this call */
  double t_lf_steps;           /* seconds spent in the filter-step launches only */
  double t_h2d;                /* coordinates host->device (colours overlap the graph build) */
  double t_d2h;                /* denoised colours device->host */
  int32_t graph_reused;        /* 1: FGBD_FLAG_REUSE_GRAPH matched the held graph */
  /* per channel: 1 when Jacobi's difference-of-sums convergence test
     (noise.py:152) never met its target but the directly summed
     off-diagonal norm did -- the reference raises NoiseEstimationError
     "Jacobi did not converge" on such a matrix (noise.py:180-185); this
     build returns the eigenvalues */
  int32_t jacobi_direct_off[3];
  /* slab ranks run by this call (fgbd_denoise_slab): per rank, seconds of
     device time in [0] upload + own sort + block lists, [1] cross-slab
     neighbours + rows, [2] NE-GBP + FSLR, [3] output + download */
  double t_slab_rank[16][4];
} fgbd_report;

/* Result of NE-GBP (noise.py:63-73). */
typedef struct fgbd_noise {
  double sigma_est;
  double per_channel_sigma[3];
  double eigenvalues[3][FGBD_MAX_PATCH];
  double covariance[3][FGBD_MAX_PATCH][FGBD_MAX_PATCH];
  int32_t m[3];
  double tau[3];
  int32_t fallback[3];
  int64_t eligible_count;
  int32_t patch_size;
  int32_t jacobi_direct_off[3]; /* see fgbd_report.jacobi_direct_off */
} fgbd_noise;

/* Shape of the graph held by a context after fgbd_build_graph. */
typedef struct fgbd_graph_info {
  int64_t n;
  int64_t n_edges;   /* E: unique undirected edges */
  int64_t nnz;       /* 2E CSR slots */
  int32_t max_degree;
  double sigma_g;    /* graph.py:227-233 */
} fgbd_graph_info;

typedef struct fgbd_ctx fgbd_ctx;

/* ---- context ---------------------------------------------------------- */
/* Owns the device scratch for frames up to max_points (grows on demand),
 * one CUDA stream and the per-context error message.  NULL on failure
 * (fgbd_last_error(NULL) then describes why). */
fgbd_ctx* fgbd_ctx_create(int32_t device, int64_t max_points);
void fgbd_ctx_destroy(fgbd_ctx* ctx);
const char* fgbd_last_error(const fgbd_ctx* ctx);
int32_t fgbd_abi_version(void);
/* cudaStream_t of the context, for callers that order work around it. */
void* fgbd_ctx_stream(fgbd_ctx* ctx);
/* device bytes currently reserved by the context */
int64_t fgbd_ctx_device_bytes(const fgbd_ctx* ctx);

/* ---- the drop-in: denoise (filtering.py:259-328) ---------------------- */
/* coords: (n,3) int64, colors: (n,3) float64, out_colors: (n,3) float64.
 * cached_q < 0 means None (full estimation + selection); otherwise the
 * cached path (filtering.py:313-326) runs cached_q filter steps.
 * cached_sigma is reported verbatim when cached_q >= 0 (NaN = None -> 0). */
int32_t fgbd_denoise(fgbd_ctx* ctx, const int64_t* coords, const double* colors,
                     int64_t n, int32_t bit_depth, const fgbd_config* cfg,
                     int32_t cached_q, double cached_sigma, double* out_colors,
                     fgbd_report* report, uint32_t flags);

/* ---- stage entry points (parity / stage API) -------------------------- */
/* radix_argsort (graph.py:154-171): stable LSD argsort of uint64 keys over
 * ceil(key_bits/8) byte passes.  perm_out: (n,) int64. */
int32_t fgbd_radix_argsort(fgbd_ctx* ctx, const uint64_t* keys, int64_t n,
                           int32_t key_bits, int64_t* perm_out, uint32_t flags);

/* scanline_codes + sort_permutation (graph.py:122-136, 174-176) for one
 * line (1..3).  codes_out (n,) uint64 and perm_out (n,) int64 may be NULL. */
int32_t fgbd_scan_line(fgbd_ctx* ctx, const int64_t* coords, int64_t n,
                       int32_t bit_depth, int32_t line, uint64_t* codes_out,
                       int64_t* perm_out, uint32_t flags);

/* build_slg / build_weighted_slg (graph.py:211-251): builds the scan-line
 * graph of the frame on the device and keeps it in the context. */
int32_t fgbd_build_graph(fgbd_ctx* ctx, const int64_t* coords, int64_t n,
                         int32_t bit_depth, fgbd_graph_info* info, uint32_t flags);

/* Export the context's graph in the reference's Graph conventions
 * (graph.py:40-107): indptr (n+1), indices/csr_edge (nnz) ascending per row,
 * edge_u/edge_v/edge_sqdist (E) lexicographic with u < v, edge_weights (E)
 * exp(-sqdist/sigma_g^2), weighted_degrees (n).  Any pointer may be NULL. */
int32_t fgbd_graph_export(fgbd_ctx* ctx, int64_t* indptr, int64_t* indices,
                          int64_t* csr_edge, int64_t* edge_u, int64_t* edge_v,
                          double* edge_sqdist, double* edge_weights,
                          double* weighted_degrees);

/* extract_patches + estimate_noise_from_patches (noise.py:82-119, 219-243)
 * on the context's graph.  fslr_stat_out (n) receives the FSLR statistic
 * mean_c std_c(patch) (filtering.py:186) for eligible points and -1 for the
 * rest; may be NULL. */
int32_t fgbd_estimate_noise(fgbd_ctx* ctx, const double* colors, int32_t patch_size,
                            int32_t tau_divisor, fgbd_noise* out,
                            double* fslr_stat_out, uint32_t flags);

/* fslr_mask (filtering.py:175-194) from the last fgbd_estimate_noise call.
 * include_out (n) uint8.  Returns FGBD_E_FILTER with all_excluded = 1 when
 * every point was excluded (the reference's AllPointsExcludedError). */
int32_t fgbd_fslr_mask(fgbd_ctx* ctx, double sigma_est, double sigma_floor,
                       uint8_t* include_out, int32_t* all_excluded);

/* filter_step x q (filtering.py:132-165) on a caller-supplied CSR graph with
 * fp64 per-slot weights (weight injection: bit-exact against scipy). */
int32_t fgbd_filter_steps_csr(fgbd_ctx* ctx, const int64_t* indptr,
                              const int64_t* indices, const double* slot_weights,
                              int64_t n, int64_t nnz, const double* colors_in,
                              int32_t q, double* colors_out, uint32_t flags);

/* apply_filter on the context's graph (the cached-q path). */
int32_t fgbd_apply_filter(fgbd_ctx* ctx, const double* colors_in, int32_t q,
                          double* colors_out, uint32_t flags);

/* select_q (filtering.py:225-256) on the context's graph with an explicit
 * include mask (NULL = all points). */
int32_t fgbd_select_q(fgbd_ctx* ctx, const double* colors, const uint8_t* include,
                      double sigma_est, const fgbd_config* cfg, int32_t* q_out,
                      double* x_out, fgbd_report* report, uint32_t flags);

/* selection_criterion (filtering.py:197-222). */
int32_t fgbd_selection_criterion(fgbd_ctx* ctx, const double* y, const double* x,
                                 const uint8_t* include, int64_t n, double sigma_est,
                                 int32_t mode, double* crit_out, uint32_t flags);

/* extract_patches (noise.py:82-119) on the context's graph: materialises
 * the distance-sorted patch vectors (3, ne, patch_size) and the eligible
 * point ids (ne).  *ne_out always receives ne; outputs may be NULL. */
int32_t fgbd_extract_patches(fgbd_ctx* ctx, const double* colors, int32_t patch_size,
                             int64_t* point_index_out, double* vectors_out, int64_t* ne_out,
                             uint32_t flags);

/* compute_sigma_g + apply_gaussian_weights (graph.py:227-245) on a
 * caller-supplied edge list: sigma = mean(sqrt(sqdist)) when sigma_g is NaN,
 * weights = exp(-sqdist / sigma^2).  weights_out may be NULL. */
int32_t fgbd_edge_weights(fgbd_ctx* ctx, const double* edge_sqdist, int64_t n_edges,
                          double sigma_g, double* sigma_out, double* weights_out,
                          uint32_t flags);

/* symmetric_eigenvalues (noise.py:133-185), host C++ Jacobi. */
int32_t fgbd_symmetric_eigenvalues(const double* s, int32_t d, double* out_desc,
                                   char* err, int32_t err_len);
/* The same, also reporting in *direct_off whether the result was accepted
 * only by the directly summed off-diagonal norm -- i.e. the reference would
 * have raised "Jacobi did not converge" (noise.py:180-185). */
int32_t fgbd_symmetric_eigenvalues_ex(const double* s, int32_t d, double* out_desc,
                                      int32_t* direct_off, char* err, int32_t err_len);
/* select_tail (noise.py:188-216). */
int32_t fgbd_select_tail(const double* lam, int32_t d, int32_t tau_divisor,
                         int32_t* m, double* tau, int32_t* fallback,
                         char* err, int32_t err_len);

/* ---- spatial slab partition of one frame over P ranks ---- */
/* The frame is cut into z-slabs (contiguous ranges of the global scan-line-1
 * order); rank r owns counts[r] points and uploads, sorts, estimates and
 * filters only those.  Cross-slab scan-line neighbours come from the peers'
 * block lists, sigma_g / the NE moments / the FSLR sums are all-gathered,
 * and halo signals are read from the owner's buffers -- all over peer memory
 * (csrc/slab.cu).  Results equal fgbd_denoise on the whole frame (q, S and
 * colours bit for bit).  Bit depths up to 15.
 *
 * FGBD_SLAB_EMULATED: all P ranks run in this process on this context's GPU
 * (the test harness of the protocol); the arrays of fgbd_denoise_slab then
 * hold every rank's points, concatenated in rank order.  Otherwise one
 * process per GPU exchanges fgbd_slab_export handles (IPC) and calls
 * fgbd_slab_import before its first fgbd_denoise_slab. */
#define FGBD_SLAB_EMULATED     0x1u
#define FGBD_SLAB_FULL_OUTPUT  0x2u  /* multi-GPU: every rank receives the full frame */
#define FGBD_SLAB_EXCHANGE     0x4u  /* emulated: run the filter's per-step cross-rank
                                        exchange (slots + ticks) of the P-GPU protocol */
typedef struct fgbd_slab fgbd_slab;
fgbd_slab* fgbd_slab_create(fgbd_ctx* ctx, int32_t world, int32_t rank, int64_t n_total,
                            int64_t max_own, uint32_t slab_flags);
void fgbd_slab_destroy(fgbd_ctx* ctx, fgbd_slab* slab);
int32_t fgbd_slab_handle_size(void);
int32_t fgbd_slab_export(fgbd_ctx* ctx, fgbd_slab* slab, uint8_t* handle_out);
int32_t fgbd_slab_import(fgbd_ctx* ctx, fgbd_slab* slab, const uint8_t* handles);
/* denoise (filtering.py:259-328) over the slab ranks.  coords / colors: the
 * own points (all ranks' points, rank-major, when emulated) in increasing
 * global index; gidx: their global indices (NULL: gidx_base + i); counts:
 * points of every rank (z-slab order).  out_colors: the own points' colours
 * in input order, or the full frame (n_total, 3) with FGBD_SLAB_FULL_OUTPUT.
 * The report describes the whole frame. */
int32_t fgbd_denoise_slab(fgbd_ctx* ctx, fgbd_slab* slab, const int64_t* coords,
                          const double* colors, const uint32_t* gidx, int64_t gidx_base,
                          const int64_t* counts, int32_t bit_depth, const fgbd_config* cfg,
                          int32_t cached_q, double cached_sigma, double* out_colors,
                          fgbd_report* report, uint32_t flags);

/* ---- PLY binary vertex records (ply.py:134-287) ---- */
/* type codes: 0 int8, 1 uint8, 2 int16, 3 uint16, 4 int32, 5 uint32,
 * 6 float32, 7 float64.  offsets/types: x, y, z, red, green, blue. */
/* decode packed little-endian records into coords (int64 when coords_int is
 * given, else float64) and colours float64; *bit_length receives the bit
 * length of the largest integer coordinate (infer_bit_depth). */
int32_t fgbd_ply_decode(fgbd_ctx* ctx, const uint8_t* body, int64_t n, int32_t stride,
                        const int32_t* offsets, const int32_t* types, int64_t* coords_int,
                        double* coords_float, double* colors, int32_t* bit_length,
                        uint32_t flags);
/* encode 15-byte records (uint32 or float32 x/y/z, colours rounded half-up
 * to uint8), byte-identical to the reference save_ply body. */
int32_t fgbd_ply_encode(fgbd_ctx* ctx, const int64_t* coords_int, const double* coords_float,
                        const double* colors, int64_t n, uint8_t* body_out, uint32_t flags);
/* decode -> denoise -> encode on the device: raw vertex records in, the
 * denoised frame's records (save_ply layout) out.  bit_depth <= 0 infers it. */
int32_t fgbd_denoise_ply(fgbd_ctx* ctx, const uint8_t* body, int64_t n, int32_t stride,
                         const int32_t* offsets, const int32_t* types, int32_t bit_depth,
                         const fgbd_config* cfg, int32_t cached_q, double cached_sigma,
                         uint8_t* body_out, fgbd_report* report, uint32_t flags);

/* ---- brute-force kNN graph (graph.py:254-298) ------ */
/* build_knn_brute: exact k nearest neighbours (ties by index), symmetrised by
 * union (_graph_from_pairs, graph.py:179-208).  Coordinates are int64
 * (coords_int, bit_depth known) or float64 (coords_float).  The graph stays
 * in the context; *n_edges receives E. */
int32_t fgbd_knn_build(fgbd_ctx* ctx, const int64_t* coords_int, const double* coords_float,
                       int64_t n, int32_t k, int32_t bit_depth, int64_t* n_edges,
                       uint32_t flags);
/* Copy the held kNN graph out in the reference's Graph conventions: indptr
 * (n+1), indices/csr_edge (2E), edge_u/edge_v/edge_sqdist (E). */
int32_t fgbd_knn_export(fgbd_ctx* ctx, int64_t* indptr, int64_t* indices, int64_t* csr_edge,
                        int64_t* edge_u, int64_t* edge_v, double* edge_sqdist);

/* ---- data-model helpers (cloud.py:89-140) --------- */
/* quantize_coordinates: per-axis [min, max] -> [0, 2^bits - 1], rint.  One of
 * coords_int / coords_float.  Integer clouds already on the grid are left
 * alone: *passthrough = 1 and out is not written. */
int32_t fgbd_quantize(fgbd_ctx* ctx, const int64_t* coords_int, const double* coords_float,
                      int64_t n, int32_t bits, int64_t* out, int32_t* passthrough,
                      uint32_t flags);
/* sum over count values of (a - b)^2 in numpy's pairwise-summation order
 * (np.mean's numerator in psnr, cloud.py:126-140). */
int32_t fgbd_sq_error_sum(fgbd_ctx* ctx, const double* a, const double* b, int64_t count,
                          double* sum_out, uint32_t flags);

/* add_gaussian_noise (cloud.py:111-123): out[k] = clip(colors[k] + (0 + sigma z_k),
 * 0, 255) for the first `count` standard normals z_k of numpy's
 * Generator(Philox(key, counter)).normal stream (Philox4x64-10 + numpy's
 * 256-level ziggurat, the same variates bit for bit).  key / counter are the
 * BitGenerator's state (np.random.Philox(seed).state) before any draw.
 * sigma < 0 -> FGBD_E_CLOUD. */
int32_t fgbd_gaussian_noise(fgbd_ctx* ctx, const double* colors, int64_t count, double sigma,
                            const uint64_t key[2], const uint64_t counter[4], double* out,
                            uint32_t flags);

/* pinned host buffers for zero-staging transfers */
void* fgbd_host_alloc(int64_t bytes);
void fgbd_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* FGBD_B200_H */
