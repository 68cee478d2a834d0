// Exact brute-force k-nearest-neighbour graph on the device (SURVEY 8(f)
// rank 4; reference graph.py:254-298) -- the baseline of the paper's Table 3
// graph-construction comparison, off the denoise path.
//
// k_knn        all-pairs scan, one query per thread (two per thread in the
//              integer path), candidates staged through shared memory in
//              ascending index order; top-k kept in registers ordered by
//              (squared distance, index) -- exactly the reference's insertion
//              rule (strict <, so equal distances keep the smaller index).
//              Integer coordinates of <= 15 bits use exact uint32 distances;
//              wider or float coordinates use fp64 with the reference's
//              operation order ((dx*dx + dy*dy) + dz*dz, no FMA).
// pairs->Graph _graph_from_pairs (graph.py:179-208): undirected keys
//              lo*n + hi, stable radix sort, unique, squared lengths, and a
//              second sort of the 2E directed slots for the CSR rows.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <string>

#include "device_util.cuh"
#include "fgbd_internal.cuh"

namespace fgbd {

constexpr int kKnnBlock = 128;
constexpr int kKnnTile = 1024;  // candidates per shared-memory stage
constexpr int kKnnMaxK = 64;

// ---- distances ----------------------------------------------------------
struct DistU32 {
  using P = int4;
  using D = unsigned;
  static __device__ __forceinline__ D inf() { return UINT_MAX; }
  static __device__ __forceinline__ D dist(const P& a, const P& b) {
    const int dx = b.x - a.x, dy = b.y - a.y, dz = b.z - a.z;
    return (unsigned)(dx * dx) + (unsigned)(dy * dy) + (unsigned)(dz * dz);
  }
};

struct DistF64 {
  using P = double4;
  using D = double;
  static __device__ __forceinline__ D inf() { return __longlong_as_double(0x7ff0000000000000LL); }
  static __device__ __forceinline__ D dist(const P& a, const P& b) {
    const double dx = __dsub_rn(b.x, a.x), dy = __dsub_rn(b.y, a.y), dz = __dsub_rn(b.z, a.z);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  }
};

// Insert (d, j) into the sorted top-K (d ascending, ties: earlier index
// first).  Called only when d < bd[K-1].  From the insertion slot on, every
// entry shifts down one place (a carried entry must not be re-compared: on
// equal distances that would reorder the tie).
template <int K, typename D>
__device__ __forceinline__ void topk_insert(D (&bd)[K], int (&bj)[K], D d, int j) {
  bool carry = false;
#pragma unroll
  for (int p = 0; p < K; ++p) {
    if (carry || d < bd[p]) {
      carry = true;
      const D td = bd[p];
      const int tj = bj[p];
      bd[p] = d;
      bj[p] = j;
      d = td;
      j = tj;
    }
  }
}

// Q queries per thread, K neighbours each.
template <class M, int K, int Q>
__global__ void __launch_bounds__(kKnnBlock) k_knn(const typename M::P* __restrict__ pts,
                                                    int64_t n, int* __restrict__ out) {
  using P = typename M::P;
  using D = typename M::D;
  __shared__ P tile[kKnnTile];
  const int64_t q0 = ((int64_t)blockIdx.x * kKnnBlock) * Q + threadIdx.x;
  P me[Q];
  int qi[Q];
  D bd[Q][K];
  int bj[Q][K];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int64_t i = q0 + (int64_t)q * kKnnBlock;
    qi[q] = i < n ? (int)i : -1;
    me[q] = pts[i < n ? i : 0];
#pragma unroll
    for (int t = 0; t < K; ++t) {
      bd[q][t] = M::inf();
      bj[q][t] = -1;
    }
  }
  for (int64_t base = 0; base < n; base += kKnnTile) {
    const int cnt = (int)std::min<int64_t>(kKnnTile, n - base);
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += kKnnBlock) tile[t] = pts[base + t];
    __syncthreads();
    for (int c = 0; c < cnt; ++c) {
      const P p = tile[c];
      const int j = (int)(base + c);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const D d = M::dist(me[q], p);
        if (d < bd[q][K - 1] && j != qi[q]) topk_insert<K, D>(bd[q], bj[q], d, j);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < Q; ++q)
    if (qi[q] >= 0)
#pragma unroll
      for (int t = 0; t < K; ++t) out[(int64_t)qi[q] * K + t] = bj[q][t];
}

// Generic k (register arrays would spill): top-k in local memory.
template <class M>
__global__ void __launch_bounds__(kKnnBlock) k_knn_any(const typename M::P* __restrict__ pts,
                                                        int64_t n, int k, int* __restrict__ out) {
  using P = typename M::P;
  using D = typename M::D;
  __shared__ P tile[kKnnTile];
  const int64_t i = (int64_t)blockIdx.x * kKnnBlock + threadIdx.x;
  const P me = pts[i < n ? i : 0];
  D bd[kKnnMaxK];
  int bj[kKnnMaxK];
  for (int t = 0; t < k; ++t) {
    bd[t] = M::inf();
    bj[t] = -1;
  }
  for (int64_t base = 0; base < n; base += kKnnTile) {
    const int cnt = (int)std::min<int64_t>(kKnnTile, n - base);
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += kKnnBlock) tile[t] = pts[base + t];
    __syncthreads();
    for (int c = 0; c < cnt; ++c) {
      D d = M::dist(me, tile[c]);
      int j = (int)(base + c);
      if (!(d < bd[k - 1]) || j == i) continue;
      bool carry = false;
      for (int p = 0; p < k; ++p) {
        if (carry || d < bd[p]) {
          carry = true;
          const D td = bd[p];
          const int tj = bj[p];
          bd[p] = d;
          bj[p] = j;
          d = td;
          j = tj;
        }
      }
    }
  }
  if (i < n)
    for (int t = 0; t < k; ++t) out[i * k + t] = bj[t];
}

// ---- packing ------------------------------------------------------------
__global__ void k_pack_i4(const int64_t* __restrict__ c, int64_t n, int4* __restrict__ p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = make_int4((int)c[3 * i], (int)c[3 * i + 1], (int)c[3 * i + 2], 0);
}

// float64 copy of the coordinates (graph.py: coords.astype(np.float64))
__global__ void k_pack_d4(const int64_t* __restrict__ ci, const double* __restrict__ cf, int64_t n,
                          double4* __restrict__ p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (ci)
      p[i] = make_double4((double)ci[3 * i], (double)ci[3 * i + 1], (double)ci[3 * i + 2], 0.0);
    else
      p[i] = make_double4(cf[3 * i], cf[3 * i + 1], cf[3 * i + 2], 0.0);
  }
}

// ---- pairs -> Graph -----------------------------------------------------
// directed (i, nearest[i][t]) -> undirected key lo*n + hi; self pairs get
// the sentinel n*n, which sorts after every real key
__global__ void k_pair_keys(const int* __restrict__ nb, int64_t n, int k,
                            unsigned long long* __restrict__ key) {
  const unsigned long long sentinel = (unsigned long long)(n * n);
  const int64_t m = n * k;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = e / k, v = nb[e];
    const int64_t lo = u < v ? u : v, hi = u < v ? v : u;
    key[e] = lo == hi ? sentinel : (unsigned long long)(lo * n + hi);
  }
}

// sorted keys + first-occurrence flags
__global__ void k_unique_flags(const unsigned long long* __restrict__ key,
                               const uint32_t* __restrict__ perm, int64_t m,
                               unsigned long long sentinel,
                               unsigned long long* __restrict__ sorted,
                               int64_t* __restrict__ flag) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long kk = key[perm[p]];
    const unsigned long long prev = p ? key[perm[p - 1]] : sentinel;
    sorted[p] = kk;
    flag[p] = (kk != sentinel && (p == 0 || kk != prev)) ? 1 : 0;
  }
}

// unique edges (lexicographic, u < v), their squared lengths, and the 2E
// directed CSR keys src*n + dst with the edge id as payload
__global__ void k_edges(const unsigned long long* __restrict__ sorted,
                        const int64_t* __restrict__ flag, const int64_t* __restrict__ eid,
                        int64_t m, int64_t n, const double4* __restrict__ pts, int64_t E,
                        int64_t* __restrict__ eu, int64_t* __restrict__ ev,
                        double* __restrict__ sq, unsigned long long* __restrict__ key2,
                        int64_t* __restrict__ slot_eid) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[p]) continue;
    const int64_t e = eid[p];
    const int64_t u = (int64_t)(sorted[p] / (unsigned long long)n);
    const int64_t v = (int64_t)(sorted[p] % (unsigned long long)n);
    eu[e] = u;
    ev[e] = v;
    const double4 a = pts[u], b = pts[v];
    const double dx = __dsub_rn(a.x, b.x), dy = __dsub_rn(a.y, b.y), dz = __dsub_rn(a.z, b.z);
    // np.einsum("ij,ij->i") order for 3 terms: (x*x + z*z) + y*y
    sq[e] = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dz, dz)), __dmul_rn(dy, dy));
    key2[e] = (unsigned long long)(u * n + v);
    key2[E + e] = (unsigned long long)(v * n + u);
    slot_eid[e] = e;
    slot_eid[E + e] = e;
  }
}

// CSR rows from the sorted directed keys
__global__ void k_csr_rows(const unsigned long long* __restrict__ key2,
                           const int64_t* __restrict__ slot_eid, const uint32_t* __restrict__ perm,
                           int64_t nnz, int64_t n, int64_t* __restrict__ indptr,
                           int64_t* __restrict__ indices, int64_t* __restrict__ csr_edge) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long kk = key2[perm[p]];
    const int64_t src = (int64_t)(kk / (unsigned long long)n);
    indices[p] = (int64_t)(kk % (unsigned long long)n);
    csr_edge[p] = slot_eid[perm[p]];
    const int64_t prev = p ? (int64_t)(key2[perm[p - 1]] / (unsigned long long)n) : -1;
    for (int64_t r = prev + 1; r <= src; ++r) indptr[r] = p;
    if (p == nnz - 1)
      for (int64_t r = src + 1; r <= n; ++r) indptr[r] = nnz;
  }
}

static int grid_n(fgbd_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + kBlock - 1) / kBlock, ctx->num_sms * 8));
}

template <class M, int K>
static void knn_fixed(fgbd_ctx* ctx, const void* pts, int64_t n, int* out) {
  constexpr int Q = sizeof(typename M::P) == 16 ? 2 : 1;
  const int64_t per = (int64_t)kKnnBlock * Q;
  const int grid = (int)((n + per - 1) / per);
  k_knn<M, K, Q><<<grid, kKnnBlock, 0, ctx->stream>>>((const typename M::P*)pts, n, out);
}

template <class M>
static int knn_dispatch(fgbd_ctx* ctx, const void* pts, int64_t n, int k, int* out) {
  switch (k) {
    case 1: knn_fixed<M, 1>(ctx, pts, n, out); break;
    case 2: knn_fixed<M, 2>(ctx, pts, n, out); break;
    case 3: knn_fixed<M, 3>(ctx, pts, n, out); break;
    case 4: knn_fixed<M, 4>(ctx, pts, n, out); break;
    case 5: knn_fixed<M, 5>(ctx, pts, n, out); break;
    case 6: knn_fixed<M, 6>(ctx, pts, n, out); break;
    case 7: knn_fixed<M, 7>(ctx, pts, n, out); break;
    case 8: knn_fixed<M, 8>(ctx, pts, n, out); break;
    default: {
      const int grid = (int)((n + kKnnBlock - 1) / kKnnBlock);
      k_knn_any<M><<<grid, kKnnBlock, 0, ctx->stream>>>((const typename M::P*)pts, n, k, out);
    }
  }
  FGBD_LAUNCH(ctx);
  return FGBD_OK;
}

}  // namespace fgbd

using namespace fgbd;

namespace {

inline size_t al(size_t b) { return (b + 255) & ~size_t(255); }

int aux_reserve(fgbd_ctx* ctx, size_t need) {
  if (ctx->aux_bytes >= need) return FGBD_OK;
  if (ctx->aux) cudaFree(ctx->aux);
  ctx->aux = nullptr;
  ctx->aux_bytes = 0;
  FGBD_CUDA(ctx, cudaMalloc(&ctx->aux, need));
  ctx->aux_bytes = need;
  return FGBD_OK;
}

}  // namespace

extern "C" {

int32_t fgbd_knn_build(fgbd_ctx* ctx, const int64_t* coords_int, const double* coords_float,
                       int64_t n, int32_t k, int32_t bit_depth, int64_t* n_edges,
                       uint32_t flags) {
  if (!ctx) return set_error(ctx, FGBD_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  ctx->knn_n = -1;
  if (k < 1 || k >= n)
    return set_error(ctx, FGBD_E_GRAPH, "k must satisfy 1 <= k < n_points, got k=" +
                                            std::to_string(k) + ", n=" + std::to_string(n));
  if (k > kKnnMaxK)
    return set_error(ctx, FGBD_E_ARG, "this build supports k <= " + std::to_string(kKnnMaxK));
  if (n >= (int64_t(1) << 31))
    return set_error(ctx, FGBD_E_GRAPH, "point count exceeds the 2^31 edge-encoding limit");
  if (!coords_int && !coords_float) return set_error(ctx, FGBD_E_ARG, "no coordinates");
  const bool dev = flags & FGBD_FLAG_DEVICE_PTRS;
  const bool narrow = coords_int && bit_depth >= 1 && bit_depth <= 15;
  const int64_t m = n * k;
  // aux layout: coords in | packed f64 points | packed i32 points | nearest |
  // keys | sorted | flags | eid | tile sums | edges (u, v, sq) | key2 | slot eid
  // | CSR (indptr, indices, csr_edge)
  const int64_t tiles = (2 * m + 2047) / 2048 + 2;
  size_t off = 0;
  auto take = [&](size_t b) { const size_t o = off; off += al(b); return o; };
  const size_t o_in = take((size_t)n * 24), o_d4 = take((size_t)n * 32),
               o_i4 = take(narrow ? (size_t)n * 16 : 0), o_nb = take((size_t)m * 4),
               o_key = take((size_t)m * 8), o_sorted = take((size_t)m * 8),
               o_flag = take((size_t)m * 8), o_eid = take((size_t)m * 8),
               o_tmp = take((size_t)tiles * 8 + 16), o_eu = take((size_t)m * 8),
               o_ev = take((size_t)m * 8), o_sq = take((size_t)m * 8),
               o_key2 = take((size_t)2 * m * 8), o_seid = take((size_t)2 * m * 8),
               o_indptr = take((size_t)(n + 1) * 8), o_ind = take((size_t)2 * m * 8),
               o_csr = take((size_t)2 * m * 8);
  int rc = aux_reserve(ctx, off);
  if (rc) return rc;
  // the sort scratch is shared with the frame pipeline: the held graph is gone
  if ((rc = ensure_capacity(ctx, 2 * m, 1))) return rc;
  ctx->g_n = -1;
  char* a = (char*)ctx->aux;
  const cudaMemcpyKind kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  FGBD_CUDA(ctx, cudaMemcpyAsync(a + o_in, coords_int ? (const void*)coords_int : (const void*)coords_float,
                                 (size_t)n * 24, kind, ctx->stream));
  double4* d4 = (double4*)(a + o_d4);
  k_pack_d4<<<grid_n(ctx, n), kBlock, 0, ctx->stream>>>(
      coords_int ? (const int64_t*)(a + o_in) : nullptr,
      coords_int ? nullptr : (const double*)(a + o_in), n, d4);
  FGBD_LAUNCH(ctx);
  int* nb = (int*)(a + o_nb);
  if (narrow) {
    int4* i4 = (int4*)(a + o_i4);
    k_pack_i4<<<grid_n(ctx, n), kBlock, 0, ctx->stream>>>((const int64_t*)(a + o_in), n, i4);
    FGBD_LAUNCH(ctx);
    if ((rc = knn_dispatch<DistU32>(ctx, i4, n, k, nb))) return rc;
  } else {
    if ((rc = knn_dispatch<DistF64>(ctx, d4, n, k, nb))) return rc;
  }
  // pairs -> unique undirected edges
  unsigned long long* key = (unsigned long long*)(a + o_key);
  k_pair_keys<<<grid_n(ctx, m), kBlock, 0, ctx->stream>>>(nb, n, k, key);
  FGBD_LAUNCH(ctx);
  // keys and the sentinel are <= n^2: only the digits below its top bit sort
  const unsigned long long n2 = (unsigned long long)(n * n);
  const int key_bits = 64 - __builtin_clzll(n2);
  uint32_t* perm = nullptr;
  if ((rc = launch_argsort64(ctx, (const uint64_t*)key, m, key_bits, &perm))) return rc;
  unsigned long long* sorted = (unsigned long long*)(a + o_sorted);
  int64_t* flag = (int64_t*)(a + o_flag);
  int64_t* eid = (int64_t*)(a + o_eid);
  int64_t* tmp = (int64_t*)(a + o_tmp);
  k_unique_flags<<<grid_n(ctx, m), kBlock, 0, ctx->stream>>>(key, perm, m, n2, sorted, flag);
  FGBD_LAUNCH(ctx);
  if ((rc = scan_exclusive(ctx, flag, m, eid, tmp, tmp + tiles))) return rc;
  int64_t E = 0;
  FGBD_CUDA(ctx, cudaMemcpyAsync(&E, tmp + tiles, 8, cudaMemcpyDeviceToHost, ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  int64_t* eu = (int64_t*)(a + o_eu);
  int64_t* ev = (int64_t*)(a + o_ev);
  double* sq = (double*)(a + o_sq);
  unsigned long long* key2 = (unsigned long long*)(a + o_key2);
  int64_t* seid = (int64_t*)(a + o_seid);
  k_edges<<<grid_n(ctx, m), kBlock, 0, ctx->stream>>>(sorted, flag, eid, m, n, d4, E, eu, ev, sq,
                                                        key2, seid);
  FGBD_LAUNCH(ctx);
  // CSR: directed slots sorted by (src, dst)
  int64_t* indptr = (int64_t*)(a + o_indptr);
  int64_t* ind = (int64_t*)(a + o_ind);
  int64_t* csr = (int64_t*)(a + o_csr);
  const int64_t nnz = 2 * E;
  if (nnz > 0) {
    if ((rc = launch_argsort64(ctx, (const uint64_t*)key2, nnz, key_bits, &perm))) return rc;
    k_csr_rows<<<grid_n(ctx, nnz), kBlock, 0, ctx->stream>>>(key2, seid, perm, nnz, n, indptr, ind,
                                                             csr);
    FGBD_LAUNCH(ctx);
  } else {
    FGBD_CUDA(ctx, cudaMemsetAsync(indptr, 0, (size_t)(n + 1) * 8, ctx->stream));
  }
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->knn_n = n;
  ctx->knn_e = E;
  ctx->knn_off[0] = o_indptr;
  ctx->knn_off[1] = o_ind;
  ctx->knn_off[2] = o_csr;
  ctx->knn_off[3] = o_eu;
  ctx->knn_off[4] = o_ev;
  ctx->knn_off[5] = o_sq;
  if (n_edges) *n_edges = E;
  return FGBD_OK;
}

int32_t fgbd_knn_export(fgbd_ctx* ctx, int64_t* indptr, int64_t* indices, int64_t* csr_edge,
                        int64_t* edge_u, int64_t* edge_v, double* edge_sqdist) {
  if (!ctx) return set_error(ctx, FGBD_E_ARG, "null context");
  cudaSetDevice(ctx->device);
  if (ctx->knn_n < 0) return set_error(ctx, FGBD_E_GRAPH, "no kNN graph held by this context");
  const int64_t n = ctx->knn_n, E = ctx->knn_e;
  const size_t bytes[6] = {(size_t)(n + 1) * 8, (size_t)E * 16, (size_t)E * 16,
                           (size_t)E * 8,       (size_t)E * 8,  (size_t)E * 8};
  void* dst[6] = {indptr, indices, csr_edge, edge_u, edge_v, edge_sqdist};
  const char* a = (const char*)ctx->aux;
  for (int t = 0; t < 6; ++t)
    if (dst[t] && bytes[t])
      FGBD_CUDA(ctx, cudaMemcpyAsync(dst[t], a + ctx->knn_off[t], bytes[t], cudaMemcpyDeviceToHost,
                                     ctx->stream));
  FGBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FGBD_OK;
}

}  // extern "C"
