// Small device helpers: warp/block reductions, lane masks, last-block tickets.
#pragma once
#include <cstdio>

#include <cuda_runtime.h>
#include <stdint.h>

namespace fgbd {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Device-side bounds checks for debug builds (-DFGBD_DEBUG_BOUNDS=1, used by
// tools/debug_bounds.sh in place of compute-sanitizer): a failed check
// prints its site and traps, so the call fails loudly.
#ifndef FGBD_DEBUG_BOUNDS
#define FGBD_DEBUG_BOUNDS 0
#endif
#if FGBD_DEBUG_BOUNDS
#define FGBD_DCHECK(cond)                                                           \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      printf("FGBD_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
             #cond, (int)blockIdx.x, (int)threadIdx.x);                             \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define FGBD_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// The ELL graph: 6 slots per point of (neighbour, payload), payload = exact
// squared length until the weight pass, then fp32 Gaussian weight bits.
// Storage is one int array, slot pairs interleaved as int4 = (nbr_2p, pay_2p,
// nbr_2p+1, pay_2p+1), pair-major [3][N]: a warp reads 512 contiguous bytes
// per pair and a row is three 16-byte loads.  `nbr` and `pay` are strided
// views of that array (pay = nbr + 1), both indexed by eslot().
struct EllRef {
  int* nbr;
  uint32_t* pay;
};

__device__ __forceinline__ int64_t eslot(int s, int64_t n, int64_t i) {
  return (int64_t)(s >> 1) * 4 * n + 4 * i + 2 * (s & 1);
}

// An ELL neighbour word is the neighbour's ROW (position) in bits 0-30 and,
// in bit 31, whether its ORIGINAL point index is below the row's own -- the
// reference's weighted degree is (sum over j > i) + (sum over j < i) of the
// original indices, whatever order the rows are stored in.
constexpr int kBelowBit = (int)0x80000000u;
__device__ __forceinline__ int ell_j(int v) { return v & 0x7fffffff; }
__device__ __forceinline__ bool ell_below(int v) { return v < 0; }

// Block-wide sum of NV doubles per thread; result valid in thread 0.
// Fixed shuffle tree + fixed warp order => deterministic.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* s_scratch /*[32*NV]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) s_scratch[warp * NV + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double acc = 0.0;
      for (int w = 0; w < nwarps; ++w) acc += s_scratch[w * NV + k];
      v[k] = acc;
    }
  }
  __syncthreads();
}

// "Last block done": every block calls this after publishing its partial;
// returns true (block-uniform) in exactly one block, after all partials are
// visible.  The caller resets *ticket to 0 when finished.
__device__ __forceinline__ bool last_block(unsigned int* ticket, bool* s_flag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned t = atomicAdd(ticket, 1u);
    *s_flag = (t == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (*s_flag) __threadfence();
  return *s_flag;
}

// Like last_block, for a counter shared by `count` blocks.
__device__ __forceinline__ bool last_block_of(unsigned int* ticket, int count, bool* s_flag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned t = atomicAdd(ticket, 1u);
    *s_flag = (t == (unsigned)count - 1);
  }
  __syncthreads();
  if (*s_flag) __threadfence();
  return *s_flag;
}

// 256-bit signal row access (LDG/STG.E.ENL2.256 on sm_100a).  The compiler
// splits a double4 load whose 4th lane is unused into 128 + 64 bits, which
// doubles the L1 wavefronts of a gather; inline PTX keeps it one sector.
__device__ __forceinline__ double4 ld_row(const double4* p) {
  double4 v;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_row(double4* p, double4 v) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z),
               "d"(v.w)
               : "memory");
}

// L2 eviction-priority policies (createpolicy, sm_80+) and hinted accesses.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double4 ld_row_hint(const double4* p, uint64_t pol) {
  double4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
#ifndef FGBD_LF_FARMODE
#define FGBD_LF_FARMODE 0  // far gathers: 0 ld.global.cg, 1 L1::no_allocate, 2 L1::evict_first
#endif
__device__ __forceinline__ double4 ld_row_cg_hint(const double4* p, uint64_t pol) {
  double4 v;
#if FGBD_LF_FARMODE == 1
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p), "l"(pol));
#elif FGBD_LF_FARMODE == 2
  asm volatile("ld.global.L1::evict_first.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p), "l"(pol));
#else
  asm volatile("ld.global.cg.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p), "l"(pol));
#endif
  return v;
}
__device__ __forceinline__ void st_row_hint(double4* p, double4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "d"(v.x),
               "d"(v.y), "d"(v.z), "d"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ int2 ld_slot_hint(const int2* p, uint64_t pol) {
  int2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ int2 ld_int2_hint(const void* p, uint64_t pol) {
  int2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int4 ld_pair_hint(const int2* p, uint64_t pol) {
  int4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// Exact, order-independent sums of doubles v = 0 or v >= 1 (the edge lengths
// sqrt(sqdist) of sigma_g, graph.py:227-233): v * 2^52 is an integer below
// 2^(53 + 74) for v < 2^75, accumulated in 128-bit integers.  Any partition
// of the edges (one GPU, P slab ranks, any grid) gives the same bits.
typedef unsigned __int128 u128;
__device__ __forceinline__ u128 fx52(double v) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  const int eb = (int)((bits >> 52) & 0x7ff);
  if (eb < 1023) return 0;  // only v == 0 occurs (v >= 1 otherwise)
  const unsigned long long mant = (bits & ((1ull << 52) - 1)) | (1ull << 52);
  return (u128)mant << (eb - 1023);
}
__device__ __forceinline__ u128 warp_sum_u128(u128 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long lo = __shfl_xor_sync(kFull, (unsigned long long)v, o);
    const unsigned long long hi = __shfl_xor_sync(kFull, (unsigned long long)(v >> 64), o);
    v += ((u128)hi << 64) | lo;
  }
  return v;
}
// Block-wide sum, valid in thread 0 (s_scratch: 2 x 32 u64).
__device__ __forceinline__ u128 block_sum_u128(u128 v, unsigned long long* s_scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  v = warp_sum_u128(v);
  if (lane == 0) {
    s_scratch[2 * warp] = (unsigned long long)v;
    s_scratch[2 * warp + 1] = (unsigned long long)(v >> 64);
  }
  __syncthreads();
  u128 t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < nwarps; ++w) t += ((u128)s_scratch[2 * w + 1] << 64) | s_scratch[2 * w];
  __syncthreads();
  return t;
}
// The fixed-point sum back to a double (deterministic: a pure function of the bits).
__device__ __forceinline__ double fx52_to_double(u128 s) {
  const double hi = (double)(unsigned long long)(s >> 64), lo = (double)(unsigned long long)s;
  return ldexp(__dadd_rn(ldexp(hi, 64), lo), -52);
}

// RN(a / b) from y = RN(1 / b) (__drcp_rn): q0 = RN(a y), r = a - b q0 (exact
// with FMA), q = RN(q0 + r y) is the correctly rounded quotient for normal
// a, b and a / b (Markstein); the guarded ranges fall back to the IEEE
// division.  Checked bit-identical to a / b on random and edge pairs
// (tools/micro/div_check.c, 3e8 pairs incl. edge ranges).  3 instructions instead of a ~20-instruction
// division when one divisor serves many quotients.
__device__ __forceinline__ double div_rcp(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  if (!(fabs(q0) < 1e300) || (a != 0.0 && fabs(a) < 1e-290)) return __ddiv_rn(a, b);
  const double r = __fma_rn(-b, q0, a);
  return __fma_rn(r, y, q0);
}
__device__ __forceinline__ bool rcp_ok(double b) { return b > 1e-290 && b < 1e290; }

// Shared-memory addresses, L2 prefetch, mbarriers and bulk copies (TMA engine).
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// Grid barrier of a cooperative launch over a zero-initialised word that
// only this launch uses: one release atomic per block (block 0 adds
// 2^31 - (blocks - 1), so the top bit flips exactly when the last block
// arrives), a RELAXED spin, then one acquire fence.  cooperative_groups'
// grid.sync() spins with acquire loads, i.e. an L1 invalidation (CCTL.IVALL)
// per poll, which keeps wiping the L1 of the blocks on the same SM that are
// still working; here each block invalidates once, on leaving.  Measured
// (tools/micro/gridbar.cu, no work between barriers): 1.26 / 1.42 / 1.80 us
// per barrier at 148 / 296 / 444 blocks, against 1.2 us for grid.sync() at
// any of those sizes.  Inside kernels that move data the order flips:
// k_slg with grid.sync() spent ~1 us more per scan phase (B + barrier 4.2 vs
// 3.3 us at 1M), so it keeps this one; k_lf_run keeps grid.sync()
// (FGBD_LF_BAR).
__device__ __forceinline__ void grid_barrier(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int nb = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
    unsigned int old, cur;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(nb) : "memory");
    do {
      asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
    } while (((cur ^ old) & 0x80000000u) == 0);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}


}  // namespace fgbd
