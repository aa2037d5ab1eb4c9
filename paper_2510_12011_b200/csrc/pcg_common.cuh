// pcg_common.cuh -- device building blocks shared by the persistent PCG kernel
// (pcg.cu) and the split-phase, partitioned PCG kernels (pcg_split.cu):
// PTX helpers (mbarrier, TMA bulk copies), deterministic reductions, the
// per-warp slice pipeline and the SELL row products.
#pragma once

#include <cooperative_groups.h>

#include "internal.h"

namespace cg = cooperative_groups;

namespace tcb {


#ifndef TCB_DIRECT_MINB
#define TCB_DIRECT_MINB (2048 / TCB_CG_THREADS)  // CTAs/SM of the direct variant: 32 registers, 64 warps/SM
#endif
constexpr int kWMax = 16;                               // widest TMA-staged slice
constexpr int kValBytes = kWMax * kSellC * 8;           // 4 KB of values
constexpr int kStageBytes = kWMax * kSellC * (8 + 4);   // + 2 KB of column indices
constexpr int kStages = 2;
constexpr int kWarpSmem = kStages * kStageBytes;        // 12 KB per warp
constexpr int kCgSmem = kCgWarps * kWarpSmem;           // 12 KB per warp: 16 warps per SM

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 1-D TMA bulk copy global -> shared, completion counted on the mbarrier.
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// Sum of v over the CTA, result valid in every thread.
__device__ __forceinline__ double2 block_sum2(double2 v, double2* sh) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_sum2(v);
  __syncthreads();  // sh may still be read from a previous call
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double2 t = make_double2(0.0, 0.0);
  if (lane < (int)(blockDim.x >> 5)) t = sh[lane];
  t = warp_sum2(t);  // every warp reduces the per-warp values identically
  return t;
}

// Grid-wide deterministic sum.  buf holds gridDim.x slots.
__device__ __forceinline__ double2 grid_sum2(double2 v, double2* buf, double2* sh,
                                             cg::grid_group& grid) {
  double2 b = block_sum2(v, sh);
  if (threadIdx.x == 0) buf[blockIdx.x] = b;
  grid.sync();
  double2 acc = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < (int)gridDim.x; t += blockDim.x) {
    double2 u = buf[t];
    acc.x += u.x;
    acc.y += u.y;
  }
  return block_sum2(acc, sh);
}

// ------------------------------------------------------------------ slice pipeline
// One warp walks its slices s = gw, gw + nw, ... ; slice s's values and column
// indices are staged in stage (j mod kStages) by lane 0's TMA copies issued
// kStages slices ahead.  Slices wider than kWMax (irregular meshes) fall back
// to direct loads.
struct SlicePipe {
  char* buf;
  uint64_t* bar;
  uint32_t phase;  // bit st = parity of the next completion of stage st
  uint64_t pol;
};

__device__ __forceinline__ void slice_bounds(const int64_t* sp, int s, int64_t& base, int& w) {
  base = __ldg(sp + s);
  w = (int)((__ldg(sp + s + 1) - base) >> 5);
}

__device__ __forceinline__ void pipe_issue(SlicePipe& P, int st, const double* A, const int* col,
                                           const int64_t* sp, int s, int ns) {
  if (s >= ns) return;
  int64_t base;
  int w;
  slice_bounds(sp, s, base, w);
  if (w <= 0 || w > kWMax) return;
  char* dst = P.buf + st * kStageBytes;
  const uint32_t bv = (uint32_t)w * kSellC * 8, bc = (uint32_t)w * kSellC * 4;
  mbar_expect_tx(P.bar + st, bv + bc);
  tma_load(dst, A + base, bv, P.bar + st, P.pol);
  tma_load(dst + kValBytes, col + base, bc, P.bar + st, P.pol);
}

// f(i, base, w, staged, As, Cs) for every slice of this warp (i = this lane's row).
template <bool TMA, class F>
__device__ __forceinline__ void for_slices(SlicePipe& P, const int64_t* sp, const double* A,
                                           const int* col, int ns, int gw, int nw, int lane, F&& f);

template <class F>
__device__ __forceinline__ void for_slices_tma(SlicePipe& P, const int64_t* sp, const double* A,
                                           const int* col, int ns, int gw, int nw, int lane, F&& f) {
  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < kStages; ++st) pipe_issue(P, st, A, col, sp, gw + st * nw, ns);
  }
  int st = 0;
  for (int s = gw; s < ns; s += nw) {
    int64_t base;
    int w;
    slice_bounds(sp, s, base, w);
    const bool staged = w > 0 && w <= kWMax;
    if (staged) {
      mbar_wait(P.bar + st, (P.phase >> st) & 1u);
      P.phase ^= 1u << st;
    }
    const char* sb = P.buf + st * kStageBytes;
    f((int64_t)s * kSellC + lane, base, w, staged, reinterpret_cast<const double*>(sb),
      reinterpret_cast<const int*>(sb + kValBytes));
    __syncwarp();
    if (lane == 0) {
      fence_proxy_async();  // generic-proxy reads of the stage before the async overwrite
      pipe_issue(P, st, A, col, sp, s + kStages * nw, ns);
    }
    st = (st + 1 == kStages) ? 0 : st + 1;
  }
}

// TCB_L2PF_MAT = D > 0 (experiment): lane 0 of a warp asks the TMA unit to
// prefetch into L2 the values and column indices of the slice it will process
// D rounds later (cp.async.bulk.prefetch.L2, two instructions per slice), so the
// streamed matrix loads of the direct variant find the data in L2 and the
// dependent index -> gather chain starts sooner.
#ifndef TCB_L2PF_MAT
#define TCB_L2PF_MAT 0
#endif
__device__ __forceinline__ void l2_prefetch_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_slice(const int64_t* sp, const double* A, const int* col, int s, int ns) {
  if (s >= ns) return;
  const int64_t base = __ldg(sp + s), end = __ldg(sp + s + 1);
  const uint32_t nv = (uint32_t)(end - base);
  if (nv == 0) return;
  l2_prefetch_bulk(A + base, nv * 8u);      // 16-byte multiples: slices hold 32 k slots
  l2_prefetch_bulk(col + base, nv * 4u);
}

template <bool TMA, class F>
__device__ __forceinline__ void for_slices(SlicePipe& P, const int64_t* sp, const double* A,
                                           const int* col, int ns, int gw, int nw, int lane, F&& f) {
  if (TMA) {
    for_slices_tma(P, sp, A, col, ns, gw, nw, lane, f);
  } else {
#if TCB_L2PF_MAT > 0
    if (lane == 0)
      for (int d = 0; d < TCB_L2PF_MAT; ++d) prefetch_slice(sp, A, col, gw + d * nw, ns);
#endif
    for (int s = gw; s < ns; s += nw) {
#if TCB_L2PF_MAT > 0
      if (lane == 0) prefetch_slice(sp, A, col, s + TCB_L2PF_MAT * nw, ns);
#endif
      int64_t base;
      int w;
      slice_bounds(sp, s, base, w);
      f((int64_t)s * kSellC + lane, base, w, false, (const double*)nullptr, (const int*)nullptr);
    }
  }
}

// TCB_STAGED_BATCH = 1: the staged row product issues every gather of a row at
// once (NB slots in flight, as the latency variant 4 does from global memory):
// with values and indices already in shared memory the row costs one L2 round
// trip.  0: an unroll-8 slot loop.
#ifndef TCB_STAGED_BATCH
#define TCB_STAGED_BATCH 0
#endif
template <bool FIRST, int NB>
__device__ __forceinline__ double row_Ap_staged_batch(int w, int lane, const double* As, const int* Cs,
                                                      const double* z, const double* pold, double beta) {
  double sum = 0.0;
#pragma unroll 1
  for (int k0 = 0; k0 < w; k0 += NB) {
    double av[NB], g[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int kk = min(k0 + j, w - 1);
      const int64_t t = sell_slot(0, w, kk, lane);
      const int c = Cs[t];
      av[j] = As[t];
      g[j] = FIRST ? z[c] : z[c] + beta * pold[c];
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (k0 + j < w) sum += av[j] * g[j];
  }
  return sum;
}

// q_i = sum_k A_ik p_c, p_c = z_c (+ beta pold_c); slots accumulated in
// ascending order (the CSR order).  Staged: operands from shared memory.
template <bool FIRST>
__device__ __forceinline__ double row_Ap_staged(int w, int lane, const double* As, const int* Cs,
                                                const double* z, const double* pold, double beta) {
#if TCB_STAGED_BATCH
  if (w <= 8) return row_Ap_staged_batch<FIRST, 8>(w, lane, As, Cs, z, pold, beta);
  return row_Ap_staged_batch<FIRST, kWMax>(w, lane, As, Cs, z, pold, beta);
#endif
  double sum = 0.0;
#pragma unroll 8
  for (int k = 0; k < w; ++k) {
    const int64_t t = sell_slot(0, w, k, lane);
    const int c = Cs[t];
    const double g = FIRST ? z[c] : z[c] + beta * pold[c];
    sum += As[t] * g;
  }
  return sum;
}

// Streamed matrix loads: evict-first (default: the matrix of a large system
// is read once per iteration and never fits in L2) or cached (experiment:
// TCB_MATRIX_LOAD = 1, __ldg) for systems whose matrix could stay in L2.
#ifndef TCB_MATRIX_LOAD
#define TCB_MATRIX_LOAD 0
#endif
template <class T>
__device__ __forceinline__ T ld_mat(const T* p) {
#if TCB_MATRIX_LOAD == 1
  return __ldg(p);
#else
  return __ldcs(p);
#endif
}

// L2-resident matrix (variant 3, systems whose matrix fits in L2): values and
// column indices loaded with an L2 evict-last policy so they survive the
// vector traffic between iterations; everything else keeps its default policy.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_keep(const double* p) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(policy_evict_last()));
  return v;
}
__device__ __forceinline__ int ld_keep(const int* p) {
  int v;
  asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy_evict_last()));
  return v;
}

// Column index of slot t (slot row k) of one slice: either the plain int32
// array, or (compressed slices) a per-(slice, k) int32 base, broadcast to the
// warp, plus a 16-bit offset per slot.
struct ColIdx {
  const int* c32;
  const uint16_t* c16;  // null: uncompressed slice
  const int* kb;
  __device__ __forceinline__ int operator()(int64_t t, int k) const {
    return c16 ? __ldg(kb + k) + (int)ld_mat(c16 + t) : ld_mat(c32 + t);
  }
};

template <bool COMP>
__device__ __forceinline__ ColIdx col_of(const CgArgs& a, int64_t i, int64_t base) {
  ColIdx ci;
  ci.c32 = a.col;
  ci.c16 = nullptr;
  ci.kb = nullptr;
  if (COMP && __ldg(a.fmt + (i >> 5)) == 0) {
    ci.c16 = a.col16;
    ci.kb = a.kbase + (base >> 5);
  }
  return ci;
}

// Unroll of the direct variant's slot loop (experiment; 4 = default).
#ifndef TCB_S_UNROLL
#define TCB_S_UNROLL 4
#endif
// TCB_COMP_SHFL = 1 (experiment): variant 2's per-(slice, slot) column bases are
// loaded once per slice (lane k holds slot k's) and broadcast with a shuffle,
// instead of one broadcast load per slot.
#ifndef TCB_COMP_SHFL
#define TCB_COMP_SHFL 0
#endif
#ifndef TCB_ROW_BATCH
#define TCB_ROW_BATCH 0   // 0: unroll-4 loop; N > 0: slots in batches of N with clamped indices
#endif
template <bool FIRST>
__device__ __forceinline__ double row_Ap_keep(int64_t base, int w, int lane, const ColIdx& ci,
                                              const double* A, const double* z, const double* pold,
                                              double beta) {
  double sum = 0.0;  // variant 3: L2-resident matrix, plain int32 indices
#pragma unroll 4
  for (int k = 0; k < w; ++k) {
    const int64_t t = sell_slot(base, w, k, lane);
    const int c = ld_keep(ci.c32 + t);
    const double g = FIRST ? z[c] : z[c] + beta * pold[c];
    sum += ld_keep(A + t) * g;
  }
  return sum;
}

template <bool FIRST>
__device__ __forceinline__ double row_Ap_stream(int64_t base, int w, int lane, const ColIdx& ci,
                                                const double* A, const double* z, const double* pold,
                                                double beta) {
  double sum = 0.0;
#if TCB_ROW_BATCH > 0
  // every load of a batch in flight together; slots past the row end reload its
  // last slot (no remainder loop), accumulation in slot order
  constexpr int NB = TCB_ROW_BATCH;
#pragma unroll 1
  for (int k0 = 0; k0 < w; k0 += NB) {
    double av[NB], g[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int kk = min(k0 + j, w - 1);
      const int64_t t = sell_slot(base, w, kk, lane);
      const int c = ci(t, kk);
      av[j] = ld_mat(A + t);
      g[j] = FIRST ? z[c] : z[c] + beta * pold[c];
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (k0 + j < w) sum += av[j] * g[j];
  }
#else
#ifndef TCB_PAIRS_S
#define TCB_PAIRS_S 1   // 16-byte pair loads in the q = A p product (else per-slot loads)
#endif
#if TCB_SELL_PAIRS && TCB_PAIRS_S
  if (!ci.c16) {  // slot pairs: one 16-byte value load + one 8-byte index load per pair
    const double2* A2 = reinterpret_cast<const double2*>(A + base) + lane;
    const int2* C2 = reinterpret_cast<const int2*>(ci.c32 + base) + lane;
    const int np = w >> 1;
#pragma unroll 2
    for (int j = 0; j < np; ++j) {
      const double2 av = ld_mat(A2 + 32 * j);
      const int2 c = ld_mat(C2 + 32 * j);
      const double g0 = FIRST ? z[c.x] : z[c.x] + beta * pold[c.x];
      const double g1 = FIRST ? z[c.y] : z[c.y] + beta * pold[c.y];
      sum += av.x * g0;
      sum += av.y * g1;
    }
    if (w & 1) {
      const int64_t t = base + (int64_t)kSellC * (w - 1) + lane;
      const int c = ld_mat(ci.c32 + t);
      sum += ld_mat(A + t) * (FIRST ? z[c] : z[c] + beta * pold[c]);
    }
    return sum;
  }
#endif
#if TCB_COMP_SHFL
  if (ci.c16 && w <= kSellC) {  // variant 2: the slice's per-slot bases held one per lane, broadcast by shuffle
    const int kbl = lane < w ? __ldg(ci.kb + lane) : 0;
#pragma unroll 4
    for (int k = 0; k < w; ++k) {
      const int64_t t = sell_slot(base, w, k, lane);
      const int c = __shfl_sync(0xffffffffu, kbl, k) + (int)ld_mat(ci.c16 + t);
      const double g = FIRST ? z[c] : z[c] + beta * pold[c];
      sum += ld_mat(A + t) * g;
    }
    return sum;
  }
#endif
#if TCB_S_UNROLL == 2
#pragma unroll 2
#elif TCB_S_UNROLL == 3
#pragma unroll 3
#elif TCB_S_UNROLL == 8
#pragma unroll 8
#else
#pragma unroll 4
#endif
  for (int k = 0; k < w; ++k) {
    const int64_t t = sell_slot(base, w, k, lane);
    const int c = ci(t, k);
    const double g = FIRST ? z[c] : z[c] + beta * pold[c];
    sum += ld_mat(A + t) * g;
  }
#endif
  return sum;
}

#ifndef TCB_BATCH_NB
#define TCB_BATCH_NB 16   // slots in flight per row in variant 4 (measured: 16 at 1 CTA/SM best)
#endif
// Latency variant (VAR 4): all slots of a row in batches of NB loads in flight
// (values, indices, then the gathers), slots past the row end reload its last
// slot; accumulation in slot order.  Needs ~100 registers: one 16-warp CTA per SM.
// TCB_BATCH_MATLOAD (experiment): the latency variant's matrix loads -- 0
// evict-first streaming (default), 1 cached (__ldg), 2 L2 evict-last (for
// mid-size systems whose matrix could stay in the 126 MB L2 across iterations).
#ifndef TCB_BATCH_MATLOAD
#define TCB_BATCH_MATLOAD 0
#endif
template <class T>
__device__ __forceinline__ T ld_bmat(const T* p) {
#if TCB_BATCH_MATLOAD == 1
  return __ldg(p);
#elif TCB_BATCH_MATLOAD == 2
  return ld_keep(p);
#else
  return ld_mat(p);
#endif
}
template <bool FIRST, int NB>
__device__ __forceinline__ double row_Ap_batch(int64_t base, int w, int lane, const int* col,
                                               const double* A, const double* z, const double* pold,
                                               double beta) {
  double sum = 0.0;
#pragma unroll 1
  for (int k0 = 0; k0 < w; k0 += NB) {
    double av[NB], g[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int kk = min(k0 + j, w - 1);
      const int64_t t = sell_slot(base, w, kk, lane);
      const int c = ld_bmat(col + t);
      av[j] = ld_bmat(A + t);
      g[j] = FIRST ? z[c] : z[c] + beta * pold[c];
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (k0 + j < w) sum += av[j] * g[j];
  }
  return sum;
}

// Narrow slices (w <= 8: triangle surface meshes, ~7 slots per row) take a batch
// of 8 instead of NB (fewer clamped reloads); TCB_BATCH_SMALL = 0 disables.
#ifndef TCB_BATCH_SMALL
#define TCB_BATCH_SMALL 1
#endif
template <bool FIRST>
__device__ __forceinline__ double row_Ap_batch_w(int64_t base, int w, int lane, const int* col,
                                                 const double* A, const double* z, const double* pold,
                                                 double beta) {
  if (TCB_BATCH_SMALL && w <= 8) return row_Ap_batch<FIRST, 8>(base, w, lane, col, A, z, pold, beta);
  return row_Ap_batch<FIRST, TCB_BATCH_NB>(base, w, lane, col, A, z, pold, beta);
}

// r_0 row (A u' - K v') of the latency variant: NB slots in flight at once.
template <int NB>
__device__ __forceinline__ double row_rhs_batch(int64_t base, int w, int lane, const int* col,
                                                const double* A, const double* K, const double* up,
                                                const double* vp) {
  double sum = 0.0;
#pragma unroll 1
  for (int k0 = 0; k0 < w; k0 += NB) {
    double av[NB], kv[NB], gu[NB], gv[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int kk = min(k0 + j, w - 1);
      const int64_t t = sell_slot(base, w, kk, lane);
      const int c = ld_mat(col + t);
      av[j] = ld_mat(A + t);
      kv[j] = ld_mat(K + t);
      gu[j] = up[c];
      gv[j] = vp[c];
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (k0 + j < w) sum += av[j] * gu[j] - kv[j] * gv[j];
  }
  return sum;
}

template <bool FIRST, bool KEEP = false>
__device__ __forceinline__ double row_Ap_direct(int64_t base, int w, int lane, const ColIdx& ci,
                                                const double* A, const double* z, const double* pold,
                                                double beta) {
  if constexpr (KEEP) return row_Ap_keep<FIRST>(base, w, lane, ci, A, z, pold, beta);
  else return row_Ap_stream<FIRST>(base, w, lane, ci, A, z, pold, beta);
}

// r_0 row of Eq. 3 as A u' - K v', slots in CSR order, plain
// int32 indices, direct evict-first loads (slot pairs when TCB_SELL_PAIRS).
__device__ __forceinline__ double row_rhs_direct(int64_t base, int w, int lane, const int* col,
                                                 const double* A, const double* K, const double* up,
                                                 const double* vp) {
  double sum = 0.0;
#if TCB_SELL_PAIRS
  const double2* A2 = reinterpret_cast<const double2*>(A + base) + lane;
  const double2* K2 = reinterpret_cast<const double2*>(K + base) + lane;
  const int2* C2 = reinterpret_cast<const int2*>(col + base) + lane;
  const int np = w >> 1;
#pragma unroll 2
  for (int j = 0; j < np; ++j) {
    const double2 av = ld_mat(A2 + 32 * j), kv = ld_mat(K2 + 32 * j);
    const int2 c = ld_mat(C2 + 32 * j);
    sum += av.x * up[c.x] - kv.x * vp[c.x];
    sum += av.y * up[c.y] - kv.y * vp[c.y];
  }
  if (w & 1) {
    const int64_t t = base + (int64_t)kSellC * (w - 1) + lane;
    const int c = ld_mat(col + t);
    sum += ld_mat(A + t) * up[c] - ld_mat(K + t) * vp[c];
  }
#else
#pragma unroll 4
  for (int k = 0; k < w; ++k) {
    const int64_t t = base + (int64_t)k * kSellC + lane;
    const int c = ld_mat(col + t);
    sum += ld_mat(A + t) * up[c] - ld_mat(K + t) * vp[c];
  }
#endif
  return sum;
}

}  // namespace tcb
