// pcg.cu -- the CG path of one monodomain step as ONE persistent cooperative
// kernel per solve: right-hand side (Eq. 3) and Algorithm 1
// with the Jacobi preconditioner, all scalars on device.
//
// Data flow per iteration (two phases, two grid barriers):
//   S: p_it = z + beta p_{it-1} is formed on the fly for every gathered column,
//      q = A p_it (SELL-32, warp per slice, thread per row), the deferred
//      x += alpha_{it-1} p_{it-1}, and the partial sums of p.q.
//   U: alpha = rho / p.q;  z -= alpha q / diag(A) (z-form: r = diag(A) z is
//      not stored);  partials r.z = sum z^2 diag(A), z.z;
//      then every CTA evaluates the stopping test of Alg. 1 identically.
// Memory pipelines (tc_config.pcg_variant, measured side
// by side): 0 direct, 1 TMA-staged, 2 16-bit offsets, 3 L2-kept matrix, 4 every
// slot of a row in flight (mid-size), 5 the CUDA-graph engine (pcg_graph.cu), and
// 6 the opt-in single-reduction recurrence (pcg1r_kernel below).  The first two:
//  * DIRECT (default, variant 0): 32 registers/thread, 64 warps/SM; every warp
//    streams its slice's values and column indices with evict-first loads and
//    gathers the vectors from L1/L2; latency is hidden by occupancy.
//    Variant 2 = the same with 16-bit column offsets (fewer bytes, more
//    instructions; measured slower, kept for the record).
//  * TMA: the streamed matrix (values and column indices of a slice are two
//    contiguous runs) is staged into shared memory by TMA bulk copies
//    (cp.async.bulk + mbarrier, L2 evict-first) two slices ahead per warp;
//    96 KB smem per CTA limits it to 16 warps/SM.
// Reductions are deterministic: per-CTA partials in a fixed slot, then every
// CTA sums all partials in the same order (bitwise-identical scalars => all
// CTAs take the same branch).
#include <algorithm>

#include "pcg_common.cuh"

namespace tcb {

// ------------------------------------------------------------------ kernels
// VAR 0: direct loads, int32 indices (default), 1: TMA-staged, 2: direct loads + 16-bit indices,
// 3: direct loads with the matrix kept in L2 (evict-last; systems whose A + col fit in L2),
// 4: latency variant for systems with few slices per resident warp: every slot
//    of a row in flight at once (row_Ap_batch), one 16-warp CTA per SM
#ifndef TCB_VEC_U
#define TCB_VEC_U 0   // 1: U phase and final x update over 16-byte row pairs (measured slower)
#endif
// TCB_XMERGE = 1 (default): the deferred x update runs every other iteration, adding the
// two pending terms in their original order, x = (x + a_{it-2} p_{it-2}) +
// a_{it-1} p_{it-1} -- bitwise the sequential result -- so x is read and written
// once per two iterations (plus one read of p_{it-2}): 4n bytes per iteration less.
// Measured (profiles/r02o_exp_xmerge.txt, PCG-path frac): 20 M MS 0.873 -> 0.889,
// 10 M TT2006 0.873-0.878 -> 0.880-0.887, BiV 3 M 0.798-0.802 -> 0.793-0.796.
#ifndef TCB_XMERGE
#define TCB_XMERGE 1
#endif
#if TCB_VEC_U && TCB_XMERGE
#error "TCB_VEC_U has only the per-iteration x update: build it with -DTCB_XMERGE=0"
#endif
#if TCB_VEC_U && TCB_ZFORM
#error "TCB_VEC_U has only the r-form U phase: build it with -DTCB_ZFORM=0"
#endif
template <bool ODD>
struct ParityTag {  // compile-time iteration parity (bool(tag) folds to a constant)
  __device__ constexpr operator bool() const { return ODD; }
};
#ifndef TCB_S_PARITY
#define TCB_S_PARITY 1   // the S phase compiled once per p-buffer parity (0: one copy, runtime parity)
#endif
#ifndef TCB_DIRECT_UU
#define TCB_DIRECT_UU 1   // slices per warp pass in the direct variants' U phase and final x update
#endif
#ifndef TCB_BATCH_UU
#define TCB_BATCH_UU 1    // slices per warp pass in variant 4's U phase (measured 1 < 2 < 4)
#endif
#define TCB_MINB(VAR) ((VAR) == 1 ? (512 / TCB_CG_THREADS > 0 ? 512 / TCB_CG_THREADS : 1) : \
                       (VAR) == 4 ? 1 : TCB_DIRECT_MINB)

__device__ __forceinline__ void setup_pipe(SlicePipe& P, char* smem, uint64_t* bars, int warp, int lane) {
  P.buf = smem + warp * kWarpSmem;
  P.bar = bars;
  P.phase = 0;
  P.pol = policy_evict_first();
  if (lane == 0) {
    for (int st = 0; st < kStages; ++st) mbar_init(P.bar + st, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
}

// r_0 = b - A x_0 (MODE 0) or A u' - K v' (MODE 1, == b - A x_0 with Eq. 3's b;
// DESIGN.md "RHS"), z_0 = r_0 / diag(A), and per-CTA partials of r.z, z.z.
// Same grid as the PCG kernel that consumes the partials.
template <int MODE, int VAR>
#ifndef TCB_RHS_BATCH_NB
#define TCB_RHS_BATCH_NB 16  // slots in flight per row in variant 4's RHS (0: direct loop; measured 16 > 8 > 4 > 0)
#endif
__global__ void __launch_bounds__(kCgThreads, VAR == 1 ? TCB_MINB(1) : VAR == 4 ? 1 : (1024 / TCB_CG_THREADS > 0 ? 1024 / TCB_CG_THREADS : 1)) rhs_kernel(CgArgs a) {
  constexpr bool TMA = VAR == 1;
  constexpr bool COMP = VAR == 2;
  constexpr bool KEEP = VAR == 3;
  extern __shared__ __align__(128) char smem[];
  __shared__ double2 sh[kCgWarps];
  __shared__ __align__(8) uint64_t bars[TMA ? kCgWarps : 1][kStages];
  if (a.flags[0]) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * kCgWarps + warp;
  const int nw = gridDim.x * kCgWarps;
  const double* __restrict__ Av = a.A;
  SlicePipe P;
  if (TMA) setup_pipe(P, smem, bars[TMA ? warp : 0], warp, lane);
  double2 acc = make_double2(0.0, 0.0);
  for_slices<TMA>(P, a.slice_ptr, Av, a.col, a.s1, a.s0 + gw, nw, lane,
             [&](int64_t i, int64_t base, int w, bool staged, const double* As, const int* Cs) {
               double sum = 0.0;
               if (MODE == 1) {
                 const double* __restrict__ Kv = a.K;
                 const ColIdx ci = col_of<COMP>(a, i, base);
                 if (VAR == 4 && TCB_RHS_BATCH_NB > 0) {
                   sum = (TCB_BATCH_SMALL && w <= 8)
                             ? row_rhs_batch<8>(base, w, lane, a.col, Av, Kv, a.up, a.vp)
                             : row_rhs_batch<(TCB_RHS_BATCH_NB > 0 ? TCB_RHS_BATCH_NB : 1)>(base, w, lane, a.col, Av,
                                                                                             Kv, a.up, a.vp);
                 } else if (KEEP) {
#pragma unroll 4
                   for (int k = 0; k < w; ++k) {
                     const int64_t t = sell_slot(base, w, k, lane);
                     const int c = ld_keep(a.col + t);
                     sum += ld_keep(Av + t) * a.up[c] - ld_mat(Kv + t) * a.vp[c];
                   }
                 } else if (TCB_SELL_PAIRS && !staged && !ci.c16) {  // slot pairs: 16-byte value loads
                   const double2* A2 = reinterpret_cast<const double2*>(Av + base) + lane;
                   const double2* K2 = reinterpret_cast<const double2*>(Kv + base) + lane;
                   const int2* C2 = reinterpret_cast<const int2*>(a.col + base) + lane;
                   const int np = w >> 1;
#pragma unroll 2
                   for (int j = 0; j < np; ++j) {
                     const double2 av = ld_mat(A2 + 32 * j), kv = ld_mat(K2 + 32 * j);
                     const int2 c = ld_mat(C2 + 32 * j);
                     sum += av.x * a.up[c.x] - kv.x * a.vp[c.x];
                     sum += av.y * a.up[c.y] - kv.y * a.vp[c.y];
                   }
                   if (w & 1) {
                     const int64_t t = base + (int64_t)kSellC * (w - 1) + lane;
                     const int c = ld_mat(a.col + t);
                     sum += ld_mat(Av + t) * a.up[c] - ld_mat(Kv + t) * a.vp[c];
                   }
                 } else {
#pragma unroll 4
                   for (int k = 0; k < w; ++k) {
                     const int64_t t = sell_slot(base, w, k, lane);
                     const int64_t ts = sell_slot(0, w, k, lane);
                     const int c = staged ? Cs[ts] : ci(t, k);
                     const double av = staged ? As[ts] : ld_mat(Av + t);
                     sum += av * a.up[c] - ld_mat(Kv + t) * a.vp[c];
                   }
                 }
               } else {
                 const double ax = staged ? row_Ap_staged<true>(w, lane, As, Cs, a.x, nullptr, 0.0)
                                          : row_Ap_direct<true, KEEP>(base, w, lane, col_of<COMP>(a, i, base), Av, a.x, nullptr, 0.0);
                 sum = a.b[i] - ax;
               }
               const double zi = __ldg(a.dinv + i) * sum;
               if (a.store_r) a.r[i] = sum;
               a.z[i] = zi;
               acc.x += sum * zi;
               acc.y += zi * zi;
             });
  const double2 b = block_sum2(acc, sh);
  if (threadIdx.x == 0) a.part[blockIdx.x] = b;
}

// Variant 4's RHS as the first phase of the cooperative kernel (fuse_rhs): the
// batched row product r_0 = A u' - K v', z_0, per-CTA partials, grid barrier.
__device__ __forceinline__ void rhs_phase_batch(const CgArgs& a, int gw, int nw, int lane, double2* sh,
                                                cg::grid_group& grid) {
  const int64_t* __restrict__ sp = a.slice_ptr;
  double2 acc0 = make_double2(0.0, 0.0);
  for (int s = a.s0 + gw; s < a.s1; s += nw) {
    const int64_t base = __ldg(sp + s);
    const int w = (int)((__ldg(sp + s + 1) - base) >> 5);
    const int64_t i = (int64_t)s * kSellC + lane;
    const double sum = (TCB_BATCH_SMALL && w <= 8)
                           ? row_rhs_batch<8>(base, w, lane, a.col, a.A, a.K, a.up, a.vp)
                           : row_rhs_batch<(TCB_RHS_BATCH_NB > 0 ? TCB_RHS_BATCH_NB : 1)>(base, w, lane, a.col, a.A,
                                                                                           a.K, a.up, a.vp);
    const double zi = __ldg(a.dinv + i) * sum;
    if (a.store_r) a.r[i] = sum;
    a.z[i] = zi;
    acc0.x += sum * zi;
    acc0.y += zi * zi;
  }
  const double2 b0 = block_sum2(acc0, sh);
  if (threadIdx.x == 0) a.part[blockIdx.x] = b0;
  grid.sync();
}

// Algorithm 1's loop from r_0, z_0 and the RHS kernel's partials.
template <int MODE, int VAR>
__global__ void __launch_bounds__(kCgThreads, TCB_MINB(VAR)) pcg_kernel(CgArgs a) {
  constexpr bool TMA = VAR == 1;
  constexpr bool COMP = VAR == 2;
  constexpr bool KEEP = VAR == 3;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) char smem[];
  __shared__ double2 sh[kCgWarps];
  __shared__ __align__(8) uint64_t bars[TMA ? kCgWarps : 1][kStages];
  if (a.flags[0]) return;  // context aborted earlier: uniform across the grid

  constexpr bool BATCH = VAR == 4;
  constexpr int UU = TMA ? 4 : BATCH ? TCB_BATCH_UU : TCB_DIRECT_UU;  // slices per warp pass in the streaming phases
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * kCgWarps + warp;
  const int nw = gridDim.x * kCgWarps;
  const int32_t ns = a.nslices;
  const int64_t* __restrict__ sp = a.slice_ptr;
  const int* __restrict__ col = a.col;
  const double* __restrict__ Av = a.A;
  const double* __restrict__ dinv = a.dinv;
  double2* partA = a.part;
  double2* partB = a.part + gridDim.x;

  SlicePipe P;
  if (TMA) setup_pipe(P, smem, bars[TMA ? warp : 0], warp, lane);
  // streaming phases over row pairs when every vector is 16-byte aligned
  const int64_t n2 = (int64_t)ns * (kSellC / 2);
  const bool vec2 = !TMA && TCB_VEC_U &&
                    ((((uintptr_t)a.r) | ((uintptr_t)a.z) | ((uintptr_t)a.q) | ((uintptr_t)dinv) |
                      ((uintptr_t)a.x) | ((uintptr_t)a.p0) | ((uintptr_t)a.p1)) & 15) == 0;

  // ---- variant 4 with fuse_rhs: the RHS phase here (rhs_kernel's batched row
  // product), then a grid barrier -- one launch and one kernel boundary per
  // solve fewer (mid-size systems are launch-latency sensitive) --------------
  if constexpr (BATCH && MODE == 1) {
    if (a.fuse_rhs) rhs_phase_batch(a, gw, nw, lane, sh, grid);
  }
  // ---- rho_0 = r.z, ||z_0|| from the RHS kernel's per-CTA partials ------------
  double2 tot;
  {
    double2 acc0 = make_double2(0.0, 0.0);
    for (int t = threadIdx.x; t < a.n_rpart; t += blockDim.x) {
      const double2 u = a.rpart[t];
      acc0.x += u.x;
      acc0.y += u.y;
    }
    tot = block_sum2(acc0, sh);
  }
  double2 acc;
  double rho = tot.x;
  double zeta = sqrt(tot.y);
  double zref = zeta;
  int it = 0;
  int conv = 0, nan = 0;
  if (isnan(rho) || isnan(zeta)) nan = 1;
  if (!nan && zeta < a.eps_a) conv = 1;  // reading C4: return x0

  double alpha = 0.0, beta = 0.0, alpha_prev = 0.0;
  bool last_valid = false;
  if (!nan && !conv) {
    for (it = 0; it < a.max_iters;) {
      // ---- S: p = z + beta p_old (on the fly), q = A p, x += alpha_prev p_old
      acc = make_double2(0.0, 0.0);
      double* __restrict__ pnew = (it & 1) ? a.p1 : a.p0;   // p_it
      const double* __restrict__ pold = (it & 1) ? a.p0 : a.p1;  // p_{it-1}
      if (it == 0) {
        for_slices<TMA>(P, sp, Av, col, ns, gw, nw, lane,
                   [&](int64_t i, int64_t base, int w, bool staged, const double* As, const int* Cs) {
                     const double pi = a.z[i];
                     const double sum = staged ? row_Ap_staged<true>(w, lane, As, Cs, a.z, nullptr, 0.0)
                                      : BATCH ? row_Ap_batch_w<true>(base, w, lane, col, Av, a.z, nullptr, 0.0)
                                               : row_Ap_direct<true, KEEP>(base, w, lane, col_of<COMP>(a, i, base), Av, a.z, nullptr, 0.0);
                     pnew[i] = pi;
                     a.q[i] = sum;
                     acc.x += pi * sum;
                   });
      } else {
        // S of iteration it >= 1 with p_it -> pn, p_{it-1} -> po_ (TCB_S_PARITY: one
        // copy per parity, so both are kernel-parameter pointers, not registers)
        auto s_iter = [&](double* __restrict__ pnew, const double* __restrict__ pold, auto odd) {
        for_slices<TMA>(P, sp, Av, col, ns, gw, nw, lane,
                   [&](int64_t i, int64_t base, int w, bool staged, const double* As, const int* Cs) {
                     const double po = pold[i];
                     const double pi = a.z[i] + beta * po;
#if TCB_XMERGE
                     if (!bool(odd)) {   // even it >= 2: p_{it-2} (still in pnew) and p_{it-1}, in order
                       const double xi = a.x[i], p2 = pnew[i];
                       a.x[i] = (xi + alpha_prev * p2) + alpha * po;
                     }
#else
                     const double xi = a.x[i];
                     a.x[i] = xi + alpha * po;
#endif
                     const double sum = staged ? row_Ap_staged<false>(w, lane, As, Cs, a.z, pold, beta)
                                      : BATCH ? row_Ap_batch_w<false>(base, w, lane, col, Av, a.z, pold, beta)
                                               : row_Ap_direct<false, KEEP>(base, w, lane, col_of<COMP>(a, i, base), Av, a.z, pold, beta);
                     pnew[i] = pi;
                     a.q[i] = sum;
                     acc.x += pi * sum;
                   });
        };
        if (TCB_S_PARITY) {
          if (it & 1) s_iter(a.p1, a.p0, ParityTag<true>{});
          else s_iter(a.p0, a.p1, ParityTag<false>{});
        } else {
          s_iter(pnew, pold, (bool)(it & 1));
        }
      }
      last_valid = true;
      tot = grid_sum2(acc, partB, sh, grid);
      const double pq = tot.x;
      if (isnan(pq)) { nan = 1; break; }
      alpha_prev = alpha;
      alpha = rho / pq;                                   // alpha_k = rho_k / p.q
      // ---- U: r -= alpha q, z = r / d, partials of r.z and z.z (UU slices / warp pass)
      acc = make_double2(0.0, 0.0);
      if (vec2) {  // row pairs: 16-byte loads and stores
        double2* __restrict__ r2 = reinterpret_cast<double2*>(a.r);
        double2* __restrict__ z2 = reinterpret_cast<double2*>(a.z);
        const double2* __restrict__ q2 = reinterpret_cast<const double2*>(a.q);
        const double2* __restrict__ d2 = reinterpret_cast<const double2*>(dinv);
        for (int64_t j = (int64_t)gw * kSellC + lane; j < n2; j += (int64_t)nw * kSellC) {
          const double2 rr = r2[j], qq = q2[j], dd = __ldg(d2 + j);
          double2 rn, zn;
          rn.x = rr.x - alpha * qq.x;
          rn.y = rr.y - alpha * qq.y;
          zn.x = dd.x * rn.x;
          zn.y = dd.y * rn.y;
          r2[j] = rn;
          z2[j] = zn;
          acc.x += rn.x * zn.x;
          acc.x += rn.y * zn.y;
          acc.y += zn.x * zn.x;
          acc.y += zn.y * zn.y;
        }
      } else
      for (int s = gw; s < ns; s += UU * nw) {
        double rr[UU], qq[UU], dd[UU];
#pragma unroll
        for (int u = 0; u < UU; ++u) {
          const int su = s + u * nw;
          if (su < ns) {
            const int64_t i = (int64_t)su * kSellC + lane;
            rr[u] = TCB_ZFORM ? a.z[i] : a.r[i];
            qq[u] = a.q[i];
            dd[u] = __ldg(dinv + i);
          }
        }
#pragma unroll
        for (int u = 0; u < UU; ++u) {
          const int su = s + u * nw;
          if (su < ns) {
            const int64_t i = (int64_t)su * kSellC + lane;
#if TCB_ZFORM
            // z-form: z_{k+1} = z_k - alpha D^-1 q (= D^-1 r_{k+1}); r.z = sum z^2 / dinv
            const double zi = rr[u] - alpha * (dd[u] * qq[u]);
            a.z[i] = zi;
            acc.x += dd[u] != 0.0 ? zi * (zi / dd[u]) : 0.0;
            acc.y += zi * zi;
#else
            const double ri = rr[u] - alpha * qq[u], zi = dd[u] * ri;
            a.r[i] = ri;
            a.z[i] = zi;
            acc.x += ri * zi;
            acc.y += zi * zi;
#endif
          }
        }
      }
      tot = grid_sum2(acc, partA, sh, grid);
      ++it;
      const double zeta_new = sqrt(tot.y);
      zeta = zeta_new;
      if (isnan(zeta_new) || isnan(tot.x)) { nan = 1; break; }
      if (zeta_new < a.eps_a || zeta_new / zref < a.eps_r) { conv = 1; break; }
      beta = tot.x / rho;                                 // beta_k = rho_{k+1} / rho_k
      rho = tot.x;
      if (a.rel_mode == 0) zref = zeta_new;
    }
  }
  // deferred x += alpha p of the last iteration (Alg. 1 updates x before the test)
  if (last_valid && !nan) {
    const double* __restrict__ plast = ((it - 1) & 1) ? a.p1 : a.p0;  // p of the last iteration
    if (vec2) {
      double2* __restrict__ x2 = reinterpret_cast<double2*>(a.x);
      const double2* __restrict__ pl2 = reinterpret_cast<const double2*>(plast);
      for (int64_t j = (int64_t)gw * kSellC + lane; j < n2; j += (int64_t)nw * kSellC) {
        const double2 xx = x2[j], pp = pl2[j];
        x2[j] = make_double2(xx.x + alpha * pp.x, xx.y + alpha * pp.y);
      }
    } else {
      // TCB_XMERGE: S(it-1) skipped its x update when it-1 was odd -> p_{it-2} pending too
      const bool two = TCB_XMERGE && !(it & 1) && it >= 2;
      const double* __restrict__ pl2 = (it & 1) ? a.p1 : a.p0;   // p_{it-2}
    for (int s = gw; s < ns; s += UU * nw) {
      double xx[UU], pp[UU], p2[UU];
#pragma unroll
      for (int u = 0; u < UU; ++u)
        if (s + u * nw < ns) {
          const int64_t i = (int64_t)(s + u * nw) * kSellC + lane;
          xx[u] = a.x[i];
          pp[u] = plast[i];
          p2[u] = two ? pl2[i] : 0.0;
        }
#pragma unroll
      for (int u = 0; u < UU; ++u)
        if (s + u * nw < ns)
          a.x[(int64_t)(s + u * nw) * kSellC + lane] = (two ? xx[u] + alpha_prev * p2[u] : xx[u]) + alpha * pp[u];
    }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.stat->iters = it;
    a.stat->converged = conv;
    a.stat->znorm = zeta;
    int32_t* f = a.flags;
    if (nan) {
      f[0] = 1; f[1] = 1; f[4] = a.step_tag;
    } else {
      f[2] = conv ? 0 : f[2] + 1;
      if (f[3] > 0 && f[2] >= f[3]) { f[0] = 1; f[4] = a.step_tag; }
    }
  }
}

// ------------------------------------------------------------------ variant 6
// Single-reduction PCG (Chronopoulos & Gear's recurrence; SURVEY 8(e) "optional
// ... not the paper's algorithm, behind a flag and parity-checked";
// tc_config.pcg_variant = 6): the iterates of Algorithm 1 in exact arithmetic,
// with the two inner products of an iteration in one reduction, so ONE grid
// barrier per iteration instead of two.  Jacobi-preconditioned, z-form:
//   u = D^-1 r (Alg. 1's z), t = D^-1 A u, sigma = D^-1 A p;
//   init:  t_0 = D^-1 A u_0,  gamma_0 = r_0.u_0,  delta_0 = (A u_0).u_0,  alpha_0 = gamma_0/delta_0
//   phase i (one pass over the rows, then the reduction):
//     sigma_i = t_i + beta_i sigma_{i-1}     p_i = u_i + beta_i p_{i-1}
//     u_{i+1} = u_i - alpha_i sigma_i        x_{i+1} = x_i + alpha_i p_i
//     w = A u_{i+1} (the gathered u_{i+1} of a neighbour is formed on the fly from
//       its u_i, t_i, sigma_{i-1} by the same expression its owner uses: bitwise equal)
//     t_{i+1} = D^-1 w;  partials gamma_{i+1} = sum u^2/D^-1, delta_{i+1} = w.u, |u_{i+1}|^2
//   then Alg. 1's stopping test on |u_{i+1}| = |z_{i+1}| (readings C1-C3), and
//     beta_{i+1} = gamma_{i+1}/gamma_i,  alpha_{i+1} = gamma_{i+1}/(delta_{i+1} - beta_{i+1} gamma_{i+1}/alpha_i).
// u, t and sigma are gathered while being rewritten, so each has two buffers
// (u: z / r, t: q / p1, sigma: e0 / e1); p and x are own-row only (in place).
// Bytes per iteration 12 nnz + 4(n+1) + 88 n (vs 72 n); for latency-bound
// mid-size systems, where a grid barrier and a phase ramp cost more than that.
#ifndef TCB_1R_NB
#define TCB_1R_NB 8   // slots in flight per row (three gathers each)
#endif
__device__ __forceinline__ double u_next(double u, double t, double so, double alpha, double beta, bool first,
                                         double& sig) {
  sig = first ? t : fma(beta, so, t);
  return fma(-alpha, sig, u);
}

template <bool FIRST, int NB>
__device__ __forceinline__ double row_Au_next(int64_t base, int w, int lane, const int* col, const double* A,
                                              const double* u, const double* t, const double* so,
                                              double alpha, double beta) {
  double sum = 0.0;
#pragma unroll 1
  for (int k0 = 0; k0 < w; k0 += NB) {
    double av[NB], g[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int kk = min(k0 + j, w - 1);
      const int64_t ts = sell_slot(base, w, kk, lane);
      const int c = ld_mat(col + ts);
      av[j] = ld_mat(A + ts);
      double sig;
      g[j] = u_next(u[c], t[c], FIRST ? 0.0 : so[c], alpha, beta, FIRST, sig);
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (k0 + j < w) sum += av[j] * g[j];
  }
  return sum;
}

// Deterministic grid sum of three values (two double2 slots per CTA per call;
// the caller alternates buf between two 2 x gridDim.x regions).
__device__ __forceinline__ double3 grid_sum3(double3 v, double2* buf, double2* sh, cg::grid_group& grid) {
  const double2 b01 = block_sum2(make_double2(v.x, v.y), sh);
  const double2 b2 = block_sum2(make_double2(v.z, 0.0), sh);
  if (threadIdx.x == 0) {
    buf[blockIdx.x] = b01;
    buf[gridDim.x + blockIdx.x] = b2;
  }
  grid.sync();
  double2 acc01 = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < (int)gridDim.x; t += blockDim.x) {
    const double2 p = buf[t], q = buf[gridDim.x + t];
    acc01.x += p.x;
    acc01.y += p.y;
    acc2.x += q.x;
  }
  const double2 s01 = block_sum2(acc01, sh);
  const double2 s2 = block_sum2(acc2, sh);
  return make_double3(s01.x, s01.y, s2.x);
}

template <int MODE>
__global__ void __launch_bounds__(kCgThreads, 1) pcg1r_kernel(CgArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double2 sh[kCgWarps];
  if (a.flags[0]) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * kCgWarps + warp;
  const int nw = gridDim.x * kCgWarps;
  const int32_t ns = a.nslices;
  const int64_t* __restrict__ sp = a.slice_ptr;
  const int* __restrict__ col = a.col;
  const double* __restrict__ Av = a.A;
  const double* __restrict__ dinv = a.dinv;
  if constexpr (MODE == 1) {
    if (a.fuse_rhs) rhs_phase_batch(a, gw, nw, lane, sh, grid);
  }
  // u_i in (z, r)[i & 1], t_i in (q, p1)[i & 1], sigma_i in (e0, e1)[i & 1]
  double* __restrict__ p = a.p0;
  double2* part = a.part;         // 4 x gridDim.x slots: two regions of 2 x gridDim.x

  // gamma_0 = r_0.z_0, |z_0| from the RHS partials
  double2 tot;
  {
    double2 acc0 = make_double2(0.0, 0.0);
    for (int t = threadIdx.x; t < a.n_rpart; t += blockDim.x) {
      const double2 u = a.rpart[t];
      acc0.x += u.x;
      acc0.y += u.y;
    }
    tot = block_sum2(acc0, sh);
  }
  double gamma = tot.x;
  double zeta = sqrt(tot.y);
  double zref = zeta;
  int it = 0, conv = 0, nan = 0;
  if (isnan(gamma) || isnan(zeta)) nan = 1;
  if (!nan && zeta < a.eps_a) conv = 1;  // reading C4: return x0
  if (!nan && !conv) {
    // init: t_0 = D^-1 A u_0, delta_0 = (A u_0).u_0
    double2 acc = make_double2(0.0, 0.0);
    for (int s = gw; s < ns; s += nw) {
      const int64_t base = __ldg(sp + s);
      const int w = (int)((__ldg(sp + s + 1) - base) >> 5);
      const int64_t i = (int64_t)s * kSellC + lane;
      const double wi = row_Ap_batch_w<true>(base, w, lane, col, Av, a.z, nullptr, 0.0);
      a.q[i] = __ldg(dinv + i) * wi;
      acc.x += wi * a.z[i];
    }
    // the RHS partials live in part[0, grid): this sum uses the second region
    tot = grid_sum2(acc, part + 2 * gridDim.x, sh, grid);
    const double delta0 = tot.x;
    if (isnan(delta0)) nan = 1;
    double alpha = gamma / delta0, beta = 0.0;
    for (it = 0; !nan && it < a.max_iters;) {
      const int c = it & 1;
      const double* __restrict__ u = c ? a.r : a.z;
      const double* __restrict__ t = c ? a.p1 : a.q;
      const double* __restrict__ so = c ? a.e0 : a.e1;   // sigma_{it-1}
      double* __restrict__ un = c ? a.z : a.r;
      double* __restrict__ tn = c ? a.q : a.p1;
      double* __restrict__ sn = c ? a.e1 : a.e0;         // sigma_it
      double3 acc3 = make_double3(0.0, 0.0, 0.0);
      for (int s = gw; s < ns; s += nw) {
        const int64_t base = __ldg(sp + s);
        const int w = (int)((__ldg(sp + s + 1) - base) >> 5);
        const int64_t i = (int64_t)s * kSellC + lane;
        const double wi = it == 0 ? row_Au_next<true, TCB_1R_NB>(base, w, lane, col, Av, u, t, so, alpha, beta)
                                  : row_Au_next<false, TCB_1R_NB>(base, w, lane, col, Av, u, t, so, alpha, beta);
        const double ui = u[i], di = __ldg(dinv + i);
        double sig;
        const double un_i = u_next(ui, t[i], it == 0 ? 0.0 : so[i], alpha, beta, it == 0, sig);
        const double pi = it == 0 ? ui : ui + beta * p[i];
        p[i] = pi;
        a.x[i] = a.x[i] + alpha * pi;
        sn[i] = sig;
        un[i] = un_i;
        tn[i] = di * wi;
        acc3.x += di != 0.0 ? un_i * (un_i / di) : 0.0;   // r.z = sum z^2 / D^-1 (z-form)
        acc3.y += wi * un_i;
        acc3.z += un_i * un_i;
      }
      const double3 r3 = grid_sum3(acc3, part + (c ? 2 * gridDim.x : 0), sh, grid);
      ++it;
      const double zeta_new = sqrt(r3.z);
      zeta = zeta_new;
      if (isnan(zeta_new) || isnan(r3.x) || isnan(r3.y)) { nan = 1; break; }
      if (zeta_new < a.eps_a || zeta_new / zref < a.eps_r) { conv = 1; break; }
      const double beta_n = r3.x / gamma;                       // gamma_{i+1} / gamma_i
      const double den = r3.y - beta_n * r3.x / alpha;          // = p_{i+1}.A p_{i+1}
      alpha = r3.x / den;
      if (isnan(alpha)) { nan = 1; break; }
      beta = beta_n;
      gamma = r3.x;
      if (a.rel_mode == 0) zref = zeta_new;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.stat->iters = it;
    a.stat->converged = conv;
    a.stat->znorm = zeta;
    int32_t* f = a.flags;
    if (nan) {
      f[0] = 1; f[1] = 1; f[4] = a.step_tag;
    } else {
      f[2] = conv ? 0 : f[2] + 1;
      if (f[3] > 0 && f[2] >= f[3]) { f[0] = 1; f[4] = a.step_tag; }
    }
  }
}


__global__ void spmv_kernel(const int64_t* __restrict__ sp, const int* __restrict__ col,
                            const double* __restrict__ Av, int32_t ns, const double* __restrict__ x,
                            double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < ns; s += nw) {
    const int64_t base = sp[s];
    const int w = (int)((sp[s + 1] - base) >> 5);
    double sum = 0.0;
#pragma unroll 4
    for (int k = 0; k < w; ++k) {
      const int64_t t = sell_slot(base, w, k, lane);
      sum += Av[t] * x[col[t]];
    }
    y[(int64_t)s * kSellC + lane] = sum;
  }
}

static int g_sm_count[64] = {0};

static int sm_count(int dev) {
  if (dev < 0 || dev >= 64) return 148;
  if (!g_sm_count[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    g_sm_count[dev] = v > 0 ? v : 148;
  }
  return g_sm_count[dev];
}

static const void* rhs_fn(int mode, int variant) {
  if (variant == 4 || variant == 6) return mode == 1 ? (const void*)rhs_kernel<1, 4> : (const void*)rhs_kernel<0, 4>;
  if (variant == 3) return mode == 1 ? (const void*)rhs_kernel<1, 3> : (const void*)rhs_kernel<0, 3>;
  if (variant == 1) return mode == 1 ? (const void*)rhs_kernel<1, 1> : (const void*)rhs_kernel<0, 1>;
  if (variant == 2) return mode == 1 ? (const void*)rhs_kernel<1, 2> : (const void*)rhs_kernel<0, 2>;
  return mode == 1 ? (const void*)rhs_kernel<1, 0> : (const void*)rhs_kernel<0, 0>;
}
static const void* pcg_fn(int mode, int variant) {
  if (variant == 6) return mode == 1 ? (const void*)pcg1r_kernel<1> : (const void*)pcg1r_kernel<0>;
  if (variant == 4) return mode == 1 ? (const void*)pcg_kernel<1, 4> : (const void*)pcg_kernel<0, 4>;
  if (variant == 3) return mode == 1 ? (const void*)pcg_kernel<1, 3> : (const void*)pcg_kernel<0, 3>;
  if (variant == 1) return mode == 1 ? (const void*)pcg_kernel<1, 1> : (const void*)pcg_kernel<0, 1>;
  if (variant == 2) return mode == 1 ? (const void*)pcg_kernel<1, 2> : (const void*)pcg_kernel<0, 2>;
  return mode == 1 ? (const void*)pcg_kernel<1, 0> : (const void*)pcg_kernel<0, 0>;
}
static int pcg_smem(int variant) { return variant == 1 ? kCgSmem : 0; }

// Variant actually launched: an explicit request, or (requested < 0, the
// default) the latency variant 4 when the system has at most kAutoBatch slices
// per resident warp of the direct variant (mid-size systems such as configs[2],
// where each warp owns 1-3 slices and the S phase is one latency chain per
// slot batch), else the direct variant 0 (measured crossover: DESIGN.md "PCG").
// The same choice for a system that gets 1/share of the GPU (cohorts of
// concurrent large members, api.cu), and that share of the variant's grid.
int cg_pick_variant_share(int requested, int32_t nslices, int device, int share) {
  if (requested >= 0) return requested;
  const int64_t warps = (int64_t)sm_count(device) * (2048 / 32) / std::max(share, 1);
  return (int64_t)nslices <= kAutoBatch * warps ? 4 : 0;
}
int cg_grid_size_share(int variant, int32_t nslices, int device, int share) {
  return std::max(1, cg_grid_size(1, variant, nslices, device) / std::max(share, 1));
}

int cg_pick_variant(int requested, int32_t nslices, int device) {
  if (requested >= 0) return requested;
  const int64_t warps = (int64_t)sm_count(device) * (2048 / 32);
  return (int64_t)nslices <= kAutoBatch * warps ? 4 : 0;
}

// Grid: enough CTAs for one slice per warp, capped at the co-resident maximum
// (cooperative launch); large problems get every SM x occupancy (2 CTAs / SM).
int cg_grid_size(int mode, int variant, int32_t nslices, int device) {
  cudaFuncSetAttribute(pcg_fn(mode, variant), cudaFuncAttributeMaxDynamicSharedMemorySize, pcg_smem(variant));
  cudaFuncSetAttribute(rhs_fn(mode, variant), cudaFuncAttributeMaxDynamicSharedMemorySize, pcg_smem(variant));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg_fn(mode, variant), kCgThreads, pcg_smem(variant));
  if (per_sm < 1) per_sm = 1;
#ifdef TCB_CG_PER_SM_CAP
  if (per_sm > TCB_CG_PER_SM_CAP) per_sm = TCB_CG_PER_SM_CAP;
#endif
  int maxg = per_sm * sm_count(device);
  int need = (nslices + kCgWarps - 1) / kCgWarps;
  if (need < 1) need = 1;
  return need < maxg ? need : maxg;
}

cudaError_t launch_pcg(int mode, int variant, const CgArgs& a, int grid, cudaStream_t s) {
  void* args[] = {(void*)&a};
  cudaError_t e = cudaLaunchKernel(rhs_fn(mode, variant), dim3(grid), dim3(kCgThreads), args,
                                   pcg_smem(variant), s);
  if (e != cudaSuccess) return e;
  return cudaLaunchCooperativeKernel(pcg_fn(mode, variant), dim3(grid), dim3(kCgThreads), args,
                                     pcg_smem(variant), s);
}

cudaError_t launch_pcg_only(int mode, int variant, const CgArgs& a, int grid, cudaStream_t s) {
  void* args[] = {(void*)&a};
  return cudaLaunchCooperativeKernel(pcg_fn(mode, variant), dim3(grid), dim3(kCgThreads), args,
                                     pcg_smem(variant), s);
}

__global__ void chunk_maxcol_kernel(const int64_t* __restrict__ sp, const int32_t* __restrict__ col,
                                    int32_t nslices, int32_t spc, int32_t* chunk_max) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t s = (int32_t)(t >> 5);
  if (s >= nslices) return;
  const int lane = threadIdx.x & 31;
  const int64_t base = sp[s];
  const int w = (int)((sp[s + 1] - base) >> 5);
  int32_t m = 0;
  for (int k = 0; k < w; ++k) m = max(m, col[base + (int64_t)k * kSellC + lane]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) atomicMax(chunk_max + s / spc, m);
}

cudaError_t launch_chunk_maxcol(const int64_t* sp, const int32_t* col, int32_t nslices, int32_t spc,
                                int32_t* chunk_max, cudaStream_t s) {
  const int64_t threads = (int64_t)nslices * 32;
  chunk_maxcol_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(sp, col, nslices, spc, chunk_max);
  return cudaGetLastError();
}

cudaError_t launch_rhs(int mode, int variant, const CgArgs& a, int grid, cudaStream_t s) {
  void* args[] = {(void*)&a};
  return cudaLaunchKernel(rhs_fn(mode, variant), dim3(grid), dim3(kCgThreads), args, pcg_smem(variant), s);
}

cudaError_t launch_spmv(const int64_t* sp, const int32_t* col, const double* A, int32_t ns,
                        const double* x, double* y, cudaStream_t s) {
  int threads = 256;
  int64_t warps = ns;
  int blocks = (int)std::min<int64_t>((warps * 32 + threads - 1) / threads, 148 * 16);
  if (blocks < 1) blocks = 1;
  spmv_kernel<<<blocks, threads, 0, s>>>(sp, col, A, ns, x, y);
  return cudaGetLastError();
}

}  // namespace tcb
