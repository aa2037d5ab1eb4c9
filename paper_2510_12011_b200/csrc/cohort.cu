// cohort.cu -- the cluster engine: every time step of a replica (ionic update,
// stimulus, RHS, Algorithm 1, rotation) runs inside ONE thread-block cluster,
// for n steps, in ONE launch; a cohort of independent replicas (SURVEY 8f row
// f1: "many independent meshes") is one grid of clusters.
//
// Why: a small mesh (configs[0], 4 305 nodes)
// under the grid engine spends its step in launch gaps and grid-wide barriers
// (~9 us per PCG iteration at 148 SMs for ~1 MB of work).  Here the replica
// owns C <= 16 CTAs of one cluster: the per-iteration barriers are hardware
// cluster barriers (barrier.cluster, ~0.2 us), the inner products are reduced
// through distributed shared memory (each CTA stores its partial into every
// CTA's slot, then every CTA sums the C slots in rank order -> bitwise-identical
// scalars, identical stopping decisions, no host round trip), and the whole
// solve stays L2-resident.  Replicas never synchronise with each other: each
// cluster stops its own PCG (per-replica stopping), and clusters beyond the
// co-resident count are scheduled as others retire.
//
// The arithmetic per node and per row is the per-step kernels' (ionic_node.cuh,
// the SELL-32 row sums of pcg.cu in the same slot order); only the grouping of
// the inner-product partial sums differs (C CTAs instead of the grid).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstring>

#include "ionic_node.cuh"
#include "pcg_common.cuh"

namespace tcb {

namespace {

constexpr int kCoWarps = kCoThreads / 32;
constexpr size_t kTTBytes = sizeof(TTParams) + sizeof(TTDerived);
constexpr size_t kCRNBytes = sizeof(CRNParams) + sizeof(CRNDerived);
constexpr int kParamDoubles = (int)(((kTTBytes > kCRNBytes ? kTTBytes : kCRNBytes) + 7) / 8);

struct CoShared {
  CoRep R;
  double prm[kParamDoubles];
  double2 sh[2][kCoWarps];
  double2 slot[2][kCoMaxCluster];
};

// Deterministic cluster-wide sum with ONE CTA barrier and ONE cluster barrier:
// each warp stores its partial in sh[par][warp]; after __syncthreads thread t < C
// adds the warp partials in warp order and stores the CTA partial into slot
// [par][my rank] of CTA t (DSMEM); after the cluster barrier every thread of
// every CTA adds the C slots in rank order (bitwise-identical results).  `par`
// alternates, so neither sh nor the slots of the next reduction can overwrite
// values still being read (a CTA reaches the reduction after next only once
// every CTA has arrived at the next cluster barrier).
__device__ __forceinline__ double2 cluster_sum2(double2 v, CoShared& S, int& par,
                                                cg::cluster_group& cl, int C, int crank) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_sum2(v);
  if (lane == 0) S.sh[par][warp] = v;
  __syncthreads();
  if ((int)threadIdx.x < C) {
    double2 b = S.sh[par][0];
#pragma unroll
    for (int w = 1; w < kCoWarps; ++w) {
      b.x += S.sh[par][w].x;
      b.y += S.sh[par][w].y;
    }
    double2* dst = cl.map_shared_rank(&S.slot[par][crank], (int)threadIdx.x);
    *dst = b;
  }
  cl.sync();
  double2 acc = S.slot[par][0];
  for (int t = 1; t < C; ++t) {
    const double2 u = S.slot[par][t];
    acc.x += u.x;
    acc.y += u.y;
  }
  par ^= 1;
  return acc;
}

}  // namespace

// Rows of a replica are cut into C contiguous blocks of whole slices, one per
// CTA; warp w of a CTA takes slices s0 + w, s0 + w + 8, ... .  Every per-row
// phase (ionic, RHS, S, U, x update, LAT) maps row i to the same thread, so a
// row's own data needs no barrier between phases; only gathered vectors (u', v',
// z, p) cross CTAs, and every phase that gathers them follows a cluster barrier.
//
// RES (cluster-resident): for the whole launch the
// replica lives in the cluster's distributed shared memory -- every vector of
// the step (three V buffers, r, q, diag^-1, z, p0, p1, u', v') as C blocks of
// own rows, one per CTA, at the same offsets in every CTA, and each CTA's
// matrix block (A, K, col: TMA bulk copies at launch).  Gathers of a column
// owned by another CTA are ld.shared::cluster loads through DSMEM (column
// indices are rewritten once to (owner CTA, local row)); nothing but the cell
// states, LAT/LRT and the per-step reports touches global memory until the
// V buffers are written back at the end.  Otherwise (STREAMING) every array
// stays in global memory / L2.
constexpr int kNVec = 11;  // V0 V1 V2 r q dinv | z p0 p1 u' v' (gathered)
enum { vV0 = 0, vR = 3, vQ = 4, vD = 5, vZ = 6, vP0 = 7, vP1 = 8, vUP = 9, vVP = 10 };
constexpr int kOwnerShift = 20;   // packed column: owner CTA << 20 | local row
constexpr int kB = 16;            // slots of a row gathered in one batch

__device__ __forceinline__ double ld_dsmem(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t map_rank(const void* p, int r) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_addr(p)), "r"(r));
  return out;
}

#ifdef TCB_COHORT_PHASES  // experiment build only (tools/exp_cohort_phases.sh)
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PH(k) do { if (ph_on) { const unsigned long long t_ = gtime(); ph[k] += t_ - ph_t; ph_t = t_; } } while (0)
#else
#define PH(k) do { } while (0)
#endif

// MINB: CTAs per SM the register allocation must allow.  1 (resident and the
// default streaming launch): up to 255 registers, no spills.  2 ("dense"
// streaming, a cohort option): 128 registers, 228-728 bytes of spills (MS ..
// CRN) for twice the resident clusters -- fewer rounds when the members
// outnumber the 1-per-SM clusters.
template <int MODEL, bool RES, int MINB = 1>
__global__ void __launch_bounds__(kCoThreads, MINB)
    cohort_kernel(const CoRep* __restrict__ reps, int64_t nsteps) {
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks();
  const int crank = (int)cl.block_rank();
  __shared__ CoShared S;
  __shared__ Exp2Table T;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t cbase[kCoMaxCluster];  // DSMEM address of every CTA's vector block
  extern __shared__ __align__(128) char dsm[];
  if (threadIdx.x == 0) S.R = reps[blockIdx.x / C];
  __syncthreads();
  const CoRep& R = S.R;
  for (int j = threadIdx.x; j < kParamDoubles; j += blockDim.x) S.prm[j] = R.params[j];
  if (MODEL != TC_ION_MS) exp2_table_init(&T, R.tab);  // includes __syncthreads
  __syncthreads();
  const TTParams& TP = *reinterpret_cast<const TTParams*>(S.prm);
  const TTDerived& TD = *reinterpret_cast<const TTDerived*>(S.prm + sizeof(TTParams) / 8);
  const MSParams& MP = *reinterpret_cast<const MSParams*>(S.prm);
  const MSDerived& MD = *reinterpret_cast<const MSDerived*>(S.prm + sizeof(MSParams) / 8);
  const CRNParams& CP = *reinterpret_cast<const CRNParams*>(S.prm);
  const CRNDerived& CD = *reinterpret_cast<const CRNDerived*>(S.prm + sizeof(CRNParams) / 8);

  // every CTA reads the same flags before any CTA can change them (the first
  // write follows a cluster barrier), so the early exit is cluster-uniform
  const int32_t flag0 = R.flags[0];
  int32_t fails = R.flags[2];
  const int32_t budget = R.flags[3];
  if (flag0) {
    if (R.status && crank == 0 && threadIdx.x == 0) *R.status = R.flags[1] ? 2 : 1;
    return;
  }
  if (R.status && crank == 0 && threadIdx.x == 0) *R.status = 0;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t ns = R.nslices, n = R.n;
  const int spc = (ns + C - 1) / C;                 // slices per CTA
  const int s0 = min(ns, crank * spc), s1 = min(ns, s0 + spc);
  const int64_t row0 = (int64_t)s0 * kSellC, rown = (int64_t)(s1 - s0) * kSellC;
  const int rpc = spc * kSellC;                     // rows per CTA block (vector stride)
  const int64_t t0 = R.slice_ptr[s0], tn = R.slice_ptr[s1] - t0;

  // matrix and own-row vectors: shared (RES, offset so global indices work) or global
  const int64_t* sp = R.slice_ptr;
  const int* col = R.col;
  const double* Av = R.A;
  const double* Kv = R.K;
  const double* dinv = R.dinv;
  double* Vb[3] = {R.V[0], R.V[1], R.V[2]};
  double* r = R.r;
  double* q = R.q;
  double* z = R.z;
  double* p0 = R.p0;
  double* p1 = R.p1;
  double* up = R.up;
  double* vp = R.vp;
  uint32_t vbase = 0;  // RES: this CTA's vector block in its own shared window
  if (RES) {
    // layout (cohort_smem_bytes): kNVec vectors x rpc | slice offsets | pad | A K col [tn]
    // (compact: col [tn] only; A and K stay in global memory and are read through L2)
    double* sv = reinterpret_cast<double*>(dsm);
    int64_t* ssp = reinterpret_cast<int64_t*>(sv + (size_t)kNVec * rpc);
    const size_t moff = ((size_t)kNVec * rpc * 8 + (size_t)(spc + 1) * 8 + 127) & ~(size_t)127;
    const bool cmp = R.compact != 0;
    double* sA = reinterpret_cast<double*>(dsm + moff);
    double* sK = sA + tn;
    int* sC = cmp ? reinterpret_cast<int*>(dsm + moff) : reinterpret_cast<int*>(sK + tn);
    if (threadIdx.x == 0 && tn > 0) {
      mbar_init(&mbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      const uint64_t pol = policy_evict_first();
      mbar_expect_tx(&mbar, (uint32_t)(tn * (cmp ? 4 : 20)));
      if (!cmp) {
        tma_load(sA, R.A + t0, (uint32_t)(tn * 8), &mbar, pol);
        tma_load(sK, R.K + t0, (uint32_t)(tn * 8), &mbar, pol);
      }
      tma_load(sC, R.col + t0, (uint32_t)(tn * 4), &mbar, pol);
    }
    if ((int)threadIdx.x < C) cbase[threadIdx.x] = map_rank(sv, (int)threadIdx.x);
    for (int j = threadIdx.x; j <= s1 - s0; j += blockDim.x) ssp[j] = R.slice_ptr[s0 + j];
    for (int j = threadIdx.x; j < rpc; j += blockDim.x) {
      const bool own = j < rown;
#pragma unroll
      for (int b = 0; b < 3; ++b) sv[(size_t)b * rpc + j] = own ? R.V[b][row0 + j] : 0.0;
      sv[(size_t)vD * rpc + j] = own ? R.dinv[row0 + j] : 0.0;
      for (int v = vR; v < kNVec; ++v)
        if (v != vD) sv[(size_t)v * rpc + j] = 0.0;
    }
    __syncthreads();
    if (tn > 0) mbar_wait(&mbar, 0);
    for (int64_t j = threadIdx.x; j < tn; j += blockDim.x) {  // column -> (owner, local row)
      const int c = sC[j];
      const int o = c / rpc;
      sC[j] = (o << kOwnerShift) | (c - o * rpc);
    }
    // pointers offset so that global slot / row indices address the shared copies
    if (!cmp) {
      Av = sA - t0;
      Kv = sK - t0;
    }
    col = sC - t0;
    sp = ssp - s0;
    for (int b = 0; b < 3; ++b) Vb[b] = sv + (size_t)b * rpc - row0;
    r = sv + (size_t)vR * rpc - row0;
    q = sv + (size_t)vQ * rpc - row0;
    dinv = sv + (size_t)vD * rpc - row0;
    z = sv + (size_t)vZ * rpc - row0;
    p0 = sv + (size_t)vP0 * rpc - row0;
    p1 = sv + (size_t)vP1 * rpc - row0;
    up = sv + (size_t)vUP * rpc - row0;
    vp = sv + (size_t)vVP * rpc - row0;
    vbase = smem_addr(sv);
    cl.sync();  // every CTA's vectors initialised and cbase set before any gather
  }
  (void)vbase;
  // DSMEM address of vector v at packed column pc (RES)
  const uint32_t vstride = (uint32_t)rpc * 8u;
  auto gaddr = [&](int pc) -> uint32_t {
    return cbase[pc >> kOwnerShift] + (uint32_t)(pc & ((1 << kOwnerShift) - 1)) * 8u;
  };
  int iVk = R.iVk, iVkm1 = R.iVkm1, iX = R.iX;
  int has_prev = R.has_prev;
  int par = 0;
  bool aborted = false;
#ifdef TCB_COHORT_PHASES
  // phases: 0 ionic, 1 stimulus + barrier, 2 RHS + reduction, 3 S, 4 p.q reduction,
  // 5 U, 6 r.z reduction, 7 rest (x update, report)
  const bool ph_on = blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ph_t = gtime();
  long long ph_iters = 0;
#endif

  for (int64_t st = 0; st < nsteps; ++st) {
    const int64_t k = R.k0 + st;
    double* Vk = Vb[iVk];
    double* Vkm1 = Vb[iVkm1];
    double* x = Vb[iX];
    IonArgs ia{};
    ia.n = n;
    ia.stride = R.stride;
    ia.Vk = Vk;
    ia.Vkm1 = Vkm1;
    ia.U = R.U;
    ia.x0 = x;
    ia.up = up;
    ia.vp = vp;
    ia.act = R.act;
    ia.lat = R.lat;
    ia.lrt = R.lrt;
    ia.t_k = k * R.dt;
    ia.lat_thr = R.lat_thr;
    ia.lrt_thr = R.lrt_thr;
    ia.dt = R.dt;
    ia.theta = R.theta;
    const bool do_lat = st > 0;  // V^k of the call's first step was tested by the last epilogue

    // ---- a1: ionic step, LAT/LRT of V^k, x0, u', v' (own rows) -------------------
    for (int s = s0 + warp; s < s1; s += kCoWarps) {
      const int64_t i = (int64_t)s * kSellC + lane;
      if (i >= n) continue;
      const double V = Vk[i];
      const double Vp = has_prev ? Vkm1[i] : V;
      if (do_lat) activation_update(ia, i, V, Vp);
      double In;
      if (MODEL == TC_ION_TT2006_EPI) {
        double u[kTTStates];
#pragma unroll
        for (int q2 = 0; q2 < kTTStates; ++q2) u[q2] = R.U[q2 * R.stride + i];
        In = tt_advance(V, u, R.dt, TP, TD, &T);
#pragma unroll
        for (int q2 = 0; q2 < kTTStates; ++q2) R.U[q2 * R.stride + i] = u[q2];
      } else if (MODEL == TC_ION_CRN) {
        double u[kCRNStates];
#pragma unroll
        for (int q2 = 0; q2 < kCRNStates; ++q2) u[q2] = R.U[q2 * R.stride + i];
        In = crn_advance(V, u, R.dt, CP, CD, &T);
#pragma unroll
        for (int q2 = 0; q2 < kCRNStates; ++q2) R.U[q2 * R.stride + i] = u[q2];
      } else {
        In = ms_advance(V, R.U + i, R.dt, MP, MD);
      }
      write_rhs(ia, i, V, Vp, In);
    }
    PH(0);
    // ---- a0: stimulus of the epoch containing step k (epochs are disjoint) -------
    for (int e = 0; e < R.n_ep; ++e) {
      const StimEpoch ep = R.ep[e];
      if (ep.k0 <= k && k < ep.k1) {
        if (RES) {  // own rows only (the list is small); after this CTA's ionic writes
          __syncthreads();
          for (int t = threadIdx.x; t < ep.m; t += kCoThreads) {
            const int32_t i = R.stim_idx[ep.off + t];
            if (i < row0 || i >= row0 + rown) continue;
            const double ds = R.dt * R.stim_s[ep.off + t];  // dt Isv / (chi Cm)
            up[i] += ds;
            vp[i] += R.theta * R.dt * ds;
          }
        } else {
          cl.sync();  // u', v' of every node written
          for (int t = crank * kCoThreads + threadIdx.x; t < ep.m; t += C * kCoThreads) {
            const int32_t i = R.stim_idx[ep.off + t];
            const double ds = R.dt * R.stim_s[ep.off + t];
            up[i] += ds;
            vp[i] += R.theta * R.dt * ds;
          }
        }
      }
    }
    cl.sync();  // the RHS gathers u', v' of neighbouring rows
    PH(1);

    // ---- a2: r0 = A u' - K v', z0 = r0 / diag(A), rho_0, ||z0||^2 -----------------
    double2 acc = make_double2(0.0, 0.0);
    for (int s = s0 + warp; s < s1; s += kCoWarps) {
      const int64_t i = (int64_t)s * kSellC + lane;
      const int64_t base = sp[s];
      const int w = (int)((sp[s + 1] - base) >> 5);
      double sum = 0.0;
      // slots in batches of kB: all loads of a batch in flight together (predicated,
      // no remainder loop), then accumulated in slot order
#pragma unroll 1
      for (int k0 = 0; k0 < w; k0 += kB) {
        double a[kB], b[kB], g1[kB], g2[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) {  // slots past the row end reload its last slot
          const int64_t t = sell_slot(base, w, min(k0 + j, w - 1), lane);
          a[j] = Av[t];
          b[j] = Kv[t];
          if (RES) {
            const uint32_t g = gaddr(col[t]);
            g1[j] = ld_dsmem(g + vUP * vstride);
            g2[j] = ld_dsmem(g + vVP * vstride);
          } else {
            const int c = col[t];
            g1[j] = up[c];
            g2[j] = vp[c];
          }
        }
#pragma unroll
        for (int j = 0; j < kB; ++j)
          if (k0 + j < w) sum += a[j] * g1[j] - b[j] * g2[j];
      }
      const double zi = dinv[i] * sum;
      r[i] = sum;
      z[i] = zi;
      acc.x += sum * zi;
      acc.y += zi * zi;
    }
    double2 tot = cluster_sum2(acc, S, par, cl, C, crank);
    PH(2);

    // ---- a3-a5: Algorithm 1 (same data flow as pcg_kernel) -------------------------
    double rho = tot.x;
    double zeta = sqrt(tot.y);
    double zref = zeta;
    int it = 0, conv = 0, nan = 0;
    if (isnan(rho) || isnan(zeta)) nan = 1;
    if (!nan && zeta < R.eps_a) conv = 1;  // reading C4: return x0
    double alpha = 0.0, beta = 0.0;
    bool last_valid = false;
    if (!nan && !conv) {
      for (it = 0; it < R.max_iters;) {
        // S: p = z + beta p_old (on the fly), q = A p, x += alpha_prev p_old
        acc = make_double2(0.0, 0.0);
        double* pnew = (it & 1) ? p1 : p0;
        const double* pold = (it & 1) ? p0 : p1;
        const uint32_t pold_off = ((it & 1) ? vP0 : vP1) * vstride;
        for (int s = s0 + warp; s < s1; s += kCoWarps) {
          const int64_t i = (int64_t)s * kSellC + lane;
          const int64_t base = sp[s];
          const int w = (int)((sp[s + 1] - base) >> 5);
          double sum = 0.0, pi;
          if (it == 0) {
            pi = z[i];
      #pragma unroll 1
      for (int k0 = 0; k0 < w; k0 += kB) {
              double a[kB], g1[kB];
#pragma unroll
              for (int j = 0; j < kB; ++j) {
                const int64_t t = sell_slot(base, w, min(k0 + j, w - 1), lane);
                a[j] = Av[t];
                g1[j] = RES ? ld_dsmem(gaddr(col[t]) + vZ * vstride) : z[col[t]];
              }
#pragma unroll
              for (int j = 0; j < kB; ++j)
                if (k0 + j < w) sum += a[j] * g1[j];
            }
          } else {
            const double po = pold[i];
            pi = z[i] + beta * po;
            x[i] = x[i] + alpha * po;
      #pragma unroll 1
      for (int k0 = 0; k0 < w; k0 += kB) {
              double a[kB], g1[kB], g2[kB];
#pragma unroll
              for (int j = 0; j < kB; ++j) {
                const int64_t t = sell_slot(base, w, min(k0 + j, w - 1), lane);
                a[j] = Av[t];
                if (RES) {
                  const uint32_t g = gaddr(col[t]);
                  g1[j] = ld_dsmem(g + vZ * vstride);
                  g2[j] = ld_dsmem(g + pold_off);
                } else {
                  const int c = col[t];
                  g1[j] = z[c];
                  g2[j] = pold[c];
                }
              }
#pragma unroll
              for (int j = 0; j < kB; ++j)
                if (k0 + j < w) sum += a[j] * (g1[j] + beta * g2[j]);
            }
          }
          pnew[i] = pi;
          q[i] = sum;
          acc.x += pi * sum;
        }
        last_valid = true;
        PH(3);
        tot = cluster_sum2(acc, S, par, cl, C, crank);
        PH(4);
        const double pq = tot.x;
        if (isnan(pq)) { nan = 1; break; }
        alpha = rho / pq;
        // U: r -= alpha q, z = r / d, partials of r.z and z.z
        acc = make_double2(0.0, 0.0);
        for (int s = s0 + warp; s < s1; s += kCoWarps) {
          const int64_t i = (int64_t)s * kSellC + lane;
          const double ri = r[i] - alpha * q[i], zi = dinv[i] * ri;
          r[i] = ri;
          z[i] = zi;
          acc.x += ri * zi;
          acc.y += zi * zi;
        }
        PH(5);
        tot = cluster_sum2(acc, S, par, cl, C, crank);
        PH(6);
        ++it;
        const double zeta_new = sqrt(tot.y);
        zeta = zeta_new;
        if (isnan(zeta_new) || isnan(tot.x)) { nan = 1; break; }
        if (zeta_new < R.eps_a || zeta_new / zref < R.eps_r) { conv = 1; break; }
        beta = tot.x / rho;
        rho = tot.x;
        if (R.rel_mode == 0) zref = zeta_new;
      }
    }
    // deferred x += alpha p of the last iteration (own rows, same mapping as S)
    if (last_valid && !nan) {
      const double* plast = ((it - 1) & 1) ? p1 : p0;
      for (int s = s0 + warp; s < s1; s += kCoWarps) {
        const int64_t i = (int64_t)s * kSellC + lane;
        x[i] = x[i] + alpha * plast[i];
      }
    }
    // ---- a6: report, failure budget, rotation ---------------------------------------
    if (crank == 0 && threadIdx.x == 0) {
      R.stats[st].iters = it;
      R.stats[st].converged = conv;
      R.stats[st].znorm = zeta;
    }
    if (nan) {
      aborted = true;
    } else {
      fails = conv ? 0 : fails + 1;
      if (budget > 0 && fails >= budget) aborted = true;
    }
    if (crank == 0 && threadIdx.x == 0) {
      int32_t* f = R.flags;
      f[2] = fails;
      if (aborted) {
        f[0] = 1;
        f[4] = (int32_t)k;
        if (nan) f[1] = 1;
      }
    }
    if (aborted) {
      if (R.status && crank == 0 && threadIdx.x == 0) *R.status = nan ? 2 : 1;
      break;
    }
    const int old = iVkm1;
    iVkm1 = iVk;
    iVk = iX;
    iX = old;
    has_prev = 1;
    PH(7);
#ifdef TCB_COHORT_PHASES
    ph_iters += it;
#endif
  }
#ifdef TCB_COHORT_PHASES
  if (ph_on)
    printf("phases_ns steps %lld iters %lld C %d res %d: ionic %llu stim %llu rhs %llu S %llu red_pq %llu U %llu red_rz %llu rest %llu\n",
           (long long)nsteps, ph_iters, C, (int)RES, ph[0], ph[1], ph[2], ph[3], ph[4], ph[5], ph[6], ph[7]);
#endif
  // LAT/LRT of the last V (time t_{k0 + nsteps}); own rows only
  if (!aborted && nsteps > 0) {
    IonArgs ia{};
    ia.act = R.act;
    ia.lat = R.lat;
    ia.lrt = R.lrt;
    ia.t_k = (R.k0 + nsteps) * R.dt;
    ia.lat_thr = R.lat_thr;
    ia.lrt_thr = R.lrt_thr;
    const double* Vk = Vb[iVk];
    const double* Vkm1 = Vb[iVkm1];
    for (int s = s0 + warp; s < s1; s += kCoWarps) {
      const int64_t i = (int64_t)s * kSellC + lane;
      if (i < n) activation_update(ia, i, Vk[i], Vkm1[i]);
    }
  }
  if (RES) {  // write the shared V buffers back (own rows; same thread mapping)
    for (int s = s0 + warp; s < s1; s += kCoWarps) {
      const int64_t i = (int64_t)s * kSellC + lane;
#pragma unroll
      for (int b = 0; b < 3; ++b) R.V[b][i] = Vb[b][i];
    }
  }
  cl.sync();  // no CTA leaves while another may still address its shared memory
}

static const void* cohort_fn(int model, bool res, bool dense = false) {
  if (model == TC_ION_TT2006_EPI)
    return res ? (const void*)cohort_kernel<TC_ION_TT2006_EPI, true>
               : dense ? (const void*)cohort_kernel<TC_ION_TT2006_EPI, false, 2>
                       : (const void*)cohort_kernel<TC_ION_TT2006_EPI, false>;
  if (model == TC_ION_CRN)
    return res ? (const void*)cohort_kernel<TC_ION_CRN, true>
               : dense ? (const void*)cohort_kernel<TC_ION_CRN, false, 2>
                       : (const void*)cohort_kernel<TC_ION_CRN, false>;
  return res ? (const void*)cohort_kernel<TC_ION_MS, true>
             : dense ? (const void*)cohort_kernel<TC_ION_MS, false, 2> : (const void*)cohort_kernel<TC_ION_MS, false>;
}

int cohort_param_doubles() { return kParamDoubles; }

void cohort_pack_params(int model, const TTParams& tp, const MSParams& mp, const CRNParams& cp,
                        double* out) {
  for (int j = 0; j < kParamDoubles; ++j) out[j] = 0.0;
  if (model == TC_ION_CRN) {
    const CRNDerived d = crn_derived(cp);
    std::memcpy(out, &cp, sizeof(CRNParams));
    std::memcpy(out + sizeof(CRNParams) / 8, &d, sizeof(CRNDerived));
  } else if (model == TC_ION_TT2006_EPI) {
    const TTDerived d = tt_derived(tp);
    std::memcpy(out, &tp, sizeof(TTParams));
    std::memcpy(out + sizeof(TTParams) / 8, &d, sizeof(TTDerived));
  } else {
    const MSDerived d = ms_derived(mp);
    std::memcpy(out, &mp, sizeof(MSParams));
    std::memcpy(out + sizeof(MSParams) / 8, &d, sizeof(MSDerived));
  }
}

// Shared memory a cluster-resident launch needs for a replica with slice
// pointers sp[0..ns] cut into C blocks (the largest block decides).
size_t cohort_smem_bytes(const int64_t* sp, int32_t ns, int C, bool compact) {
  const int spc = (ns + C - 1) / C;
  if ((int64_t)spc * kSellC >= (1 << kOwnerShift)) return (size_t)1 << 40;  // packed columns overflow
  const size_t moff = ((size_t)kNVec * spc * kSellC * 8 + (size_t)(spc + 1) * 8 + 127) & ~(size_t)127;
  size_t tmax = 0;
  for (int r = 0; r < C; ++r) {
    const int s0 = std::min(ns, r * spc), s1 = std::min(ns, s0 + spc);
    tmax = std::max(tmax, (size_t)(sp[s1] - sp[s0]));
  }
  return moff + tmax * (compact ? 4 : 20);
}

// Largest dynamic shared memory a cluster-resident launch may use.
size_t cohort_smem_limit(int model) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, cohort_fn(model, true));
  const size_t stat = fa.sharedSizeBytes;
  return optin > (int)stat + 1024 ? (size_t)optin - stat - 1024 : 0;
}

static cudaLaunchConfig_t cohort_cfg(int nrep, int csize, size_t smem, cudaStream_t s,
                                     cudaLaunchAttribute* at) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(nrep * csize));
  cfg.blockDim = dim3(kCoThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cfg;
}

static void prepare(const void* fn, size_t smem) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

int cohort_active_clusters(int model, int csize, size_t smem, bool dense) {
  const void* fn = cohort_fn(model, smem > 0, dense && smem == 0);
  prepare(fn, smem);
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = cohort_cfg(1, csize, smem, nullptr, at);
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return ncl;
}

// Largest power-of-two cluster size <= want (<= 16) of which at least one
// cluster can be resident; 0 if none.
int cohort_cluster_size(int model, int want) {
  for (int c = kCoMaxCluster; c >= 1; c >>= 1)
    if (c <= want && cohort_active_clusters(model, c, 0) > 0) return c;
  return 0;
}

cudaError_t launch_cohort(int model, const CoRep* d_reps, int nrep, int csize, size_t smem,
                          int64_t nsteps, cudaStream_t s, bool dense) {
  if (nrep <= 0 || nsteps <= 0) return cudaSuccess;
  const void* fn = cohort_fn(model, smem > 0, dense && smem == 0);
  prepare(fn, smem);
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = cohort_cfg(nrep, csize, smem, s, at);
  void* args[] = {(void*)&d_reps, (void*)&nsteps};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace tcb
