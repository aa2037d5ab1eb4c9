// ionic.cu -- per-node kernels of one step: the explicit ionic update (Eq. 2
// row 1) fused with the LAT/LRT test, the extrapolated guess
// x0 = 2V^k - V^{k-1} and the two RHS vectors u', v' that let the
// PCG kernel form r_0 = b - A x0 = A u' - K v'.
//
// Per node (one thread, SoA state, coalesced):
//   y  = V^k - dt I_n                       (I_n = I_ion(V^k, u^{k+1}) / C_m, mV/ms)
//   x0 = 2V^k - V^{k-1}
//   u' = y - x0,   v' = dt (V^k + theta (y - V^k))
// Stimuli add dt s and theta dt^2 s (s = Isv / (chi C_m)) in stimulus_kernel.
#include <cmath>
#include <cstring>
#include <algorithm>
#include <map>
#include <mutex>

#include "ionic_node.cuh"

namespace tcb {


#ifndef TCB_ION_THREADS
#define TCB_ION_THREADS 128   // measured: 128 / 256
#endif
constexpr int kIonThreads = TCB_ION_THREADS;
// minimum resident CTAs per SM for the FP64-bound TT2006 / CRN kernels (register
// cap 65536 / (threads x this)): 4 = 128 registers (no cap), 5 = 96, 6 = 80.
// Measured at 10 M nodes (profiles/r02b_exp_ionic.txt, ionic ms/step):
// TT2006 4 / 5 / 6 = 1.19 / 1.13 / 1.17 (5: 96 registers, no spills);
// CRN 4 / 5 / 6 = 1.20 / 1.20 / 1.20 (5 spills 32 bytes) -> 5 and 4.
#ifndef TCB_ION_MINB
#define TCB_ION_MINB 5
#endif
#ifndef TCB_ION_MINB_CRN
#define TCB_ION_MINB_CRN 4
#endif

// The exp / log tables (fp64math.cuh): filled once per device and process into
// global memory (read-only, 3 KB).  TCB_ION_TAB_SMEM = 1 (default): every CTA
// copies them into shared memory (384 coalesced 8-byte loads, one barrier);
// 0: the kernels read them from global memory (L1).  r01 computed them per CTA
// (2 exp2 and half a log per thread plus a barrier: ~5 % of the kernel, ncu
// r02c).  Measured at 10 M nodes (profiles/r02d_exp_ionic.txt, ionic ms/step):
// TT2006 1.015 (shared) vs 1.060 (global), CRN 1.148 vs 1.211.
#ifndef TCB_ION_TAB_SMEM
#define TCB_ION_TAB_SMEM 1
#endif
__global__ void tables_fill_kernel(Exp2Table* T) { exp2_table_fill(T); }

const Exp2Table* device_tables() {
  static std::mutex mu;
  static std::map<int, Exp2Table*> tabs;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  Exp2Table*& t = tabs[dev];
  if (!t) {
    Exp2Table* d = nullptr;
    if (cudaMalloc(&d, sizeof(Exp2Table)) != cudaSuccess) return nullptr;
    tables_fill_kernel<<<1, 256>>>(d);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      cudaFree(d);
      return nullptr;
    }
    t = d;
  }
  return t;
}

// Load-latency hiding (ncu r02f: 16 % of the warp samples wait on the state
// loads at the top of the kernel).  TCB_ION_EARLY_LOADS = 1: the node's V and
// states are loaded BEFORE the per-CTA table copy and its barrier, so the DRAM
// latency overlaps them.  TCB_ION_L2PF = 1: every thread also prefetches (into
// L2, no registers) the V and states of the node one resident wave ahead
// (pf_dist nodes), which a CTA of the next wave then finds in L2.
// Measured (profiles/r02h_exp_ionic.txt, 10 M nodes, ionic ms/step, 1965 MHz):
// TT2006 early 0.952-0.957 vs late 0.962; CRN early 1.087 vs late 1.062 -> early
// loads for TT2006 only (TCB_ION_EARLY_LOADS_CRN); the L2 prefetch costs 2-4 %.
#ifndef TCB_ION_EARLY_LOADS
#define TCB_ION_EARLY_LOADS 1
#endif
#ifndef TCB_ION_EARLY_LOADS_CRN
#define TCB_ION_EARLY_LOADS_CRN 0
#endif
#ifndef TCB_ION_L2PF
#define TCB_ION_L2PF 0
#endif
__device__ __forceinline__ void pf_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// nodes of one resident wave of a one-node-per-thread ionic kernel (the L2
// prefetch distance)
template <class K>
static int64_t ion_wave(K kernel) {
  static int64_t wave = 0;  // per kernel (B200 only: one SM count)
  if (!wave) {
    int per = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kIonThreads, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    wave = (int64_t)std::max(per, 1) * sms * kIonThreads;
  }
  return wave;
}

template <int NS>
__device__ __forceinline__ void ion_prefetch(const IonArgs& a, int64_t j) {
#if TCB_ION_L2PF
  if (j < a.n && ((threadIdx.x & 3) == 0)) {   // one 32-byte sector per 4 nodes
    pf_l2(a.Vk + j);
    if (a.has_prev) pf_l2(a.Vkm1 + j);
#pragma unroll
    for (int s = 0; s < NS; ++s) pf_l2(a.U + s * a.stride + j);
  }
#else
  (void)a;
  (void)j;
#endif
}

// TCB_ION_NPT = k > 1 (experiment): k nodes per thread, processed one after the
// other (the per-CTA table copy and the per-thread constant set-up amortised
// over k nodes); TCB_ION_NPT_PF = 1 also prefetches the later nodes' V and states
// into L2 at the start.
#ifndef TCB_ION_NPT
#define TCB_ION_NPT 1
#endif
#ifndef TCB_ION_NPT_PF
#define TCB_ION_NPT_PF 0
#endif
#if TCB_ION_NPT > 1
__global__ void __launch_bounds__(kIonThreads, TCB_ION_MINB)
    ionic_tt_kernel(IonArgs a, TTParams P, TTDerived D, const Exp2Table* __restrict__ G, int64_t pf_dist) {
  (void)pf_dist;
  if (a.flags[0]) return;
  const int64_t i0 = (int64_t)blockIdx.x * (blockDim.x * TCB_ION_NPT) + threadIdx.x;
  double V = 0.0, Vp = 0.0;
  double u[kTTStates];
  if (i0 < a.n) {
    V = a.Vk[i0];
    Vp = a.has_prev ? a.Vkm1[i0] : V;
#pragma unroll
    for (int s = 0; s < kTTStates; ++s) u[s] = a.U[s * a.stride + i0];
  }
#if TCB_ION_NPT_PF
  for (int q = 1; q < TCB_ION_NPT; ++q) {
    const int64_t j = i0 + (int64_t)q * blockDim.x;
    if (j < a.n && (threadIdx.x & 3) == 0) {
      pf_l2(a.Vk + j);
      if (a.has_prev) pf_l2(a.Vkm1 + j);
#pragma unroll
      for (int s = 0; s < kTTStates; ++s) pf_l2(a.U + s * a.stride + j);
    }
  }
#endif
  __shared__ Exp2Table Ts;
  exp2_table_init(&Ts, G);
  const Exp2Table* T = &Ts;
#pragma unroll 1
  for (int q = 0; q < TCB_ION_NPT; ++q) {
    const int64_t i = i0 + (int64_t)q * blockDim.x;
    if (i >= a.n) break;
    if (q > 0) {
      V = a.Vk[i];
      Vp = a.has_prev ? a.Vkm1[i] : V;
#pragma unroll
      for (int s = 0; s < kTTStates; ++s) u[s] = a.U[s * a.stride + i];
    }
    if (a.do_lat) activation_update(a, i, V, Vp);
    const double In = tt_advance(V, u, a.dt, P, D, T);
#pragma unroll
    for (int s = 0; s < kTTStates; ++s) a.U[s * a.stride + i] = u[s];
    write_rhs(a, i, V, Vp, In);
  }
}
#else
__global__ void __launch_bounds__(kIonThreads, TCB_ION_MINB)
    ionic_tt_kernel(IonArgs a, TTParams P, TTDerived D, const Exp2Table* __restrict__ G, int64_t pf_dist) {
  if (a.flags[0]) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double V = 0.0, Vp = 0.0;
  double u[kTTStates];
#if TCB_ION_EARLY_LOADS
  if (i < a.n) {
    V = a.Vk[i];
    Vp = a.has_prev ? a.Vkm1[i] : V;
#pragma unroll
    for (int s = 0; s < kTTStates; ++s) u[s] = a.U[s * a.stride + i];
  }
#endif
  ion_prefetch<kTTStates>(a, i + pf_dist);
#if TCB_ION_TAB_SMEM
  __shared__ Exp2Table Ts;
  exp2_table_init(&Ts, G);
  const Exp2Table* T = &Ts;
#else
  const Exp2Table* __restrict__ T = G;
#endif
  if (i >= a.n) return;
#if !TCB_ION_EARLY_LOADS
  V = a.Vk[i];
  Vp = a.has_prev ? a.Vkm1[i] : V;
#pragma unroll
  for (int s = 0; s < kTTStates; ++s) u[s] = a.U[s * a.stride + i];
#endif
  if (a.do_lat) activation_update(a, i, V, Vp);
  const double In = tt_advance(V, u, a.dt, P, D, T);
#pragma unroll
  for (int s = 0; s < kTTStates; ++s) a.U[s * a.stride + i] = u[s];
  write_rhs(a, i, V, Vp, In);
}
#endif

// ---- persistent variant with asynchronous state prefetch (TCB_ION_PERSIST) ----
// One wave of CTAs walks the node tiles (128 nodes each) in a grid-stride loop;
// while a tile computes, the next tile's V^k, V^{k-1} and cell states travel
// from HBM into this thread's own shared-memory slots by cp.async (no register
// cost, no barrier: every thread reads and refills only its own slots), so the
// start-of-CTA load stall of the one-node-per-thread kernel (12 % of the warp
// samples, ncu r02c) and the per-CTA table copy are paid once per CTA.
#ifndef TCB_ION_PERSIST
#define TCB_ION_PERSIST 0
#endif
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// fields of a node in the stage: [0] V^k, [1] V^{k-1}, [2 ..) states
template <int NS>
__device__ __forceinline__ void prefetch_node(const IonArgs& a, int64_t i, double* st) {
  if (i >= a.n) return;
  cp_async8(st, a.Vk + i);
  cp_async8(st + kIonThreads, (a.has_prev ? a.Vkm1 : a.Vk) + i);
#pragma unroll
  for (int s = 0; s < NS; ++s) cp_async8(st + (2 + s) * kIonThreads, a.U + s * a.stride + i);
}

template <int MODEL>
__global__ void __launch_bounds__(kIonThreads, MODEL == TC_ION_CRN ? TCB_ION_MINB_CRN : TCB_ION_MINB)
    ionic_persist_kernel(IonArgs a, TTParams P, TTDerived D, CRNParams CP, CRNDerived CD,
                         const Exp2Table* __restrict__ G) {
  constexpr int NS = MODEL == TC_ION_CRN ? kCRNStates : kTTStates;
  extern __shared__ __align__(16) double stage[];   // (2 + NS) x kIonThreads
  __shared__ Exp2Table Ts;
  exp2_table_init(&Ts, G);
  if (a.flags[0]) return;
  double* my = stage + threadIdx.x;
  const int64_t ntiles = ((int64_t)a.n + kIonThreads - 1) / kIonThreads;
  int64_t tile = blockIdx.x;
  if (tile < ntiles) prefetch_node<NS>(a, tile * kIonThreads + threadIdx.x, my);
  cp_async_commit();
  for (; tile < ntiles; tile += gridDim.x) {
    const int64_t i = tile * kIonThreads + threadIdx.x;
    cp_async_wait0();
    double u[NS];
    const double V = my[0], Vp = my[kIonThreads];
#pragma unroll
    for (int s = 0; s < NS; ++s) u[s] = my[(2 + s) * kIonThreads];
    // the slots are free again: start the next tile's loads, then compute this one
    const int64_t inext = (tile + gridDim.x) * kIonThreads + threadIdx.x;
    if (tile + gridDim.x < ntiles) prefetch_node<NS>(a, inext, my);
    cp_async_commit();
    if (i < a.n) {
      if (a.do_lat) activation_update(a, i, V, Vp);
      double In;
      if constexpr (MODEL == TC_ION_CRN) In = crn_advance(V, u, a.dt, CP, CD, &Ts);
      else In = tt_advance(V, u, a.dt, P, D, &Ts);
#pragma unroll
      for (int s = 0; s < NS; ++s) a.U[s * a.stride + i] = u[s];
      write_rhs(a, i, V, Vp, In);
    }
  }
  cp_async_wait0();
}

template <int MODEL>
static cudaError_t launch_persist(const IonArgs& a, const TTParams& tp, const CRNParams& cp, cudaStream_t s) {
  const Exp2Table* G = device_tables();
  if (!G) return cudaErrorMemoryAllocation;
  constexpr int NS = MODEL == TC_ION_CRN ? kCRNStates : kTTStates;
  const size_t smem = (size_t)(2 + NS) * kIonThreads * 8;
  static int grid_cache[2] = {0, 0};
  int& per = grid_cache[MODEL == TC_ION_CRN ? 1 : 0];
  if (!per) {
    cudaFuncSetAttribute(ionic_persist_kernel<MODEL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ionic_persist_kernel<MODEL>, kIonThreads, smem);
    if (per < 1) per = 1;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = ((int64_t)a.n + kIonThreads - 1) / kIonThreads;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)per * sms);
  TTDerived td{};
  CRNDerived cd{};
  if (MODEL == TC_ION_CRN) cd = crn_derived(cp);
  else td = tt_derived(tp);
  ionic_persist_kernel<MODEL><<<grid, kIonThreads, smem, s>>>(a, tp, td, cp, cd, G);
  return cudaGetLastError();
}

TTDerived tt_derived(const TTParams& P) {
  TTDerived D;
  D.frt = P.F / (P.R * P.T);
  D.rtf = P.R * P.T / P.F;
  D.sq_ko = std::sqrt(P.Ko / 5.4);
  D.ecal0 = std::exp(-30.0 * D.frt);
  D.gcal4 = 4.0 * P.GCaL * P.F * D.frt;
  D.inaca_k = P.kNaCa / ((P.KmNai * P.KmNai * P.KmNai + P.Nao * P.Nao * P.Nao) * (P.KmCa + P.Cao));
  D.nao3_alpha = P.Nao * P.Nao * P.Nao * P.alpha;
  D.inak_k = P.PNaK * P.Ko / (P.Ko + P.KmK);
  D.eks_num = P.Ko + P.pKNa * P.Nao;
  D.vc_vss = P.Vc / P.Vss;
  D.vsr_vss = P.Vsr / P.Vss;
  D.vsr_vc = P.Vsr / P.Vc;
  D.cap_2vssf = P.CAP / (2.0 * P.Vss * P.F);
  D.cap_2vcf = P.CAP / (2.0 * P.Vc * P.F);
  D.cap_vcf = P.CAP / (P.Vc * P.F);
  D.kup2 = P.Kup * P.Kup;
  D.log_ko = std::log(P.Ko);
  D.log_nao = std::log(P.Nao);
  D.log_eks_num = std::log(D.eks_num);
  D.log_cao = std::log(P.Cao);
  D.x_m12 = std::exp(-12.0);        // (-60 - V)/5   = -12 - V/5
  D.x_7 = std::exp(7.0);            // (V + 35)/5    =   7 + V/5
  D.x_m3_2 = std::exp(-3.2);        // -0.1 (V + 32) = -3.2 - V/10
  D.x_m26_7 = std::exp(-26.0 / 7.0);  // (-26 - V)/7
  D.x_m4_5 = std::exp(-4.5);        // (-45 - V)/10
  D.x_m3 = std::exp(-3.0);          // (-60 - V)/20, (V - 60)/20
  D.x_5_6 = std::exp(5.0 / 6.0);    // (5 - V)/6
  D.x_20_6 = std::exp(20.0 / 6.0);  // (20 - V)/6
  D.x_4 = std::exp(4.0);            // (V + 20)/5
  D.x_m4 = std::exp(-4.0);          // (V - 20)/5
  D.x_1 = std::exp(1.0);            // (V + 5)/5
  D.x_2_5 = std::exp(2.5);          // (50 - V)/20, (25 - V)/10
  D.x_3 = std::exp(3.0);            // (V + 30)/10
  D.x_20_7 = std::exp(20.0 / 7.0);  // (V + 20)/7
  D.x_1_3 = std::exp(1.3);          // (13 - V)/10
  D.x_5 = std::exp(5.0);            // (V + 35)/7
  D.x_m1 = std::exp(-1.0);          // 0.1 (V - EK - 10) = -1 + 0.1 (V - EK)
  return D;
}

// ------------------------------------------------------------------ Mitchell-Schaeffer
MSDerived ms_derived(const MSParams& p) {
  return MSDerived{p.V_max - p.V_min, 1.0 / p.tau_open, 1.0 / p.tau_close, 1.0 / p.tau_in,
                   1.0 / p.tau_out};
}

__global__ void ionic_ms_kernel(IonArgs a, MSParams P, MSDerived D) {
  if (a.flags[0]) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const double V = a.Vk[i];
  const double Vp = a.has_prev ? a.Vkm1[i] : V;
  if (a.do_lat) activation_update(a, i, V, Vp);
  const double In = ms_advance(V, a.U + i, a.dt, P, D);
  write_rhs(a, i, V, Vp, In);
}

// ------------------------------------------------------------------ MMS source
// chi = Cm = 1, I_ion = 0; source r(x,y,t_k + theta dt) of Eq. 8;
// Dirichlet nodes take x0 = w(t_{k+1}) (reading M3).
__device__ __forceinline__ double mms_w(double x, double y, double t, const MMSParams& p) {
  return exp(-p.k * t) * cos(p.w1 * x + p.w2 * y - p.lam * t);
}

__global__ void ionic_mms_kernel(IonArgs a, MMSParams P) {
  if (a.flags[0]) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const double V = a.Vk[i];
  const double Vp = a.has_prev ? a.Vkm1[i] : V;
  const double X = a.xyz[3 * i], Y = a.xyz[3 * i + 1];
  const double ph = P.w1 * X + P.w2 * Y - P.lam * a.t_src;
  const double r = exp(-P.k * a.t_src) * (-P.k * cos(ph) + P.lam * sin(ph)) +
                   (P.w1 * P.w1 + P.w2 * P.w2) * exp(-P.k * a.t_src) * cos(ph);
  const double dv = a.dt * r;  // y - V^k
  const double x0 = a.dirichlet[i] ? mms_w(X, Y, a.t_next, P) : 2.0 * V - Vp;
  a.x0[i] = x0;
  a.up[i] = (V + dv) - x0;
  a.vp[i] = a.dt * (V + a.theta * dv);
}

// ------------------------------------------------------------------ stimulus, LAT epilogue
__global__ void stimulus_kernel(int32_t m, const int32_t* __restrict__ idx,
                                const double* __restrict__ s, double* up, double* vp, double dt,
                                double theta, const int32_t* flags) {
  if (flags[0]) return;
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int32_t i = idx[t];
  const double ds = dt * s[t];  // dt Isv / (chi Cm)
  up[i] += ds;
  vp[i] += theta * dt * ds;
}

__global__ void lat_epilogue_kernel(IonArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  activation_update(a, i, a.Vk[i], a.Vkm1[i]);
}

__global__ void gather_kernel(int64_t n, const int32_t* __restrict__ idx,
                              const double* __restrict__ in, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[idx[i]];
}
// every field of a host-layout state (tc_set_state: V^k | V^{k-1} | u_0 .. u_{S-1},
// field stride in_stride, original order) into the internal order: one launch,
// blockIdx.y = field.
__global__ void gather_state_kernel(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ in,
                                    int64_t in_stride, double* __restrict__ v0, double* __restrict__ v1,
                                    double* __restrict__ U, int64_t upad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int f = blockIdx.y;
  double* out = f == 0 ? v0 : f == 1 ? v1 : U + (int64_t)(f - 2) * upad;
  out[i] = in[(int64_t)f * in_stride + idx[i]];
}
__global__ void scatter_kernel(int64_t n, const int32_t* __restrict__ idx,
                               const double* __restrict__ in, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[idx[i]] = in[i];
}

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

cudaError_t launch_ionic_tt(const IonArgs& a, const TTParams& p, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  if (TCB_ION_PERSIST) return launch_persist<TC_ION_TT2006_EPI>(a, p, CRNParams{}, s);
  const Exp2Table* G = device_tables();
  if (!G) return cudaErrorMemoryAllocation;
  ionic_tt_kernel<<<nblk(a.n, kIonThreads * TCB_ION_NPT), kIonThreads, 0, s>>>(a, p, tt_derived(p), G,
                                                                              ion_wave(ionic_tt_kernel));
  return cudaGetLastError();
}
cudaError_t launch_ionic_ms(const IonArgs& a, const MSParams& p, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  ionic_ms_kernel<<<nblk(a.n, 256), 256, 0, s>>>(a, p, ms_derived(p));
  return cudaGetLastError();
}
cudaError_t launch_ionic_mms(const IonArgs& a, const MMSParams& p, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  ionic_mms_kernel<<<nblk(a.n, 256), 256, 0, s>>>(a, p);
  return cudaGetLastError();
}
// ------------------------------------------------------------------ CRN 1998
CRNDerived crn_derived(const CRNParams& P) {
  CRNDerived D;
  D.rtf = P.R * P.T / P.F;
  D.frt = P.F / (P.R * P.T);
  D.sigma_k = 0.0365 * (std::exp(P.Nao / 67.3) - 1.0) / 7.0;
  D.cm_vif = P.Cm / (P.Vi * P.F);
  D.cm_2vif = P.Cm / (2.0 * P.Vi * P.F);
  D.inak_k = P.INaKmax * P.Ko / (P.Ko + P.KmKo);
  D.inaca_k = P.INaCamax / ((P.KmNa * P.KmNa * P.KmNa + P.Nao * P.Nao * P.Nao) * (P.KmCa + P.Cao));
  D.nao3 = P.Nao * P.Nao * P.Nao;
  D.inv_tautr = 1.0 / P.tautr;
  D.iupleak_k = P.Iupmax / P.Caupmax;
  D.vup_vi = P.Vup / P.Vi;
  D.vrel_vi = P.Vrel / P.Vi;
  D.vrel_vup = P.Vrel / P.Vup;
  D.inv_kq10 = 1.0 / P.KQ10;
  D.kq10 = P.KQ10;
  D.inv_tauu = 1.0 / P.tauu;
  D.fn_c = 1e-15 / (2.0 * P.F) * P.Cm;  // currents per capacitance -> pA
  D.log_nao = std::log(P.Nao);
  D.log_ko = std::log(P.Ko);
  D.log_cao = std::log(P.Cao);
  return D;
}

__global__ void __launch_bounds__(kIonThreads, TCB_ION_MINB_CRN)
    ionic_crn_kernel(IonArgs a, CRNParams P, CRNDerived D, const Exp2Table* __restrict__ G, int64_t pf_dist) {
  if (a.flags[0]) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double V = 0.0, Vp = 0.0;
  double u[kCRNStates];
#if TCB_ION_EARLY_LOADS_CRN
  if (i < a.n) {
    V = a.Vk[i];
    Vp = a.has_prev ? a.Vkm1[i] : V;
#pragma unroll
    for (int s = 0; s < kCRNStates; ++s) u[s] = a.U[s * a.stride + i];
  }
#endif
  ion_prefetch<kCRNStates>(a, i + pf_dist);
#if TCB_ION_TAB_SMEM
  __shared__ Exp2Table Ts;
  exp2_table_init(&Ts, G);
  const Exp2Table* T = &Ts;
#else
  const Exp2Table* __restrict__ T = G;
#endif
  if (i >= a.n) return;
#if !TCB_ION_EARLY_LOADS_CRN
  V = a.Vk[i];
  Vp = a.has_prev ? a.Vkm1[i] : V;
#pragma unroll
  for (int s = 0; s < kCRNStates; ++s) u[s] = a.U[s * a.stride + i];
#endif
  if (a.do_lat) activation_update(a, i, V, Vp);
  const double In = crn_advance(V, u, a.dt, P, D, T);
#pragma unroll
  for (int s = 0; s < kCRNStates; ++s) a.U[s * a.stride + i] = u[s];
  write_rhs(a, i, V, Vp, In);
}

cudaError_t launch_ionic_crn(const IonArgs& a, const CRNParams& p, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  if (TCB_ION_PERSIST) return launch_persist<TC_ION_CRN>(a, TTParams{}, p, s);
  const Exp2Table* G = device_tables();
  if (!G) return cudaErrorMemoryAllocation;
  ionic_crn_kernel<<<nblk(a.n, kIonThreads), kIonThreads, 0, s>>>(a, p, crn_derived(p), G, ion_wave(ionic_crn_kernel));
  return cudaGetLastError();
}

cudaError_t launch_stimulus(int32_t m, const int32_t* idx, const double* sv, double* up, double* vp,
                            double dt, double theta, const int32_t* flags, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  stimulus_kernel<<<nblk(m, 256), 256, 0, st>>>(m, idx, sv, up, vp, dt, theta, flags);
  return cudaGetLastError();
}
cudaError_t launch_lat_epilogue(const IonArgs& a, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  lat_epilogue_kernel<<<nblk(a.n, 256), 256, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_gather(int64_t n, const int32_t* idx, const double* in, double* out,
                          cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  gather_kernel<<<nblk(n, 256), 256, 0, s>>>(n, idx, in, out);
  return cudaGetLastError();
}
cudaError_t launch_gather_state(int64_t n, const int32_t* idx, const double* in, int64_t in_stride, double* v0,
                                double* v1, double* U, int64_t upad, int32_t nstates, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  gather_state_kernel<<<dim3((unsigned)nblk(n, 256), (unsigned)(2 + nstates)), 256, 0, s>>>(n, idx, in, in_stride,
                                                                                         v0, v1, U, upad);
  return cudaGetLastError();
}
cudaError_t launch_scatter(int64_t n, const int32_t* idx, const double* in, double* out,
                           cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  scatter_kernel<<<nblk(n, 256), 256, 0, s>>>(n, idx, in, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ parameters
void tt_defaults(TTParams* p, double* V0, double u0[kTTStates]) {
  *p = TTParams{8314.472, 310.0, 96485.3415, 0.185, 0.016404, 0.001094, 0.00005468, 5.4, 140.0, 2.0,
                14.838, 5.405, 0.294, 0.153, 0.392, 0.03, 3.98e-5, 2.9e-4, 5.92e-4, 0.1238, 5e-4, 0.0146,
                2.724, 1.0, 40.0, 1000.0, 87.5, 1.38, 0.1, 0.35, 2.5,
                0.2, 0.001, 10.0, 0.3, 0.4, 0.00025,
                0.006375, 0.00025, 0.102, 0.15, 0.045, 0.06, 0.005, 1.5, 2.5, 1.0, 3.6e-4, 0.0038};
  *V0 = -85.23;
  const double ic[kTTStates] = {136.89, 8.604, 1.26e-4, 3.6e-4, 3.64, 0.9073, 0.00172, 0.7444, 0.7045,
                                0.00621, 0.4712, 0.0095, 2.42e-8, 0.999998, 3.373e-5, 0.7888, 0.9755,
                                0.9953};
  for (int s = 0; s < kTTStates; ++s) u0[s] = ic[s];
}

void ms_defaults(MSParams* p) { *p = MSParams{0.3, 6.0, 120.0, 150.0, 0.13, -80.0, 20.0}; }

void crn_defaults(CRNParams* p, double* V0, double u0[kCRNStates]) {
  *p = CRNParams{8.3143, 310.0, 96.4867, 100.0, 13668.0, 1109.52, 96.48, 5.4, 140.0, 1.8,
                 7.8, 0.09, 0.1652, 0.029411765, 0.12941176, 0.12375, 6.744375e-4, 1.131e-3,
                 0.59933874, 10.0, 1.5, 1600.0, 87.5, 1.38, 0.1, 0.35, 0.275, 30.0, 180.0,
                 0.005, 0.00092, 15.0, 0.05, 0.07, 10.0, 0.00238, 0.0005, 0.8, 8.0, 3.0};
  *V0 = -81.18;
  const double ic[kCRNStates] = {11.17, 139.0, 1.013e-4, 1.488, 1.488, 2.908e-3, 0.9649, 0.9775,
                                 3.043e-2, 0.9992, 4.966e-3, 0.9986, 3.296e-5, 1.869e-2, 1.367e-4,
                                 0.9996, 0.7755, 2.35e-112, 1.0, 0.9992};
  for (int s = 0; s < kCRNStates; ++s) u0[s] = ic[s];
}

static const char* kTTNames[] = {
    "R", "T", "F", "CAP", "Vc", "Vsr", "Vss", "Ko", "Nao", "Cao", "GNa", "GK1", "Gto", "GKr", "GKs",
    "pKNa", "GCaL", "GbNa", "GbCa", "GpCa", "KpCa", "GpK", "PNaK", "KmK", "KmNa", "kNaCa", "KmNai",
    "KmCa", "ksat", "gamma", "alpha", "Bufc", "Kbufc", "Bufsr", "Kbufsr", "Bufss", "Kbufss",
    "Vmaxup", "Kup", "Vrel", "k1p", "k2p", "k3", "k4", "EC", "maxsr", "minsr", "Vleak", "Vxfer"};
static const char* kMSNames[] = {"tau_in", "tau_out", "tau_open", "tau_close", "v_gate", "V_min",
                                 "V_max"};

double* tt_param_slot(TTParams* p, const char* name) {
  static_assert(sizeof(TTParams) == sizeof(kTTNames) / sizeof(kTTNames[0]) * sizeof(double), "");
  for (size_t k = 0; k < sizeof(kTTNames) / sizeof(kTTNames[0]); ++k)
    if (!strcmp(kTTNames[k], name)) return reinterpret_cast<double*>(p) + k;
  return nullptr;
}
static const char* kCRNNames[] = {
    "R", "T", "F", "Cm", "Vi", "Vup", "Vrel", "Ko", "Nao", "Cao", "gNa", "gK1", "gto", "gKr",
    "gKs", "gCaL", "gbNa", "gbCa", "INaKmax", "KmNai", "KmKo", "INaCamax", "KmNa", "KmCa", "ksat",
    "gamma", "IpCamax", "Krel", "tautr", "Iupmax", "Kup", "Caupmax", "CMDNmax", "TRPNmax",
    "CSQNmax", "KmCMDN", "KmTRPN", "KmCSQN", "tauu", "KQ10"};

double* crn_param_slot(CRNParams* p, const char* name) {
  static_assert(sizeof(CRNParams) == sizeof(kCRNNames) / sizeof(kCRNNames[0]) * sizeof(double), "");
  for (size_t k = 0; k < sizeof(kCRNNames) / sizeof(kCRNNames[0]); ++k)
    if (!strcmp(kCRNNames[k], name)) return reinterpret_cast<double*>(p) + k;
  return nullptr;
}

double* ms_param_slot(MSParams* p, const char* name) {
  for (size_t k = 0; k < sizeof(kMSNames) / sizeof(kMSNames[0]); ++k)
    if (!strcmp(kMSNames[k], name)) return reinterpret_cast<double*>(p) + k;
  return nullptr;
}

}  // namespace tcb
