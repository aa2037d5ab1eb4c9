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
#include <cstring>

#include "internal.h"

namespace tcb {

// ------------------------------------------------------------------ LAT / LRT
__device__ __forceinline__ void activation_update(const IonArgs& a, int64_t i, double Vnow,
                                                  double Vprev) {
  const uint8_t st = a.act[i];
  if (st == 0) {
    if (Vnow > a.lat_thr) { a.lat[i] = a.t_k; a.act[i] = 1; }      // first V > 0
  } else if (st == 1) {
    if (Vnow < a.lrt_thr && Vnow - Vprev < 0.0) { a.lrt[i] = a.t_k; a.act[i] = 2; }
  }
}

__device__ __forceinline__ void write_rhs(const IonArgs& a, int64_t i, double V, double Vp,
                                          double In) {
  const double x0 = 2.0 * V - Vp;
  const double dv = -a.dt * In;            // y - V^k
  a.x0[i] = x0;
  a.up[i] = (V + dv) - x0;
  a.vp[i] = a.dt * (V + a.theta * dv);
}

// ------------------------------------------------------------------ TT2006 epi
// ten Tusscher & Panfilov 2006 (cited P:98), epicardial cell; states in the
// order Ki Nai Cai CaSS CaSR Rbar m h j xr1 xr2 xs r s d f f2 fCass.
enum { sKi, sNai, sCai, sCaSS, sCaSR, sRbar, sm, sh, sj, sxr1, sxr2, sxs, sr, ss, sd, sf, sf2, sfc };

struct TTVolt {     // factors that depend on V only (shared by both current evaluations)
  double ecal;      // exp(2 (V-15) F/RT)
  double enaca_a;   // exp(gamma V F/RT)
  double enaca_b;   // exp((gamma-1) V F/RT)
  double fnak;      // 1 / (1 + 0.1245 exp(-0.1 V F/RT) + 0.0353 exp(-V F/RT))
  double fpk;       // 1 / (1 + exp((25 - V)/5.98))
};

struct TTCur {
  double ina, ik1, ito, ikr, iks, ical, inaca, inak, ipca, ipk, ibna, ibca;
};

__device__ __forceinline__ TTVolt tt_volt(double V, const TTParams& P) {
  const double frt = P.F / (P.R * P.T);
  TTVolt f;
  f.ecal = exp(2.0 * (V - 15.0) * frt);
  f.enaca_a = exp(P.gamma * V * frt);
  f.enaca_b = exp((P.gamma - 1.0) * V * frt);
  f.fnak = 1.0 / (1.0 + 0.1245 * exp(-0.1 * V * frt) + 0.0353 * exp(-V * frt));
  f.fpk = 1.0 / (1.0 + exp((25.0 - V) / 5.98));
  return f;
}

__device__ __forceinline__ TTCur tt_cur(double V, const double* u, const TTParams& P,
                                        const TTVolt& f) {
  const double rtf = P.R * P.T / P.F;
  const double ek = rtf * log(P.Ko / u[sKi]);
  const double ena = rtf * log(P.Nao / u[sNai]);
  const double eks = rtf * log((P.Ko + P.pKNa * P.Nao) / (u[sKi] + P.pKNa * u[sNai]));
  const double eca = 0.5 * rtf * log(P.Cao / u[sCai]);
  TTCur c;
  c.ina = P.GNa * u[sm] * u[sm] * u[sm] * u[sh] * u[sj] * (V - ena);
  {
    const double dvk = V - ek;
    const double a1 = 0.1 / (1.0 + exp(0.06 * (dvk - 200.0)));
    const double b1 = (3.0 * exp(0.0002 * (dvk + 100.0)) + exp(0.1 * (dvk - 10.0))) /
                      (1.0 + exp(-0.5 * dvk));
    c.ik1 = P.GK1 * (a1 / (a1 + b1)) * dvk;
  }
  c.ito = P.Gto * u[sr] * u[ss] * (V - ek);
  c.ikr = P.GKr * sqrt(P.Ko / 5.4) * u[sxr1] * u[sxr2] * (V - ek);
  c.iks = P.GKs * u[sxs] * u[sxs] * (V - eks);
  {
    const double frt = P.F / (P.R * P.T);
    c.ical = P.GCaL * u[sd] * u[sf] * u[sf2] * u[sfc] * 4.0 * (V - 15.0) * (P.F * frt) *
             (0.25 * u[sCaSS] * f.ecal - P.Cao) / (f.ecal - 1.0);
  }
  {
    const double nai3 = u[sNai] * u[sNai] * u[sNai];
    const double nao3 = P.Nao * P.Nao * P.Nao;
    const double kmn3 = P.KmNai * P.KmNai * P.KmNai;
    c.inaca = P.kNaCa * (f.enaca_a * nai3 * P.Cao - f.enaca_b * nao3 * u[sCai] * P.alpha) /
              ((kmn3 + nao3) * (P.KmCa + P.Cao) * (1.0 + P.ksat * f.enaca_b));
  }
  c.inak = P.PNaK * P.Ko * u[sNai] * f.fnak / ((P.Ko + P.KmK) * (u[sNai] + P.KmNa));
  c.ipca = P.GpCa * u[sCai] / (P.KpCa + u[sCai]);
  c.ipk = P.GpK * f.fpk * (V - ek);
  c.ibna = P.GbNa * (V - ena);
  c.ibca = P.GbCa * (V - eca);
  return c;
}

__device__ __forceinline__ double tt_total(const TTCur& c) {
  return c.ina + c.ik1 + c.ito + c.ikr + c.iks + c.ical + c.inaca + c.inak + c.ipca + c.ipk +
         c.ibna + c.ibca;
}

// c_new of a rapidly buffered pool: c + B c/(c+K) grows by delta.
__device__ __forceinline__ double buffered(double c, double delta, double B, double K) {
  const double bound = B * c / (c + K);
  const double bb = B - bound - delta - c + K;
  const double cc = K * (bound + delta + c);
  return 0.5 * (sqrt(bb * bb + 4.0 * cc) - bb);
}

__device__ __forceinline__ double rl(double y, double yinf, double tau, double dt) {
  return yinf - (yinf - y) * exp(-dt / tau);
}

__device__ __forceinline__ double sig(double x) { return 1.0 / (1.0 + exp(x)); }

// Advances u in place; returns I_n(V, u^{k+1}).
__device__ __forceinline__ double tt_advance(double V, double* u, double dt, const TTParams& P) {
  const TTVolt f = tt_volt(V, P);
  const TTCur c = tt_cur(V, u, P, f);
  // -- calcium dynamics (currents and fluxes at (V^k, u^k)) --
  const double casr = u[sCaSR], cass = u[sCaSS], cai = u[sCai];
  const double ec = P.EC / casr;
  const double kcasr = P.maxsr - (P.maxsr - P.minsr) / (1.0 + ec * ec);
  const double k1 = P.k1p / kcasr, k2 = P.k2p * kcasr;
  const double rbar = u[sRbar] + dt * (P.k4 * (1.0 - u[sRbar]) - k2 * cass * u[sRbar]);
  const double oo = k1 * cass * cass * rbar / (P.k3 + k1 * cass * cass);
  const double irel = P.Vrel * oo * (casr - cass);
  const double ileak = P.Vleak * (casr - cai);
  const double iup = P.Vmaxup / (1.0 + (P.Kup * P.Kup) / (cai * cai));
  const double ixfer = P.Vxfer * (cass - cai);
  const double nu_sr = dt * (iup - irel - ileak);
  const double nu_ss = dt * (-ixfer * (P.Vc / P.Vss) + irel * (P.Vsr / P.Vss) -
                             c.ical * P.CAP / (2.0 * P.Vss * P.F));
  const double nu_i = dt * (-(c.ibca + c.ipca - 2.0 * c.inaca) * P.CAP / (2.0 * P.Vc * P.F) -
                            (iup - ileak) * (P.Vsr / P.Vc) + ixfer);
  u[sRbar] = rbar;
  u[sCaSR] = buffered(casr, nu_sr, P.Bufsr, P.Kbufsr);
  u[sCaSS] = buffered(cass, nu_ss, P.Bufss, P.Kbufss);
  u[sCai] = buffered(cai, nu_i, P.Bufc, P.Kbufc);
  const double vcf = P.CAP / (P.Vc * P.F);
  u[sNai] = u[sNai] - dt * (c.ina + c.ibna + 3.0 * c.inak + 3.0 * c.inaca) * vcf;
  u[sKi] = u[sKi] - dt * (c.ik1 + c.ito + c.ikr + c.iks - 2.0 * c.inak + c.ipk) * vcf;

  // -- gates, Rush-Larsen at V^k (fCass with the new CaSS) --
  {
    const double am = sig((-60.0 - V) / 5.0);
    const double bm = 0.1 * sig((V + 35.0) / 5.0) + 0.1 * sig((V - 50.0) / 200.0);
    const double mi = sig((-56.86 - V) / 9.03);
    u[sm] = rl(u[sm], mi * mi, am * bm, dt);
  }
  {
    const double hi = sig((V + 71.55) / 7.43);
    const double hinf = hi * hi;
    double ah, bh, aj, bj;
    if (V >= -40.0) {
      ah = 0.0;
      bh = 0.77 / (0.13 * (1.0 + exp(-(V + 10.66) / 11.1)));
      aj = 0.0;
      bj = 0.6 * exp(0.057 * V) / (1.0 + exp(-0.1 * (V + 32.0)));
    } else {
      ah = 0.057 * exp(-(V + 80.0) / 6.8);
      bh = 2.7 * exp(0.079 * V) + 3.1e5 * exp(0.3485 * V);
      aj = (-2.5428e4 * exp(0.2444 * V) - 6.948e-6 * exp(-0.04391 * V)) * (V + 37.78) /
           (1.0 + exp(0.311 * (V + 79.23)));
      bj = 0.02424 * exp(-0.01052 * V) / (1.0 + exp(-0.1378 * (V + 40.14)));
    }
    u[sh] = rl(u[sh], hinf, 1.0 / (ah + bh), dt);
    u[sj] = rl(u[sj], hinf, 1.0 / (aj + bj), dt);
  }
  u[sxr1] = rl(u[sxr1], sig((-26.0 - V) / 7.0),
               (450.0 * sig((-45.0 - V) / 10.0)) * (6.0 * sig((V + 30.0) / 11.5)), dt);
  u[sxr2] = rl(u[sxr2], sig((V + 88.0) / 24.0),
               (3.0 * sig((-60.0 - V) / 20.0)) * (1.12 * sig((V - 60.0) / 20.0)), dt);
  u[sxs] = rl(u[sxs], sig((-5.0 - V) / 14.0),
              (1400.0 / sqrt(1.0 + exp((5.0 - V) / 6.0))) * sig((V - 35.0) / 15.0) + 80.0, dt);
  u[sr] = rl(u[sr], sig((20.0 - V) / 6.0), 9.5 * exp(-(V + 40.0) * (V + 40.0) / 1800.0) + 0.8, dt);
  u[ss] = rl(u[ss], sig((V + 20.0) / 5.0),
             85.0 * exp(-(V + 45.0) * (V + 45.0) / 320.0) + 5.0 * sig((V - 20.0) / 5.0) + 3.0, dt);
  u[sd] = rl(u[sd], sig((-8.0 - V) / 7.5),
             (1.4 * sig((-35.0 - V) / 13.0) + 0.25) * (1.4 * sig((V + 5.0) / 5.0)) +
                 sig((50.0 - V) / 20.0),
             dt);
  u[sf] = rl(u[sf], sig((V + 20.0) / 7.0),
             1102.5 * exp(-(V + 27.0) * (V + 27.0) / 225.0) + 200.0 * sig((13.0 - V) / 10.0) +
                 180.0 * sig((V + 30.0) / 10.0) + 20.0,
             dt);
  u[sf2] = rl(u[sf2], 0.67 * sig((V + 35.0) / 7.0) + 0.33,
              600.0 * exp(-(V + 25.0) * (V + 25.0) / 170.0) + 31.0 * sig((25.0 - V) / 10.0) +
                  16.0 * sig((V + 30.0) / 10.0),
              dt);
  {
    const double q = u[sCaSS] / 0.05;
    const double den = 1.0 / (1.0 + q * q);
    u[sfc] = rl(u[sfc], 0.6 * den + 0.4, 80.0 * den + 2.0, dt);
  }
  return tt_total(tt_cur(V, u, P, f));  // I_ion(V^k, u^{k+1}) (reading I2)
}

__global__ void __launch_bounds__(128) ionic_tt_kernel(IonArgs a, TTParams P) {
  if (a.flags[0]) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const double V = a.Vk[i];
  const double Vp = a.has_prev ? a.Vkm1[i] : V;
  if (a.do_lat) activation_update(a, i, V, Vp);
  double u[kTTStates];
#pragma unroll
  for (int s = 0; s < kTTStates; ++s) u[s] = a.U[s * a.stride + i];
  const double In = tt_advance(V, u, a.dt, P);
#pragma unroll
  for (int s = 0; s < kTTStates; ++s) a.U[s * a.stride + i] = u[s];
  write_rhs(a, i, V, Vp, In);
}

// ------------------------------------------------------------------ Mitchell-Schaeffer
__global__ void ionic_ms_kernel(IonArgs a, MSParams P) {
  if (a.flags[0]) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const double V = a.Vk[i];
  const double Vp = a.has_prev ? a.Vkm1[i] : V;
  if (a.do_lat) activation_update(a, i, V, Vp);
  const double span = P.V_max - P.V_min;
  const double v = (V - P.V_min) / span;
  double h = a.U[i];
  h = (v < P.v_gate) ? h + a.dt * ((1.0 - h) / P.tau_open) : h + a.dt * (-h / P.tau_close);
  a.U[i] = h;
  const double In = -span * (h * v * v * (1.0 - v) / P.tau_in - v / P.tau_out);
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
__global__ void scatter_kernel(int64_t n, const int32_t* __restrict__ idx,
                               const double* __restrict__ in, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[idx[i]] = in[i];
}

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

cudaError_t launch_ionic_tt(const IonArgs& a, const TTParams& p, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  ionic_tt_kernel<<<nblk(a.n, 128), 128, 0, s>>>(a, p);
  return cudaGetLastError();
}
cudaError_t launch_ionic_ms(const IonArgs& a, const MSParams& p, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  ionic_ms_kernel<<<nblk(a.n, 256), 256, 0, s>>>(a, p);
  return cudaGetLastError();
}
cudaError_t launch_ionic_mms(const IonArgs& a, const MMSParams& p, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  ionic_mms_kernel<<<nblk(a.n, 256), 256, 0, s>>>(a, p);
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
double* ms_param_slot(MSParams* p, const char* name) {
  for (size_t k = 0; k < sizeof(kMSNames) / sizeof(kMSNames[0]); ++k)
    if (!strcmp(kMSNames[k], name)) return reinterpret_cast<double*>(p) + k;
  return nullptr;
}

}  // namespace tcb
