// ionic_node.cuh -- per-node device code of the ionic step (Eq. 2 row 1, P:128;
// P:139), the LAT/LRT test and the RHS vectors x0, u', v' (P:200-203,
// DESIGN.md "RHS"), shared by the per-step kernels (ionic.cu) and the cohort
// engine (cohort.cu), so both paths run the same arithmetic per node.
#pragma once

#include "fp64math.cuh"
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
//
// Arithmetic layout: exact in exact arithmetic to
// the model equations, rearranged for the FP64 pipe -- branch-free exp /
// reciprocal (fp64math.cuh), division by constants as multiplication by
// their reciprocals, parameter-only factors folded on the host (TTDerived),
// and voltage exponentials that share a slope computed from one exponential,
// e.g. exp((V+35)/5) = e^7 exp(V/5), exp((-60-V)/5) = e^-12 / exp(V/5).
enum { sKi, sNai, sCai, sCaSS, sCaSR, sRbar, sm, sh, sj, sxr1, sxr2, sxs, sr, ss, sd, sf, sf2, sfc };

struct TTDerived {      // parameter-only factors (host-computed per launch)
  double frt, rtf;      // F/RT, RT/F
  double sq_ko;         // sqrt(Ko / 5.4)
  double ecal0;         // exp(-30 F/RT)
  double gcal4;         // 4 GCaL F^2/RT
  double inaca_k;       // kNaCa / ((KmNai^3 + Nao^3)(KmCa + Cao))
  double nao3_alpha;    // Nao^3 alpha
  double inak_k;        // PNaK Ko / (Ko + KmK)
  double eks_num;       // Ko + pKNa Nao
  double vc_vss, vsr_vss, vsr_vc;
  double cap_2vssf, cap_2vcf, cap_vcf;
  double kup2;          // Kup^2
  double log_ko, log_nao, log_eks_num, log_cao;   // logs of the Nernst numerators
  // e^c of the constant offsets of the shared-slope voltage exponentials
  double x_m12, x_7, x_m3_2, x_m26_7, x_m4_5, x_m3, x_5_6, x_20_6, x_4, x_m4, x_1, x_2_5, x_3,
      x_20_7, x_1_3, x_5, x_m1;
};

struct TTVolt {         // factors that depend on V only (shared by both current evaluations)
  double ecal;          // exp(2 (V-15) F/RT)
  double enaca_a;       // exp(gamma V F/RT)
  double enaca_b;       // exp((gamma-1) V F/RT)
  double fnak;          // 1 / (1 + 0.1245 exp(-0.1 V F/RT) + 0.0353 exp(-V F/RT))
  double fpk;           // 1 / (1 + exp((25 - V)/5.98))
};

struct TTCur {
  double ina, ik1, ito, ikr, iks, ical, inaca, inak, ipca, ipk, ibna, ibca;
};

#define EXP(x) tc_exp((x), T)

// TCB_ION_FOLD = 1 (default): quotients of the model's rate expressions merged
// over a common denominator where only their combination is used (e.g. 1/tau_m
// = 1/(alpha_m beta_m) with alpha_m = 1/A, beta_m = 0.1/B1 + 0.1/B2 is
// 10 A B1 B2 / (B1 + B2)), so one reciprocal replaces up to four; every merged
// term is a sum of positive factors (no cancellation).  0: the literal forms.
#ifndef TCB_ION_FOLD
#define TCB_ION_FOLD 1
#endif

__device__ __forceinline__ double sig(double x, const Exp2Table* T) {  // 1 / (1 + e^x)
  return tc_rcp(1.0 + EXP(x));
}

__device__ __forceinline__ TTVolt tt_volt(double V, const TTParams& P, const TTDerived& D,
                                          const Exp2Table* T) {
  TTVolt f;
  const double E = EXP(V * D.frt);          // exp(V F/RT)
  const double iE = tc_rcp(E);
  f.ecal = E * E * D.ecal0;                 // exp(2 (V - 15) F/RT)
  f.enaca_a = EXP(P.gamma * V * D.frt);
  f.enaca_b = f.enaca_a * iE;               // exp((gamma - 1) V F/RT)
  f.fnak = tc_rcp(1.0 + 0.1245 * EXP(-0.1 * V * D.frt) + 0.0353 * iE);
  f.fpk = tc_rcp(1.0 + EXP((25.0 - V) * (1.0 / 5.98)));
  return f;
}

// The current evaluation runs twice per step (at u^k and u^{k+1}); TCB_CUR_NOINLINE
// keeps one copy of its code (instruction-cache experiment).
#ifndef TCB_CUR_NOINLINE
#define TCB_CUR_NOINLINE 0
#endif
#if TCB_CUR_NOINLINE
#define TCB_CUR_ATTR static __device__ __noinline__
#else
#define TCB_CUR_ATTR __device__ __forceinline__
#endif

TCB_CUR_ATTR TTCur tt_cur(double V, const double* u, const TTParams& P,
                                        const TTDerived& D, const TTVolt& f, const Exp2Table* T) {
  // Nernst potentials RT/F log(c_o / c_i) = RT/F (log c_o - log c_i): the
  // numerators' logs come from the host, the branch-free tc_log does the rest
  const double ek = D.rtf * (D.log_ko - tc_log(u[sKi], T));
  const double ena = D.rtf * (D.log_nao - tc_log(u[sNai], T));
  const double eks = D.rtf * (D.log_eks_num - tc_log(u[sKi] + P.pKNa * u[sNai], T));
  const double eca = 0.5 * D.rtf * (D.log_cao - tc_log(u[sCai], T));
  TTCur c;
  c.ina = P.GNa * u[sm] * u[sm] * u[sm] * u[sh] * u[sj] * (V - ena);
  {
    const double dvk = V - ek;
    const double e1 = EXP(0.1 * dvk);                 // exp(0.1 (V - EK))
    const double e2 = e1 * e1, e5 = e2 * e2 * e1;     // exp(0.5 (V - EK))
#if TCB_ION_FOLD
    // a1 = 0.1/Q, b1 = N e5/(1 + e5):  a1/(a1 + b1) = 0.1 (1 + e5) / (0.1 (1 + e5) + N e5 Q)
    const double Q = 1.0 + EXP(0.06 * (dvk - 200.0));
    const double N = 3.0 * EXP(0.0002 * (dvk + 100.0)) + e1 * D.x_m1;
    const double a1 = 0.1 * (1.0 + e5);
    c.ik1 = P.GK1 * (a1 * tc_rcp(fma(N * e5, Q, a1))) * dvk;
#else
    const double a1 = 0.1 * tc_rcp(1.0 + EXP(0.06 * (dvk - 200.0)));
    const double b1 = (3.0 * EXP(0.0002 * (dvk + 100.0)) + e1 * D.x_m1) *
                      tc_rcp(1.0 + tc_rcp(e5));
    c.ik1 = P.GK1 * (a1 * tc_rcp(a1 + b1)) * dvk;
#endif
  }
  c.ito = P.Gto * u[sr] * u[ss] * (V - ek);
  c.ikr = P.GKr * D.sq_ko * u[sxr1] * u[sxr2] * (V - ek);
  c.iks = P.GKs * u[sxs] * u[sxs] * (V - eks);
  c.ical = D.gcal4 * u[sd] * u[sf] * u[sf2] * u[sfc] * (V - 15.0) *
           (0.25 * u[sCaSS] * f.ecal - P.Cao) * tc_rcp(f.ecal - 1.0);
  {
    const double nai3 = u[sNai] * u[sNai] * u[sNai];
    c.inaca = D.inaca_k * (f.enaca_a * nai3 * P.Cao - f.enaca_b * D.nao3_alpha * u[sCai]) *
              tc_rcp(1.0 + P.ksat * f.enaca_b);
  }
  c.inak = D.inak_k * u[sNai] * f.fnak * tc_rcp(u[sNai] + P.KmNa);
  c.ipca = P.GpCa * u[sCai] * tc_rcp(P.KpCa + u[sCai]);
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
  const double bound = B * c * tc_rcp(c + K);
  const double bb = B - bound - delta - c + K;
  const double cc = K * (bound + delta + c);
  return 0.5 * (sqrt(bb * bb + 4.0 * cc) - bb);
}

// Rush-Larsen with the rate 1/tau given
__device__ __forceinline__ double rl_rate(double y, double yinf, double inv_tau, double dt,
                                          const Exp2Table* T) {
  return yinf - (yinf - y) * EXP(-dt * inv_tau);
}

// TCB_CUR_LOOP = 1: the two current evaluations of a step (at u^k for the
// concentration updates, at u^{k+1} for I_n, reading I2) are one copy of the
// code run twice (a two-pass loop) -- half the current code in the instruction
// cache (ncu r02c: 9 % of warp stalls were instruction fetch); 0 (default): two
// inlined copies -- the loop keeps the currents, states and V-factors live across
// the back edge and spills 630-720 bytes (ptxas, r02), and its code is larger.
#ifndef TCB_CUR_LOOP
#define TCB_CUR_LOOP 0
#endif

// Advances u in place; returns I_n(V, u^{k+1}).
__device__ __forceinline__ double tt_advance(double V, double* u, double dt, const TTParams& P,
                                             const TTDerived& D, const Exp2Table* T) {
  const TTVolt f = tt_volt(V, P, D, T);
#if TCB_CUR_LOOP
  TTCur c;
#pragma unroll 1
  for (int pass = 0;; ++pass) {
  c = tt_cur(V, u, P, D, f, T);
  if (pass) break;
#else
  const TTCur c = tt_cur(V, u, P, D, f, T);
#endif
  // -- calcium dynamics (currents and fluxes at (V^k, u^k)) --
  const double casr = u[sCaSR], cass = u[sCaSS], cai = u[sCai];
#if TCB_ION_FOLD
  // 1/(1 + (EC/casr)^2) = casr^2/(casr^2 + EC^2);  k1 = k1p/kcasr only enters
  // oo = k1 cass^2 rbar/(k3 + k1 cass^2) = k1p cass^2 rbar/(k3 kcasr + k1p cass^2);
  // iup = Vmaxup/(1 + Kup^2/cai^2) = Vmaxup cai^2/(cai^2 + Kup^2)
  const double casr2 = casr * casr;
  const double kcasr = P.maxsr - (P.maxsr - P.minsr) * (casr2 * tc_rcp(fma(P.EC, P.EC, casr2)));
  const double k2 = P.k2p * kcasr;
  const double rbar = u[sRbar] + dt * (P.k4 * (1.0 - u[sRbar]) - k2 * cass * u[sRbar]);
  const double k1c = P.k1p * cass * cass;
  const double oo = k1c * rbar * tc_rcp(fma(P.k3, kcasr, k1c));
  const double irel = P.Vrel * oo * (casr - cass);
  const double ileak = P.Vleak * (casr - cai);
  const double cai2 = cai * cai;
  const double iup = P.Vmaxup * cai2 * tc_rcp(cai2 + D.kup2);
#else
  const double ec = P.EC * tc_rcp(casr);
  const double kcasr = P.maxsr - (P.maxsr - P.minsr) * tc_rcp(1.0 + ec * ec);
  const double k1 = P.k1p * tc_rcp(kcasr), k2 = P.k2p * kcasr;
  const double rbar = u[sRbar] + dt * (P.k4 * (1.0 - u[sRbar]) - k2 * cass * u[sRbar]);
  const double oo = k1 * cass * cass * rbar * tc_rcp(P.k3 + k1 * cass * cass);
  const double irel = P.Vrel * oo * (casr - cass);
  const double ileak = P.Vleak * (casr - cai);
  const double iup = P.Vmaxup * tc_rcp(1.0 + D.kup2 * tc_rcp(cai * cai));
#endif
  const double ixfer = P.Vxfer * (cass - cai);
  const double nu_sr = dt * (iup - irel - ileak);
  const double nu_ss = dt * (-ixfer * D.vc_vss + irel * D.vsr_vss - c.ical * D.cap_2vssf);
  const double nu_i = dt * (-(c.ibca + c.ipca - 2.0 * c.inaca) * D.cap_2vcf -
                            (iup - ileak) * D.vsr_vc + ixfer);
  u[sRbar] = rbar;
  u[sCaSR] = buffered(casr, nu_sr, P.Bufsr, P.Kbufsr);
  u[sCaSS] = buffered(cass, nu_ss, P.Bufss, P.Kbufss);
  u[sCai] = buffered(cai, nu_i, P.Bufc, P.Kbufc);
  u[sNai] = u[sNai] - dt * (c.ina + c.ibna + 3.0 * c.inak + 3.0 * c.inaca) * D.cap_vcf;
  u[sKi] = u[sKi] - dt * (c.ik1 + c.ito + c.ikr + c.iks - 2.0 * c.inak + c.ipk) * D.cap_vcf;

  // -- gates, Rush-Larsen at V^k (fCass with the new CaSS) --
  // shared-slope exponentials
  const double e5 = EXP(V * (1.0 / 5.0)), ie5 = tc_rcp(e5);
  const double e7 = EXP(V * (1.0 / 7.0)), ie7 = tc_rcp(e7);
  const double e10 = EXP(V * (1.0 / 10.0)), ie10 = tc_rcp(e10);
  const double e20 = EXP(V * (1.0 / 20.0)), ie20 = tc_rcp(e20);
  const double e6 = EXP(V * (1.0 / 6.0)), ie6 = tc_rcp(e6);
  {
#if TCB_ION_FOLD
    // am = 1/A, bm = 0.1/B1 + 0.1/B2:  1/(am bm) = 10 A B1 B2/(B1 + B2)
    const double A = 1.0 + D.x_m12 * ie5;                // (-60-V)/5: e^-12
    const double B1 = 1.0 + D.x_7 * e5;                  // (V+35)/5: e^7
    const double B2 = 1.0 + EXP((V - 50.0) * (1.0 / 200.0));
    const double inv_tau = 10.0 * A * B1 * B2 * tc_rcp(B1 + B2);
#else
    const double am = tc_rcp(1.0 + D.x_m12 * ie5);     // (-60-V)/5: e^-12
    const double bm = 0.1 * tc_rcp(1.0 + D.x_7 * e5)    // (V+35)/5: e^7
                      + 0.1 * sig((V - 50.0) * (1.0 / 200.0), T);
    const double inv_tau = tc_rcp(am * bm);
#endif
    const double mi = sig((-56.86 - V) * (1.0 / 9.03), T);
    u[sm] = rl_rate(u[sm], mi * mi, inv_tau, dt, T);
  }
  {
    const double hi = sig((V + 71.55) * (1.0 / 7.43), T);
    const double hinf = hi * hi;
    double ah, bh, aj, bj;
    if (V >= -40.0) {
      ah = 0.0;
      bh = 0.77 * tc_rcp(0.13 * (1.0 + EXP(-(V + 10.66) * (1.0 / 11.1))));
      aj = 0.0;
      bj = 0.6 * EXP(0.057 * V) * tc_rcp(1.0 + D.x_m3_2 * ie10);   // e^-3.2
    } else {
      ah = 0.057 * EXP(-(V + 80.0) * (1.0 / 6.8));
      bh = 2.7 * EXP(0.079 * V) + 3.1e5 * EXP(0.3485 * V);
      aj = (-2.5428e4 * EXP(0.2444 * V) - 6.948e-6 * EXP(-0.04391 * V)) * (V + 37.78) *
           tc_rcp(1.0 + EXP(0.311 * (V + 79.23)));
      bj = 0.02424 * EXP(-0.01052 * V) * tc_rcp(1.0 + EXP(-0.1378 * (V + 40.14)));
    }
    u[sh] = rl_rate(u[sh], hinf, ah + bh, dt, T);
    u[sj] = rl_rate(u[sj], hinf, aj + bj, dt, T);
  }
  {
    const double xr1_inf = tc_rcp(1.0 + D.x_m26_7 * ie7);       // (-26-V)/7: e^(-26/7)
#if TCB_ION_FOLD
    // a = 450/A, b = 6/B:  1/(a b) = A B/2700
    const double inv_tau = (1.0 + D.x_m4_5 * ie10) *            // (-45-V)/10: e^-4.5
                           (1.0 + EXP((V + 30.0) * (1.0 / 11.5))) * (1.0 / 2700.0);
#else
    const double a = 450.0 * tc_rcp(1.0 + D.x_m4_5 * ie10);    // (-45-V)/10: e^-4.5
    const double b = 6.0 * sig((V + 30.0) * (1.0 / 11.5), T);
    const double inv_tau = tc_rcp(a * b);
#endif
    u[sxr1] = rl_rate(u[sxr1], xr1_inf, inv_tau, dt, T);
  }
  {
    const double xr2_inf = sig((V + 88.0) * (1.0 / 24.0), T);
#if TCB_ION_FOLD
    // a = 3/A, b = 1.12/B:  1/(a b) = A B/3.36
    const double inv_tau = (1.0 + D.x_m3 * ie20) * (1.0 + D.x_m3 * e20) * (1.0 / 3.36);
#else
    const double a = 3.0 * tc_rcp(1.0 + D.x_m3 * ie20);      // (-60-V)/20: e^-3
    const double b = 1.12 * tc_rcp(1.0 + D.x_m3 * e20);      // (V-60)/20: e^-3
    const double inv_tau = tc_rcp(a * b);
#endif
    u[sxr2] = rl_rate(u[sxr2], xr2_inf, inv_tau, dt, T);
  }
  {
    const double xs_inf = sig((-5.0 - V) * (1.0 / 14.0), T);
#if TCB_ION_FOLD
    // tau = 1400/(sqrt(C) E) + 80, E = 1 + e^((V-35)/15):  1/tau = E/(1400/sqrt(C) + 80 E)
    const double E = 1.0 + EXP((V - 35.0) * (1.0 / 15.0));
    const double inv_tau = E * tc_rcp(fma(1400.0, rsqrt(1.0 + D.x_5_6 * ie6), 80.0 * E));  // (5-V)/6: e^(5/6)
#else
    const double tau = 1400.0 * tc_rcp(sqrt(1.0 + D.x_5_6 * ie6))  // (5-V)/6: e^(5/6)
                       * sig((V - 35.0) * (1.0 / 15.0), T) + 80.0;
    const double inv_tau = tc_rcp(tau);
#endif
    u[sxs] = rl_rate(u[sxs], xs_inf, inv_tau, dt, T);
  }
  {
    const double r_inf = tc_rcp(1.0 + D.x_20_6 * ie6);              // (20-V)/6: e^(10/3)
    const double d40 = V + 40.0;
    const double tau = 9.5 * EXP(-d40 * d40 * (1.0 / 1800.0)) + 0.8;
    u[sr] = rl_rate(u[sr], r_inf, tc_rcp(tau), dt, T);
  }
  {
    const double s_inf = tc_rcp(1.0 + D.x_4 * e5);              // (V+20)/5: e^4
    const double d45 = V + 45.0;
#if TCB_ION_FOLD
    // tau = G + 5/S:  1/tau = S/(G S + 5)
    const double S = 1.0 + D.x_m4 * e5;                          // (V-20)/5: e^-4
    const double G = 85.0 * EXP(-d45 * d45 * (1.0 / 320.0)) + 3.0;
    const double inv_tau = S * tc_rcp(fma(G, S, 5.0));
#else
    const double tau = 85.0 * EXP(-d45 * d45 * (1.0 / 320.0)) +
                       5.0 * tc_rcp(1.0 + D.x_m4 * e5) + 3.0;   // (V-20)/5: e^-4
    const double inv_tau = tc_rcp(tau);
#endif
    u[ss] = rl_rate(u[ss], s_inf, inv_tau, dt, T);
  }
  {
    const double d_inf = sig((-8.0 - V) * (1.0 / 7.5), T);
#if TCB_ION_FOLD
    // tau = (1.4/S1 + 0.25)(1.4/D2) + 1/D3:
    //   1/tau = S1 D2 D3 / (1.4 D3 (1.4 + 0.25 S1) + S1 D2)
    const double S1 = 1.0 + EXP((-35.0 - V) * (1.0 / 13.0));
    const double D2 = 1.0 + D.x_1 * e5;                          // (V+5)/5: e
    const double D3 = 1.0 + D.x_2_5 * ie20;                      // (50-V)/20: e^2.5
    const double S1D2 = S1 * D2;
    const double inv_tau = S1D2 * D3 * tc_rcp(fma(1.4 * D3, fma(0.25, S1, 1.4), S1D2));
#else
    const double tau = (1.4 * sig((-35.0 - V) * (1.0 / 13.0), T) + 0.25) *
                           (1.4 * tc_rcp(1.0 + D.x_1 * e5)) +     // (V+5)/5: e
                       tc_rcp(1.0 + D.x_2_5 * ie20);               // (50-V)/20: e^2.5
    const double inv_tau = tc_rcp(tau);
#endif
    u[sd] = rl_rate(u[sd], d_inf, inv_tau, dt, T);
  }
  const double s30 = tc_rcp(1.0 + D.x_3 * e10);                 // (V+30)/10: e^3
  {
    const double f_inf = tc_rcp(1.0 + D.x_20_7 * e7);                // (V+20)/7: e^(20/7)
    const double d27 = V + 27.0;
#if TCB_ION_FOLD
    // tau = G + 200/F1:  1/tau = F1/(G F1 + 200)
    const double F1 = 1.0 + D.x_1_3 * ie10;                      // (13-V)/10: e^1.3
    const double G = 1102.5 * EXP(-d27 * d27 * (1.0 / 225.0)) + 180.0 * s30 + 20.0;
    const double inv_tau = F1 * tc_rcp(fma(G, F1, 200.0));
#else
    const double tau = 1102.5 * EXP(-d27 * d27 * (1.0 / 225.0)) +
                       200.0 * tc_rcp(1.0 + D.x_1_3 * ie10) +      // (13-V)/10: e^1.3
                       180.0 * s30 + 20.0;
    const double inv_tau = tc_rcp(tau);
#endif
    u[sf] = rl_rate(u[sf], f_inf, inv_tau, dt, T);
  }
  {
    const double f2_inf = 0.67 * tc_rcp(1.0 + D.x_5 * e7) + 0.33; // (V+35)/7: e^5
    const double d25 = V + 25.0;
#if TCB_ION_FOLD
    // tau = G + 31/F2:  1/tau = F2/(G F2 + 31)
    const double F2 = 1.0 + D.x_2_5 * ie10;                      // (25-V)/10: e^2.5
    const double G = 600.0 * EXP(-d25 * d25 * (1.0 / 170.0)) + 16.0 * s30;
    const double inv_tau = F2 * tc_rcp(fma(G, F2, 31.0));
#else
    const double tau = 600.0 * EXP(-d25 * d25 * (1.0 / 170.0)) +
                       31.0 * tc_rcp(1.0 + D.x_2_5 * ie10) +        // (25-V)/10: e^2.5
                       16.0 * s30;
    const double inv_tau = tc_rcp(tau);
#endif
    u[sf2] = rl_rate(u[sf2], f2_inf, inv_tau, dt, T);
  }
  {
    const double q = u[sCaSS] * (1.0 / 0.05);
    const double den = tc_rcp(1.0 + q * q);
    u[sfc] = rl_rate(u[sfc], 0.6 * den + 0.4, tc_rcp(80.0 * den + 2.0), dt, T);
  }
#if TCB_CUR_LOOP
  }
  return tt_total(c);  // I_ion(V^k, u^{k+1}) (reading I2): the second pass
#else
  return tt_total(tt_cur(V, u, P, D, f, T));  // I_ion(V^k, u^{k+1}) (reading I2)
#endif
}

// ------------------------------------------------------------------ Mitchell-Schaeffer
struct MSDerived {  // reciprocals of the time constants (host-computed)
  double span, inv_open, inv_close, inv_in, inv_out;
};

// Advances the gate h in place (forward Euler at V^k); returns I_n(V^k, h^{k+1}).
__device__ __forceinline__ double ms_advance(double V, double* h_io, double dt, const MSParams& P,
                                             const MSDerived& D) {
  // the gate decision uses the same correctly rounded division as the oracle
  const double v = (V - P.V_min) / D.span;
  double h = *h_io;
  h = (v < P.v_gate) ? h + dt * ((1.0 - h) * D.inv_open) : h + dt * (-h * D.inv_close);
  *h_io = h;
  return -D.span * (h * v * v * (1.0 - v) * D.inv_in - v * D.inv_out);
}


// ------------------------------------------------------------------ CRN 1998 (atrial)
// Courtemanche, Ramirez & Nattel 1998 (named among the paper's models, P:98;
// SURVEY 8f row f4; reading I6), the same equations as the oracle
// (oracle.c 6c): Rush-Larsen for the 15 gates, forward Euler for Na_i, K_i,
// Ca_i (instantaneous TRPN/CMDN buffering factor), Ca_up, Ca_rel -- all at
// (V^k, u^k); I_n = I_ion(V^k, u^{k+1}) (reading I2).  20 states in the order
// Nai Ki Cai Caup Carel m h j oa oi ua ui xr xs d f fCa u v w.
enum { cNai, cKi, cCai, cCaup, cCarel, cm, chh, cj, coa, coi, cua, cui, cxr, cxs, cd, cf, cfCa,
       cu, cv, cw };

struct CRNDerived {   // parameter-only factors (host-computed)
  double rtf, frt, sigma_k;   // RT/F, F/RT, 0.0365 sigma
  double cm_vif, cm_2vif;     // Cm / (Vi F), Cm / (2 Vi F)
  double inak_k;              // INaK_max Ko / (Ko + KmKo)
  double inaca_k;             // INaCa_max / ((KmNa^3 + Nao^3)(KmCa + Cao))
  double nao3, inv_tautr, iupleak_k, vup_vi, vrel_vi, vrel_vup, inv_kq10, kq10, inv_tauu, fn_c;
  double log_nao, log_ko, log_cao;   // logs of the Nernst numerators
};

struct CRNCur {
  double ina, ik1, ito, ikur, ikr, iks, ical, inak, inaca, ibna, ibca, ipca;
};

TCB_CUR_ATTR CRNCur crn_cur(double V, const double* u, const CRNParams& P,
                                          const CRNDerived& D, const Exp2Table* T) {
  CRNCur c;
  const double nai = u[cNai], ki = u[cKi], cai = u[cCai];
  const double ena = D.rtf * (D.log_nao - tc_log(nai, T)), ek = D.rtf * (D.log_ko - tc_log(ki, T));
  const double eca = 0.5 * D.rtf * (D.log_cao - tc_log(cai, T));
  const double m = u[cm], oa = u[coa], ua = u[cua], xs = u[cxs];
  c.ina = P.gNa * m * m * m * u[chh] * u[cj] * (V - ena);
  c.ik1 = P.gK1 * (V - ek) * tc_rcp(1.0 + EXP(0.07 * (V + 80.0)));
  c.ito = P.gto * oa * oa * oa * u[coi] * (V - ek);
  const double gkur = 0.005 + 0.05 * tc_rcp(1.0 + EXP((V - 15.0) * (1.0 / -13.0)));
  c.ikur = gkur * ua * ua * ua * u[cui] * (V - ek);
  c.ikr = P.gKr * u[cxr] * (V - ek) * tc_rcp(1.0 + EXP((V + 15.0) * (1.0 / 22.4)));
  c.iks = P.gKs * xs * xs * (V - ek);
  c.ical = P.gCaL * u[cd] * u[cf] * u[cfCa] * (V - 65.0);
  const double e = EXP(-V * D.frt);                         // exp(-F V / RT)
  const double fnak = tc_rcp(1.0 + 0.1245 * EXP(-0.1 * V * D.frt) + D.sigma_k * e);
  const double q = P.KmNai * tc_rcp(nai);
  c.inak = D.inak_k * fnak * tc_rcp(1.0 + q * sqrt(q));
  const double eg = EXP(P.gamma * V * D.frt), eg1 = eg * e;  // exp((gamma-1) F V / RT)
  c.inaca = D.inaca_k * (eg * nai * nai * nai * P.Cao - eg1 * D.nao3 * cai) *
            tc_rcp(1.0 + P.ksat * eg1);
  c.ibna = P.gbNa * (V - ena);
  c.ibca = P.gbCa * (V - eca);
  c.ipca = P.IpCamax * cai * tc_rcp(0.0005 + cai);
  return c;
}

__device__ __forceinline__ double crn_total(const CRNCur& c) {
  return c.ina + c.ik1 + c.ito + c.ikur + c.ikr + c.iks + c.ical + c.inak + c.inaca + c.ibna +
         c.ibca + c.ipca;
}

// 1 / (1 + e^x) for the release-flux sigmoids, whose arguments (Fn / 1.367e-15)
// reach |x| ~ 1e4: outside |x| <= 700 (the range of tc_exp) the value is 0 or 1
// to double precision (what 1/(1 + exp(x)) gives with libm: inf -> 0, 0 -> 1).
__device__ __forceinline__ double crn_sig(double x, const Exp2Table* T) {
  if (x > 700.0) return 0.0;
  if (x < -700.0) return 1.0;
  return tc_rcp(1.0 + EXP(x));
}

__device__ __forceinline__ double rl_tau(double y, double yinf, double tau, double dt,
                                         const Exp2Table* T) {
  return yinf - (yinf - y) * EXP(-dt * tc_rcp(tau));
}

// Gate with tau = 1/R, given as the rate R (TCB_ION_FOLD: 1/tau = R without the
// reciprocal of a reciprocal) or, literally, as tau = 1/R.
#if TCB_ION_FOLD
#define CRN_RL_RATE(y, yinf, R) rl_rate((y), (yinf), (R), dt, T)
#else
#define CRN_RL_RATE(y, yinf, R) rl_tau((y), (yinf), tc_rcp(R), dt, T)
#endif

// Advances u in place; returns I_n(V, u^{k+1}).
__device__ __forceinline__ double crn_advance(double V, double* u, double dt, const CRNParams& P,
                                              const CRNDerived& D, const Exp2Table* T) {
#if TCB_CUR_LOOP
  CRNCur c;
#pragma unroll 1
  for (int pass = 0;; ++pass) {
  c = crn_cur(V, u, P, D, T);
  if (pass) break;
#else
  const CRNCur c = crn_cur(V, u, P, D, T);
#endif
  const double cai = u[cCai], caup = u[cCaup], carel = u[cCarel];
  const double irel = P.Krel * u[cu] * u[cu] * u[cv] * u[cw] * (carel - cai);
  const double itr = (caup - carel) * D.inv_tautr;
  const double iupleak = D.iupleak_k * caup;
#if TCB_ION_FOLD
  const double iup = P.Iupmax * cai * tc_rcp(cai + P.Kup);     // Iupmax/(1 + Kup/cai)
#else
  const double iup = P.Iupmax * tc_rcp(1.0 + P.Kup * tc_rcp(cai));
#endif
  // gates at (V^k, u^k), each Rush-Larsen update applied as soon as its
  // steady state and time constant are known (nothing below reads a gate)
  {
    double a, b, ti;
    a = (V == -47.13) ? 3.2 : 0.32 * (V + 47.13) * tc_rcp(1.0 - EXP(-0.1 * (V + 47.13)));
    b = 0.08 * EXP(V * (-1.0 / 11.0));
    ti = tc_rcp(a + b);
    u[cm] = CRN_RL_RATE(u[cm], a * ti, a + b);
    if (V < -40.0) {
      a = 0.135 * EXP((V + 80.0) * (1.0 / -6.8));
      b = 3.56 * EXP(0.079 * V) + 3.1e5 * EXP(0.35 * V);
    } else {
      a = 0.0;
      b = tc_rcp(0.13 * (1.0 + EXP((V + 10.66) * (1.0 / -11.1))));
    }
    ti = tc_rcp(a + b);
    u[chh] = CRN_RL_RATE(u[chh], a * ti, a + b);
    if (V < -40.0) {
      a = (-127140.0 * EXP(0.2444 * V) - 3.474e-5 * EXP(-0.04391 * V)) * (V + 37.78) *
          tc_rcp(1.0 + EXP(0.311 * (V + 79.23)));
      b = 0.1212 * EXP(-0.01052 * V) * tc_rcp(1.0 + EXP(-0.1378 * (V + 40.14)));
    } else {
      a = 0.0;
      b = 0.3 * EXP(-2.535e-7 * V) * tc_rcp(1.0 + EXP(-0.1 * (V + 32.0)));
    }
    ti = tc_rcp(a + b);
    u[cj] = CRN_RL_RATE(u[cj], a * ti, a + b);
    // oa and ua share their rate functions
    a = 0.65 * tc_rcp(EXP((V + 10.0) * (1.0 / -8.5)) + EXP((V - 30.0) * (1.0 / -59.0)));
    b = 0.65 * tc_rcp(2.5 + EXP((V + 82.0) * (1.0 / 17.0)));
    const double rq = (a + b) * D.kq10;                       // 1/tau = (a + b) KQ10
    u[coa] = CRN_RL_RATE(u[coa], tc_rcp(1.0 + EXP((V + 20.47) * (1.0 / -17.54))), rq);
    u[cua] = CRN_RL_RATE(u[cua], tc_rcp(1.0 + EXP((V + 30.3) * (1.0 / -9.6))), rq);
    a = tc_rcp(18.53 + EXP((V + 113.7) * (1.0 / 10.95)));
    b = tc_rcp(35.56 + EXP((V + 1.26) * (1.0 / -7.44)));
    u[coi] = CRN_RL_RATE(u[coi], tc_rcp(1.0 + EXP((V + 43.1) * (1.0 / 5.3))), (a + b) * D.kq10);
    a = tc_rcp(21.0 + EXP((V - 185.0) * (1.0 / -28.0)));
    b = EXP((V - 158.0) * (1.0 / 16.0));
    u[cui] = CRN_RL_RATE(u[cui], tc_rcp(1.0 + EXP((V - 99.45) * (1.0 / 27.48))), (a + b) * D.kq10);
    a = (V == -14.1) ? 0.0015 : 0.0003 * (V + 14.1) * tc_rcp(1.0 - EXP((V + 14.1) * (1.0 / -5.0)));
    b = (V == 3.3328) ? 3.7836118e-4
                      : 7.3898e-5 * (V - 3.3328) * tc_rcp(EXP((V - 3.3328) * (1.0 / 5.1237)) - 1.0);
    u[cxr] = CRN_RL_RATE(u[cxr], tc_rcp(1.0 + EXP((V + 14.1) * (1.0 / -6.5))), a + b);
    a = (V == 19.9) ? 0.00068 : 4e-5 * (V - 19.9) * tc_rcp(1.0 - EXP((V - 19.9) * (1.0 / -17.0)));
    b = (V == 19.9) ? 0.000315 : 3.5e-5 * (V - 19.9) * tc_rcp(EXP((V - 19.9) * (1.0 / 9.0)) - 1.0);
#if TCB_ION_FOLD
    u[cxs] = rl_rate(u[cxs], rsqrt(1.0 + EXP((V - 19.9) * (1.0 / -12.7))), 2.0 * (a + b), dt, T);
#else
    u[cxs] = rl_tau(u[cxs], tc_rcp(sqrt(1.0 + EXP((V - 19.9) * (1.0 / -12.7)))), 0.5 * tc_rcp(a + b), dt, T);
#endif
    {
      const double ed = EXP((V + 10.0) * (1.0 / -6.24));
      const double td = (V == -10.0) ? 4.579 * tc_rcp(1.0 + ed)
                                     : (1.0 - ed) * tc_rcp(0.035 * (V + 10.0) * (1.0 + ed));
      u[cd] = rl_tau(u[cd], tc_rcp(1.0 + EXP((V + 10.0) * (1.0 / -8.0))), td, dt, T);
    }
    {
      const double ef = EXP(-(V + 28.0) * (1.0 / 6.9));
      const double v10 = V + 10.0;
      // tau = 9/X
      u[cf] = CRN_RL_RATE(u[cf], ef * tc_rcp(1.0 + ef),
                          (0.0197 * EXP(-0.0337 * 0.0337 * v10 * v10) + 0.02) * (1.0 / 9.0));
    }
    u[cfCa] = CRN_RL_RATE(u[cfCa], tc_rcp(1.0 + cai * (1.0 / 0.00035)), 0.5);   // tau = 2 ms
    const double fn = 1000.0 * (1e-15 * P.Vrel * irel - D.fn_c * (0.5 * c.ical - 0.2 * c.inaca));
    const double su = crn_sig(-(fn - 3.4175e-13) * (1.0 / 13.67e-16), T);
    u[cu] = CRN_RL_RATE(u[cu], su, D.inv_tauu);
    u[cv] = rl_tau(u[cv], 1.0 - crn_sig(-(fn - 6.835e-14) * (1.0 / 13.67e-16), T), 1.91 + 2.09 * su, dt, T);
    const double ew = EXP(-(V - 7.9) * (1.0 / 5.0));
    const double tw = (V == 7.9) ? 6.0 * 0.2 / 1.3 : 6.0 * (1.0 - ew) * tc_rcp((1.0 + 0.3 * ew) * (V - 7.9));
    u[cw] = rl_tau(u[cw], 1.0 - tc_rcp(1.0 + EXP(-(V - 40.0) * (1.0 / 17.0))), tw, dt, T);
  }
  // concentrations: forward Euler at (V^k, u^k)
  const double dnai = (-3.0 * c.inak - 3.0 * c.inaca - c.ibna - c.ina) * D.cm_vif;
  const double dki = (2.0 * c.inak - c.ik1 - c.ito - c.ikur - c.ikr - c.iks) * D.cm_vif;
  const double b1 = (2.0 * c.inaca - c.ipca - c.ical - c.ibca) * D.cm_2vif +
                    (iupleak - iup) * D.vup_vi + irel * D.vrel_vi;
  const double t1 = cai + P.KmTRPN, t2 = cai + P.KmCMDN;
  const double b2 = 1.0 + P.TRPNmax * P.KmTRPN * tc_rcp(t1 * t1) + P.CMDNmax * P.KmCMDN * tc_rcp(t2 * t2);
  const double dcaup = iup - iupleak - itr * D.vrel_vup;
  const double t3 = carel + P.KmCSQN;
  const double dcarel = (itr - irel) * tc_rcp(1.0 + P.CSQNmax * P.KmCSQN * tc_rcp(t3 * t3));
  u[cNai] += dt * dnai;
  u[cKi] += dt * dki;
  u[cCai] += dt * (b1 * tc_rcp(b2));
  u[cCaup] += dt * dcaup;
  u[cCarel] += dt * dcarel;
#if TCB_CUR_LOOP
  }
  return crn_total(c);  // I_ion(V^k, u^{k+1}) (reading I2): the second pass
#else
  return crn_total(crn_cur(V, u, P, D, T));  // I_ion(V^k, u^{k+1}) (reading I2)
#endif
}

TTDerived tt_derived(const TTParams& P);
MSDerived ms_derived(const MSParams& P);
CRNDerived crn_derived(const CRNParams& P);

}  // namespace tcb
