// fp64math.cuh -- branch-free FP64 exp / reciprocal / division for the ionic
// kernels.  The CUDA math library versions carry
// special-case branches and materialise their 64-bit constants through uniform
// registers (~20 % of the TT2006 kernel's instructions were UMOV); these
// versions keep the FP64 pipe busy instead.  Accuracy ~1 ulp for |x| < 708;
// below, 0 (exp_range).
#pragma once

#include <cstdint>

namespace tcb {

// Exp table size: TCB_EXP_TAB = 256 (default): 256-entry table and a degree-4
// polynomial (|r| <= ln2/512, truncation r^5/120 < 3.8e-17 relative); 64: degree 5
// (r01 default, truncation < 3.5e-17); 32: degree 6.
// 1024 (default since r02l): degree 3 (|r| <= ln2/2048, truncation r^4/24 <
// 5.8e-16 relative, ~3 ulp).  Measured with TCB_EXP_CW1 (profiles/r02l_exp_ionic.txt,
// ionic cycles = ms x SM MHz at 10 M nodes): TT2006 1.91k -> 1.78k, CRN 2.14k -> 2.06k.
#ifndef TCB_EXP_TAB
#define TCB_EXP_TAB 1024
#endif
constexpr int kExpTab = TCB_EXP_TAB;
constexpr int kExpShift = TCB_EXP_TAB == 1024 ? 10 : TCB_EXP_TAB == 256 ? 8 : (TCB_EXP_TAB == 64 ? 6 : 5);
// TCB_EXP_CW1 = 1 (default): one-constant argument reduction r = x - k ln2/N
// (ln2/N rounded to double): error |x| 2^-54 relative, < 6e-15 for the |x| <= 100
// of the ionic models' exponentials (below -708 the result is 0 anyway); 0:
// Cody-Waite hi/lo pair, exact for |k| < 2^20.
#ifndef TCB_EXP_CW1
#define TCB_EXP_CW1 1
#endif
// TCB_EXP_IRANGE = 1 (experiment, unsafe): the x >= -708 range test on the
// integer k (INT pipe) instead of a DSETP (FP64 pipe) -- k wraps for |x| > ~2e6
// (Rush-Larsen exponents at V = -150 mV, dt 0.05: NaN in
// test_ionic_voltage_range_one_step), so the default keeps the FP64 compare.
#ifndef TCB_EXP_IRANGE
#define TCB_EXP_IRANGE 0
#endif

constexpr int kLogTab = 64;

// Per-CTA shared-memory tables of the branch-free exp and log:
//   t[j]  = 2^(j/N), j = 0..N-1 (tc_exp);
//   lg[j] = {c_j, -log c_j}, c_j = 1/(1 + (j + 1/2)/64) (tc_log; one 16-byte load).
struct Exp2Table {
  double t[kExpTab];
  double2 lg[kLogTab];
};

// Fill the tables (libm exp2 / log, once per device: ionic.cu device_tables).
__device__ __forceinline__ void exp2_table_fill(Exp2Table* T) {
  for (int j = threadIdx.x; j < kExpTab; j += blockDim.x) T->t[j] = exp2((double)j / kExpTab);
  for (int j = threadIdx.x; j < kLogTab; j += blockDim.x) {
    const double c = 1.0 / (1.0 + (j + 0.5) / kLogTab);
    T->lg[j] = make_double2(c, -log(c));
  }
}

// Per-CTA shared-memory copy of the device tables G (long-running kernels).
__device__ __forceinline__ void exp2_table_init(Exp2Table* T, const Exp2Table* __restrict__ G) {
  const double* g = reinterpret_cast<const double*>(G);
  double* t = reinterpret_cast<double*>(T);
  for (int j = threadIdx.x; j < (int)(sizeof(Exp2Table) / 8); j += blockDim.x) t[j] = __ldg(g + j);
  __syncthreads();
}

// log(x) for positive normal x, branch-free (replaces libm log: ~80 SASS
// instructions with special-case branches and 29 FP64 ops -> ~20 and 12).
//   x = 2^e m, m in [1, 2);  j = top 6 mantissa bits;  r = m c_j - 1, |r| < 2^-7
//   log x = e ln2 + (-log c_j) + log(1 + r),  log(1 + r) by its degree-7 Taylor
//   polynomial (truncation |r|^8/8 < 1.7e-18 absolute, < 2.2e-16 of log(1 + r)).
//   Accuracy ~2 ulp.  NaN / inf in,
//   NaN out (the x * 0 term); zero, negative and denormal inputs are not
//   handled (concentrations of the ionic models; a blown-up state still trips
//   the NaN checks through V).
__device__ __forceinline__ double tc_log(double x, const Exp2Table* __restrict__ T) {
  const int hi = __double2hiint(x);
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(x));
  const double2 cl = T->lg[(hi >> 14) & 63];
  // e + 2^52 + 1023 as a double (biased exponent in the low word), x*0 carries NaN
  const double eb = fma(x, 0.0, __hiloint2double(0x43300000, (unsigned)hi >> 20));
  const double e = eb - 4503599627371519.0;             // - (2^52 + 1023)
  const double r = fma(m, cl.x, -1.0);
  double q = 1.0 / 7.0;
  q = fma(q, r, -1.0 / 6.0);
  q = fma(q, r, 0.2);
  q = fma(q, r, -0.25);
  q = fma(q, r, 1.0 / 3.0);
  q = fma(q, r, -0.5);
  const double l1p = fma(q, r * r, r);
  const double kLn2Hi = 6.93147180369123816490e-01;     // 0x3FE62E42FEE00000: e * hi exact
  const double kLn2Lo = 1.90821492927058770002e-10;
  return fma(e, kLn2Hi, cl.y) + fma(e, kLn2Lo, l1p);
}

// Range.  The scale 2^m is added to the exponent field of v = 2^(j/N) P(r),
// which wraps for x < -708 (into the sign bit: the TT2006 m gate near -99 mV at
// dt 0.05 gave -1e300, Rush-Larsen e^{-dt/tau} with tiny tau) and, for
// |x| > 2.3e7 (V ~ -150 mV at dt 0.1), the integer m itself overflows.  So
// anything but x >= -708 returns 0 (one FP64 compare and two selects, the cost
// the former NaN test had) and m is clamped to <= 1023 (integer min; above
// x ~ 709.8 a finite value below 2^1024 instead of inf).  Accepted: e^x for
// -745 < x < -708 is 0 instead of a denormal (< 3.3e-308); NaN x gives 0 (a NaN
// state still reaches the currents directly -- y in yinf - (yinf - y) e^x, V in
// g (V - E) -- and the PCG NaN test); x > 2.3e7 is not handled.
// TCB_EXP_SCALE (experiment): scale by a DMUL with 2^m built from the clamped m,
// m in [-1022, 1023] (no compare / selects; e^x below -708 is a value below
// 2.3e-308 instead of 0, NaN x stays NaN).
#ifndef TCB_EXP_SCALE
#define TCB_EXP_SCALE 0
#endif
__device__ __forceinline__ double exp_range(double x, double v, int m, int k) {
#if TCB_EXP_SCALE
  const int mc = max(min(m, 1023), -1022);
  return v * __hiloint2double((mc + 1023) << 20, 0);
#else
  const double s = __hiloint2double(__double2hiint(v) + (min(m, 1023) << 20), __double2loint(v));
#if TCB_EXP_IRANGE
  // k = round(x N / ln2): x >= -708 <=> k >= ceil(-708 N / ln2) up to rounding at the edge
  constexpr int kMin = (int)(-708.0 * kExpTab / 0.69314718055994530942);
  (void)x;
  return k >= kMin ? s : 0.0;
#else
  (void)k;
  return x >= -708.0 ? s : 0.0;
#endif
#endif
}

// e^x = 2^m 2^(j/N) P(r),  x = (N m + j) ln2/N + r,  |r| <= ln2/(2N) (Cody-Waite);
// N = 64 with P of degree 5 (default) or N = 32 with degree 6.
// TCB_EXP_NOINLINE (experiment): one out-of-line copy instead of ~40 inlined ones
// per ionic kernel (instruction-cache pressure vs call overhead): measured slower,
// 1.76 vs 1.37 ms (TT2006, 10 M nodes).
#ifndef TCB_EXP_NOINLINE
#define TCB_EXP_NOINLINE 0
#endif
#if TCB_EXP_NOINLINE
static __device__ __noinline__ double tc_exp(double x, const Exp2Table* __restrict__ T) {
#else
__device__ __forceinline__ double tc_exp(double x, const Exp2Table* __restrict__ T) {
#endif
  const double kShift = 6755399441055744.0;             // 1.5 * 2^52
  // x = (N m + j) ln2/N + r (Cody-Waite: ln2/N in a hi part exact for |k| < 2^20 and a lo part)
  const double kInvLn2N = kExpTab / 0.69314718055994530942;
  const double kLn2N_hi = 0.69314718036912381649 / kExpTab;   // ln2_hi (0x3FE62E42FEE00000) / N
  const double kLn2N_lo = 1.9082149292705877000e-10 / kExpTab;
  const double kd = fma(x, kInvLn2N, kShift);
  const int k = __double2loint(kd);                     // round-to-nearest integer
  const double kf = kd - kShift;
#if TCB_EXP_CW1
  const double r = fma(-kf, 0.69314718055994530942 / kExpTab, x);
  (void)kLn2N_hi;
  (void)kLn2N_lo;
#else
  double r = fma(-kf, kLn2N_hi, x);
  r = fma(-kf, kLn2N_lo, r);
#endif
#if TCB_EXP_TAB == 1024
  double p = 1.0 / 6.0;
#elif TCB_EXP_TAB == 256
  double p = 1.0 / 24.0;
  p = fma(p, r, 1.0 / 6.0);
#elif TCB_EXP_TAB == 64
  double p = 1.0 / 120.0;
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
#else
  double p = 1.0 / 720.0;
  p = fma(p, r, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
#endif
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double v = T->t[k & (kExpTab - 1)] * p;
  return exp_range(x, v, k >> kExpShift, k);
}

// 1/b: hardware approximation r0 (MUFU.RCP64H, ~2^-22 relative) refined by
// r = r0 (1 + e + e^2), e = 1 - b r0 (error e^3 ~ 2^-66 plus rounding: as
// accurate as two Newton steps, 3 dependent DFMA instead of 4).
// TCB_RCP_NEWTON2 = 1: the two Newton steps of r01.
#ifndef TCB_RCP_NEWTON2
#define TCB_RCP_NEWTON2 0
#endif
__device__ __forceinline__ double tc_rcp(double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
#if TCB_RCP_NEWTON2
  double e = fma(-b, r, 1.0);
  r = fma(r, e, r);
  e = fma(-b, r, 1.0);
  return fma(r, e, r);
#else
  const double e = fma(-b, r, 1.0);
  return fma(r, fma(e, e, e), r);
#endif
}

// a/b with one residual correction.
__device__ __forceinline__ double tc_div(double a, double b) {
  const double r = tc_rcp(b);
  const double q = a * r;
  return fma(r, fma(-b, q, a), q);
}

}  // namespace tcb
