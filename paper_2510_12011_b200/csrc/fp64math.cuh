// fp64math.cuh -- branch-free FP64 exp / reciprocal / division for the ionic
// kernels.  The CUDA math library versions carry
// special-case branches and materialise their 64-bit constants through uniform
// registers (~20 % of the TT2006 kernel's instructions were UMOV); these
// versions keep the FP64 pipe busy instead.  Accuracy ~1 ulp over the range
// the cell models use (|x| < 700); NaN propagates (blow-up detection).
#pragma once

#include <cstdint>

namespace tcb {

// 2^(j/32), j = 0..31, filled once per CTA into shared memory.
struct Exp2Table {
  double t[32];
};

__device__ __forceinline__ void exp2_table_init(Exp2Table* T) {
  for (int j = threadIdx.x; j < 32; j += blockDim.x) T->t[j] = exp2((double)j / 32.0);
  __syncthreads();
}

// e^x = 2^m 2^(j/32) P6(r),  x = (32 m + j) ln2/32 + r,  |r| <= ln2/64 (Cody-Waite).
__device__ __forceinline__ double tc_exp(double x, const Exp2Table* __restrict__ T) {
  const double kShift = 6755399441055744.0;             // 1.5 * 2^52
  const double kInvLn2_32 = 46.16624130844683;          // 32 / ln 2
  const double kLn2_32_hi = 0.02166084938653512;        // (ln 2)_hi / 32, 32 significant bits
  const double kLn2_32_lo = 5.9631716539705866e-12;     // (ln 2)_lo / 32
  const double kd = fma(x, kInvLn2_32, kShift);
  const int k = __double2loint(kd);                     // round-to-nearest integer
  const double kf = kd - kShift;
  double r = fma(-kf, kLn2_32_hi, x);
  r = fma(-kf, kLn2_32_lo, r);
  double p = 1.0 / 720.0;
  p = fma(p, r, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double v = T->t[k & 31] * p;
  const double s = __hiloint2double(__double2hiint(v) + ((k >> 5) << 20), __double2loint(v));
  return (x != x) ? x : s;
}

// 1/b: hardware approximation + two Newton steps (relative error ~1e-16).
__device__ __forceinline__ double tc_rcp(double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = fma(-b, r, 1.0);
  r = fma(r, e, r);
  e = fma(-b, r, 1.0);
  return fma(r, e, r);
}

// a/b with one residual correction.
__device__ __forceinline__ double tc_div(double a, double b) {
  const double r = tc_rcp(b);
  const double q = a * r;
  return fma(r, fma(-b, q, a), q);
}

}  // namespace tcb
