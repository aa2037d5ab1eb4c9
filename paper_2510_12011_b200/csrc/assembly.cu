// assembly.cu -- GPU assembly of the P1 FEM matrices into
// the SELL-32 layout of a row block [row0, row0 + n) (col = internal indices
// during assembly): one thread per row gathers the contributions of the
// elements incident to its node in ascending element order, so every stored
// entry is summed in the same order as an element-order scatter-add, without
// atomics (deterministic).  Boundary (one-time) work, not on the step path.
//
//   tets:      |e| = |det J| / 6,  grad phi_a from the adjugate of J (columns
//              x_a - x_0),  M_e = |e|/20 (1 + delta_ab);
//   triangles: |e| = |n|/2 with n = e1 x e2, in-plane gradients, M_e = |e|/12 (1 + delta_ab);
//   K_e = |e| grad phi_a . sigma grad phi_b,
//   sigma = sigma_t I + (sigma_l - sigma_t) f f^T   (reading A13),
//   A = chi Cm M + theta dt K (Eq. 3),  dinv = 1 / A_ii (Jacobi).
#include <cstring>

#include "internal.h"

namespace tcb {

__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

__global__ void assemble_kernel(AsmArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const int64_t s = i / kSellC, lane = i % kSellC;
  const int64_t base = a.slice_ptr[s];
  const int len = a.rowlen[i];
  const int w = (int)((a.slice_ptr[s + 1] - a.slice_ptr[s]) / kSellC);
  for (int k = 0; k < w; ++k) {
    a.A[sell_slot(base, w, k, lane)] = 0.0;  // accumulates M first
    a.K[sell_slot(base, w, k, lane)] = 0.0;
  }
  for (int64_t t = a.inc_ptr[i]; t < a.inc_ptr[i + 1]; ++t) {
    const int32_t code = a.inc[t];
    const int64_t e = code >> 2;
    const int la = code & 3;
    const int kel = a.k;
    const int32_t* v = a.tets + (int64_t)kel * e;
    double X[4][3];
    for (int q = 0; q < kel; ++q)
      for (int c = 0; c < 3; ++c) X[q][c] = a.xyz[3 * (int64_t)v[q] + c];
    double g[4][3];
    double vol, mass_w;  // |e| and the mass weight: |e|/20 (tet), |e|/12 (triangle)
    if (kel == 4) {
      double d1[3], d2[3], d3[3];
      for (int c = 0; c < 3; ++c) {
        d1[c] = X[1][c] - X[0][c];
        d2[c] = X[2][c] - X[0][c];
        d3[c] = X[3][c] - X[0][c];
      }
      cross3(d2, d3, g[1]);
      cross3(d3, d1, g[2]);
      cross3(d1, d2, g[3]);
      const double det = d1[0] * g[1][0] + d1[1] * g[1][1] + d1[2] * g[1][2];
      if (det == 0.0) { atomicExch(a.err, 1); return; }
      for (int c = 0; c < 3; ++c) {
        g[1][c] /= det;
        g[2][c] /= det;
        g[3][c] /= det;
        g[0][c] = -(g[1][c] + g[2][c] + g[3][c]);
      }
      vol = fabs(det) / 6.0;
      mass_w = vol / 20.0;
    } else {
      // triangle embedded in 3-D: n = e1 x e2, |e| = |n|/2,
      // grad phi_1 = (e2 x n)/|n|^2, grad phi_2 = (n x e1)/|n|^2 (in-plane).
      double e1[3], e2[3], nv[3];
      for (int c = 0; c < 3; ++c) {
        e1[c] = X[1][c] - X[0][c];
        e2[c] = X[2][c] - X[0][c];
      }
      cross3(e1, e2, nv);
      const double nn = nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2];
      if (nn == 0.0) { atomicExch(a.err, 1); return; }
      cross3(e2, nv, g[1]);
      cross3(nv, e1, g[2]);
      for (int c = 0; c < 3; ++c) {
        g[1][c] /= nn;
        g[2][c] /= nn;
        g[0][c] = -(g[1][c] + g[2][c]);
      }
      vol = sqrt(nn) / 2.0;
      mass_w = vol / 12.0;
    }
    // conductivity tensor of the element
    const int r = a.ereg[e];
    const double sl = a.sig_l[r], st = a.sig_t[r];
    double f[3] = {a.fibre[3 * e], a.fibre[3 * e + 1], a.fibre[3 * e + 2]};
    const double fn = sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
    f[0] /= fn; f[1] /= fn; f[2] /= fn;
    // sigma grad phi_a
    double sg[3];
    for (int c = 0; c < 3; ++c) {
      double acc = st * g[la][c];
      double fd = f[0] * g[la][0] + f[1] * g[la][1] + f[2] * g[la][2];
      sg[c] = acc + (sl - st) * f[c] * fd;
    }
    for (int lb = 0; lb < kel; ++lb) {
      const int32_t j = v[lb];
      int k = 0;
      while (k < len && a.col[sell_slot(base, w, k, lane)] != j) ++k;
      if (k == len) { atomicExch(a.err, 2); return; }
      const double Kab = vol * (sg[0] * g[lb][0] + sg[1] * g[lb][1] + sg[2] * g[lb][2]);
      const double Mab = mass_w * (la == lb ? 2.0 : 1.0);
      const int64_t t = sell_slot(base, w, k, lane);
      a.A[t] += Mab;
      a.K[t] += Kab;
    }
  }
  double diag = 0.0;
  for (int k = 0; k < w; ++k) {
    const int64_t t = sell_slot(base, w, k, lane);
    const double Aval = a.c_mass * a.A[t] + a.c_stiff * a.K[t];
    a.A[t] = Aval;
    if (k < len && a.col[t] == (int32_t)(a.row0 + i)) diag = Aval;
  }
  const bool dir = a.dirichlet && a.dirichlet[i];
  a.dinv[i] = dir ? 0.0 : 1.0 / diag;  // Dirichlet rows never move (reading M3)
}

cudaError_t launch_assemble(const AsmArgs& a, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  assemble_kernel<<<(int)((a.n + 127) / 128), 128, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace tcb
