/*
 * oracle.c -- the plain, slow, obviously-correct CPU ORACLE of the TorchCor
 * monodomain step (arXiv 2510.12011).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load this file's shared library.  It shares no code, header, table or
 * constant generator with the CUDA path in paper_2510_12011_b200/ and neither
 * side includes or links the other.
 *
 * Everything is IEEE double, no blocking or fusion; built with -O2
 * -ffp-contract=off (no FMA contraction, no fast-math) and -fopenmp.  OpenMP
 * pragmas sit ONLY on loops whose iterations are independent (one output row /
 * node per iteration: SpMV rows, PCG elementwise updates, per-node ionic
 * steps), so every result is bitwise the same at any thread count
 * (tests/test_oracle_solver.py::test_oracle_threads_bitwise); reductions (dot
 * products), assembly and RCM stay sequential.  Thread count: or_set_threads.
 *
 * Citation convention: "P:n" = line n of the paper text,
 * "S:n" = line n of SPEC.md (used only for interfaces / tie rules), "SURVEY"
 * = SURVEY.md section of this repo (the readings are listed in DESIGN.md).
 *
 * Parity pins for every function live in tests/test_oracle_*.py; functions
 * without a pin say "parity unpinned" below (only the biology of TT2006 is).
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Error codes (mirrors nothing; oracle-local)                              */
/* ------------------------------------------------------------------------ */
#define OR_OK 0
#define OR_EINVAL 1     /* bad argument / index out of range */
#define OR_EDEGEN 2     /* zero-measure element */
#define OR_ENAN 3       /* NaN in a PCG inner product */
#define OR_ENOMEM 4
#define OR_EREGION 5    /* region tag without a conductivity entry */
#define OR_EFIBRE 6     /* zero fibre vector */

/* ======================================================================== */
/* 1. Conductivity tensor and P1 tetrahedron element matrices               */
/*    P:70 "longitudinal and the transverse conductivities"; the            */
/*    transversely-isotropic construction sigma_t I + (sigma_l-sigma_t) f f^T */
/*    is SPEC S:103-111 (paper silent, reading A13).               */
/* ======================================================================== */
int or_conductivity_tensor(const double f_in[3], double sigma_l, double sigma_t,
                           double sig[9]) {
  double nrm = sqrt(f_in[0] * f_in[0] + f_in[1] * f_in[1] + f_in[2] * f_in[2]);
  if (!(nrm > 0.0)) return OR_EFIBRE;
  double f[3] = {f_in[0] / nrm, f_in[1] / nrm, f_in[2] / nrm};
  for (int c = 0; c < 3; ++c)
    for (int d = 0; d < 3; ++d)
      sig[3 * c + d] = (c == d ? sigma_t : 0.0) + (sigma_l - sigma_t) * f[c] * f[d];
  return OR_OK;
}

/* Local P1 matrices of one tetrahedron ("linear Finite Elements").
 *   |e|  = |det[x1-x0, x2-x0, x3-x0]| / 6
 *   grad phi_1..3 = rows of J^{-1} (J has columns x_a - x_0), computed by the
 *   adjugate: (d2 x d3)/det, (d3 x d1)/det, (d1 x d2)/det;
 *   grad phi_0 = -(grad phi_1 + grad phi_2 + grad phi_3).
 *   M_e[a][b] = |e|/20 (1 + delta_ab)               (consistent mass)
 *   K_e[a][b] = |e| grad phi_a^T sigma grad phi_b                 */
int or_tet_local(const double x[12], const double sig[9], double Me[16],
                 double Ke[16], double* vol_out) {
  double d1[3], d2[3], d3[3];
  for (int c = 0; c < 3; ++c) {
    d1[c] = x[3 + c] - x[c];
    d2[c] = x[6 + c] - x[c];
    d3[c] = x[9 + c] - x[c];
  }
  double c23[3] = {d2[1] * d3[2] - d2[2] * d3[1], d2[2] * d3[0] - d2[0] * d3[2],
                   d2[0] * d3[1] - d2[1] * d3[0]};
  double c31[3] = {d3[1] * d1[2] - d3[2] * d1[1], d3[2] * d1[0] - d3[0] * d1[2],
                   d3[0] * d1[1] - d3[1] * d1[0]};
  double c12[3] = {d1[1] * d2[2] - d1[2] * d2[1], d1[2] * d2[0] - d1[0] * d2[2],
                   d1[0] * d2[1] - d1[1] * d2[0]};
  double det = d1[0] * c23[0] + d1[1] * c23[1] + d1[2] * c23[2];
  if (det == 0.0 || !isfinite(det)) return OR_EDEGEN;
  double vol = fabs(det) / 6.0;
  double G[4][3];
  for (int c = 0; c < 3; ++c) {
    G[1][c] = c23[c] / det;
    G[2][c] = c31[c] / det;
    G[3][c] = c12[c] / det;
    G[0][c] = -(G[1][c] + G[2][c] + G[3][c]);
  }
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      double s = 0.0;
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d) s += G[a][c] * sig[3 * c + d] * G[b][d];
      Ke[4 * a + b] = vol * s;
      Me[4 * a + b] = vol / 20.0 * (a == b ? 2.0 : 1.0);
    }
  if (vol_out) *vol_out = vol;
  return OR_OK;
}

/* Local P1 matrices of one triangle embedded in 3-D (surface meshes, P:68
 * "triangular or tetrahedral elements"; "gradients are taken in the
 * element's tangent plane").  With e1 = x1-x0, e2 = x2-x0, n = e1 x e2:
 *   |e| = |n|/2,  grad phi_1 = (e2 x n)/|n|^2,  grad phi_2 = (n x e1)/|n|^2,
 *   grad phi_0 = -(grad phi_1 + grad phi_2)   (in-plane vectors)
 *   M_e[a][b] = |e|/12 (1 + delta_ab)
 *   K_e[a][b] = |e| grad phi_a^T sigma grad phi_b (only the in-plane part of
 *   sigma acts, since the gradients lie in the plane).                      */
int or_tri_local(const double x[9], const double sig[9], double Me[9], double Ke[9],
                 double* area_out) {
  double e1[3], e2[3], nv[3];
  for (int c = 0; c < 3; ++c) {
    e1[c] = x[3 + c] - x[c];
    e2[c] = x[6 + c] - x[c];
  }
  nv[0] = e1[1] * e2[2] - e1[2] * e2[1];
  nv[1] = e1[2] * e2[0] - e1[0] * e2[2];
  nv[2] = e1[0] * e2[1] - e1[1] * e2[0];
  double nn = nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2];
  if (nn == 0.0 || !isfinite(nn)) return OR_EDEGEN;
  double area = sqrt(nn) / 2.0;
  double G[3][3];
  G[1][0] = (e2[1] * nv[2] - e2[2] * nv[1]) / nn;
  G[1][1] = (e2[2] * nv[0] - e2[0] * nv[2]) / nn;
  G[1][2] = (e2[0] * nv[1] - e2[1] * nv[0]) / nn;
  G[2][0] = (nv[1] * e1[2] - nv[2] * e1[1]) / nn;
  G[2][1] = (nv[2] * e1[0] - nv[0] * e1[2]) / nn;
  G[2][2] = (nv[0] * e1[1] - nv[1] * e1[0]) / nn;
  for (int c = 0; c < 3; ++c) G[0][c] = -(G[1][c] + G[2][c]);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double sum = 0.0;
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d) sum += G[a][c] * sig[3 * c + d] * G[b][d];
      Ke[3 * a + b] = area * sum;
      Me[3 * a + b] = area / 12.0 * (a == b ? 2.0 : 1.0);
    }
  if (area_out) *area_out = area;
  return OR_OK;
}

/* ======================================================================== */
/* 2. Sparsity pattern and global assembly           */
/*    Pattern: (i,j) stored iff some element contains both i and j (i==j    */
/*    included); columns strictly increasing per row.  M and K are   */
/*    assembled on this one pattern, keeping structural zeros of K.         */
/* ======================================================================== */
static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* Two calls: col == NULL -> fills rowptr (n+1) and returns nnz;
 * col != NULL -> fills col (rowptr must be the result of the first call).
 * k = nodes per element (3 triangles, 4 tetrahedra).
 * Returns -1 on an out-of-range index. */
int64_t or_pattern_k(int64_t n, int64_t E, int k, const int32_t* tets, int32_t* rowptr,
                     int32_t* col) {
  for (int64_t e = 0; e < (int64_t)k * E; ++e)
    if (tets[e] < 0 || tets[e] >= n) return -1;
  /* node -> element incidence */
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t* inc = (int64_t*)malloc(sizeof(int64_t) * (size_t)(k * E + 1));
  int32_t* mark = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* buf = (int32_t*)malloc(sizeof(int32_t) * (size_t)(k * E + 4));
  if (!cnt || !inc || !mark || !buf) { free(cnt); free(inc); free(mark); free(buf); return -1; }
  for (int64_t e = 0; e < E; ++e)
    for (int a = 0; a < k; ++a) cnt[tets[k * e + a] + 1]++;
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  memcpy(pos, cnt, sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t e = 0; e < E; ++e)
    for (int a = 0; a < k; ++a) inc[pos[tets[k * e + a]]++] = e;
  for (int64_t i = 0; i < n; ++i) mark[i] = -1;
  int64_t nnz = 0;
  for (int64_t i = 0; i < n; ++i) {
    int32_t m = 0;
    buf[m++] = (int32_t)i; /* the diagonal is always stored */
    mark[i] = (int32_t)i;
    for (int64_t t = cnt[i]; t < cnt[i + 1]; ++t) {
      int64_t e = inc[t];
      for (int a = 0; a < k; ++a) {
        int32_t j = tets[k * e + a];
        if (mark[j] != (int32_t)i) { mark[j] = (int32_t)i; buf[m++] = j; }
      }
    }
    qsort(buf, (size_t)m, sizeof(int32_t), cmp_i32);
    if (col == NULL) {
      rowptr[i] = (int32_t)nnz;
    } else {
      memcpy(col + rowptr[i], buf, sizeof(int32_t) * (size_t)m);
    }
    nnz += m;
  }
  if (col == NULL) rowptr[n] = (int32_t)nnz;
  free(cnt); free(inc); free(mark); free(buf); free(pos);
  return nnz;
}

int64_t or_pattern(int64_t n, int64_t E, const int32_t* tets, int32_t* rowptr, int32_t* col) {
  return or_pattern_k(n, E, 4, tets, rowptr, col);
}

/* slot of column j in row i (binary search over the sorted row), or -1 */
static int64_t find_slot(const int32_t* rowptr, const int32_t* col, int32_t i, int32_t j) {
  int64_t lo = rowptr[i], hi = (int64_t)rowptr[i + 1] - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) / 2;
    if (col[mid] == j) return mid;
    if (col[mid] < j) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

/* Global M and K by scatter-add in ELEMENT ORDER ("global scatter-add").
 * Region r of element e picks (sigma_l, sigma_t) from the (reg_ids -> sl, st)
 * table; fibre[e] is normalised here.  k = 4 for
 * tetrahedra, 3 for surface triangles. */
int or_assemble_k(int64_t n, const double* xyz, int64_t E, int k, const int32_t* tets,
                  const int32_t* region, const double* fibre, int32_t nreg,
                  const int32_t* reg_ids, const double* sig_l, const double* sig_t,
                  const int32_t* rowptr, const int32_t* col, double* Mval, double* Kval) {
  if (k != 3 && k != 4) return OR_EINVAL;
  int64_t nnz = rowptr[n];
  for (int64_t s = 0; s < nnz; ++s) { Mval[s] = 0.0; Kval[s] = 0.0; }
  for (int64_t e = 0; e < E; ++e) {
    int32_t r = -1;
    for (int32_t q = 0; q < nreg; ++q)
      if (reg_ids[q] == region[e]) { r = q; break; }
    if (r < 0) return OR_EREGION;
    double sig[9];
    if (or_conductivity_tensor(fibre + 3 * e, sig_l[r], sig_t[r], sig) != OR_OK)
      return OR_EFIBRE;
    double xl[12], Me[16], Ke[16];
    for (int a = 0; a < k; ++a) {
      int32_t v = tets[k * e + a];
      if (v < 0 || v >= n) return OR_EINVAL;
      for (int c = 0; c < 3; ++c) xl[3 * a + c] = xyz[3 * (int64_t)v + c];
    }
    int st = (k == 4) ? or_tet_local(xl, sig, Me, Ke, NULL) : or_tri_local(xl, sig, Me, Ke, NULL);
    if (st != OR_OK) return st;
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) {
        int64_t s = find_slot(rowptr, col, tets[k * e + a], tets[k * e + b]);
        if (s < 0) return OR_EINVAL;
        Mval[s] += Me[k * a + b];
        Kval[s] += Ke[k * a + b];
      }
  }
  return OR_OK;
}

int or_assemble(int64_t n, const double* xyz, int64_t E, const int32_t* tets,
                const int32_t* region, const double* fibre, int32_t nreg,
                const int32_t* reg_ids, const double* sig_l, const double* sig_t,
                const int32_t* rowptr, const int32_t* col, double* Mval,
                double* Kval) {
  return or_assemble_k(n, xyz, E, 4, tets, region, fibre, nreg, reg_ids, sig_l, sig_t, rowptr,
                       col, Mval, Kval);
}

/* ======================================================================== */
/* 3. Reverse Cuthill-McKee ("reordering ... using the Reverse         */
/*    Cuthill-McKee (RCM) algorithm to minimise the bandwidth"); tie rules   */
/*    from S:146: start = lowest-degree unvisited node (ties: lowest index)  */
/*    per connected component; neighbours enqueued by ascending degree, ties */
/*    by ascending index; the whole Cuthill-McKee order is reversed.          */
/*    Output perm[new] = old.                                                */
/* ======================================================================== */
static const int32_t* g_deg; /* qsort context (single-threaded oracle) */
static int cmp_deg_idx(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  if (g_deg[x] != g_deg[y]) return (g_deg[x] > g_deg[y]) - (g_deg[x] < g_deg[y]);
  return (x > y) - (x < y);
}

int or_rcm(int32_t n, const int32_t* rowptr, const int32_t* col, int32_t* perm) {
  int32_t* deg = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* byd = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  char* seen = (char*)calloc((size_t)n + 1, 1);
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* nb = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  if (!deg || !byd || !seen || !order || !nb) return OR_ENOMEM;
  for (int32_t i = 0; i < n; ++i) {
    int32_t d = 0;
    for (int32_t t = rowptr[i]; t < rowptr[i + 1]; ++t) d += (col[t] != i);
    deg[i] = d;
    byd[i] = i;
  }
  g_deg = deg;
  qsort(byd, (size_t)n, sizeof(int32_t), cmp_deg_idx);
  int32_t head = 0, tail = 0, scan = 0;
  while (tail < n) {
    while (seen[byd[scan]]) ++scan;
    int32_t s = byd[scan];
    seen[s] = 1;
    order[tail++] = s;
    while (head < tail) {
      int32_t v = order[head++];
      int32_t m = 0;
      for (int32_t t = rowptr[v]; t < rowptr[v + 1]; ++t) {
        int32_t w = col[t];
        if (!seen[w]) { seen[w] = 1; nb[m++] = w; }
      }
      qsort(nb, (size_t)m, sizeof(int32_t), cmp_deg_idx);
      for (int32_t q = 0; q < m; ++q) order[tail++] = nb[q];
    }
  }
  for (int32_t i = 0; i < n; ++i) perm[i] = order[n - 1 - i];
  free(deg); free(byd); free(seen); free(order); free(nb);
  return OR_OK;
}

/* ======================================================================== */
/* 4. CSR SpMV ("exact CSR row-wise product in float64")              */
/* ======================================================================== */
/* threads for the per-row / per-node loops (1 = the sequential oracle) */
void or_set_threads(int32_t k) {
#ifdef _OPENMP
  omp_set_num_threads(k > 0 ? k : 1);
#else
  (void)k;
#endif
}
int32_t or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void or_spmv(int32_t n, const int32_t* rowptr, const int32_t* col, const double* val,
             const double* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int32_t t = rowptr[i]; t < rowptr[i + 1]; ++t) s += val[t] * x[col[t]];
    y[i] = s;
  }
}

static double dot(int32_t n, const double* a, const double* b) {
  double s = 0.0;
  for (int32_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* ======================================================================== */
/* 5. PCG, Algorithm 1 of the paper, line by line.              */
/*    Preconditioner "M" = diag(A) (Jacobi) when jacobi != 0,  */
/*    identity otherwise.  Readings: C2 -- z_{k+1} = M^{-1}      */
/*    r_{k+1} is formed before the stopping test that uses it; C1 -- the     */
/*    relative test divides by the previous ||z|| (rel_mode 0, literal) or  */
/*    by ||z_0|| (rel_mode 1); C3 -- Euclidean norm; C4 -- ||z_0|| < eps_a   */
/*    returns x0 after 0 iterations.  trace (nullable, m+1 entries) receives */
/*    ||z_0||, ||z_1||, ... as computed.                                     */
/* ======================================================================== */
int or_pcg(int32_t n, const int32_t* rowptr, const int32_t* col, const double* val,
           const double* b, const double* x0, int32_t jacobi, double eps_a,
           double eps_r, int32_t m, int32_t rel_mode, double* x, int32_t* iters,
           double* znorm, int32_t* converged, double* trace) {
  double* r = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* z = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* p = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* q = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* d = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  if (!r || !z || !p || !q || !d) return OR_ENOMEM;
  int status = OR_OK;
  for (int32_t i = 0; i < n; ++i) {           /* M = diag(A) */
    double di = 1.0;
    if (jacobi) {
      int64_t s = find_slot(rowptr, col, i, i);
      di = (s >= 0) ? val[s] : 0.0;
      if (di == 0.0) { status = OR_EINVAL; goto done; }
    }
    d[i] = di;
  }
  /* r_0 = b - A x_0 ; M z_0 = r_0 ; p_0 = z_0 ; x = x_0 ; rho_0 = r_0^T z_0 */
  or_spmv(n, rowptr, col, val, x0, q);
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < n; ++i) {
    r[i] = b[i] - q[i];
    z[i] = r[i] / d[i];
    p[i] = z[i];
    x[i] = x0[i];
  }
  double rho = dot(n, r, z);
  double zeta = sqrt(dot(n, z, z));          /* ||z_k|| */
  double zref = zeta;
  if (trace) trace[0] = zeta;
  *iters = 0; *converged = 0; *znorm = zeta;
  if (isnan(rho) || isnan(zeta)) { status = OR_ENAN; goto done; }
  if (zeta < eps_a) { *converged = 1; goto done; }   /* reading C4 */
  for (int32_t k = 0; k < m; ++k) {
    or_spmv(n, rowptr, col, val, p, q);           /* q_k = A p_k */
    double pq = dot(n, p, q);
    if (isnan(pq)) { status = OR_ENAN; goto done; }
    double alpha = rho / pq;                      /* alpha_k = rho_k / p_k^T q_k */
#pragma omp parallel for schedule(static)
    for (int32_t i = 0; i < n; ++i) x[i] += alpha * p[i];    /* x = x + alpha p */
#pragma omp parallel for schedule(static)
    for (int32_t i = 0; i < n; ++i) r[i] -= alpha * q[i];    /* r_{k+1} */
#pragma omp parallel for schedule(static)
    for (int32_t i = 0; i < n; ++i) z[i] = r[i] / d[i];      /* M z_{k+1} = r_{k+1} (C2) */
    double zeta_new = sqrt(dot(n, z, z));
    if (trace) trace[k + 1] = zeta_new;
    *iters = k + 1; *znorm = zeta_new;
    if (isnan(zeta_new)) { status = OR_ENAN; goto done; }
    if (zeta_new < eps_a || zeta_new / zref < eps_r) { *converged = 1; goto done; }
    double rho_new = dot(n, r, z);                /* rho_{k+1} = r^T z */
    if (isnan(rho_new)) { status = OR_ENAN; goto done; }
    double beta = rho_new / rho;                  /* beta_k */
#pragma omp parallel for schedule(static)
    for (int32_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rho = rho_new;
    if (rel_mode == 0) zref = zeta_new;           /* literal consecutive ratio (C1) */
  }
done:
  free(r); free(z); free(p); free(q); free(d);
  return status;
}

/* ======================================================================== */
/* 6. Ionic models.  The paper prints no ionic equations (P:98 cites them); */
/*    both are transcribed from their primary publications (I1,  */
/*    I4, I5).  Per Eq. (2) row 1 the states advance explicitly at  */
/*    (V^k, u^k); I_n = I_ion(V^k, u^{k+1}) per unit capacitance (mV/ms),    */
/*    Eq. (2)'s argument order (reading I2; units reading U1).        */
/* ======================================================================== */

/* ---- 6a. Mitchell-Schaeffer 2003 ("Mitchell-Schaeffer") ----------- */
/* params: [tau_in, tau_out, tau_open, tau_close, v_gate, V_min, V_max]      */
/* state : h ; v = (V - V_min)/(V_max - V_min)  (S:305 mapping)              */
void or_ms_default_params(double* p) {
  p[0] = 0.3; p[1] = 6.0; p[2] = 120.0; p[3] = 150.0; p[4] = 0.13;
  p[5] = -80.0; p[6] = 20.0;
}
void or_ms_step(int64_t n, const double* V, double* h, double dt, const double* p,
                double* In) {
  double tin = p[0], tout = p[1], topen = p[2], tclose = p[3], vg = p[4];
  double vmin = p[5], vrange = p[6] - p[5];
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double v = (V[i] - vmin) / vrange;
    double dh = (v < vg) ? (1.0 - h[i]) / topen : -h[i] / tclose;  /* g(V^k,u^k) */
    h[i] = h[i] + dt * dh;                                          /* forward Euler */
    double Jin = h[i] * v * v * (1.0 - v) / tin;                    /* at u^{k+1} */
    double Jout = -v / tout;
    In[i] = -vrange * (Jin + Jout);                                 /* mV/ms */
  }
}

/* ---- 6b. ten Tusscher-Panfilov 2006, epicardial ----------- */
/* 18 states (SoA, state-major U[s*n + i]):                                   */
enum { TT_Ki, TT_Nai, TT_Cai, TT_CaSS, TT_CaSR, TT_Rbar, TT_m, TT_h, TT_j,
       TT_xr1, TT_xr2, TT_xs, TT_r, TT_s, TT_d, TT_f, TT_f2, TT_fCass, TT_NS };
/* parameter vector (49 entries, names in or_tt_param_name) */
enum { P_R, P_T, P_F, P_CAP, P_Vc, P_Vsr, P_Vss, P_Ko, P_Nao, P_Cao, P_GNa, P_GK1,
       P_Gto, P_GKr, P_GKs, P_pKNa, P_GCaL, P_GbNa, P_GbCa, P_GpCa, P_KpCa, P_GpK,
       P_PNaK, P_KmK, P_KmNa, P_kNaCa, P_KmNai, P_KmCa, P_ksat, P_gamma, P_alpha,
       P_Bufc, P_Kbufc, P_Bufsr, P_Kbufsr, P_Bufss, P_Kbufss, P_Vmaxup, P_Kup,
       P_Vrel, P_k1p, P_k2p, P_k3, P_k4, P_EC, P_maxsr, P_minsr, P_Vleak, P_Vxfer,
       P_N };
static const char* TT_PNAMES[P_N] = {
    "R", "T", "F", "CAP", "Vc", "Vsr", "Vss", "Ko", "Nao", "Cao", "GNa", "GK1",
    "Gto", "GKr", "GKs", "pKNa", "GCaL", "GbNa", "GbCa", "GpCa", "KpCa", "GpK",
    "PNaK", "KmK", "KmNa", "kNaCa", "KmNai", "KmCa", "ksat", "gamma", "alpha",
    "Bufc", "Kbufc", "Bufsr", "Kbufsr", "Bufss", "Kbufss", "Vmaxup", "Kup",
    "Vrel", "k1p", "k2p", "k3", "k4", "EC", "maxsr", "minsr", "Vleak", "Vxfer"};
static const char* TT_SNAMES[TT_NS] = {"Ki", "Nai", "Cai", "CaSS", "CaSR", "Rbar",
                                       "m", "h", "j", "xr1", "xr2", "xs", "r", "s",
                                       "d", "f", "f2", "fCass"};
int32_t or_tt_nparams(void) { return P_N; }
int32_t or_tt_nstates(void) { return TT_NS; }
const char* or_tt_param_name(int32_t k) { return (k >= 0 && k < P_N) ? TT_PNAMES[k] : 0; }
const char* or_tt_state_name(int32_t k) { return (k >= 0 && k < TT_NS) ? TT_SNAMES[k] : 0; }

/* Constants of the published TT2006 model, epicardial cell (Gto, GKs epi). */
void or_tt_default_params(double* p) {
  p[P_R] = 8314.472; p[P_T] = 310.0; p[P_F] = 96485.3415; p[P_CAP] = 0.185;
  p[P_Vc] = 0.016404; p[P_Vsr] = 0.001094; p[P_Vss] = 0.00005468;
  p[P_Ko] = 5.4; p[P_Nao] = 140.0; p[P_Cao] = 2.0;
  p[P_GNa] = 14.838; p[P_GK1] = 5.405; p[P_Gto] = 0.294; p[P_GKr] = 0.153;
  p[P_GKs] = 0.392; p[P_pKNa] = 0.03; p[P_GCaL] = 3.98e-5; p[P_GbNa] = 2.9e-4;
  p[P_GbCa] = 5.92e-4; p[P_GpCa] = 0.1238; p[P_KpCa] = 5e-4; p[P_GpK] = 0.0146;
  p[P_PNaK] = 2.724; p[P_KmK] = 1.0; p[P_KmNa] = 40.0;
  p[P_kNaCa] = 1000.0; p[P_KmNai] = 87.5; p[P_KmCa] = 1.38; p[P_ksat] = 0.1;
  p[P_gamma] = 0.35; p[P_alpha] = 2.5;
  p[P_Bufc] = 0.2; p[P_Kbufc] = 0.001; p[P_Bufsr] = 10.0; p[P_Kbufsr] = 0.3;
  p[P_Bufss] = 0.4; p[P_Kbufss] = 0.00025;
  p[P_Vmaxup] = 0.006375; p[P_Kup] = 0.00025; p[P_Vrel] = 0.102;
  p[P_k1p] = 0.15; p[P_k2p] = 0.045; p[P_k3] = 0.06; p[P_k4] = 0.005;
  p[P_EC] = 1.5; p[P_maxsr] = 2.5; p[P_minsr] = 1.0; p[P_Vleak] = 3.6e-4;
  p[P_Vxfer] = 0.0038;
}
/* Epicardial initial conditions (published steady state; I4). */
double or_tt_initial_state(double* u) {
  u[TT_Ki] = 136.89; u[TT_Nai] = 8.604; u[TT_Cai] = 1.26e-4; u[TT_CaSS] = 3.6e-4;
  u[TT_CaSR] = 3.64; u[TT_Rbar] = 0.9073; u[TT_m] = 0.00172; u[TT_h] = 0.7444;
  u[TT_j] = 0.7045; u[TT_xr1] = 0.00621; u[TT_xr2] = 0.4712; u[TT_xs] = 0.0095;
  u[TT_r] = 2.42e-8; u[TT_s] = 0.999998; u[TT_d] = 3.373e-5; u[TT_f] = 0.7888;
  u[TT_f2] = 0.9755; u[TT_fCass] = 0.9953;
  return -85.23; /* V_0 in mV */
}

/* The 12 membrane currents (pA/pF = mV/ms) of TT2006 at (V, u).            */
typedef struct {
  double INa, IK1, Ito, IKr, IKs, ICaL, INaCa, INaK, IpCa, IpK, IbNa, IbCa;
} tt_currents;

static tt_currents tt_eval_currents(double V, const double* u, const double* p) {
  tt_currents c;
  double RTONF = p[P_R] * p[P_T] / p[P_F];
  double FRT = p[P_F] / (p[P_R] * p[P_T]);
  double Ki = u[TT_Ki], Nai = u[TT_Nai], Cai = u[TT_Cai], CaSS = u[TT_CaSS];
  double Ko = p[P_Ko], Nao = p[P_Nao], Cao = p[P_Cao];
  /* reversal potentials */
  double EK = RTONF * log(Ko / Ki);
  double ENa = RTONF * log(Nao / Nai);
  double EKs = RTONF * log((Ko + p[P_pKNa] * Nao) / (Ki + p[P_pKNa] * Nai));
  double ECa = 0.5 * RTONF * log(Cao / Cai);
  /* I_Na */
  double m = u[TT_m];
  c.INa = p[P_GNa] * m * m * m * u[TT_h] * u[TT_j] * (V - ENa);
  /* I_K1 with its instantaneous rectification */
  double ak1 = 0.1 / (1.0 + exp(0.06 * (V - EK - 200.0)));
  double bk1 = (3.0 * exp(0.0002 * (V - EK + 100.0)) + exp(0.1 * (V - EK - 10.0))) /
               (1.0 + exp(-0.5 * (V - EK)));
  double xk1 = ak1 / (ak1 + bk1);
  c.IK1 = p[P_GK1] * xk1 * (V - EK);
  /* I_to, I_Kr, I_Ks */
  c.Ito = p[P_Gto] * u[TT_r] * u[TT_s] * (V - EK);
  c.IKr = p[P_GKr] * sqrt(Ko / 5.4) * u[TT_xr1] * u[TT_xr2] * (V - EK);
  c.IKs = p[P_GKs] * u[TT_xs] * u[TT_xs] * (V - EKs);
  /* I_CaL (GHK form, shifted by 15 mV) */
  double e2 = exp(2.0 * (V - 15.0) * FRT);
  c.ICaL = p[P_GCaL] * u[TT_d] * u[TT_f] * u[TT_f2] * u[TT_fCass] * 4.0 * (V - 15.0) *
           (p[P_F] * FRT) * (0.25 * CaSS * e2 - Cao) / (e2 - 1.0);
  /* I_NaCa */
  double eg = exp(p[P_gamma] * V * FRT), eg1 = exp((p[P_gamma] - 1.0) * V * FRT);
  double KmNai3 = p[P_KmNai] * p[P_KmNai] * p[P_KmNai];
  double Nao3 = Nao * Nao * Nao;
  c.INaCa = p[P_kNaCa] * (eg * Nai * Nai * Nai * Cao - eg1 * Nao3 * Cai * p[P_alpha]) /
            ((KmNai3 + Nao3) * (p[P_KmCa] + Cao) * (1.0 + p[P_ksat] * eg1));
  /* I_NaK */
  c.INaK = p[P_PNaK] * Ko * Nai /
           ((Ko + p[P_KmK]) * (Nai + p[P_KmNa]) *
            (1.0 + 0.1245 * exp(-0.1 * V * FRT) + 0.0353 * exp(-V * FRT)));
  /* pumps and background currents */
  c.IpCa = p[P_GpCa] * Cai / (p[P_KpCa] + Cai);
  c.IpK = p[P_GpK] * (V - EK) / (1.0 + exp((25.0 - V) / 5.98));
  c.IbNa = p[P_GbNa] * (V - ENa);
  c.IbCa = p[P_GbCa] * (V - ECa);
  return c;
}

static double tt_sum(const tt_currents* c) {
  return c->INa + c->IK1 + c->Ito + c->IKr + c->IKs + c->ICaL + c->INaCa + c->INaK +
         c->IpCa + c->IpK + c->IbNa + c->IbCa;
}

/* I_n for one cell at (V,u): the sum of the 12 currents (no I_stim: reading I3) */
double or_tt_current(double V, const double* u, const double* p) {
  tt_currents c = tt_eval_currents(V, u, p);
  return tt_sum(&c);
}

/* Rapid-buffer update of a buffered concentration (reference-code algebra):
 * solves c + B c/(c+K) = c_old + B c_old/(c_old+K) + delta for c > 0.       */
double or_tt_buffer(double c_old, double delta, double B, double K) {
  double cbuf = B * c_old / (c_old + K);
  double bq = B - cbuf - delta - c_old + K;
  double cq = K * (cbuf + delta + c_old);
  return (sqrt(bq * bq + 4.0 * cq) - bq) / 2.0;
}

/* Rush-Larsen update of a gate y with steady state yinf and time constant tau */
double or_rush_larsen(double y, double yinf, double tau, double dt) {
  return yinf - (yinf - y) * exp(-dt / tau);
}

/* One TT2006 step of one cell: u -> u^{k+1}; returns I_n(V, u^{k+1}).
 * Order = the model's reference code: concentrations first with currents at
 * (V^k,u^k), then gates (Rush-Larsen, reading I1) with V^k and the updated
 * CaSS; then currents re-evaluated at (V^k, u^{k+1}) (reading I2).          */
static double tt_cell_step(double V, double* u, double dt, const double* p) {
  tt_currents c = tt_eval_currents(V, u, p);
  double F = p[P_F], CAP = p[P_CAP], Vc = p[P_Vc], Vsr = p[P_Vsr], Vss = p[P_Vss];
  double Cai = u[TT_Cai], CaSS = u[TT_CaSS], CaSR = u[TT_CaSR];
  /* RyR: R-bar by forward Euler, open probability O */
  double kCaSR = p[P_maxsr] - (p[P_maxsr] - p[P_minsr]) /
                                  (1.0 + (p[P_EC] / CaSR) * (p[P_EC] / CaSR));
  double k1 = p[P_k1p] / kCaSR, k2 = p[P_k2p] * kCaSR;
  double Rbar = u[TT_Rbar] + dt * (p[P_k4] * (1.0 - u[TT_Rbar]) - k2 * CaSS * u[TT_Rbar]);
  double O = k1 * CaSS * CaSS * Rbar / (p[P_k3] + k1 * CaSS * CaSS);
  /* SR fluxes */
  double Irel = p[P_Vrel] * O * (CaSR - CaSS);
  double Ileak = p[P_Vleak] * (CaSR - Cai);
  double Iup = p[P_Vmaxup] / (1.0 + (p[P_Kup] * p[P_Kup]) / (Cai * Cai));
  double Ixfer = p[P_Vxfer] * (CaSS - Cai);
  /* buffered calcium compartments */
  double CaSR_n = or_tt_buffer(CaSR, dt * (Iup - Irel - Ileak), p[P_Bufsr], p[P_Kbufsr]);
  double CaSS_n = or_tt_buffer(
      CaSS, dt * (-Ixfer * (Vc / Vss) + Irel * (Vsr / Vss) - c.ICaL * CAP / (2.0 * Vss * F)),
      p[P_Bufss], p[P_Kbufss]);
  double Cai_n = or_tt_buffer(
      Cai, dt * (-(c.IbCa + c.IpCa - 2.0 * c.INaCa) * CAP / (2.0 * Vc * F) -
                 (Iup - Ileak) * (Vsr / Vc) + Ixfer),
      p[P_Bufc], p[P_Kbufc]);
  /* sodium and potassium (no I_stim in K_i: reading I3) */
  double Nai_n = u[TT_Nai] - dt * (c.INa + c.IbNa + 3.0 * c.INaK + 3.0 * c.INaCa) * CAP / (Vc * F);
  double Ki_n = u[TT_Ki] - dt * (c.IK1 + c.Ito + c.IKr + c.IKs - 2.0 * c.INaK + c.IpK) * CAP / (Vc * F);
  u[TT_Rbar] = Rbar; u[TT_CaSR] = CaSR_n; u[TT_CaSS] = CaSS_n; u[TT_Cai] = Cai_n;
  u[TT_Nai] = Nai_n; u[TT_Ki] = Ki_n;

  /* gates: steady states and time constants at V^k */
  double am = 1.0 / (1.0 + exp((-60.0 - V) / 5.0));
  double bm = 0.1 / (1.0 + exp((V + 35.0) / 5.0)) + 0.1 / (1.0 + exp((V - 50.0) / 200.0));
  double tau_m = am * bm;
  double em = 1.0 + exp((-56.86 - V) / 9.03);
  double m_inf = 1.0 / (em * em);
  double eh = 1.0 + exp((V + 71.55) / 7.43);
  double h_inf = 1.0 / (eh * eh);
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
  double tau_h = 1.0 / (ah + bh);
  double tau_j = 1.0 / (aj + bj);
  double j_inf = h_inf;
  double xr1_inf = 1.0 / (1.0 + exp((-26.0 - V) / 7.0));
  double tau_xr1 = (450.0 / (1.0 + exp((-45.0 - V) / 10.0))) * (6.0 / (1.0 + exp((V + 30.0) / 11.5)));
  double xr2_inf = 1.0 / (1.0 + exp((V + 88.0) / 24.0));
  double tau_xr2 = (3.0 / (1.0 + exp((-60.0 - V) / 20.0))) * (1.12 / (1.0 + exp((V - 60.0) / 20.0)));
  double xs_inf = 1.0 / (1.0 + exp((-5.0 - V) / 14.0));
  double tau_xs = (1400.0 / sqrt(1.0 + exp((5.0 - V) / 6.0))) * (1.0 / (1.0 + exp((V - 35.0) / 15.0))) + 80.0;
  double r_inf = 1.0 / (1.0 + exp((20.0 - V) / 6.0));                       /* epi */
  double tau_r = 9.5 * exp(-(V + 40.0) * (V + 40.0) / 1800.0) + 0.8;
  double s_inf = 1.0 / (1.0 + exp((V + 20.0) / 5.0));                        /* epi */
  double tau_s = 85.0 * exp(-(V + 45.0) * (V + 45.0) / 320.0) + 5.0 / (1.0 + exp((V - 20.0) / 5.0)) + 3.0;
  double d_inf = 1.0 / (1.0 + exp((-8.0 - V) / 7.5));
  double tau_d = (1.4 / (1.0 + exp((-35.0 - V) / 13.0)) + 0.25) * (1.4 / (1.0 + exp((V + 5.0) / 5.0))) +
                 1.0 / (1.0 + exp((50.0 - V) / 20.0));
  double f_inf = 1.0 / (1.0 + exp((V + 20.0) / 7.0));
  double tau_f = 1102.5 * exp(-(V + 27.0) * (V + 27.0) / 225.0) + 200.0 / (1.0 + exp((13.0 - V) / 10.0)) +
                 180.0 / (1.0 + exp((V + 30.0) / 10.0)) + 20.0;
  double f2_inf = 0.67 / (1.0 + exp((V + 35.0) / 7.0)) + 0.33;
  double tau_f2 = 600.0 * exp(-(V + 25.0) * (V + 25.0) / 170.0) + 31.0 / (1.0 + exp((25.0 - V) / 10.0)) +
                  16.0 / (1.0 + exp((V + 30.0) / 10.0));
  double cs = CaSS_n / 0.05;
  double fcass_inf = 0.6 / (1.0 + cs * cs) + 0.4;
  double tau_fcass = 80.0 / (1.0 + cs * cs) + 2.0;
  u[TT_m] = or_rush_larsen(u[TT_m], m_inf, tau_m, dt);
  u[TT_h] = or_rush_larsen(u[TT_h], h_inf, tau_h, dt);
  u[TT_j] = or_rush_larsen(u[TT_j], j_inf, tau_j, dt);
  u[TT_xr1] = or_rush_larsen(u[TT_xr1], xr1_inf, tau_xr1, dt);
  u[TT_xr2] = or_rush_larsen(u[TT_xr2], xr2_inf, tau_xr2, dt);
  u[TT_xs] = or_rush_larsen(u[TT_xs], xs_inf, tau_xs, dt);
  u[TT_r] = or_rush_larsen(u[TT_r], r_inf, tau_r, dt);
  u[TT_s] = or_rush_larsen(u[TT_s], s_inf, tau_s, dt);
  u[TT_d] = or_rush_larsen(u[TT_d], d_inf, tau_d, dt);
  u[TT_f] = or_rush_larsen(u[TT_f], f_inf, tau_f, dt);
  u[TT_f2] = or_rush_larsen(u[TT_f2], f2_inf, tau_f2, dt);
  u[TT_fCass] = or_rush_larsen(u[TT_fCass], fcass_inf, tau_fcass, dt);

  return or_tt_current(V, u, p);   /* I_ion(V^k, u^{k+1}) */
}

/* Field version: U is state-major SoA (U[s*n + i]). */
void or_tt_step(int64_t n, const double* V, double* U, double dt, const double* p,
                double* In) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double u[TT_NS];
    for (int s = 0; s < TT_NS; ++s) u[s] = U[(int64_t)s * n + i];
    In[i] = tt_cell_step(V[i], u, dt, p);
    for (int s = 0; s < TT_NS; ++s) U[(int64_t)s * n + i] = u[s];
  }
}

/* ---- 6c. Courtemanche-Ramirez-Nattel 1998 human atrial cell ("CRN",      */
/*      named among the supported models).           */
/* The paper gives no equations; they are the published model (Am J Physiol */
/* 275:H301, 1998; the CellML transcription), reading I6:          */
/* "parity unpinned" for the biological constants, pinned for quiescence,   */
/* the action potential, Nernst potentials and the integrator.               */
/* Integrator (as TT2006, readings I1/I2/I3): Rush-Larsen for the 15 gates,  */
/* forward Euler for the 5 concentrations with the instantaneous-buffer      */
/* factor of Ca_i and Ca_rel, all at (V^k, u^k); I_n = I_ion(V^k, u^{k+1}).  */
/* 20 states, state-major: */
enum { CR_Nai, CR_Ki, CR_Cai, CR_Caup, CR_Carel, CR_m, CR_h, CR_j, CR_oa, CR_oi,
       CR_ua, CR_ui, CR_xr, CR_xs, CR_d, CR_f, CR_fCa, CR_u, CR_v, CR_w, CR_NS };
enum { Q_R, Q_T, Q_F, Q_Cm, Q_Vi, Q_Vup, Q_Vrel, Q_Ko, Q_Nao, Q_Cao, Q_gNa, Q_gK1,
       Q_gto, Q_gKr, Q_gKs, Q_gCaL, Q_gbNa, Q_gbCa, Q_INaKmax, Q_KmNai, Q_KmKo,
       Q_INaCamax, Q_KmNa, Q_KmCa, Q_ksat, Q_gamma, Q_IpCamax, Q_Krel, Q_tautr,
       Q_Iupmax, Q_Kup, Q_Caupmax, Q_CMDNmax, Q_TRPNmax, Q_CSQNmax, Q_KmCMDN,
       Q_KmTRPN, Q_KmCSQN, Q_tauu, Q_KQ10, Q_N };
static const char* CR_PNAMES[Q_N] = {
    "R", "T", "F", "Cm", "Vi", "Vup", "Vrel", "Ko", "Nao", "Cao", "gNa", "gK1",
    "gto", "gKr", "gKs", "gCaL", "gbNa", "gbCa", "INaKmax", "KmNai", "KmKo",
    "INaCamax", "KmNa", "KmCa", "ksat", "gamma", "IpCamax", "Krel", "tautr",
    "Iupmax", "Kup", "Caupmax", "CMDNmax", "TRPNmax", "CSQNmax", "KmCMDN",
    "KmTRPN", "KmCSQN", "tauu", "KQ10"};
static const char* CR_SNAMES[CR_NS] = {"Nai", "Ki", "Cai", "Caup", "Carel", "m", "h", "j",
                                       "oa", "oi", "ua", "ui", "xr", "xs", "d", "f",
                                       "fCa", "u", "v", "w"};
int32_t or_crn_nparams(void) { return Q_N; }
int32_t or_crn_nstates(void) { return CR_NS; }
const char* or_crn_param_name(int32_t k) { return (k >= 0 && k < Q_N) ? CR_PNAMES[k] : 0; }
const char* or_crn_state_name(int32_t k) { return (k >= 0 && k < CR_NS) ? CR_SNAMES[k] : 0; }

void or_crn_default_params(double* p) {
  p[Q_R] = 8.3143; p[Q_T] = 310.0; p[Q_F] = 96.4867; p[Q_Cm] = 100.0;
  p[Q_Vi] = 13668.0; p[Q_Vup] = 1109.52; p[Q_Vrel] = 96.48;
  p[Q_Ko] = 5.4; p[Q_Nao] = 140.0; p[Q_Cao] = 1.8;
  p[Q_gNa] = 7.8; p[Q_gK1] = 0.09; p[Q_gto] = 0.1652; p[Q_gKr] = 0.029411765;
  p[Q_gKs] = 0.12941176; p[Q_gCaL] = 0.12375; p[Q_gbNa] = 6.744375e-4; p[Q_gbCa] = 1.131e-3;
  p[Q_INaKmax] = 0.59933874; p[Q_KmNai] = 10.0; p[Q_KmKo] = 1.5;
  p[Q_INaCamax] = 1600.0; p[Q_KmNa] = 87.5; p[Q_KmCa] = 1.38; p[Q_ksat] = 0.1;
  p[Q_gamma] = 0.35; p[Q_IpCamax] = 0.275; p[Q_Krel] = 30.0; p[Q_tautr] = 180.0;
  p[Q_Iupmax] = 0.005; p[Q_Kup] = 0.00092; p[Q_Caupmax] = 15.0;
  p[Q_CMDNmax] = 0.05; p[Q_TRPNmax] = 0.07; p[Q_CSQNmax] = 10.0;
  p[Q_KmCMDN] = 0.00238; p[Q_KmTRPN] = 0.0005; p[Q_KmCSQN] = 0.8;
  p[Q_tauu] = 8.0; p[Q_KQ10] = 3.0;
}
/* Published initial conditions (resting cell). */
double or_crn_initial_state(double* u) {
  u[CR_Nai] = 11.17; u[CR_Ki] = 139.0; u[CR_Cai] = 1.013e-4; u[CR_Caup] = 1.488;
  u[CR_Carel] = 1.488; u[CR_m] = 2.908e-3; u[CR_h] = 0.9649; u[CR_j] = 0.9775;
  u[CR_oa] = 3.043e-2; u[CR_oi] = 0.9992; u[CR_ua] = 4.966e-3; u[CR_ui] = 0.9986;
  u[CR_xr] = 3.296e-5; u[CR_xs] = 1.869e-2; u[CR_d] = 1.367e-4; u[CR_f] = 0.9996;
  u[CR_fCa] = 0.7755; u[CR_u] = 2.35e-112; u[CR_v] = 1.0; u[CR_w] = 0.9992;
  return -81.18;
}

/* membrane currents per unit capacitance (pA/pF = mV/ms) at (V, u) */
typedef struct {
  double INa, IK1, Ito, IKur, IKr, IKs, ICaL, INaK, INaCa, IbNa, IbCa, IpCa;
} crn_currents;

static crn_currents crn_eval_currents(double V, const double* u, const double* p) {
  crn_currents c;
  const double RTF = p[Q_R] * p[Q_T] / p[Q_F], FRT = p[Q_F] / (p[Q_R] * p[Q_T]);
  const double Nai = u[CR_Nai], Ki = u[CR_Ki], Cai = u[CR_Cai];
  const double Ko = p[Q_Ko], Nao = p[Q_Nao], Cao = p[Q_Cao];
  const double ENa = RTF * log(Nao / Nai), EK = RTF * log(Ko / Ki);
  const double ECa = RTF / 2.0 * log(Cao / Cai);
  const double m = u[CR_m], oa = u[CR_oa], ua = u[CR_ua], xs = u[CR_xs];
  c.INa = p[Q_gNa] * m * m * m * u[CR_h] * u[CR_j] * (V - ENa);
  c.IK1 = p[Q_gK1] * (V - EK) / (1.0 + exp(0.07 * (V + 80.0)));
  c.Ito = p[Q_gto] * oa * oa * oa * u[CR_oi] * (V - EK);
  const double gKur = 0.005 + 0.05 / (1.0 + exp((V - 15.0) / -13.0));
  c.IKur = gKur * ua * ua * ua * u[CR_ui] * (V - EK);
  c.IKr = p[Q_gKr] * u[CR_xr] * (V - EK) / (1.0 + exp((V + 15.0) / 22.4));
  c.IKs = p[Q_gKs] * xs * xs * (V - EK);
  c.ICaL = p[Q_gCaL] * u[CR_d] * u[CR_f] * u[CR_fCa] * (V - 65.0);
  const double sigma = (exp(Nao / 67.3) - 1.0) / 7.0;
  const double fNaK = 1.0 / (1.0 + 0.1245 * exp(-0.1 * V * FRT) + 0.0365 * sigma * exp(-V * FRT));
  c.INaK = p[Q_INaKmax] * fNaK / (1.0 + pow(p[Q_KmNai] / Nai, 1.5)) * Ko / (Ko + p[Q_KmKo]);
  const double g = p[Q_gamma];
  c.INaCa = p[Q_INaCamax] *
            (exp(g * V * FRT) * Nai * Nai * Nai * Cao - exp((g - 1.0) * V * FRT) * Nao * Nao * Nao * Cai) /
            ((p[Q_KmNa] * p[Q_KmNa] * p[Q_KmNa] + Nao * Nao * Nao) * (p[Q_KmCa] + Cao) *
             (1.0 + p[Q_ksat] * exp((g - 1.0) * V * FRT)));
  c.IbNa = p[Q_gbNa] * (V - ENa);
  c.IbCa = p[Q_gbCa] * (V - ECa);
  c.IpCa = p[Q_IpCamax] * Cai / (0.0005 + Cai);
  return c;
}

static double crn_sum(const crn_currents* c) {
  return c->INa + c->IK1 + c->Ito + c->IKur + c->IKr + c->IKs + c->ICaL + c->INaK +
         c->INaCa + c->IbNa + c->IbCa + c->IpCa;
}

double or_crn_current(double V, const double* u, const double* p) {
  crn_currents c = crn_eval_currents(V, u, p);
  return crn_sum(&c);
}

/* steady states and time constants of the 15 gates at (V, u) */
typedef struct { double inf[15], tau[15]; } crn_gates;
enum { G_m, G_h, G_j, G_oa, G_oi, G_ua, G_ui, G_xr, G_xs, G_d, G_f, G_fCa, G_u, G_v, G_w };

static void crn_eval_gates(double V, const double* u, const double* p, const crn_currents* c,
                           double Irel, crn_gates* G) {
  double a, b;
  /* I_Na gates */
  a = (V == -47.13) ? 3.2 : 0.32 * (V + 47.13) / (1.0 - exp(-0.1 * (V + 47.13)));
  b = 0.08 * exp(-V / 11.0);
  G->inf[G_m] = a / (a + b); G->tau[G_m] = 1.0 / (a + b);
  if (V < -40.0) {
    a = 0.135 * exp((V + 80.0) / -6.8);
    b = 3.56 * exp(0.079 * V) + 3.1e5 * exp(0.35 * V);
  } else {
    a = 0.0;
    b = 1.0 / (0.13 * (1.0 + exp((V + 10.66) / -11.1)));
  }
  G->inf[G_h] = a / (a + b); G->tau[G_h] = 1.0 / (a + b);
  if (V < -40.0) {
    a = (-127140.0 * exp(0.2444 * V) - 3.474e-5 * exp(-0.04391 * V)) * (V + 37.78) /
        (1.0 + exp(0.311 * (V + 79.23)));
    b = 0.1212 * exp(-0.01052 * V) / (1.0 + exp(-0.1378 * (V + 40.14)));
  } else {
    a = 0.0;
    b = 0.3 * exp(-2.535e-7 * V) / (1.0 + exp(-0.1 * (V + 32.0)));
  }
  G->inf[G_j] = a / (a + b); G->tau[G_j] = 1.0 / (a + b);
  /* I_to, I_Kur gates (time constants divided by K_Q10) */
  const double KQ = p[Q_KQ10];
  a = 0.65 / (exp((V + 10.0) / -8.5) + exp((V - 30.0) / -59.0));
  b = 0.65 / (2.5 + exp((V + 82.0) / 17.0));
  G->tau[G_oa] = 1.0 / (a + b) / KQ;
  G->inf[G_oa] = 1.0 / (1.0 + exp((V + 20.47) / -17.54));
  a = 1.0 / (18.53 + exp((V + 113.7) / 10.95));
  b = 1.0 / (35.56 + exp((V + 1.26) / -7.44));
  G->tau[G_oi] = 1.0 / (a + b) / KQ;
  G->inf[G_oi] = 1.0 / (1.0 + exp((V + 43.1) / 5.3));
  a = 0.65 / (exp((V + 10.0) / -8.5) + exp((V - 30.0) / -59.0));
  b = 0.65 / (2.5 + exp((V + 82.0) / 17.0));
  G->tau[G_ua] = 1.0 / (a + b) / KQ;
  G->inf[G_ua] = 1.0 / (1.0 + exp((V + 30.3) / -9.6));
  a = 1.0 / (21.0 + exp((V - 185.0) / -28.0));
  b = exp((V - 158.0) / 16.0);
  G->tau[G_ui] = 1.0 / (a + b) / KQ;
  G->inf[G_ui] = 1.0 / (1.0 + exp((V - 99.45) / 27.48));
  /* I_Kr, I_Ks */
  a = (V == -14.1) ? 0.0015 : 0.0003 * (V + 14.1) / (1.0 - exp((V + 14.1) / -5.0));
  b = (V == 3.3328) ? 3.7836118e-4 : 7.3898e-5 * (V - 3.3328) / (exp((V - 3.3328) / 5.1237) - 1.0);
  G->tau[G_xr] = 1.0 / (a + b);
  G->inf[G_xr] = 1.0 / (1.0 + exp((V + 14.1) / -6.5));
  a = (V == 19.9) ? 0.00068 : 4e-5 * (V - 19.9) / (1.0 - exp((V - 19.9) / -17.0));
  b = (V == 19.9) ? 0.000315 : 3.5e-5 * (V - 19.9) / (exp((V - 19.9) / 9.0) - 1.0);
  G->tau[G_xs] = 0.5 / (a + b);
  G->inf[G_xs] = 1.0 / sqrt(1.0 + exp((V - 19.9) / -12.7));
  /* I_CaL */
  G->inf[G_d] = 1.0 / (1.0 + exp((V + 10.0) / -8.0));
  G->tau[G_d] = (V == -10.0) ? 4.579 / (1.0 + exp((V + 10.0) / -6.24))
                             : (1.0 - exp((V + 10.0) / -6.24)) /
                                   (0.035 * (V + 10.0) * (1.0 + exp((V + 10.0) / -6.24)));
  G->inf[G_f] = exp(-(V + 28.0) / 6.9) / (1.0 + exp(-(V + 28.0) / 6.9));
  G->tau[G_f] = 9.0 / (0.0197 * exp(-0.0337 * 0.0337 * (V + 10.0) * (V + 10.0)) + 0.02);
  G->inf[G_fCa] = 1.0 / (1.0 + u[CR_Cai] / 0.00035);
  G->tau[G_fCa] = 2.0;
  /* SR release gates: flux Fn in the release junction (pA -> femtomoles) */
  const double Cm = p[Q_Cm];
  const double Fn = 1000.0 * (1e-15 * p[Q_Vrel] * Irel -
                              1e-15 / (2.0 * p[Q_F]) * (0.5 * c->ICaL * Cm - 0.2 * c->INaCa * Cm));
  G->inf[G_u] = 1.0 / (1.0 + exp(-(Fn - 3.4175e-13) / 13.67e-16));
  G->tau[G_u] = p[Q_tauu];
  G->tau[G_v] = 1.91 + 2.09 / (1.0 + exp(-(Fn - 3.4175e-13) / 13.67e-16));
  G->inf[G_v] = 1.0 - 1.0 / (1.0 + exp(-(Fn - 6.835e-14) / 13.67e-16));
  G->tau[G_w] = (V == 7.9) ? 6.0 * 0.2 / 1.3
                           : 6.0 * (1.0 - exp(-(V - 7.9) / 5.0)) /
                                 ((1.0 + 0.3 * exp(-(V - 7.9) / 5.0)) * (V - 7.9));
  G->inf[G_w] = 1.0 - 1.0 / (1.0 + exp(-(V - 40.0) / 17.0));
}

/* One CRN step of one cell: u -> u^{k+1}; returns I_n(V, u^{k+1}). */
static double crn_cell_step(double V, double* u, double dt, const double* p) {
  crn_currents c = crn_eval_currents(V, u, p);
  const double F = p[Q_F], Cm = p[Q_Cm], Vi = p[Q_Vi], Vup = p[Q_Vup], Vrel = p[Q_Vrel];
  const double Cai = u[CR_Cai], Caup = u[CR_Caup], Carel = u[CR_Carel];
  /* SR fluxes (mM/ms) */
  const double Irel = p[Q_Krel] * u[CR_u] * u[CR_u] * u[CR_v] * u[CR_w] * (Carel - Cai);
  const double Itr = (Caup - Carel) / p[Q_tautr];
  const double Iupleak = p[Q_Iupmax] * Caup / p[Q_Caupmax];
  const double Iup = p[Q_Iupmax] / (1.0 + p[Q_Kup] / Cai);
  crn_gates G;
  crn_eval_gates(V, u, p, &c, Irel, &G);
  /* concentrations: forward Euler (currents in pA = per-capacitance x Cm) */
  const double dNai = (-3.0 * c.INaK - 3.0 * c.INaCa - c.IbNa - c.INa) * Cm / (Vi * F);
  const double dKi = (2.0 * c.INaK - c.IK1 - c.Ito - c.IKur - c.IKr - c.IKs) * Cm / (Vi * F);
  const double B1 = (2.0 * c.INaCa - c.IpCa - c.ICaL - c.IbCa) * Cm / (2.0 * Vi * F) +
                    (Vup * (Iupleak - Iup) + Irel * Vrel) / Vi;
  const double B2 = 1.0 + p[Q_TRPNmax] * p[Q_KmTRPN] / ((Cai + p[Q_KmTRPN]) * (Cai + p[Q_KmTRPN])) +
                    p[Q_CMDNmax] * p[Q_KmCMDN] / ((Cai + p[Q_KmCMDN]) * (Cai + p[Q_KmCMDN]));
  const double dCaup = Iup - Iupleak - Itr * Vrel / Vup;
  const double dCarel = (Itr - Irel) /
                        (1.0 + p[Q_CSQNmax] * p[Q_KmCSQN] / ((Carel + p[Q_KmCSQN]) * (Carel + p[Q_KmCSQN])));
  u[CR_Nai] += dt * dNai;
  u[CR_Ki] += dt * dKi;
  u[CR_Cai] += dt * (B1 / B2);
  u[CR_Caup] += dt * dCaup;
  u[CR_Carel] += dt * dCarel;
  /* gates: Rush-Larsen at (V^k, u^k) */
  for (int g = 0; g < 15; ++g)
    u[CR_m + g] = or_rush_larsen(u[CR_m + g], G.inf[g], G.tau[g], dt);
  return or_crn_current(V, u, p);   /* I_ion(V^k, u^{k+1}) (reading I2) */
}

void or_crn_step(int64_t n, const double* V, double* U, double dt, const double* p, double* In) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double u[CR_NS];
    for (int s = 0; s < CR_NS; ++s) u[s] = U[(int64_t)s * n + i];
    In[i] = crn_cell_step(V[i], u, dt, p);
    for (int s = 0; s < CR_NS; ++s) U[(int64_t)s * n + i] = u[s];
  }
}
