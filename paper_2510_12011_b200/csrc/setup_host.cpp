// setup_host.cpp -- one-time host setup of libtcb200 (not on the per-step path):
// orientation fix, node->element incidence, the sparsity pattern of
// M u K, Reverse Cuthill-McKee (tie rules S:146), the
// permuted CSR and its SELL-32 layout.  OpenMP over rows where independent.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "internal.h"

namespace tcb {

// k = 4: swap tet vertices 1,2 when the signed volume is negative; k = 3
// (surface triangles in 3-D): no orientation.  Reports the first zero-measure
// or out-of-range element.
std::string orient_and_validate(int64_t n, int64_t E, int k, int32_t* tets, const double* xyz) {
  int64_t bad_idx = -1, bad_vol = -1;
#pragma omp parallel for schedule(static) reduction(max : bad_idx, bad_vol)
  for (int64_t e = 0; e < E; ++e) {
    int32_t* t = tets + (int64_t)k * e;
    bool ok = true;
    for (int a = 0; a < k; ++a)
      if (t[a] < 0 || t[a] >= n) ok = false;
    if (!ok) {
      bad_idx = std::max(bad_idx, e);
      continue;
    }
    if (k == 3) {
      double e1[3], e2[3];
      for (int c = 0; c < 3; ++c) {
        e1[c] = xyz[3 * (int64_t)t[1] + c] - xyz[3 * (int64_t)t[0] + c];
        e2[c] = xyz[3 * (int64_t)t[2] + c] - xyz[3 * (int64_t)t[0] + c];
      }
      const double nx = e1[1] * e2[2] - e1[2] * e2[1], ny = e1[2] * e2[0] - e1[0] * e2[2],
                   nz = e1[0] * e2[1] - e1[1] * e2[0];
      const double nn = nx * nx + ny * ny + nz * nz;
      if (!(nn > 0.0) || !std::isfinite(nn)) bad_vol = std::max(bad_vol, e);
      continue;
    }
    const double* p0 = xyz + 3 * (int64_t)t[0];
    double d[3][3];
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) d[a][c] = xyz[3 * (int64_t)t[a + 1] + c] - p0[c];
    double det = d[0][0] * (d[1][1] * d[2][2] - d[1][2] * d[2][1]) -
                 d[0][1] * (d[1][0] * d[2][2] - d[1][2] * d[2][0]) +
                 d[0][2] * (d[1][0] * d[2][1] - d[1][1] * d[2][0]);
    if (!(det != 0.0) || !std::isfinite(det)) {
      bad_vol = std::max(bad_vol, e);
      continue;
    }
    if (det < 0) std::swap(t[1], t[2]);
  }
  if (bad_idx >= 0) return "EINVAL:tet " + std::to_string(bad_idx) + " has a node index out of range";
  if (bad_vol >= 0) return "EDEGEN:tet " + std::to_string(bad_vol) + " has zero volume";
  return "";
}

// node -> (4*e + a) incidence (k nodes per element, a < k); entries of a node
// in ascending element order.
void build_incidence(int64_t n, int64_t E, int k, const int32_t* tets, std::vector<int64_t>& ptr,
                     std::vector<int32_t>& inc) {
  ptr.assign(n + 1, 0);
  for (int64_t e = 0; e < (int64_t)k * E; ++e) ptr[tets[e] + 1]++;
  for (int64_t i = 0; i < n; ++i) ptr[i + 1] += ptr[i];
  std::vector<int64_t> pos(ptr.begin(), ptr.end() - 1);
  inc.resize((int64_t)k * E);
  for (int64_t e = 0; e < E; ++e)
    for (int a = 0; a < k; ++a) inc[pos[tets[(int64_t)k * e + a]]++] = (int32_t)(4 * e + a);
}

// Row i holds i and every node sharing an element with i, ascending.
void build_pattern(int64_t n, int k, const int32_t* tets, const std::vector<int64_t>& ptr,
                   const std::vector<int32_t>& inc, std::vector<int64_t>& rowptr,
                   std::vector<int32_t>& col) {
  rowptr.assign(n + 1, 0);
  auto gather = [&](int64_t i, std::vector<int32_t>& buf) {
    buf.clear();
    buf.push_back((int32_t)i);
    for (int64_t t = ptr[i]; t < ptr[i + 1]; ++t) {
      int64_t e = inc[t] >> 2;
      for (int a = 0; a < k; ++a) buf.push_back(tets[(int64_t)k * e + a]);
    }
    std::sort(buf.begin(), buf.end());
    buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
  };
#pragma omp parallel
  {
    std::vector<int32_t> buf;
#pragma omp for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
      gather(i, buf);
      rowptr[i + 1] = (int64_t)buf.size();
    }
  }
  for (int64_t i = 0; i < n; ++i) rowptr[i + 1] += rowptr[i];
  col.resize(rowptr[n]);
#pragma omp parallel
  {
    std::vector<int32_t> buf;
#pragma omp for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
      gather(i, buf);
      std::copy(buf.begin(), buf.end(), col.begin() + rowptr[i]);
    }
  }
}

// Reverse Cuthill-McKee: per connected component start at the lowest-degree
// unvisited node (ties: lowest index); enqueue unvisited neighbours by
// ascending (degree, index); reverse the whole order.  perm[new] = old.
void rcm_order(int64_t n, const std::vector<int64_t>& rowptr, const std::vector<int32_t>& col,
               std::vector<int32_t>& perm) {
  std::vector<int32_t> deg(n);
  int32_t maxdeg = 0;
  for (int64_t i = 0; i < n; ++i) {
    int32_t d = 0;
    for (int64_t t = rowptr[i]; t < rowptr[i + 1]; ++t) d += (col[t] != i);
    deg[i] = d;
    maxdeg = std::max(maxdeg, d);
  }
  // nodes by (degree, index): counting sort, stable in index
  std::vector<int64_t> cnt(maxdeg + 2, 0);
  for (int64_t i = 0; i < n; ++i) cnt[deg[i] + 1]++;
  for (int d = 0; d <= maxdeg; ++d) cnt[d + 1] += cnt[d];
  std::vector<int32_t> byd(n);
  for (int64_t i = 0; i < n; ++i) byd[cnt[deg[i]]++] = (int32_t)i;
  std::vector<uint8_t> seen(n, 0);
  std::vector<int32_t> order;
  order.reserve(n);
  std::vector<int32_t> nb;
  int64_t head = 0, scan = 0;
  auto less = [&](int32_t a, int32_t b) { return deg[a] != deg[b] ? deg[a] < deg[b] : a < b; };
  while ((int64_t)order.size() < n) {
    while (seen[byd[scan]]) ++scan;
    int32_t s = byd[scan];
    seen[s] = 1;
    order.push_back(s);
    while (head < (int64_t)order.size()) {
      int32_t v = order[head++];
      nb.clear();
      for (int64_t t = rowptr[v]; t < rowptr[v + 1]; ++t) {
        int32_t w = col[t];
        if (!seen[w]) {
          seen[w] = 1;
          nb.push_back(w);
        }
      }
      std::sort(nb.begin(), nb.end(), less);
      order.insert(order.end(), nb.begin(), nb.end());
    }
  }
  perm.resize(n);
  for (int64_t i = 0; i < n; ++i) perm[i] = order[n - 1 - i];
}

// CSR of P A P^T: new row r = old row perm[r], columns inv[], sorted.
void permute_csr(int64_t n, const std::vector<int64_t>& rowptr, const std::vector<int32_t>& col,
                 const std::vector<int32_t>& perm, const std::vector<int32_t>& inv,
                 std::vector<int64_t>& rowptr2, std::vector<int32_t>& col2) {
  rowptr2.assign(n + 1, 0);
  for (int64_t r = 0; r < n; ++r) rowptr2[r + 1] = rowptr2[r] + (rowptr[perm[r] + 1] - rowptr[perm[r]]);
  col2.resize(rowptr2[n]);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t r = 0; r < n; ++r) {
    int64_t o = perm[r], d = rowptr2[r];
    for (int64_t t = rowptr[o]; t < rowptr[o + 1]; ++t) col2[d++] = inv[col[t]];
    std::sort(col2.begin() + rowptr2[r], col2.begin() + rowptr2[r + 1]);
  }
}

// SELL-32 layout of a CSR pattern.  csr_slot (optional) maps CSR entry -> slot.
void csr_to_sell(int32_t n, const int64_t* rowptr, const int32_t* col, HostSell& s,
                 std::vector<int64_t>* csr_slot) {
  s.n = n;
  s.nslices = (n + kSellC - 1) / kSellC;
  s.n_pad = (int64_t)s.nslices * kSellC;
  s.slice_ptr.assign(s.nslices + 1, 0);
  s.rowlen.resize(n);
  for (int32_t sl = 0; sl < s.nslices; ++sl) {
    int64_t w = 0;
    for (int32_t l = 0; l < kSellC; ++l) {
      int64_t i = (int64_t)sl * kSellC + l;
      if (i < n) w = std::max<int64_t>(w, rowptr[i + 1] - rowptr[i]);
    }
    s.slice_ptr[sl + 1] = s.slice_ptr[sl] + w * kSellC;
  }
  s.col.resize(s.slice_ptr[s.nslices]);
  if (csr_slot) csr_slot->resize(rowptr[n]);
#pragma omp parallel for schedule(static)
  for (int32_t sl = 0; sl < s.nslices; ++sl) {
    int64_t base = s.slice_ptr[sl], w = (s.slice_ptr[sl + 1] - base) / kSellC;
    for (int32_t l = 0; l < kSellC; ++l) {
      int64_t i = (int64_t)sl * kSellC + l;
      int64_t len = (i < n) ? rowptr[i + 1] - rowptr[i] : 0;
      if (i < n) s.rowlen[i] = (int32_t)len;
      for (int64_t k = 0; k < w; ++k) {
        int64_t slot = sell_slot(base, w, k, l);
        if (k < len) {
          s.col[slot] = col[rowptr[i] + k];
          if (csr_slot) (*csr_slot)[rowptr[i] + k] = slot;
        } else {
          s.col[slot] = (int32_t)i;  // padding: self, value 0
        }
      }
    }
  }
}

// 16-bit column compression per (slice, slot row): base = min over the 32
// lanes, offsets < 2^16; slices where any slot row spans more stay int32.
void compress_sell(HostSell& s) {
  const int64_t total = s.slice_ptr[s.nslices];
  s.col16.assign(total, 0);
  s.kbase.assign(total / kSellC, 0);
  s.fmt.assign(s.nslices, 0);
  int64_t wide = 0;
#pragma omp parallel for schedule(static) reduction(+ : wide)
  for (int32_t sl = 0; sl < s.nslices; ++sl) {
    const int64_t base = s.slice_ptr[sl], w = (s.slice_ptr[sl + 1] - base) / kSellC;
    bool ok = true;
    for (int64_t k = 0; k < w && ok; ++k) {
      int32_t mn = s.col[sell_slot(base, w, k, 0)], mx = mn;
      for (int l = 1; l < kSellC; ++l) {
        const int32_t c = s.col[sell_slot(base, w, k, l)];
        mn = std::min(mn, c);
        mx = std::max(mx, c);
      }
      if ((int64_t)mx - mn > 65535) ok = false;
      s.kbase[base / kSellC + k] = mn;
    }
    if (!ok) {
      s.fmt[sl] = 1;
      wide += 1;
      continue;
    }
    for (int64_t k = 0; k < w; ++k)
      for (int l = 0; l < kSellC; ++l) {
        const int64_t t = sell_slot(base, w, k, l);
        s.col16[t] = (uint16_t)(s.col[t] - s.kbase[base / kSellC + k]);
      }
  }
  s.n_wide = wide;
}

// Balanced contiguous row blocks of the internal (RCM) order: block p owns
// [g0, g1) = [floor(n p / P), floor(n (p+1) / P)).  With RCM's level structure
// the ghosts of a block come from its neighbouring blocks.
int64_t block_start(int64_t n, int nparts, int p) { return (n * p) / nparts; }

// The plan of block p from ITS OWN ROWS alone (lrp: rowptr of rows [g0, g1)
// rebased to 0, lcol: their columns, internal indices).  The pattern is
// structurally symmetric (P1 FEM), so what neighbour q needs from p -- q's
// ghosts inside p's block -- is the set of p's rows with a column in q's block;
// both sides list it in ascending internal index.  Each rank can plan itself
// (and its neighbours) without the others' rows.
PartPlan plan_from_rows(int64_t n, int nparts, int p, const int64_t* lrp, const int32_t* lcol) {
  PartPlan P;
  P.g0 = block_start(n, nparts, p);
  P.g1 = block_start(n, nparts, p + 1);
  const int64_t m = P.g1 - P.g0;
  auto owner = [&](int64_t g) {
    int q = (int)((g * nparts) / n);
    while (q + 1 < nparts && block_start(n, nparts, q + 1) <= g) ++q;
    while (q > 0 && block_start(n, nparts, q) > g) --q;
    return q;
  };
  std::vector<int32_t> gh;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t t = lrp[i]; t < lrp[i + 1]; ++t)
      if (lcol[t] < P.g0 || lcol[t] >= P.g1) gh.push_back(lcol[t]);
  std::sort(gh.begin(), gh.end());
  gh.erase(std::unique(gh.begin(), gh.end()), gh.end());
  P.ghosts = std::move(gh);
  P.recv_off.push_back(0);
  for (size_t t = 0; t < P.ghosts.size(); ++t) {
    const int q = owner(P.ghosts[t]);
    if (P.nbr.empty() || P.nbr.back() != q) {
      if (!P.nbr.empty()) P.recv_off.push_back((int64_t)t);
      P.nbr.push_back(q);
    }
  }
  if (!P.nbr.empty()) P.recv_off.push_back((int64_t)P.ghosts.size());
  // send lists, neighbour by neighbour (ascending), rows ascending
  P.send_off.assign(1, 0);
  for (int q : P.nbr) {
    const int64_t b0 = block_start(n, nparts, q), b1 = block_start(n, nparts, q + 1);
    for (int64_t i = 0; i < m; ++i)
      for (int64_t t = lrp[i]; t < lrp[i + 1]; ++t)
        if (lcol[t] >= b0 && lcol[t] < b1) {
          P.send_g.push_back((int32_t)(P.g0 + i));
          break;
        }
    P.send_off.push_back((int64_t)P.send_g.size());
  }
  return P;
}

void plan_partitions(int64_t n, const int64_t* rowptr, const int32_t* col, int nparts,
                     std::vector<PartPlan>& plans) {
  plans.assign(nparts, PartPlan());
#pragma omp parallel for schedule(dynamic, 1)
  for (int p = 0; p < nparts; ++p) {
    const int64_t g0 = block_start(n, nparts, p), g1 = block_start(n, nparts, p + 1);
    std::vector<int64_t> lrp(g1 - g0 + 1);
    for (int64_t i = g0; i <= g1; ++i) lrp[i - g0] = rowptr[i] - rowptr[g0];
    plans[p] = plan_from_rows(n, nparts, p, lrp.data(), col + rowptr[g0]);
  }
}

// Interior-first order of the row blocks of plan_partitions (DESIGN.md
// "Multi-GPU"): inside block [g0, g1) the rows with no column outside the block
// come first, then the boundary rows (the ones that read ghosts), each group in
// the incoming order.  order[new] = old (internal indices); n_int[p] = interior
// rows of block p.  The blocks and their ghost sets are unchanged.
void interior_first(int64_t n, const int64_t* rowptr, const int32_t* col, int nparts,
                    std::vector<int32_t>& order, std::vector<int64_t>& n_int) {
  order.resize(n);
  n_int.assign(nparts, 0);
#pragma omp parallel for schedule(dynamic, 1)
  for (int p = 0; p < nparts; ++p) {
    const int64_t g0 = (n * p) / nparts, g1 = (n * (p + 1)) / nparts;  // plan_partitions' bounds
    std::vector<uint8_t> inner(g1 - g0, 1);
    for (int64_t i = g0; i < g1; ++i)
      for (int64_t t = rowptr[i]; t < rowptr[i + 1]; ++t)
        if (col[t] < g0 || col[t] >= g1) {
          inner[i - g0] = 0;
          break;
        }
    int64_t w = g0;
    for (int64_t i = g0; i < g1; ++i)
      if (inner[i - g0]) order[w++] = (int32_t)i;
    n_int[p] = w - g0;
    for (int64_t i = g0; i < g1; ++i)
      if (!inner[i - g0]) order[w++] = (int32_t)i;
  }
}

}  // namespace tcb
