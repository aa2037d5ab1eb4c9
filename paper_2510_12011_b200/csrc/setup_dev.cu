// setup_dev.cu -- device-side setup of a single-partition system (SURVEY 8f
// row f3): the CSR pattern of M u K, Reverse Cuthill-McKee (SPEC
// S:146 tie rules), the permuted pattern, its SELL-32 layout and the element
// incidence the assembly kernel gathers from -- all on the GPU, from the element
// list alone.  Results are identical to the host path (setup_host.cpp), which
// the CPU tests pin against the oracle:
//  * pattern: row i = {i} u {nodes sharing an element with i}, ascending -- here
//    the sorted, de-duplicated (row, col) keys of every element's k x k node
//    pairs plus the n diagonal keys (one radix sort + unique);
//  * RCM: the host algorithm is Cuthill-McKee BFS -- per component start at the
//    lowest (degree, index) unvisited node, append each dequeued node's unseen
//    neighbours in ascending (degree, index) -- reversed.  Level-synchronously:
//    a node of level L+1 is appended by its FIRST level-L neighbour in CM order,
//    so level L+1 in CM order is its nodes sorted by (position of that first
//    neighbour, degree, index); one 64-bit key sort per level reproduces the
//    sequential order exactly;
//  * incidence: a stable sort of (node, element slot) pairs keeps each node's
//    elements in ascending element order (the assembly's summation order);
//  * partitioned systems (nparts > 1, SURVEY 8f f3 "RCM/partition on device"):
//    the interior-first order of the row blocks (setup_host.cpp interior_first)
//    as one 64-bit key sort (block, reads-a-ghost, row), and the global permuted
//    CSR as output instead of a SELL layout; each part's plan and SELL are then
//    built from its own rows (api.cu assemble_device_parts).
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <vector>

#include "internal.h"

namespace tcb {

namespace {

__global__ void k_pair_keys(int64_t E, int k, const int32_t* __restrict__ tets, int sh,
                            uint64_t* __restrict__ keys) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t kk = (int64_t)k * k;
  if (t >= E * kk) return;
  const int64_t e = t / kk;
  const int ab = (int)(t - e * kk), a = ab / k, b = ab - a * k;
  keys[t] = ((uint64_t)tets[k * e + a] << sh) | (uint64_t)tets[k * e + b];
}

__global__ void k_diag_keys(int64_t n, int sh, uint64_t* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = ((uint64_t)i << sh) | (uint64_t)i;
}

// sorted unique (row, col) keys -> CSR (every row holds its diagonal, so every
// row occurs and rows are contiguous)
__global__ void k_keys_to_csr(int64_t nnz, int sh, const uint64_t* __restrict__ keys,
                              int64_t* __restrict__ rowptr, int32_t* __restrict__ col) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnz) return;
  const uint64_t key = keys[t];
  const int64_t r = (int64_t)(key >> sh);
  col[t] = (int32_t)(key & ((1ull << sh) - 1));
  if (t == 0 || (int64_t)(keys[t - 1] >> sh) != r) rowptr[r] = t;
  if (t == nnz - 1) rowptr[r + 1] = nnz;
}

__global__ void k_degree_keys(int64_t n, const int64_t* __restrict__ rowptr, uint64_t* __restrict__ keys,
                              int32_t* __restrict__ ids) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t deg = (uint64_t)(rowptr[i + 1] - rowptr[i] - 1);  // off-diagonal entries
  keys[i] = (deg << 32) | (uint64_t)i;
  ids[i] = (int32_t)i;
}

__global__ void k_rank(int64_t n, const int32_t* __restrict__ byd, int32_t* __restrict__ rank) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) rank[byd[j]] = (int32_t)j;
}

// one warp per frontier node: every unvisited neighbour records the smallest
// frontier position that reaches it and is appended once to `next`
// (state: 0 unseen, 1 discovered in this level, 2 in an earlier level / frontier)
__global__ void k_expand(int64_t fs, int64_t fe, const int32_t* __restrict__ order,
                         const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                         int32_t* state, int32_t* parent, int32_t* next, unsigned int* cnt) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (fs + w >= fe) return;
  const int32_t p = (int32_t)(fs + w);
  const int32_t v = order[p];
  for (int64_t t = rowptr[v] + lane; t < rowptr[v + 1]; t += 32) {
    const int32_t u = col[t];
    if (state[u] == 2) continue;
    atomicMin(parent + u, p);
    if (atomicCAS(state + u, 0, 1) == 0) next[atomicAdd(cnt, 1u)] = u;
  }
}

__global__ void k_level_keys(int64_t m, const int32_t* __restrict__ next, const int32_t* __restrict__ parent,
                             const int32_t* __restrict__ rank, uint64_t* __restrict__ keys) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int32_t u = next[j];
  keys[j] = ((uint64_t)(uint32_t)parent[u] << 32) | (uint64_t)(uint32_t)rank[u];
}

__global__ void k_mark(int64_t m, const int32_t* __restrict__ nodes, int32_t* state) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < m) state[nodes[j]] = 2;
}

__global__ void k_first_unvisited(int64_t from, int64_t n, const int32_t* __restrict__ byd,
                                  const int32_t* __restrict__ state, unsigned long long* best) {
  const int64_t j = from + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n && state[byd[j]] == 0) atomicMin(best, (unsigned long long)j);
}

__global__ void k_reverse_inv(int64_t n, const int32_t* __restrict__ order, int32_t* __restrict__ perm,
                              int32_t* __restrict__ inv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t o = order[n - 1 - i];
  perm[i] = o;
  inv[o] = (int32_t)i;
}

__global__ void k_identity(int64_t n, int32_t* __restrict__ perm, int32_t* __restrict__ inv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) perm[i] = inv[i] = (int32_t)i;
}

__global__ void k_permuted_keys(int64_t n, int sh, const int64_t* __restrict__ rowptr,
                                const int32_t* __restrict__ col, const int32_t* __restrict__ inv,
                                uint64_t* __restrict__ keys) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint64_t ri = (uint64_t)inv[r] << sh;
  for (int64_t t = rowptr[r]; t < rowptr[r + 1]; ++t) keys[t] = ri | (uint64_t)inv[col[t]];
}

__global__ void k_slice_width(int64_t n, int32_t nslices, const int64_t* __restrict__ rowptr,
                              int32_t* __restrict__ rowlen, int64_t* __restrict__ width) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one thread per padded row
  if (i >= (int64_t)nslices * kSellC) return;
  const int32_t len = i < n ? (int32_t)(rowptr[i + 1] - rowptr[i]) : 0;
  if (i < n) rowlen[i] = len;
  int32_t m = len;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) width[i / kSellC] = (int64_t)m * kSellC;
}

__global__ void k_fill_sell(int64_t n, int32_t nslices, const int64_t* __restrict__ rowptr,
                            const int32_t* __restrict__ col, const int64_t* __restrict__ sp,
                            int32_t* __restrict__ scol) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)nslices * kSellC) return;
  const int64_t s = i / kSellC, l = i - s * kSellC;
  const int64_t base = sp[s], w = (sp[s + 1] - base) / kSellC;
  const int64_t len = i < n ? rowptr[i + 1] - rowptr[i] : 0;
  for (int64_t k = 0; k < w; ++k)
    scol[sell_slot(base, w, k, l)] = k < len ? col[rowptr[i] + k] : (int32_t)i;  // padding: self
}

__global__ void k_tets_perm(int64_t m, const int32_t* __restrict__ tets, const int32_t* __restrict__ inv,
                            int32_t* __restrict__ tets2, int32_t* __restrict__ slot) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  tets2[t] = inv[tets[t]];
  slot[t] = (int32_t)t;
}

__global__ void k_count(int64_t m, const int32_t* __restrict__ keys, int64_t* __restrict__ cnt) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + keys[t] + 1), 1ull);
}

__global__ void k_inc_code(int64_t m, int k, const int32_t* __restrict__ slot, int32_t* __restrict__ inc) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int32_t s = slot[t], e = s / k, a = s - e * k;
  inc[t] = 4 * e + a;
}

// block of plan_partitions' bounds g0(p) = floor(n p / P) holding row i
__device__ __forceinline__ int block_of(int64_t i, int64_t n, int P) {
  int p = (int)((i * P) / n);
  while (p + 1 < P && (n * (p + 1)) / P <= i) ++p;
  while (p > 0 && (n * p) / P > i) --p;
  return p;
}

// interior-first keys: (block, reads-a-ghost flag, row);
// sorting them gives, per block, the interior rows then the boundary rows, each
// in the incoming order.  Interior rows are counted per block.
__global__ void k_interior_keys(int64_t n, int P, const int64_t* __restrict__ rowptr,
                                const int32_t* __restrict__ col, uint64_t* __restrict__ keys,
                                unsigned long long* __restrict__ n_int) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int p = block_of(i, n, P);
  const int64_t g0 = (n * p) / P, g1 = (n * (p + 1)) / P;
  uint64_t out = 0;
  for (int64_t t = rowptr[i]; t < rowptr[i + 1]; ++t)
    if (col[t] < g0 || col[t] >= g1) {
      out = 1;
      break;
    }
  keys[i] = ((uint64_t)p << 33) | (out << 32) | (uint64_t)i;
  if (!out) atomicAdd(n_int + p, 1ull);
}

// perm2[new] = perm[order[new]] (order = low 32 bits of the sorted keys), inv2
__global__ void k_compose(int64_t n, const uint64_t* __restrict__ keys, const int32_t* __restrict__ perm,
                          int32_t* __restrict__ perm2, int32_t* __restrict__ inv2) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int32_t o = perm[(int64_t)(keys[j] & 0xffffffffull)];
  perm2[j] = o;
  inv2[o] = (int32_t)j;
}

inline unsigned nb(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

struct Scratch {  // cudaMalloc'ed temporaries freed on scope exit
  std::vector<void*> p;
  template <class T>
  cudaError_t get(T** out, int64_t count) {
    void* v = nullptr;
    cudaError_t e = cudaMalloc(&v, (size_t)std::max<int64_t>(count, 1) * sizeof(T));
    if (e == cudaSuccess) {
      p.push_back(v);
      *out = (T*)v;
    }
    return e;
  }
  void drop(void* v) {
    auto it = std::find(p.begin(), p.end(), v);
    if (it != p.end()) {
      cudaFree(v);
      p.erase(it);
    }
  }
  ~Scratch() {
    for (void* v : p) cudaFree(v);
  }
};

#define DS_TRY(x)                        \
  do {                                   \
    cudaError_t e_ = (x);                \
    if (e_ != cudaSuccess) return e_;    \
  } while (0)

template <class F>
cudaError_t cub_call(Scratch& S, F&& f) {  // f(temp, bytes) twice: size query, run
  size_t bytes = 0;
  DS_TRY(f(nullptr, bytes));
  char* tmp = nullptr;
  DS_TRY(S.get(&tmp, (int64_t)bytes));
  cudaError_t e = f(tmp, bytes);
  S.drop(tmp);
  return e;
}

// sorted unique keys of `m` raw keys (in place in `a`, b scratch) -> count
cudaError_t sort_unique(Scratch& S, uint64_t* a, uint64_t* b, int64_t m, int bits, int64_t* count,
                        cudaStream_t s) {
  cub::DoubleBuffer<uint64_t> db(a, b);
  DS_TRY(cub_call(S, [&](void* t, size_t& by) {
    return cub::DeviceRadixSort::SortKeys(t, by, db, m, 0, bits, s);
  }));
  uint64_t* sorted = db.Current();
  uint64_t* other = db.Alternate();
  int64_t* d_cnt = nullptr;
  DS_TRY(S.get(&d_cnt, 1));
  DS_TRY(cub_call(S, [&](void* t, size_t& by) {
    return cub::DeviceSelect::Unique(t, by, sorted, other, d_cnt, m, s);
  }));
  DS_TRY(cudaMemcpyAsync(count, d_cnt, 8, cudaMemcpyDeviceToHost, s));
  DS_TRY(cudaStreamSynchronize(s));
  if (other != a) DS_TRY(cudaMemcpyAsync(a, other, (size_t)*count * 8, cudaMemcpyDeviceToDevice, s));
  S.drop(d_cnt);
  return cudaSuccess;
}

}  // namespace

cudaError_t dev_setup(int64_t n, int64_t E, int k, const int32_t* d_tets, int use_rcm, int nparts,
                      bool reorder_parts, bool csr_out, DevPattern& out, cudaStream_t s) {
  Scratch S;
  int sh = 1;
  while ((1ll << sh) < n) ++sh;
  // ---- pattern of the original numbering --------------------------------------
  const int64_t m = E * k * k + n;
  uint64_t *ka = nullptr, *kb = nullptr;
  DS_TRY(S.get(&ka, m));
  DS_TRY(S.get(&kb, m));
  if (E > 0) k_pair_keys<<<nb(E * k * k), 256, 0, s>>>(E, k, d_tets, sh, ka);
  k_diag_keys<<<nb(n), 256, 0, s>>>(n, sh, ka + E * k * k);
  DS_TRY(cudaGetLastError());
  int64_t nnz = 0;
  DS_TRY(sort_unique(S, ka, kb, m, 2 * sh, &nnz, s));
  int64_t* rp = nullptr;
  int32_t* cl = nullptr;
  DS_TRY(S.get(&rp, n + 1));
  DS_TRY(S.get(&cl, nnz));
  k_keys_to_csr<<<nb(nnz), 256, 0, s>>>(nnz, sh, ka, rp, cl);
  DS_TRY(cudaGetLastError());
  // ---- RCM (perm: internal -> original) ----------------------------------------
  DS_TRY(cudaMalloc(&out.perm, n * 4));
  DS_TRY(cudaMalloc(&out.inv, n * 4));
  if (use_rcm) {
    int32_t *ids = nullptr, *byd = nullptr, *rank = nullptr, *order = nullptr, *parent = nullptr,
            *next = nullptr, *nsorted = nullptr;
    int32_t* state = nullptr;
    unsigned int* cnt = nullptr;
    unsigned long long* best = nullptr;
    DS_TRY(S.get(&ids, n));
    DS_TRY(S.get(&byd, n));
    DS_TRY(S.get(&rank, n));
    DS_TRY(S.get(&order, n));
    DS_TRY(S.get(&parent, n));
    DS_TRY(S.get(&next, n));
    DS_TRY(S.get(&nsorted, n));
    DS_TRY(S.get(&state, n));
    DS_TRY(S.get(&cnt, 1));
    DS_TRY(S.get(&best, 1));
    // nodes by (degree, index)
    k_degree_keys<<<nb(n), 256, 0, s>>>(n, rp, kb, ids);
    uint64_t* kc = ka;  // the pattern keys are no longer needed
    DS_TRY(cub_call(S, [&](void* t, size_t& by) {
      return cub::DeviceRadixSort::SortPairs(t, by, kb, kc, ids, byd, n, 0, 64, s);
    }));
    k_rank<<<nb(n), 256, 0, s>>>(n, byd, rank);
    DS_TRY(cudaMemsetAsync(state, 0, n * 4, s));
    DS_TRY(cudaMemsetAsync(parent, 0x7f, n * 4, s));  // 0x7f7f7f7f: larger than any position
    int64_t fs = 0, fe = 0, scan = 0;
    while (fe < n) {
      if (fs == fe) {  // new component: lowest (degree, index) unvisited node
        const unsigned long long init = ULLONG_MAX;
        DS_TRY(cudaMemcpyAsync(best, &init, 8, cudaMemcpyHostToDevice, s));
        k_first_unvisited<<<nb(n - scan), 256, 0, s>>>(scan, n, byd, state, best);
        unsigned long long j = 0;
        DS_TRY(cudaMemcpyAsync(&j, best, 8, cudaMemcpyDeviceToHost, s));
        DS_TRY(cudaStreamSynchronize(s));
        if (j == ULLONG_MAX) return cudaErrorUnknown;  // cannot happen: fe < n
        scan = (int64_t)j;
        DS_TRY(cudaMemcpyAsync(order + fe, byd + scan, 4, cudaMemcpyDeviceToDevice, s));
        k_mark<<<1, 32, 0, s>>>(1, order + fe, state);
        fe += 1;
      }
      DS_TRY(cudaMemsetAsync(cnt, 0, 4, s));
      k_expand<<<nb((fe - fs) * 32), 256, 0, s>>>(fs, fe, order, rp, cl, state, parent, next, cnt);
      unsigned int mnext = 0;
      DS_TRY(cudaMemcpyAsync(&mnext, cnt, 4, cudaMemcpyDeviceToHost, s));
      DS_TRY(cudaStreamSynchronize(s));
      fs = fe;
      if (mnext == 0) continue;
      k_level_keys<<<nb(mnext), 256, 0, s>>>(mnext, next, parent, rank, kb);
      DS_TRY(cub_call(S, [&](void* t, size_t& by) {
        return cub::DeviceRadixSort::SortPairs(t, by, kb, kc, next, order + fe, (int64_t)mnext, 0, 64, s);
      }));
      k_mark<<<nb(mnext), 256, 0, s>>>(mnext, order + fe, state);
      fe += mnext;
    }
    k_reverse_inv<<<nb(n), 256, 0, s>>>(n, order, out.perm, out.inv);
  } else {
    k_identity<<<nb(n), 256, 0, s>>>(n, out.perm, out.inv);
  }
  DS_TRY(cudaGetLastError());
  // ---- permuted pattern (P A P^T) -------------------------------------------------
  // (rp, cl) = original pattern; the permuted one goes to (rp2, cl2), which is
  // (rp, cl) itself for a single partition (the original is no longer needed)
  // partitioned output (csr_out): the global permuted CSR; reorder_parts: the
  // interior-first order of the nparts blocks first (off: plain RCM order, A/B)
  const bool reorder = csr_out && reorder_parts && nparts > 1;
  int64_t* rp2 = rp;
  int32_t* cl2 = cl;
  if (csr_out) {
    DS_TRY(cudaMalloc(&out.rowptr, (n + 1) * 8));
    DS_TRY(cudaMalloc(&out.colidx, nnz * 4));
    rp2 = out.rowptr;
    cl2 = out.colidx;
  }
  auto permute = [&]() -> cudaError_t {
    k_permuted_keys<<<nb(n), 256, 0, s>>>(n, sh, rp, cl, out.inv, kb);
    DS_TRY(cudaGetLastError());
    cub::DoubleBuffer<uint64_t> db(kb, ka);
    DS_TRY(cub_call(S, [&](void* t, size_t& by) {
      return cub::DeviceRadixSort::SortKeys(t, by, db, nnz, 0, 2 * sh, s);
    }));
    k_keys_to_csr<<<nb(nnz), 256, 0, s>>>(nnz, sh, db.Current(), rp2, cl2);
    return cudaGetLastError();
  };
  DS_TRY(permute());
  if (reorder) {
    // interior-first order inside each row block (setup_host.cpp interior_first),
    // then the pattern again in the final order
    unsigned long long* cnt_int = nullptr;
    int32_t *perm2 = nullptr, *inv2 = nullptr;
    DS_TRY(S.get(&cnt_int, nparts));
    DS_TRY(S.get(&perm2, n));
    DS_TRY(S.get(&inv2, n));
    DS_TRY(cudaMemsetAsync(cnt_int, 0, nparts * 8, s));
    k_interior_keys<<<nb(n), 256, 0, s>>>(n, nparts, rp2, cl2, kb, cnt_int);
    DS_TRY(cudaGetLastError());
    int pbits = 1;
    while ((1 << pbits) < nparts) ++pbits;
    cub::DoubleBuffer<uint64_t> db(kb, ka);
    DS_TRY(cub_call(S, [&](void* t, size_t& by) {
      return cub::DeviceRadixSort::SortKeys(t, by, db, n, 0, 33 + pbits, s);
    }));
    k_compose<<<nb(n), 256, 0, s>>>(n, db.Current(), out.perm, perm2, inv2);
    DS_TRY(cudaGetLastError());
    DS_TRY(cudaMemcpyAsync(out.perm, perm2, n * 4, cudaMemcpyDeviceToDevice, s));
    DS_TRY(cudaMemcpyAsync(out.inv, inv2, n * 4, cudaMemcpyDeviceToDevice, s));
    std::vector<unsigned long long> h(nparts);
    DS_TRY(cudaMemcpyAsync(h.data(), cnt_int, nparts * 8, cudaMemcpyDeviceToHost, s));
    DS_TRY(cudaStreamSynchronize(s));
    out.n_int.assign(h.begin(), h.end());
    DS_TRY(permute());
  }
  S.drop(ka);
  S.drop(kb);
  out.n = n;
  out.nnz = nnz;
  if (csr_out) {  // partitioned: the global CSR is the output; SELL is per part (host)
    S.drop(rp);
    S.drop(cl);
    out.nslices = 0;
    out.nnz_pad = 0;
  } else {
  out.nslices = (int32_t)((n + kSellC - 1) / kSellC);
  DS_TRY(cudaMalloc(&out.rowlen, n * 4));
  DS_TRY(cudaMalloc(&out.slice_ptr, (out.nslices + 1) * 8));
  int64_t* width = nullptr;
  DS_TRY(S.get(&width, out.nslices + 1));
  k_slice_width<<<nb((int64_t)out.nslices * kSellC), 256, 0, s>>>(n, out.nslices, rp, out.rowlen, width);
  DS_TRY(cudaMemsetAsync(width + out.nslices, 0, 8, s));
  DS_TRY(cub_call(S, [&](void* t, size_t& by) {
    return cub::DeviceScan::ExclusiveSum(t, by, width, out.slice_ptr, out.nslices + 1, s);
  }));
  DS_TRY(cudaMemcpyAsync(&out.nnz_pad, out.slice_ptr + out.nslices, 8, cudaMemcpyDeviceToHost, s));
  DS_TRY(cudaStreamSynchronize(s));
  DS_TRY(cudaMalloc(&out.col, out.nnz_pad * 4));
  k_fill_sell<<<nb((int64_t)out.nslices * kSellC), 256, 0, s>>>(n, out.nslices, rp, cl, out.slice_ptr, out.col);
  DS_TRY(cudaGetLastError());
  S.drop(rp);
  S.drop(cl);
  }
  // ---- permuted elements and their incidence (ascending element order per node) ----
  const int64_t ke = E * k;
  DS_TRY(cudaMalloc(&out.tets2, std::max<int64_t>(ke, 1) * 4));
  DS_TRY(cudaMalloc(&out.inc, std::max<int64_t>(ke, 1) * 4));
  DS_TRY(cudaMalloc(&out.iptr, (n + 1) * 8));
  int32_t *slot = nullptr, *key2 = nullptr, *slot2 = nullptr;
  DS_TRY(S.get(&slot, ke));
  DS_TRY(S.get(&key2, ke));
  DS_TRY(S.get(&slot2, ke));
  DS_TRY(cudaMemsetAsync(out.iptr, 0, (n + 1) * 8, s));
  if (ke > 0) {
    k_tets_perm<<<nb(ke), 256, 0, s>>>(ke, d_tets, out.inv, out.tets2, slot);
    k_count<<<nb(ke), 256, 0, s>>>(ke, out.tets2, out.iptr);
    DS_TRY(cub_call(S, [&](void* t, size_t& by) {  // stable: slots stay ascending per node
      return cub::DeviceRadixSort::SortPairs(t, by, out.tets2, key2, slot, slot2, ke, 0, sh, s);
    }));
    k_inc_code<<<nb(ke), 256, 0, s>>>(ke, k, slot2, out.inc);
    DS_TRY(cub_call(S, [&](void* t, size_t& by) {
      return cub::DeviceScan::InclusiveSum(t, by, out.iptr, out.iptr, n + 1, s);
    }));
  }
  DS_TRY(cudaGetLastError());
  return cudaStreamSynchronize(s);
}

__global__ void k_gather3(int64_t n, const int32_t* __restrict__ perm, const double* __restrict__ in,
                          double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t o = perm[i];
#pragma unroll
  for (int q = 0; q < 3; ++q) out[3 * i + q] = in[3 * o + q];
}

cudaError_t dev_gather3(int64_t n, const int32_t* perm, const double* in, double* out, cudaStream_t s) {
  if (n > 0) k_gather3<<<nb(n), 256, 0, s>>>(n, perm, in, out);
  return cudaGetLastError();
}

void dev_setup_free(DevPattern& p) {
  cudaFree(p.rowptr);
  cudaFree(p.colidx);
  cudaFree(p.perm);
  cudaFree(p.inv);
  cudaFree(p.slice_ptr);
  cudaFree(p.col);
  cudaFree(p.rowlen);
  cudaFree(p.iptr);
  cudaFree(p.inc);
  cudaFree(p.tets2);
  p = DevPattern{};
}

}  // namespace tcb
