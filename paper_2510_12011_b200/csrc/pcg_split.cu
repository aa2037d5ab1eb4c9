// pcg_split.cu -- Algorithm 1 for a row-partitioned system
// (multi-GPU over NCCL, or several partitions of one GPU): the same data flow
// as the persistent kernel, cut at the two global reductions so that a
// collective can sit between the phases.
//
// Per partition and iteration:
//   pack_p : p_it = z + beta p_{it-1} of the owned nodes other partitions need
//   (halo) : received into the ghost region of z (the ghost region of p stays 0,
//            so z_c + beta p_c == p_c for every ghost column c)
//   S      : q = A p_it, x += alpha_{it-1} p_{it-1}, rank partial of p.q
//   (allreduce p.q)
//   U      : alpha = rho / p.q, z -= alpha q / diag (z-form), rank partials r.z, z.z
//   (allreduce)
//   scalar : one thread: stopping test, beta, rho (identical on every partition,
//            because the all-reduced sums are bitwise identical)
// Every kernel returns at once when the scalar state says "done".
#include "pcg_common.cuh"

namespace tcb {

constexpr int kSplitThreads = 256;
constexpr int kSplitWarps = kSplitThreads / 32;

// CTA partial -> part[blockIdx]; the last CTA to finish sums all partials in
// index order (deterministic) into *out and re-arms the ticket.
__device__ __forceinline__ void reduce_to_rank(double2 acc, double2* part, unsigned int* ticket,
                                               double2* out, double2* sh) {
  __shared__ bool last;
  const double2 b = block_sum2(acc, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = b;
    __threadfence();
    const unsigned int t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double2 s = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < (int)gridDim.x; t += blockDim.x) {
    const double2 u = __ldcg(part + t);
    s.x += u.x;
    s.y += u.y;
  }
  s = block_sum2(s, sh);
  if (threadIdx.x == 0) {
    *out = s;
    *ticket = 0u;
  }
}

// Halo overlap: the rows of a partition are numbered
// interior-first, so an S / RHS pass runs as two launches on the same grid --
// phase 0 over the interior slices [0, nslices_int) while the halo is in
// flight, phase 1 over the rest once it has landed.  Phase 0 leaves each CTA's
// partial in part[grid + blockIdx]; phase 1 adds it to its own before the
// deterministic reduction (the same per-CTA order at any timing).  Phase 2 =
// one launch over every slice (no halo).
__device__ __forceinline__ void reduce_phase(const SplitArgs& a, double2 acc, double2* out, double2* sh) {
  if (a.phase == 0) {
    const double2 b = block_sum2(acc, sh);
    if (threadIdx.x == 0) a.part[gridDim.x + blockIdx.x] = b;
    return;
  }
  if (a.phase == 1 && threadIdx.x == 0) {
    const double2 b0 = a.part[gridDim.x + blockIdx.x];
    acc.x += b0.x;   // thread 0 carries the interior partial into the block sum
    acc.y += b0.y;
  }
  reduce_to_rank(acc, a.part, a.ticket, out, sh);
}

template <int MODE>
__global__ void __launch_bounds__(kSplitThreads, 4) split_rhs_kernel(SplitArgs a) {
  __shared__ double2 sh[kSplitWarps];
  if (a.flags[0]) return;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kSplitWarps + (threadIdx.x >> 5), nw = gridDim.x * kSplitWarps;
  double2 acc = make_double2(0.0, 0.0);
  for (int s = a.s0 + gw; s < a.s1; s += nw) {
    const int64_t base = __ldg(a.slice_ptr + s);
    const int w = (int)((__ldg(a.slice_ptr + s + 1) - base) >> 5);
    const int64_t i = (int64_t)s * kSellC + lane;
    const double sum = row_rhs_direct(base, w, lane, a.col, a.A, a.K, a.up, a.vp);  // r_0 = A u' - K v'
    const double zi = __ldg(a.dinv + i) * sum;
    a.r[i] = sum;
    a.z[i] = zi;
    acc.x += sum * zi;
    acc.y += zi * zi;
  }
  reduce_phase(a, acc, a.red, sh);
}

// rho_0 = r.z, ||z_0|| from the all-reduced sums (reading C4: ||z_0|| < eps_a -> done)
__global__ void split_init_kernel(SplitArgs a) {
  Scalars s{};
  const double2 g = a.red[0];
  s.rho = g.x;
  s.zeta = sqrt(g.y);
  s.zref = s.zeta;
  s.plast = -1;
  if (isnan(s.rho) || isnan(s.zeta)) { s.nan = 1; s.done = 1; }
  else if (s.zeta < a.eps_a) { s.conv = 1; s.done = 1; }
  if (a.flags[0]) s.done = 1;
  *a.sc = s;
}

__global__ void split_pack_p_kernel(SplitArgs a) {
  const Scalars s = *a.sc;
  if (s.done) return;
  const double* pold = (s.it & 1) ? a.p0 : a.p1;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < a.n_send;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = a.send_idx[j];
    a.send_buf[j] = s.it == 0 ? a.z[i] : a.z[i] + s.beta * pold[i];
  }
}

__global__ void pack_gather_kernel(int64_t m, const int32_t* __restrict__ idx,
                                   const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * blockDim.x)
    dst[j] = src[idx[j]];
}

__global__ void __launch_bounds__(kSplitThreads, 8) split_S_kernel(SplitArgs a) {
  __shared__ double2 sh[kSplitWarps];
  const Scalars s = *a.sc;
  if (s.done) return;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kSplitWarps + (threadIdx.x >> 5), nw = gridDim.x * kSplitWarps;
  double* __restrict__ pnew = (s.it & 1) ? a.p1 : a.p0;
  const double* __restrict__ pold = (s.it & 1) ? a.p0 : a.p1;
  const bool first = s.it == 0;
  double2 acc = make_double2(0.0, 0.0);
  for (int sl = a.s0 + gw; sl < a.s1; sl += nw) {
    const int64_t base = __ldg(a.slice_ptr + sl);
    const int w = (int)((__ldg(a.slice_ptr + sl + 1) - base) >> 5);
    const int64_t i = (int64_t)sl * kSellC + lane;
    double pi = a.z[i];
    if (!first) {
      const double po = pold[i];
      pi += s.beta * po;
      a.x[i] += s.alpha * po;            // deferred x += alpha_{it-1} p_{it-1}
    }
    ColIdx ci;
    ci.c32 = a.col;
    ci.c16 = nullptr;
    ci.kb = nullptr;
    const double sum = first ? row_Ap_direct<true>(base, w, lane, ci, a.A, a.z, nullptr, 0.0)
                             : row_Ap_direct<false>(base, w, lane, ci, a.A, a.z, pold, s.beta);
    pnew[i] = pi;
    a.q[i] = sum;
    acc.x += pi * sum;
  }
  reduce_phase(a, acc, a.red + 1, sh);
}

__global__ void __launch_bounds__(kSplitThreads, 8) split_U_kernel(SplitArgs a) {
  __shared__ double2 sh[kSplitWarps];
  const Scalars s = *a.sc;
  if (s.done) return;
  const double alpha = s.rho / a.red[1].x;   // alpha_k = rho_k / p.q (all-reduced)
  double2 acc = make_double2(0.0, 0.0);
  const int64_t n = (int64_t)a.nslices * kSellC;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // z-form (pcg.cu TCB_ZFORM): z -= alpha D^-1 q, r.z = sum z^2 / d^-1
    const double di = __ldg(a.dinv + i);
    const double zi = a.z[i] - alpha * (di * a.q[i]);
    a.z[i] = zi;
    acc.x += di != 0.0 ? zi * (zi / di) : 0.0;
    acc.y += zi * zi;
  }
  reduce_to_rank(acc, a.part, a.ticket, a.red, sh);
}

// The stopping test of Algorithm 1 and the scalar recurrences (one thread).
__global__ void split_scalar_kernel(SplitArgs a) {
  Scalars s = *a.sc;
  if (s.done) return;
  const double pq = a.red[1].x;
  const double2 g = a.red[0];
  s.plast = s.it & 1;                  // p buffer written by this iteration
  s.it += 1;
  if (isnan(pq)) { s.nan = 1; s.done = 1; *a.sc = s; return; }
  s.alpha = s.rho / pq;
  const double zeta = sqrt(g.y);
  s.zeta = zeta;
  if (isnan(zeta) || isnan(g.x)) { s.nan = 1; s.done = 1; }
  else if (zeta < a.eps_a || zeta / s.zref < a.eps_r) { s.conv = 1; s.done = 1; }
  else if (s.it >= a.max_iters) { s.done = 1; }
  else {
    s.beta = g.x / s.rho;
    s.rho = g.x;
    if (a.rel_mode == 0) s.zref = zeta;
  }
  *a.sc = s;
}

// x += alpha p_last (Alg. 1 updates x before its test), step report, fail budget.
__global__ void split_final_kernel(SplitArgs a) {
  const Scalars s = *a.sc;
  if (!s.nan && s.plast >= 0) {
    const double* __restrict__ pl = s.plast ? a.p1 : a.p0;
    const int64_t n = (int64_t)a.nslices * kSellC;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
      a.x[i] += s.alpha * pl[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && !a.flags[0]) {
    a.stat->iters = s.it;
    a.stat->converged = s.conv;
    a.stat->znorm = s.zeta;
    int32_t* f = a.flags;
    if (s.nan) {
      f[0] = 1; f[1] = 1; f[4] = a.step_tag;
    } else {
      f[2] = s.conv ? 0 : f[2] + 1;
      if (f[3] > 0 && f[2] >= f[3]) { f[0] = 1; f[4] = a.step_tag; }
    }
  }
}

// loopback "allreduce": the partitions' rank partials summed in partition order
__global__ void sum_partials_kernel(double2* const* reds, int nparts, int slot) {
  double2 t = make_double2(0.0, 0.0);
  for (int p = 0; p < nparts; ++p) {
    const double2 u = reds[p][slot];
    t.x += u.x;
    t.y += u.y;
  }
  for (int p = 0; p < nparts; ++p) reds[p][slot] = t;
}

static int sm_count_split() {
  static int v = 0;
  if (!v) {
    int d = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    if (v <= 0) v = 148;
  }
  return v;
}

// one full wave of the S kernel (grid-stride over slices)
int split_grid(int32_t nslices) {
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, split_S_kernel, kSplitThreads, 0);
    if (per_sm < 1) per_sm = 1;
  }
  int need = (nslices + kSplitWarps - 1) / kSplitWarps;
  int cap = sm_count_split() * per_sm;
  return need < 1 ? 1 : (need < cap ? need : cap);
}

static int small_grid(int64_t m) {
  int64_t b = (m + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 592 ? 592 : b));
}

cudaError_t launch_split_rhs(const SplitArgs& a, int grid, cudaStream_t s) {
  split_rhs_kernel<1><<<grid, kSplitThreads, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_split_init(const SplitArgs& a, cudaStream_t s) {
  split_init_kernel<<<1, 1, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_split_pack_p(const SplitArgs& a, cudaStream_t s) {
  if (a.n_send == 0) return cudaSuccess;
  split_pack_p_kernel<<<small_grid(a.n_send), 256, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_pack_gather(int64_t m, const int32_t* idx, const double* src, double* dst,
                               cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  pack_gather_kernel<<<small_grid(m), 256, 0, s>>>(m, idx, src, dst);
  return cudaGetLastError();
}
cudaError_t launch_split_S(const SplitArgs& a, int grid, cudaStream_t s) {
  split_S_kernel<<<grid, kSplitThreads, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_split_U(const SplitArgs& a, int grid, cudaStream_t s) {
  split_U_kernel<<<grid, kSplitThreads, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_split_scalar(const SplitArgs& a, cudaStream_t s) {
  split_scalar_kernel<<<1, 1, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_split_final(const SplitArgs& a, int grid, cudaStream_t s) {
  split_final_kernel<<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_sum_partials(double2* const* reds, int nparts, int slot, cudaStream_t s) {
  sum_partials_kernel<<<1, 1, 0, s>>>(reds, nparts, slot);
  return cudaGetLastError();
}

}  // namespace tcb
