// pcg_graph.cu -- Algorithm 1 (Jacobi preconditioner P:151) for
// large single-partition systems as a CUDA graph whose loop is a conditional
// WHILE node (variant 5):
//
//   [init] -> [S first] -> [U] -> WHILE(continue) { [S] -> [U] } -> [final]
//
//   init : rho_0 = r_0.z_0 and ||z_0|| from the RHS kernel's per-CTA partials;
//          early exit (reading C4); sets the loop condition.
//   S    : p_it = z + beta p_{it-1} formed on the fly for every gathered column,
//          q = A p_it (row_Ap_direct: plain SELL-32 or, TCB_SELL_PAIRS, slot pairs),
//          the deferred x += alpha_{it-1} p_{it-1}, per-CTA partials of p.q.
//   U    : every CTA sums the p.q partials in the same order (alpha identical
//          everywhere); r -= alpha q; z = r / diag(A) over 16-byte row pairs;
//          per-CTA partials of r.z, z.z; the last CTA to finish (ticket) sums
//          them in fixed order, applies the stopping test, updates the scalars
//          and sets the WHILE condition on the device.
//   final: the deferred x += alpha p of the last iteration; report and flags.
//
// The persistent kernel (pcg.cu) holds every loop scalar in registers across
// two grid barriers and is capped at 32 registers for 64 warps/SM; here each
// phase is a plain kernel with only its own state, so that the S phase could
// use the slot-pair loads without spilling (a stand-alone S phase on synthetic
// banded columns: 0.75 vs 0.96 ms at 20 M rows, tools/probe_bw.cu).  Kernel
// boundaries replace the grid barriers; the loop never returns to the host.
// Measured on the real systems it matches the persistent kernel with the plain
// layout and loses with slot pairs (profiles/r01e_exp_graph.txt), and ncu
// cannot profile kernel nodes of graphs with conditional nodes -- so it is an
// explicit option (pcg_variant = 5), parity-tested, not the default.
#include "pcg_common.cuh"

namespace tcb {

constexpr int kGThreads = 512;
constexpr int kGWarps = kGThreads / 32;
#ifndef TCB_G_MINB
#define TCB_G_MINB 4   // CTAs/SM of the S and U kernels (32 registers, 64 warps/SM)
#endif

__device__ __forceinline__ double2 cta_sum2(double2 v, double2* sh) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_sum2(v);
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double2 t = make_double2(0.0, 0.0);
  if (lane < kGWarps) t = sh[lane];
  return warp_sum2(t);
}

// Sum of m per-CTA partials, same order in every caller (deterministic).
__device__ __forceinline__ double2 sum_parts(const double2* p, int m, double2* sh) {
  double2 acc = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < m; t += blockDim.x) {
    const double2 u = __ldcg(p + t);   // written by other CTAs: read at L2
    acc.x += u.x;
    acc.y += u.y;
  }
  return cta_sum2(acc, sh);
}

__global__ void g_setstep_kernel(GStep* gs, double* x, tc_step_stat* stat, int32_t tag) {
  gs->x = x;
  gs->stat = stat;
  gs->tag = tag;
}

__global__ void __launch_bounds__(kGThreads) g_init_kernel(GArgs a) {
  __shared__ double2 sh[kGWarps];
  const double2 tot = sum_parts(a.part0, a.n_part0, sh);
  if (threadIdx.x == 0) {
    GScal s{};
    s.rho = tot.x;
    s.zeta = sqrt(tot.y);
    s.zref = s.zeta;
    s.nan = (isnan(s.rho) || isnan(s.zeta)) ? 1 : 0;
    s.conv = (!s.nan && s.zeta < a.eps_a) ? 1 : 0;   // reading C4: return x0
    s.done = (a.flags[0] || s.nan || s.conv || a.max_iters <= 0) ? 1 : 0;
    *a.sc = s;
    *a.ticket = 0u;
    cudaGraphSetConditional(a.cond, s.done ? 0u : 1u);
  }
}

// FIRST: the peeled first iteration (p_0 = z_0), outside the WHILE node.
template <bool FIRST>
__global__ void __launch_bounds__(kGThreads, TCB_G_MINB) g_S_kernel(GArgs a) {
  __shared__ double2 sh[kGWarps];
  const GScal s = *a.sc;
  if (s.done) return;   // converged / aborted before the first iteration (uniform)
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kGWarps + (threadIdx.x >> 5), nw = gridDim.x * kGWarps;
  const int32_t ns = a.nslices;
  double* __restrict__ x = a.gs->x;
  double* __restrict__ pnew = (s.it & 1) ? a.p1 : a.p0;        // p_it
  const double* __restrict__ pold = (s.it & 1) ? a.p0 : a.p1;  // p_{it-1}
  const ColIdx ci{a.col, nullptr, nullptr};
  double2 acc = make_double2(0.0, 0.0);
  if (FIRST) {
    for (int sl = gw; sl < ns; sl += nw) {
      const int64_t base = __ldg(a.slice_ptr + sl);
      const int w = (int)((__ldg(a.slice_ptr + sl + 1) - base) >> 5);
      const int64_t i = (int64_t)sl * kSellC + lane;
      const double pi = a.z[i];
      const double sum = row_Ap_direct<true>(base, w, lane, ci, a.A, a.z, nullptr, 0.0);
      pnew[i] = pi;
      a.q[i] = sum;
      acc.x += pi * sum;
    }
  } else {
    const double alpha = s.alpha, beta = s.beta;
    for (int sl = gw; sl < ns; sl += nw) {
      const int64_t base = __ldg(a.slice_ptr + sl);
      const int w = (int)((__ldg(a.slice_ptr + sl + 1) - base) >> 5);
      const int64_t i = (int64_t)sl * kSellC + lane;
      const double po = pold[i];
      const double pi = a.z[i] + beta * po;
      x[i] = x[i] + alpha * po;                                  // deferred x += alpha p_{it-1}
      const double sum = row_Ap_direct<false>(base, w, lane, ci, a.A, a.z, pold, beta);
      pnew[i] = pi;
      a.q[i] = sum;
      acc.x += pi * sum;
    }
  }
  const double2 b = cta_sum2(acc, sh);
  if (threadIdx.x == 0) a.partS[blockIdx.x] = b;
}

__global__ void __launch_bounds__(kGThreads, TCB_G_MINB) g_U_kernel(GArgs a) {
  __shared__ double2 sh[kGWarps];
  __shared__ bool last;
  const GScal s = *a.sc;
  if (s.done) return;   // only after init's early exit (the peeled first iteration)
  const double pq = sum_parts(a.partS, a.n_part, sh).x;
  const double alpha = s.rho / pq;                               // alpha_k = rho_k / p.q
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kGWarps + (threadIdx.x >> 5), nw = gridDim.x * kGWarps;
  const int64_t n2 = (int64_t)a.nslices * (kSellC / 2);
  double2* __restrict__ r2 = reinterpret_cast<double2*>(a.r);
  double2* __restrict__ z2 = reinterpret_cast<double2*>(a.z);
  const double2* __restrict__ q2 = reinterpret_cast<const double2*>(a.q);
  const double2* __restrict__ d2 = reinterpret_cast<const double2*>(a.dinv);
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t j = (int64_t)gw * kSellC + lane; j < n2; j += (int64_t)nw * kSellC) {
    const double2 rr = r2[j], qq = q2[j], dd = __ldg(d2 + j);
    double2 rn, zn;
    rn.x = rr.x - alpha * qq.x;
    rn.y = rr.y - alpha * qq.y;
    zn.x = dd.x * rn.x;
    zn.y = dd.y * rn.y;
    r2[j] = rn;
    z2[j] = zn;
    acc.x += rn.x * zn.x;
    acc.x += rn.y * zn.y;
    acc.y += zn.x * zn.x;
    acc.y += zn.y * zn.y;
  }
  const double2 b = cta_sum2(acc, sh);
  if (threadIdx.x == 0) {
    a.partU[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double2 tot = sum_parts(a.partU, gridDim.x, sh);         // fixed order: deterministic
  if (threadIdx.x == 0) {
    *a.ticket = 0u;
    GScal t = s;
    t.alpha = alpha;
    t.it = s.it + 1;
    t.last_valid = 1;
    const double zeta_new = sqrt(tot.y);
    t.zeta = zeta_new;
    if (isnan(pq) || isnan(zeta_new) || isnan(tot.x)) {
      t.nan = 1;
      t.done = 1;
    } else if (zeta_new < a.eps_a || zeta_new / s.zref < a.eps_r) {
      t.conv = 1;
      t.done = 1;
    } else {
      t.beta = tot.x / s.rho;                                    // beta_k = rho_{k+1} / rho_k
      t.rho = tot.x;
      if (a.rel_mode == 0) t.zref = zeta_new;
      t.done = t.it >= a.max_iters ? 1 : 0;
    }
    *a.sc = t;
    cudaGraphSetConditional(a.cond, t.done ? 0u : 1u);
  }
}

__global__ void __launch_bounds__(kGThreads) g_final_kernel(GArgs a) {
  const GScal s = *a.sc;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kGWarps + (threadIdx.x >> 5), nw = gridDim.x * kGWarps;
  if (s.last_valid && !s.nan && !a.flags[0]) {   // Alg. 1 updates x before its test
    double2* __restrict__ x2 = reinterpret_cast<double2*>(a.gs->x);
    const double2* __restrict__ pl2 = reinterpret_cast<const double2*>(((s.it - 1) & 1) ? a.p1 : a.p0);
    const int64_t n2 = (int64_t)a.nslices * (kSellC / 2);
    for (int64_t j = (int64_t)gw * kSellC + lane; j < n2; j += (int64_t)nw * kSellC) {
      const double2 xx = x2[j], pp = pl2[j];
      x2[j] = make_double2(xx.x + s.alpha * pp.x, xx.y + s.alpha * pp.y);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int32_t* f = a.flags;
    if (f[0]) return;            // aborted before this step: the report stays untouched
    tc_step_stat* st = a.gs->stat;
    st->iters = s.it;
    st->converged = s.conv;
    st->znorm = s.zeta;
    if (s.nan) {
      f[0] = 1; f[1] = 1; f[4] = a.gs->tag;
    } else {
      f[2] = s.conv ? 0 : f[2] + 1;
      if (f[3] > 0 && f[2] >= f[3]) { f[0] = 1; f[4] = a.gs->tag; }
    }
  }
}

int g_grid_size(int device) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)g_S_kernel<false>, kGThreads, 0);
  if (per_sm < 1) per_sm = 1;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return per_sm * sms;
}

static cudaError_t add_kernel(cudaGraphNode_t* node, cudaGraph_t g, const cudaGraphNode_t* dep, size_t ndep,
                              const void* fn, int grid, GArgs* args) {
  cudaKernelNodeParams p = {};
  p.func = const_cast<void*>(fn);
  p.gridDim = dim3(grid);
  p.blockDim = dim3(kGThreads);
  p.sharedMemBytes = 0;
  void* kargs[] = {(void*)args};
  p.kernelParams = kargs;
  return cudaGraphAddKernelNode(node, g, dep, ndep, &p);
}

// Builds and instantiates the solve graph.  `a` is completed with the
// conditional handle; kernel parameters are copied into the graph.
cudaError_t g_build(GArgs a, int grid, cudaGraphExec_t* exec) {
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaGraphCreate(&g, 0);
  if (e != cudaSuccess) return e;
  cudaGraphConditionalHandle h;
  e = cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault);
  if (e == cudaSuccess) {
    a.cond = h;
    a.n_part = grid;
    cudaGraphNode_t n_init, n_S0, n_U0, n_loop, n_final, n_S, n_U;
    e = add_kernel(&n_init, g, nullptr, 0, (const void*)g_init_kernel, 1, &a);
    if (e == cudaSuccess) e = add_kernel(&n_S0, g, &n_init, 1, (const void*)g_S_kernel<true>, grid, &a);
    if (e == cudaSuccess) e = add_kernel(&n_U0, g, &n_S0, 1, (const void*)g_U_kernel, grid, &a);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    if (e == cudaSuccess) e = cudaGraphAddNode(&n_loop, g, &n_U0, 1, &cp);
    if (e == cudaSuccess) {
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      e = add_kernel(&n_S, body, nullptr, 0, (const void*)g_S_kernel<false>, grid, &a);
      if (e == cudaSuccess) e = add_kernel(&n_U, body, &n_S, 1, (const void*)g_U_kernel, grid, &a);
    }
    if (e == cudaSuccess) e = add_kernel(&n_final, g, &n_loop, 1, (const void*)g_final_kernel, grid, &a);
    if (e == cudaSuccess) e = cudaGraphInstantiate(exec, g, 0);
  }
  cudaGraphDestroy(g);
  return e;
}

cudaError_t g_launch(cudaGraphExec_t exec, GStep* gs, double* x, tc_step_stat* stat, int32_t tag, cudaStream_t s) {
  g_setstep_kernel<<<1, 1, 0, s>>>(gs, x, stat, tag);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cudaGraphLaunch(exec, s);
}

}  // namespace tcb
