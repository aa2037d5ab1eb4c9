// pcg.cu -- the CG path of one monodomain step as ONE persistent cooperative
// kernel per solve: right-hand side (Eq. 3) and Algorithm 1
// with the Jacobi preconditioner, all scalars on device.
//
// Data flow per iteration (two phases, two grid barriers):
//   S: p_it = z + beta p_{it-1} is formed on the fly for every gathered column,
//      q = A p_it (SELL-32, warp per slice, thread per row), the deferred
//      x += alpha_{it-1} p_{it-1}, and the partial sums of p.q.
//   U: alpha = rho / p.q;  r -= alpha q;  z = r / diag(A);  partials r.z, z.z;
//      then every CTA evaluates the stopping test of Alg. 1 identically.
// Reductions are deterministic: per-CTA partials in a fixed slot, then every
// CTA sums all partials in the same order (bitwise-identical scalars => all
// CTAs take the same branch).
#include <cooperative_groups.h>

#include "internal.h"

namespace cg = cooperative_groups;

namespace tcb {

__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// Sum of v over the CTA, result valid in every thread.
__device__ __forceinline__ double2 block_sum2(double2 v, double2* sh) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_sum2(v);
  __syncthreads();  // sh may still be read from a previous call
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double2 t = make_double2(0.0, 0.0);
  if (lane < kCgWarps) t = sh[lane];
  t = warp_sum2(t);  // every warp reduces the 8 values identically
  return t;
}

// Grid-wide deterministic sum.  buf holds gridDim.x slots.
__device__ __forceinline__ double2 grid_sum2(double2 v, double2* buf, double2* sh,
                                             cg::grid_group& grid) {
  double2 b = block_sum2(v, sh);
  if (threadIdx.x == 0) buf[blockIdx.x] = b;
  grid.sync();
  double2 acc = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < (int)gridDim.x; t += blockDim.x) {
    double2 u = buf[t];
    acc.x += u.x;
    acc.y += u.y;
  }
  return block_sum2(acc, sh);
}

template <int MODE>
__global__ void __launch_bounds__(kCgThreads) pcg_kernel(CgArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double2 sh[kCgWarps];
  if (a.flags[0]) return;  // context aborted earlier: uniform across the grid

  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kCgWarps + (threadIdx.x >> 5);
  const int nw = gridDim.x * kCgWarps;
  const int32_t ns = a.nslices;
  const int64_t* __restrict__ sp = a.slice_ptr;
  const int32_t* __restrict__ col = a.col;
  const double* __restrict__ Av = a.A;
  const double* __restrict__ dinv = a.dinv;
  double2* partA = a.part;
  double2* partB = a.part + gridDim.x;

  // ---- r_0, z_0 = M^{-1} r_0, rho_0 = r.z, ||z_0||^2 ------------------------
  double2 acc = make_double2(0.0, 0.0);
  for (int s = gw; s < ns; s += nw) {
    const int64_t base = __ldg(sp + s);
    const int w = (int)((__ldg(sp + s + 1) - base) >> 5);
    const int64_t i = (int64_t)s * kSellC + lane;
    double sum = 0.0;
    if (MODE == 1) {
      const double* __restrict__ Kv = a.K;
      // r_0 = A u' - K v'  (== b - A x_0 with Eq. 3's b)
#pragma unroll 4
      for (int k = 0; k < w; ++k) {
        const int64_t t = base + (int64_t)k * kSellC + lane;
        const int c = __ldg(col + t);
        sum += __ldg(Av + t) * a.up[c] - __ldg(Kv + t) * a.vp[c];
      }
    } else {
#pragma unroll 4
      for (int k = 0; k < w; ++k) {
        const int64_t t = base + (int64_t)k * kSellC + lane;
        sum += __ldg(Av + t) * a.x[__ldg(col + t)];
      }
      sum = a.b[i] - sum;
    }
    const double zi = __ldg(dinv + i) * sum;
    a.r[i] = sum;
    a.z[i] = zi;
    acc.x += sum * zi;
    acc.y += zi * zi;
  }
  double2 tot = grid_sum2(acc, partA, sh, grid);
  double rho = tot.x;
  double zeta = sqrt(tot.y);
  double zref = zeta;
  int it = 0;
  int conv = 0, nan = 0;
  if (isnan(rho) || isnan(zeta)) nan = 1;
  if (!nan && zeta < a.eps_a) conv = 1;  // reading C4: return x0

  double alpha = 0.0, beta = 0.0;
  double* pold = a.p1;
  double* pnew = a.p0;
  bool last_valid = false;
  double* plast = a.p0;
  if (!nan && !conv) {
    for (it = 0; it < a.max_iters;) {
      // ---- S: p = z + beta p_old (on the fly), q = A p, x += alpha_prev p_old
      acc = make_double2(0.0, 0.0);
      const bool first = (it == 0);
      for (int s = gw; s < ns; s += nw) {
        const int64_t base = __ldg(sp + s);
        const int w = (int)((__ldg(sp + s + 1) - base) >> 5);
        const int64_t i = (int64_t)s * kSellC + lane;
        double pi = a.z[i];
        if (!first) {
          const double po = pold[i];
          pi += beta * po;
          a.x[i] += alpha * po;
        }
        double sum = 0.0;
        if (first) {
#pragma unroll 4
          for (int k = 0; k < w; ++k) {
            const int64_t t = base + (int64_t)k * kSellC + lane;
            sum += __ldg(Av + t) * a.z[__ldg(col + t)];
          }
        } else {
#pragma unroll 4
          for (int k = 0; k < w; ++k) {
            const int64_t t = base + (int64_t)k * kSellC + lane;
            const int c = __ldg(col + t);
            sum += __ldg(Av + t) * (a.z[c] + beta * pold[c]);
          }
        }
        pnew[i] = pi;
        a.q[i] = sum;
        acc.x += pi * sum;
      }
      plast = pnew;
      last_valid = true;
      tot = grid_sum2(acc, partB, sh, grid);
      const double pq = tot.x;
      if (isnan(pq)) { nan = 1; break; }
      alpha = rho / pq;                                   // alpha_k = rho_k / p.q
      // ---- U: r -= alpha q, z = r / d, partials of r.z and z.z
      acc = make_double2(0.0, 0.0);
      for (int s = gw; s < ns; s += nw) {
        const int64_t i = (int64_t)s * kSellC + lane;
        const double ri = a.r[i] - alpha * a.q[i];
        const double zi = __ldg(dinv + i) * ri;
        a.r[i] = ri;
        a.z[i] = zi;
        acc.x += ri * zi;
        acc.y += zi * zi;
      }
      tot = grid_sum2(acc, partA, sh, grid);
      ++it;
      const double zeta_new = sqrt(tot.y);
      zeta = zeta_new;
      if (isnan(zeta_new) || isnan(tot.x)) { nan = 1; break; }
      if (zeta_new < a.eps_a || zeta_new / zref < a.eps_r) { conv = 1; break; }
      beta = tot.x / rho;                                 // beta_k = rho_{k+1} / rho_k
      rho = tot.x;
      if (a.rel_mode == 0) zref = zeta_new;
      double* t = pold; pold = pnew; pnew = t;
    }
  }
  // deferred x += alpha p of the last iteration (Alg. 1 updates x before the test)
  if (last_valid && !nan) {
    for (int s = gw; s < ns; s += nw) {
      const int64_t i = (int64_t)s * kSellC + lane;
      a.x[i] += alpha * plast[i];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.stat->iters = it;
    a.stat->converged = conv;
    a.stat->znorm = zeta;
    int32_t* f = a.flags;
    if (nan) {
      f[0] = 1; f[1] = 1; f[4] = a.step_tag;
    } else {
      f[2] = conv ? 0 : f[2] + 1;
      if (f[3] > 0 && f[2] >= f[3]) { f[0] = 1; f[4] = a.step_tag; }
    }
  }
}

__global__ void spmv_kernel(const int64_t* __restrict__ sp, const int32_t* __restrict__ col,
                            const double* __restrict__ Av, int32_t ns, const double* __restrict__ x,
                            double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < ns; s += nw) {
    const int64_t base = sp[s];
    const int w = (int)((sp[s + 1] - base) >> 5);
    double sum = 0.0;
#pragma unroll 4
    for (int k = 0; k < w; ++k) {
      const int64_t t = base + (int64_t)k * kSellC + lane;
      sum += Av[t] * x[col[t]];
    }
    y[(int64_t)s * kSellC + lane] = sum;
  }
}

static int g_sm_count[64] = {0};

static int sm_count(int dev) {
  if (dev < 0 || dev >= 64) return 148;
  if (!g_sm_count[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    g_sm_count[dev] = v > 0 ? v : 148;
  }
  return g_sm_count[dev];
}

// Grid: enough CTAs for one slice per warp, capped at the co-resident maximum
// (cooperative launch); large problems get every SM x occupancy.
int cg_grid_size(int mode, int32_t nslices, int device) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, mode == 1 ? (const void*)pcg_kernel<1> : (const void*)pcg_kernel<0>, kCgThreads, 0);
  if (per_sm < 1) per_sm = 1;
  int maxg = per_sm * sm_count(device);
  int need = (nslices + kCgWarps - 1) / kCgWarps;
  if (need < 1) need = 1;
  return need < maxg ? need : maxg;
}

cudaError_t launch_pcg(int mode, const CgArgs& a, int grid, cudaStream_t s) {
  void* args[] = {(void*)&a};
  const void* fn = mode == 1 ? (const void*)pcg_kernel<1> : (const void*)pcg_kernel<0>;
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kCgThreads), args, 0, s);
}

cudaError_t launch_spmv(const int64_t* sp, const int32_t* col, const double* A, int32_t ns,
                        const double* x, double* y, cudaStream_t s) {
  int threads = 256;
  int64_t warps = ns;
  int blocks = (int)std::min<int64_t>((warps * 32 + threads - 1) / threads, 148 * 16);
  if (blocks < 1) blocks = 1;
  spmv_kernel<<<blocks, threads, 0, s>>>(sp, col, A, ns, x, y);
  return cudaGetLastError();
}

}  // namespace tcb
