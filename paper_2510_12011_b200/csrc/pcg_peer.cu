// pcg_peer.cu -- the multi-GPU PCG as ONE persistent kernel per GPU, with the
// halo exchange and the cross-GPU reductions done by the kernel itself over
// NVLink peer memory (CUDA IPC mappings), DESIGN.md "Multi-GPU".
//
// Each rank ("group" of CTAs) owns a row block.  Per iteration of Alg. 1:
//   halo  : p_it = z + beta p_{it-1} of the send-list nodes is stored straight
//           into the neighbours' ghost regions of z (remote stores), then a
//           per-neighbour flag carries the epoch; readers wait on their flags
//   S     : q = A p, x += alpha p_{it-1}, p.q partial -> rank sum (group barrier);
//           rows are numbered interior-first, so in the one grid-stride pass a
//           warp meets the boundary slices (the ones that read ghosts) only in
//           its last round(s): it waits for the halo flags there (per warp, no
//           CTA barrier), its interior slices overlap the transfer
//   reduce: the rank sum is stored into slot [epoch&1][rank] of EVERY rank's
//           inbox, then every CTA waits for all ranks' slots of this epoch and
//           sums them in rank order -> bitwise-identical scalars on all ranks
//   U     : z (z-form: z -= alpha D^-1 q), (r.z, z.z) partials -> rank sum ->
//           cross-rank reduce, test, beta
// Memory ordering: data stores, __threadfence_system(), then the flag/epoch
// store; readers poll with volatile loads, then __threadfence() (which also
// drops stale L1 lines) before touching the data.  Slots are double-buffered
// by epoch parity (a rank can be at most one reduction ahead of another).
// Every wait is bounded in wall-clock time (%globaltimer; tc_config.peer_timeout_s,
// default 300 s, like a collective timeout): on timeout the kernel records an
// error flag in the context's flags, skips all further waits and finishes its
// iterations; tc_step reports TC_ENCCL.  The launch state (PeerRun) is built
// per call and every flag pointer belongs to the launching context, so
// independent contexts never share launch state.  With several groups in one cooperative launch on one GPU the same
// code runs the partitions of a single device ("peer emulation"), which is how
// the protocol is tested without 8 GPUs.
#include <memory>

#include "pcg_common.cuh"

namespace tcb {

constexpr int kPeerThreads = kPeerThreadsHost;
constexpr int kPeerWarps = kPeerThreads / 32;

constexpr int kMaxGroups = 8;  // partitions of one GPU in a peer launch (kernel-parameter space)

struct PeerRun {
  XPart parts[kMaxGroups];  // one per group, in kernel-parameter (constant) space
  int groups;          // groups in this launch (1 on real multi-GPU)
  int bpg;             // CTAs per group
  int iX, iVk;         // rotating V buffers
  double eps_a, eps_r;
  int32_t max_iters, rel_mode;
  tc_step_stat* stat;
  int32_t* flags;      // [0] abort [1] nan [2] fails [3] budget [4] step [5] peer timeout
  int32_t step_tag;
};

__device__ __forceinline__ unsigned long long vload(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void vstore(unsigned long long* p, unsigned long long v) {
  *reinterpret_cast<volatile unsigned long long*>(p) = v;
}
__device__ __forceinline__ double2 vload2(const double2* p) {
  const volatile double* q = reinterpret_cast<const volatile double*>(p);
  return make_double2(q[0], q[1]);
}
__device__ __forceinline__ void vstore2(double2* p, double2 v) {
  volatile double* q = reinterpret_cast<volatile double*>(p);
  q[0] = v.x;
  q[1] = v.y;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Barrier of the CTAs of one group (sense-reversing generation counter),
// bounded like every other wait.
__device__ __forceinline__ void group_barrier(const XPart& X, int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vg = X.bar_gen;
    const unsigned int g = *vg;
    __threadfence();
    if (atomicAdd(X.bar_count, 1u) == (unsigned int)nblocks - 1) {
      *X.bar_count = 0u;
      __threadfence();
      atomicAdd(X.bar_gen, 1u);
    } else {
      const unsigned long long t0 = gtimer();
      while (*vg == g) {
        if (gtimer() - t0 > X.timeout_ns) {
          atomicExch(X.flags + 5, 1);
          break;
        }
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Deterministic sum over the group's CTAs (valid in every thread of every CTA).
// part: 2 x nb slots, alternated by the caller's reduction counter (a CTA can be
// one reduction ahead of another, never two: the next barrier separates them).
__device__ __forceinline__ double2 group_sum2(const XPart& X, double2 v, double2* part, int lb, int nb,
                                              double2* sh) {
  const double2 b = block_sum2(v, sh);
  if (threadIdx.x == 0) part[lb] = b;
  group_barrier(X, nb);
  double2 acc = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    const double2 u = __ldcg(part + t);
    acc.x += u.x;
    acc.y += u.y;
  }
  return block_sum2(acc, sh);
}

// Bounded spin until *p == want (GE: *p >= want), thread 0 of a CTA; false on timeout.
template <bool GE>
__device__ __forceinline__ bool wait_for(const unsigned long long* p, unsigned long long want,
                                         const XPart& X) {
  const unsigned long long t0 = gtimer();
  while (GE ? vload(p) < want : vload(p) != want) {
    if (*reinterpret_cast<volatile int32_t*>(X.flags + 5)) return false;
    if (gtimer() - t0 > X.timeout_ns) {
      atomicExch(X.flags + 5, 1);
      return false;
    }
  }
  return true;
}

// Cross-rank sum of the rank value v (identical in all CTAs of the group).
// Slot parity follows the reduction count `nr` (not the epoch, which halos also
// advance): a rank cannot start reduction nr+2 before every rank has read nr.
__device__ __forceinline__ double2 cross_sum2(const XPart& X, double2 v, unsigned long long epoch,
                                              unsigned long long nr, int lb, double2* sh1) {
  const int slot = (int)(nr & 1ull);
  if (lb == 0 && threadIdx.x == 0) {
    for (int r = 0; r < X.world; ++r) {
      RedSlot* d = X.rred[r] + slot * X.world + X.rank;
      vstore2(&d->v, v);
      __threadfence_system();
      vstore(&d->e, epoch);
    }
  }
  if (threadIdx.x == 0) {
    for (int r = 0; r < X.world; ++r) wait_for<false>(&X.myred[slot * X.world + r].e, epoch, X);
    __threadfence();
    double2 s = make_double2(0.0, 0.0);
    for (int r = 0; r < X.world; ++r) {
      const double2 u = vload2(&X.myred[slot * X.world + r].v);
      s.x += u.x;
      s.y += u.y;
    }
    *sh1 = s;
  }
  __syncthreads();
  const double2 s = *sh1;
  __syncthreads();
  return s;
}

// Remote halo: for send entry j, value(j) lands in neighbour send_nbr[j]'s ghost
// region of the vector selected by `which` (0 z, 1 u', 2 v'); then the flags.
// TCB_PEER_PUSH_ARRIVE = 1 (experiment, off): arrive-only -- every CTA fences its stores
// and increments the group's push counter; the LAST CTA to arrive (it sees the
// count of this launch's push `npush` complete) fences and stores the flags, and
// nobody waits (0: a full group barrier, then CTA 0 stores the flags).  Ordering:
// each CTA's remote stores -> fence.sys -> counter RMW; the last RMW -> fence.sys
// -> flag stores, so a neighbour that sees the flag sees every CTA's data (and a
// later push's flag can never land before an earlier one's: the thread that
// stored the earlier flag fences before its next counter RMW).  The counter is
// reset by CTA 0 after the launch's final group barrier.  Measured neutral on one
// GPU (emulated partitions, world 1: profiles/r02ap_exp_peer_sync.txt), so the
// barrier version -- the one exercised since r01 -- stays the default.
#ifndef TCB_PEER_PUSH_ARRIVE
#define TCB_PEER_PUSH_ARRIVE 0
#endif
template <class ValF>
__device__ __forceinline__ void halo_push(const XPart& X, int which, unsigned long long epoch, int lb,
                                          int nb, unsigned int& npush, ValF val) {
  bool wrote = false;
  for (int64_t j = (int64_t)lb * blockDim.x + threadIdx.x; j < X.n_send; j += (int64_t)nb * blockDim.x) {
    const int q = X.send_nbr[j];
    double* base = which == 0 ? X.rz[q] : (which == 1 ? X.rup[q] : X.rvp[q]);
    base[X.send_off[j]] = val(X.send_idx[j]);
    wrote = true;
  }
  if (wrote) __threadfence_system();   // this thread's remote stores before the flag
#if TCB_PEER_PUSH_ARRIVE
  if (X.nbr_count > 0) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      const unsigned int old = atomicAdd(X.push_count, 1u);
      if (old == (npush + 1u) * (unsigned int)nb - 1u) {   // every CTA of the group has pushed
        __threadfence_system();
        for (int q = 0; q < X.nbr_count; ++q) vstore(X.rflag[q], epoch);
      }
    }
  }
  ++npush;
#else
  (void)npush;
  group_barrier(X, nb);
  if (lb == 0 && threadIdx.x < X.nbr_count) vstore(X.rflag[threadIdx.x], epoch);
#endif
}

// Per-warp halo wait (no CTA barrier): lane 0 polls the flags, then the fence
// orders the flag reads before the data reads and __syncwarp hands that order to
// the other lanes.  A warp calls it once, before its first boundary slice.
__device__ __forceinline__ void halo_wait_warp(const XPart& X, unsigned long long epoch) {
  if ((threadIdx.x & 31) == 0) {
    for (int q = 0; q < X.nbr_count; ++q) wait_for<true>(X.myflag[q], epoch, X);
    __threadfence();
  }
  __syncwarp();
}

__device__ __forceinline__ void halo_wait(const XPart& X, unsigned long long epoch) {
  if (threadIdx.x == 0) {
    for (int q = 0; q < X.nbr_count; ++q) wait_for<true>(X.myflag[q], epoch, X);
    __threadfence();
  }
  __syncthreads();
}

// RHS of the step on the partitioned system: halo of u', v' (remote stores),
// r_0 = A u' - K v' (== b - A x_0), z_0, and the cross-rank
// sums rho_0, ||z_0||^2 -> X.red0.  Own launch (64 registers); cooperative so
// that every group's CTAs are resident while they wait for their neighbours.
__global__ void __launch_bounds__(kPeerThreads, 1024 / kPeerThreads) rhs_peer_kernel(const __grid_constant__ PeerRun R) {
  __shared__ double2 sh[kPeerWarps];
  __shared__ double2 sh1;
  const int group = blockIdx.x / R.bpg;
  const int lb = blockIdx.x - group * R.bpg;
  const int nb = R.bpg;
  const XPart& X = R.parts[group];
  if (R.flags[0]) return;
  const int lane = threadIdx.x & 31;
  const int gw = lb * kPeerWarps + (threadIdx.x >> 5), nw = nb * kPeerWarps;
  unsigned long long ep = X.epoch[0];
  unsigned long long nrx = X.epoch[1];
  unsigned int npush = 0;   // halo pushes of this launch (TCB_PEER_PUSH_ARRIVE)
  ++ep;
  halo_push(X, 1, ep, lb, nb, npush, [&](int32_t i) { return X.up[i]; });
  ++ep;
  halo_push(X, 2, ep, lb, nb, npush, [&](int32_t i) { return X.vp[i]; });
  double2 acc = make_double2(0.0, 0.0);
  auto row = [&](int s) {
    const int64_t base = __ldg(X.slice_ptr + s);
    const int w = (int)((__ldg(X.slice_ptr + s + 1) - base) >> 5);
    const int64_t i = (int64_t)s * kSellC + lane;
    const double sum = row_rhs_direct(base, w, lane, X.col, X.A, X.K, X.up, X.vp);
    const double zi = __ldg(X.dinv + i) * sum;
    X.r[i] = sum;
    X.z[i] = zi;
    acc.x += sum * zi;
    acc.y += zi * zi;
  };
  // one grid-stride pass; rows are interior-first, so a warp reaches the
  // boundary slices (the ones that read ghosts) only in its last round(s): it
  // waits for the halo there, the interior slices before it overlap the transfer
  // (flags are monotone: >= ep covers both halos)
  bool waited = false;
  for (int s = gw; s < X.nslices; s += nw) {
    if (!waited && s >= X.nslices_int) {
      halo_wait_warp(X, ep);
      waited = true;
    }
    row(s);
  }
  double2 tot = group_sum2(X, acc, X.part, lb, nb, sh);
  ++ep;
  tot = cross_sum2(X, tot, ep, nrx++, lb, &sh1);
  group_barrier(X, nb);  // every CTA is done with the counters
  if (lb == 0 && threadIdx.x == 0) {
    *X.push_count = 0u;
    *X.red0 = tot;
    X.epoch[0] = ep;
    X.epoch[1] = nrx;
  }
}

// TCB_PEER_XMERGE = 1: x updated every other iteration (two pending terms added in
// their original order, bitwise the sequential result), as the single-GPU kernel does.
#ifndef TCB_PEER_XMERGE
#define TCB_PEER_XMERGE 0
#endif
// Algorithm 1's loop on the partitioned system (after rhs_peer_kernel).
// BATCH: the latency variant's row product (row_Ap_batch, every slot of a row in
// flight; ~128 registers, 2 CTAs of 8 warps per SM) for partitions with few
// slices per resident warp (variant 4).
template <bool BATCH>
__global__ void __launch_bounds__(kPeerThreads, BATCH ? (512 / kPeerThreads > 0 ? 512 / kPeerThreads : 1) : 2048 / kPeerThreads) pcg_peer_kernel(const __grid_constant__ PeerRun R) {
  __shared__ double2 sh[kPeerWarps];
  __shared__ double2 sh1;
  const int group = blockIdx.x / R.bpg;
  const int lb = blockIdx.x - group * R.bpg;  // CTA index inside the group
  const int nb = R.bpg;
  const XPart& X = R.parts[group];
  if (R.flags[0]) return;  // aborted earlier: uniform over the launch
  const int lane = threadIdx.x & 31;
  const int gw = lb * kPeerWarps + (threadIdx.x >> 5), nw = nb * kPeerWarps;
  const int ns = X.nslices;
  double* __restrict__ x = X.V[R.iX];
  unsigned long long ep = X.epoch[0];   // epoch counter (halos and reductions), same in every CTA
  unsigned long long nrx = X.epoch[1];  // cross-rank reductions done (slot parity)
  unsigned int nred = 0;                // partial-buffer parity
  double2 acc;
  double2 tot = *X.red0;
  double rho = tot.x, zeta = sqrt(tot.y), zref = zeta, alpha = 0.0, beta = 0.0, alpha_prev = 0.0;
  int it = 0, conv = 0, nan = 0, plast = -1;
  unsigned int npush = 0;   // halo pushes of this launch (TCB_PEER_PUSH_ARRIVE)
  if (isnan(rho) || isnan(zeta)) nan = 1;
  if (!nan && zeta < R.eps_a) conv = 1;
  if (!nan && !conv) {
    for (it = 0; it < R.max_iters;) {
      double* __restrict__ pnew = (it & 1) ? X.p1 : X.p0;
      const double* __restrict__ pold = (it & 1) ? X.p0 : X.p1;
      const bool first = it == 0;
      // halo of p_it into the neighbours' z ghosts
      ++ep;
      halo_push(X, 0, ep, lb, nb, npush, [&](int32_t i) { return first ? X.z[i] : X.z[i] + beta * pold[i]; });
      // S (separate first / later loops, as in the single-GPU kernel): the
      // interior slices overlap the halo, the boundary slices wait for it
      acc = make_double2(0.0, 0.0);
      const ColIdx ci{X.col, nullptr, nullptr};
      const int ni = X.nslices_int;
      if (first) {
        auto row = [&](int s) {
          const int64_t base = __ldg(X.slice_ptr + s);
          const int w = (int)((__ldg(X.slice_ptr + s + 1) - base) >> 5);
          const int64_t i = (int64_t)s * kSellC + lane;
          const double pi = X.z[i];
          const double sum = BATCH ? row_Ap_batch_w<true>(base, w, lane, X.col, X.A, X.z, nullptr, 0.0)
                                   : row_Ap_direct<true>(base, w, lane, ci, X.A, X.z, nullptr, 0.0);
          pnew[i] = pi;
          X.q[i] = sum;
          acc.x += pi * sum;
        };
        bool waited = false;
        for (int s = gw; s < ns; s += nw) {
          if (!waited && s >= ni) {
            halo_wait_warp(X, ep);
            waited = true;
          }
          row(s);
        }
      } else {
        auto row = [&](int s) {
          const int64_t base = __ldg(X.slice_ptr + s);
          const int w = (int)((__ldg(X.slice_ptr + s + 1) - base) >> 5);
          const int64_t i = (int64_t)s * kSellC + lane;
          const double po = pold[i];
          const double pi = X.z[i] + beta * po;
#if TCB_PEER_XMERGE
          if (!(it & 1)) {   // even it >= 2: p_{it-2} (still in pnew) and p_{it-1}, in order (pcg.cu TCB_XMERGE)
            const double xi = x[i], p2 = pnew[i];
            x[i] = (xi + alpha_prev * p2) + alpha * po;
          }
#else
          const double xi = x[i];
          x[i] = xi + alpha * po;
#endif
          const double sum = BATCH ? row_Ap_batch_w<false>(base, w, lane, X.col, X.A, X.z, pold, beta)
                                   : row_Ap_direct<false>(base, w, lane, ci, X.A, X.z, pold, beta);
          pnew[i] = pi;
          X.q[i] = sum;
          acc.x += pi * sum;
        };
        bool waited = false;
        for (int s = gw; s < ns; s += nw) {
          if (!waited && s >= ni) {
            halo_wait_warp(X, ep);
            waited = true;
          }
          row(s);
        }
      }
      plast = it & 1;
      tot = group_sum2(X, acc, X.part + (nred++ & 1) * nb, lb, nb, sh);
      ++ep;
      tot = cross_sum2(X, tot, ep, nrx++, lb, &sh1);
      const double pq = tot.x;
      if (isnan(pq)) { nan = 1; break; }
      alpha_prev = alpha;
      alpha = rho / pq;
      // U
      acc = make_double2(0.0, 0.0);
      for (int s = gw; s < ns; s += nw) {
        const int64_t i = (int64_t)s * kSellC + lane;
        // z-form (pcg.cu TCB_ZFORM): z -= alpha D^-1 q, r.z = sum z^2 / d^-1
        const double di = __ldg(X.dinv + i);
        const double zi = X.z[i] - alpha * (di * X.q[i]);
        X.z[i] = zi;
        acc.x += di != 0.0 ? zi * (zi / di) : 0.0;
        acc.y += zi * zi;
      }
      tot = group_sum2(X, acc, X.part + (nred++ & 1) * nb, lb, nb, sh);
      ++ep;
      tot = cross_sum2(X, tot, ep, nrx++, lb, &sh1);
      ++it;
      zeta = sqrt(tot.y);
      if (isnan(zeta) || isnan(tot.x)) { nan = 1; break; }
      if (zeta < R.eps_a || zeta / zref < R.eps_r) { conv = 1; break; }
      beta = tot.x / rho;
      rho = tot.x;
      if (R.rel_mode == 0) zref = zeta;
    }
  }
  if (plast >= 0 && !nan) {
    const double* __restrict__ pl = plast ? X.p1 : X.p0;
    // TCB_PEER_XMERGE: S(it-1) skipped its x update when it-1 was odd -> p_{it-2} pending too
    const bool two = TCB_PEER_XMERGE && !(it & 1) && it >= 2;
    const double* __restrict__ pl2 = plast ? X.p0 : X.p1;   // p_{it-2}
    for (int s = gw; s < ns; s += nw) {
      const int64_t i = (int64_t)s * kSellC + lane;
      const double xi = x[i];
      x[i] = (two ? xi + alpha_prev * pl2[i] : xi) + alpha * pl[i];
    }
  }
  // all CTAs of the group are past their last use of the epoch / push counters
  group_barrier(X, nb);
  if (lb == 0 && threadIdx.x == 0) {
    *X.push_count = 0u;
    X.epoch[0] = ep;
    X.epoch[1] = nrx;
    if (group == 0) {
      R.stat->iters = it;
      R.stat->converged = conv;
      R.stat->znorm = zeta;
      int32_t* f = R.flags;
      if (f[5]) {
        f[0] = 1; f[4] = R.step_tag;
      } else if (nan) {
        f[0] = 1; f[1] = 1; f[4] = R.step_tag;
      } else {
        f[2] = conv ? 0 : f[2] + 1;
        if (f[3] > 0 && f[2] >= f[3]) { f[0] = 1; f[4] = R.step_tag; }
      }
    }
  }
}

static const void* peer_fn(int which) {
  return which == 1 ? (const void*)rhs_peer_kernel
                    : which == 2 ? (const void*)pcg_peer_kernel<true> : (const void*)pcg_peer_kernel<false>;
}

int peer_blocks_per_sm(int which) {
  static int v[3] = {0, 0, 0};
  if (!v[which]) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v[which], peer_fn(which), kPeerThreads, 0);
    if (v[which] < 1) v[which] = 1;
  }
  return v[which];
}

int peer_max_groups() { return kMaxGroups; }

cudaError_t launch_pcg_peer(const XPart* parts, int groups, int bpg, int bpg_rhs, bool batch, int iX, int iVk,
                            unsigned long long timeout_ns, double eps_a, double eps_r, int32_t max_iters,
                            int32_t rel_mode, tc_step_stat* stat, int32_t* flags, int32_t step_tag, cudaStream_t s) {
  if (groups < 1 || groups > kMaxGroups) return cudaErrorInvalidValue;
  // per call (kernel parameters are copied at launch): no state shared between
  // contexts or host threads (large: heap, not stack)
  std::unique_ptr<PeerRun> Rp(new PeerRun());
  PeerRun& R = *Rp;
  for (int g = 0; g < groups; ++g) {
    R.parts[g] = parts[g];
    R.parts[g].flags = flags;
    R.parts[g].timeout_ns = timeout_ns;
  }
  R.groups = groups; R.iX = iX; R.iVk = iVk; R.eps_a = eps_a; R.eps_r = eps_r;
  R.max_iters = max_iters; R.rel_mode = rel_mode; R.stat = stat; R.flags = flags; R.step_tag = step_tag;
  void* args[] = {(void*)&R};
  R.bpg = bpg_rhs;
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)rhs_peer_kernel, dim3(groups * bpg_rhs),
                                              dim3(kPeerThreads), args, 0, s);
  if (e != cudaSuccess) return e;
  R.bpg = bpg;
  return cudaLaunchCooperativeKernel(peer_fn(batch ? 2 : 0), dim3(groups * bpg), dim3(kPeerThreads),
                                     args, 0, s);
}

}  // namespace tcb
