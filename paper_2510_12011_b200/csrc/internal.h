// internal.h -- private declarations of libtcb200 (B200-native TorchCor step).
// Nothing here crosses the C ABI (include/tcb200.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/tcb200.h"

namespace tcb {

// ---------------------------------------------------------------------------
// SELL-32 sparse layout (one warp = one slice of 32 consecutive rows of width w).
// Slot pairs (TCB_SELL_PAIRS=1, measured slower in situ: DESIGN.md): slots 2j and 2j+1 of a lane's row are
// adjacent, so a warp reads a slot pair as one 16-byte value load and one
// 8-byte index load per lane (measured: 16-byte streaming loads reach 7.1 TB/s
// on B200, 8-byte loads 4.9 TB/s; tools/probe_bw.cu):
//   slot k < (w & ~1) of row 32*s + lane at slice_ptr[s] + 64*(k/2) + 2*lane + k%2,
//   the odd last slot (w odd)          at slice_ptr[s] + 32*(w-1) + lane.
// TCB_SELL_PAIRS=0 (default): plain SELL, slot k at slice_ptr[s] + 32*k + lane.
// Rows keep the ascending column order of CSR, and every kernel sums a row's
// slots in that order, so the SpMV sums every row as a CSR loop does.
// Padding slots point at the row itself with value 0.
// ---------------------------------------------------------------------------
constexpr int kSellC = 32;
constexpr int kAutoBatch = 4;          // PCG variant 4 up to this many slices per resident warp (pcg.cu)
#ifndef TCB_PEER_THREADS
#define TCB_PEER_THREADS 256
#endif
constexpr int kPeerThreadsHost = TCB_PEER_THREADS;  // threads per CTA of the peer-memory PCG kernels (pcg_peer.cu)
#ifndef TCB_SELL_PAIRS
#define TCB_SELL_PAIRS 0
#endif
// Offset of slot k of lane `lane`'s row in a slice at `base` of width w.
__host__ __device__ __forceinline__ int64_t sell_slot(int64_t base, int64_t w, int64_t k, int64_t lane) {
#if TCB_SELL_PAIRS
  return k < (w & ~(int64_t)1) ? base + 64 * (k >> 1) + 2 * lane + (k & 1) : base + 32 * k + lane;
#else
  (void)w;
  return base + 32 * k + lane;
#endif
}
#ifndef TCB_CG_THREADS
#define TCB_CG_THREADS 512
#endif
constexpr int kCgThreads = TCB_CG_THREADS;  // threads per CTA of the PCG kernels (16 warps; measured best of 256/512/1024)
constexpr int kCgWarps = kCgThreads / 32;

struct HostSell {
  int32_t n = 0;
  int32_t nslices = 0;
  int64_t n_pad = 0;
  std::vector<int64_t> slice_ptr;  // nslices + 1
  std::vector<int32_t> col;        // slice_ptr[nslices]
  std::vector<int32_t> rowlen;     // n
  // 16-bit index compression: col = kbase[slice_ptr[s]/32 + k] + col16[slot]
  // for slices with fmt[s] == 0 (every slot row of the slice spans < 2^16).
  std::vector<uint16_t> col16;     // slice_ptr[nslices]
  std::vector<int32_t> kbase;      // slice_ptr[nslices] / 32
  std::vector<uint8_t> fmt;        // nslices: 0 compressed, 1 plain int32
  int64_t n_wide = 0;
};

// ---- TT2006 parameters (kernel-argument struct; names for tc_set_ionic_param)
struct TTParams {
  double R, T, F, CAP, Vc, Vsr, Vss, Ko, Nao, Cao;
  double GNa, GK1, Gto, GKr, GKs, pKNa, GCaL, GbNa, GbCa, GpCa, KpCa, GpK;
  double PNaK, KmK, KmNa, kNaCa, KmNai, KmCa, ksat, gamma, alpha;
  double Bufc, Kbufc, Bufsr, Kbufsr, Bufss, Kbufss;
  double Vmaxup, Kup, Vrel, k1p, k2p, k3, k4, EC, maxsr, minsr, Vleak, Vxfer;
};
constexpr int kTTStates = 18;
struct MSParams {
  double tau_in, tau_out, tau_open, tau_close, v_gate, V_min, V_max;
};
struct MMSParams {
  double k, w1, w2, lam;
};
// ---- CRN 1998 atrial model parameters (names for tc_set_ionic_param, oracle order)
struct CRNParams {
  double R, T, F, Cm, Vi, Vup, Vrel, Ko, Nao, Cao, gNa, gK1, gto, gKr, gKs, gCaL, gbNa, gbCa;
  double INaKmax, KmNai, KmKo, INaCamax, KmNa, KmCa, ksat, gamma, IpCamax, Krel, tautr;
  double Iupmax, Kup, Caupmax, CMDNmax, TRPNmax, CSQNmax, KmCMDN, KmTRPN, KmCSQN, tauu, KQ10;
};
constexpr int kCRNStates = 20;

void tt_defaults(TTParams* p, double* V0, double u0[kTTStates]);
void ms_defaults(MSParams* p);
void crn_defaults(CRNParams* p, double* V0, double u0[kCRNStates]);
double* crn_param_slot(CRNParams* p, const char* name);
double* tt_param_slot(TTParams* p, const char* name);
double* ms_param_slot(MSParams* p, const char* name);

// ---------------------------------------------------------------------------
// Kernel argument blocks
// ---------------------------------------------------------------------------
// TCB_ZFORM = 1 (default): the U phase keeps z only -- z_{k+1} = z_k - alpha
// D^-1 q_k and r.z = sum z^2 / d^-1 -- instead of r and z (Alg. 1 literal, 0):
// 32 instead of 40 bytes per row, the iteration 80n + 12 nnz instead of 88n.
// Same iterates in exact arithmetic; rounding differs from the oracle's at the
// 1e-16 level (parity unchanged, profiles/r02g_zform_tests.log).  Measured
// (profiles/r02g_exp_zform.txt, ms per PCG iteration): 20 M MS 1.100 -> 1.070,
// 10 M TT2006 0.508 -> 0.501; PCG-path frac 0.844 -> 0.869 / 0.863 -> 0.876.
#ifndef TCB_ZFORM
#define TCB_ZFORM 1
#endif
// TCB_FUSE_RHS4 = 1 (default): the latency variant (4) computes the RHS inside
// its cooperative kernel (one launch per solve instead of two).  Measured
// (profiles/r02ab_exp_fuse4.txt, ms/step): configs[2] 0.3627 -> 0.3603,
// sphere655k 0.1870 -> 0.1848.
#ifndef TCB_FUSE_RHS4
#define TCB_FUSE_RHS4 1
#endif
struct CgArgs {
  const int64_t* slice_ptr;
  const int32_t* col;
  const uint16_t* col16;  // nullable: 16-bit compressed indices
  const int32_t* kbase;
  const uint8_t* fmt;
  const double* A;
  const double* K;     // RHS mode only
  const double* dinv;  // 1 / A_ii (0 on Dirichlet and padding rows)
  int32_t nslices;
  double* x;           // in: x0, out: V^{k+1}
  double* r;
  double* z;
  double* q;
  double* p0;
  double* p1;
  const double* up;    // u' (RHS mode)
  const double* vp;    // v' (RHS mode)
  const double* b;     // plain mode: r0 = b - A x0
  double2* part;       // 2 * gridDim.x partial sums (double-buffered)
  double eps_a, eps_r;
  int32_t max_iters, rel_mode;
  tc_step_stat* stat;  // where this solve's report goes
  int32_t* flags;      // [0] abort [1] nan [2] consecutive fails [3] fail budget [4] step of abort
  int32_t step_tag;    // step index recorded on abort
  int32_t store_r;     // RHS kernel: also store r_0 (the r-form U phases: variant 5); z-form reads z only
  int32_t s0, s1;      // RHS kernel: slice range [s0, s1) (chunked RHS; default [0, nslices))
  const double2* rpart;  // PCG kernel: the RHS partials it sums first (default part) ...
  int32_t n_rpart;       // ... and how many (default gridDim.x)
  int32_t fuse_rhs;      // PCG kernel, variant 4: compute the RHS itself first (one launch per solve)
  double* e0;            // variant 6: the two sigma buffers (u', v' of the RHS: free once r_0 is formed)
  double* e1;
};
constexpr int kPartSlots = 4;  // double2 partial-sum slots per CTA (variant 6: two regions of 2 per CTA)

// ---- split-phase (partitioned) PCG: device scalar state of Algorithm 1 -----
struct Scalars {
  double rho, zeta, zref, alpha, beta;
  int32_t it, conv, nan, done, plast;  // plast: p buffer (0/1) written by the last iteration
};

struct SplitArgs {
  const int64_t* slice_ptr;
  const int32_t* col;    // local column indices (owned [0,n), ghosts n_pad + g)
  const double* A;
  const double* K;
  const double* dinv;
  int32_t nslices;
  int32_t s0, s1;        // slice range of this S / RHS launch ([0, nslices_int) interior, then the rest)
  int32_t phase;         // S / RHS: 0 interior launch (partials kept per CTA), 1 boundary launch (+ reduce), 2 both
  double* x;
  double* r;
  double* z;             // ghost region receives the neighbours' p
  double* q;
  double* p0;            // ghost regions stay 0
  double* p1;
  const double* up;      // ghost regions filled by the per-step halo exchange
  const double* vp;
  double2* part;         // per-CTA partials
  unsigned int* ticket;  // last-CTA-done counter (self-resetting)
  double2* red;          // [0] (r.z, z.z) and [1] (p.q, 0): rank partials, all-reduced in place
  Scalars* sc;
  double eps_a, eps_r;
  int32_t max_iters, rel_mode;
  const int32_t* send_idx;
  double* send_buf;
  int64_t n_send;
  tc_step_stat* stat;
  int32_t* flags;
  int32_t step_tag;
};

// ---- persistent multi-rank PCG over peer memory (pcg_peer.cu) -------------
constexpr int kMaxNbr = 16;
constexpr int kMaxRanks = 64;
struct RedSlot {
  double2 v;
  unsigned long long e;
  unsigned long long pad;
};
struct XPart {
  const int64_t* slice_ptr;
  const int32_t* col;
  const double* A;
  const double* K;
  const double* dinv;
  int32_t nslices, nbr_count;
  int32_t nslices_int;           // leading slices whose rows have no ghost column (no halo wait)
  double* V[3];
  double *r, *z, *q, *p0, *p1, *up, *vp;
  double2* part;                 // 2 x CTAs-per-group partials
  const int32_t* send_idx;       // send entry -> local node
  const int32_t* send_nbr;       // send entry -> neighbour slot
  const int32_t* send_off;       // send entry -> offset in that neighbour's ghost region
  int64_t n_send;
  double* rz[kMaxNbr];           // neighbours' ghost-region bases (z, u', v'), remote
  double* rup[kMaxNbr];
  double* rvp[kMaxNbr];
  unsigned long long* rflag[kMaxNbr];   // neighbour's inbox flag slot for this rank, remote
  unsigned long long* myflag[kMaxNbr];  // this rank's inbox flag slot of each neighbour
  RedSlot* rred[kMaxRanks];      // every rank's reduction slots (2 x world), remote
  RedSlot* myred;
  unsigned int* bar_count;
  unsigned int* bar_gen;
  unsigned int* push_count;       // arrive-only halo pushes of the running launch (pcg_peer.cu)
  unsigned long long* epoch;      // [0] epoch counter, [1] cross-rank reductions done
  double2* red0;                  // rho_0, ||z_0||^2 handed from the RHS kernel to the loop
  int32_t rank, world;
  int32_t* flags;                 // the context's flags ([5] peer timeout), set per launch
  unsigned long long timeout_ns;  // bound of every wait (%globaltimer), set per launch
};

struct IonArgs {
  int32_t n;
  int64_t stride;      // n_pad (SoA state stride)
  const double* Vk;
  const double* Vkm1;
  double* U;
  double* x0;
  double* up;
  double* vp;
  uint8_t* act;        // 0 none, 1 LAT set, 2 LRT set
  double* lat;
  double* lrt;
  int32_t do_lat;
  int32_t has_prev;
  double t_k;          // time of V^k (for LAT/LRT)
  double lat_thr, lrt_thr;
  double dt, theta;
  const int32_t* flags;
  // MMS only
  const double* xyz;
  const uint8_t* dirichlet;
  double t_src, t_next;
};

struct AsmArgs {
  int32_t n;
  int32_t row0;        // global (internal) index of local row 0
  int32_t k;           // nodes per element: 4 tetrahedra, 3 surface triangles
  const double* xyz;
  const int32_t* tets;
  const int32_t* ereg;
  const double* fibre;
  const double* sig_l;
  const double* sig_t;
  const int64_t* inc_ptr;
  const int32_t* inc;  // 4*e + a
  const int64_t* slice_ptr;
  const int32_t* col;
  const int32_t* rowlen;
  double* A;
  double* K;
  double* dinv;
  const uint8_t* dirichlet;  // nullable
  double c_mass, c_stiff;
  int32_t* err;
};

// ---- cluster engine / cohorts (cohort.cu) ------------------------------------
#ifndef TCB_CO_THREADS
#define TCB_CO_THREADS 256
#endif
constexpr int kCoThreads = TCB_CO_THREADS;  // threads per CTA of the cluster engine
constexpr int kCoMaxCluster = 16;   // CTAs per cluster (non-portable size 16 where allowed)
constexpr int kClusterAutoSlices = 256;   // TC_ENGINE_AUTO: cluster engine up to 8 192 rows (measured crossover between 4.3k and 30k nodes)
struct StimEpoch {
  int64_t k0, k1;  // step window [k0, k1)
  int32_t off, m;  // slice of the (local index, s) list
};
// Device descriptor of one replica: a single-partition context's buffers and
// settings at the start of a cluster-engine launch.
struct Exp2Table;
struct CoRep {
  const int64_t* slice_ptr;
  const int32_t* col;
  const double* A;
  const double* K;
  const double* dinv;
  int32_t nslices, n;
  int64_t stride;                // n_pad (SoA state stride)
  double* V[3];
  double *U, *r, *z, *q, *p0, *p1, *up, *vp;
  uint8_t* act;
  double *lat, *lrt;
  int32_t* flags;
  tc_step_stat* stats;           // nsteps entries
  int32_t* status;               // nullable: 0 ran, 1 stopped by the fail budget, 2 NaN
  const StimEpoch* ep;
  const int32_t* stim_idx;
  const double* stim_s;
  int32_t n_ep;
  int32_t iVk, iVkm1, iX, has_prev, max_iters, rel_mode;
  int32_t compact;               // resident launch: 1 = only column indices in shared memory (A, K from L2)
  int64_t k0;
  double dt, theta, eps_a, eps_r, lat_thr, lrt_thr;
  const double* params;          // cohort_pack_params block (device)
  const Exp2Table* tab;          // device_tables() (exp / log tables, copied to shared memory)
};
int cohort_param_doubles();
void cohort_pack_params(int model, const TTParams& tp, const MSParams& mp, const CRNParams& cp,
                        double* out);
int cohort_cluster_size(int model, int want);
int cohort_active_clusters(int model, int csize, size_t smem, bool dense = false);  // smem 0 = streaming launch
size_t cohort_smem_bytes(const int64_t* sp, int32_t ns, int C, bool compact = false);
size_t cohort_smem_limit(int model);
// smem > 0: cluster-resident launch with that much dynamic shared memory per CTA
cudaError_t launch_cohort(int model, const CoRep* d_reps, int nrep, int csize, size_t smem,
                          int64_t nsteps, cudaStream_t s, bool dense = false);

// ---- launchers (return cudaError_t of the launch) --------------------------
cudaError_t launch_assemble(const AsmArgs& a, cudaStream_t s);
struct Exp2Table;
// exp / log tables of the ionic kernels, filled once per device (ionic.cu); null on failure
const Exp2Table* device_tables();
cudaError_t launch_ionic_tt(const IonArgs& a, const TTParams& p, cudaStream_t s);
cudaError_t launch_ionic_ms(const IonArgs& a, const MSParams& p, cudaStream_t s);
cudaError_t launch_ionic_mms(const IonArgs& a, const MMSParams& p, cudaStream_t s);
cudaError_t launch_ionic_crn(const IonArgs& a, const CRNParams& p, cudaStream_t s);
cudaError_t launch_stimulus(int32_t m, const int32_t* idx, const double* s, double* up, double* vp,
                            double dt, double theta, const int32_t* flags, cudaStream_t st);
cudaError_t launch_lat_epilogue(const IonArgs& a, cudaStream_t s);
cudaError_t launch_gather(int64_t n, const int32_t* idx, const double* in, double* out, cudaStream_t s);
cudaError_t launch_scatter(int64_t n, const int32_t* idx, const double* in, double* out, cudaStream_t s);
cudaError_t launch_gather_state(int64_t n, const int32_t* idx, const double* in, int64_t in_stride, double* v0,
                                double* v1, double* U, int64_t upad, int32_t nstates, cudaStream_t s);
cudaError_t launch_spmv(const int64_t* slice_ptr, const int32_t* col, const double* A, int32_t nslices,
                        const double* x, double* y, cudaStream_t s);
// PCG: mode 0 = plain (r0 = b - A x0), 1 = monodomain RHS (r0 = A u' - K v')
// variant 0 = direct loads at full occupancy, 1 = TMA-staged matrix stream
int cg_grid_size(int mode, int variant, int32_t nslices, int device);
// ---- graph engine (pcg_graph.cu, variant 5): Algorithm 1 as a CUDA graph with a
// device-driven WHILE node; scalars live in device memory between the kernels
struct GScal {
  double rho, zeta, zref, alpha, beta;
  int32_t it, conv, nan, done, last_valid;
};
struct GStep {            // per-step arguments, written by a one-thread kernel before each launch
  double* x;              // in: x0, out: V^{k+1}
  tc_step_stat* stat;
  int32_t tag;
};
struct GArgs {
  const int64_t* slice_ptr;
  const int32_t* col;
  const double* A;
  const double* dinv;
  int32_t nslices;
  double *r, *z, *q, *p0, *p1;
  const double2* part0;   // RHS kernel partials (rho_0, ||z_0||^2)
  int32_t n_part0;
  double2* partS;         // S kernel partials (p.q)
  double2* partU;         // U kernel partials (r.z, z.z)
  int32_t n_part;         // S / U grid
  GScal* sc;
  GStep* gs;
  unsigned int* ticket;
  int32_t* flags;
  double eps_a, eps_r;
  int32_t max_iters, rel_mode;
  cudaGraphConditionalHandle cond;
};
int g_grid_size(int device);
cudaError_t g_build(GArgs a, int grid, cudaGraphExec_t* exec);
cudaError_t g_launch(cudaGraphExec_t exec, GStep* gs, double* x, tc_step_stat* stat, int32_t tag, cudaStream_t s);

int cg_pick_variant(int requested, int32_t nslices, int device);
int cg_pick_variant_share(int requested, int32_t nslices, int device, int share);
int cg_grid_size_share(int variant, int32_t nslices, int device, int share);
cudaError_t launch_rhs(int mode, int variant, const CgArgs& a, int grid, cudaStream_t s);
cudaError_t launch_pcg(int mode, int variant, const CgArgs& a, int grid, cudaStream_t s);
cudaError_t launch_pcg_only(int mode, int variant, const CgArgs& a, int grid, cudaStream_t s);
// per-chunk maximum column of the rows of a single-partition SELL layout
cudaError_t launch_chunk_maxcol(const int64_t* sp, const int32_t* col, int32_t nslices, int32_t slices_per_chunk,
                                int32_t* chunk_max, cudaStream_t s);

// split-phase PCG launchers (pcg_split.cu); grid = split_grid(nslices)
int split_grid(int32_t nslices);
cudaError_t launch_split_rhs(const SplitArgs& a, int grid, cudaStream_t s);
cudaError_t launch_split_init(const SplitArgs& a, cudaStream_t s);
cudaError_t launch_split_pack_p(const SplitArgs& a, cudaStream_t s);
cudaError_t launch_pack_gather(int64_t m, const int32_t* idx, const double* src, double* dst,
                               cudaStream_t s);
cudaError_t launch_split_S(const SplitArgs& a, int grid, cudaStream_t s);
cudaError_t launch_split_U(const SplitArgs& a, int grid, cudaStream_t s);
cudaError_t launch_split_scalar(const SplitArgs& a, cudaStream_t s);
cudaError_t launch_split_final(const SplitArgs& a, int grid, cudaStream_t s);
cudaError_t launch_sum_partials(double2* const* reds, int nparts, int slot, cudaStream_t s);
int peer_blocks_per_sm(int which);  // 0 loop kernel, 1 RHS kernel, 2 loop kernel (batch variant)
int peer_max_groups();
// parts: HOST array of `groups` XParts (passed by value in kernel-parameter space)
cudaError_t launch_pcg_peer(const XPart* parts, int groups, int bpg, int bpg_rhs, bool batch, int iX, int iVk,
                            unsigned long long timeout_ns, double eps_a,
                            double eps_r, int32_t max_iters, int32_t rel_mode, tc_step_stat* stat,
                            int32_t* flags, int32_t step_tag, cudaStream_t s);

// ---- host setup (setup_host.cpp) --------------------------------------------
struct HostMesh;
std::string orient_and_validate(int64_t n, int64_t E, int k, int32_t* tets, const double* xyz);
void build_incidence(int64_t n, int64_t E, int k, const int32_t* tets, std::vector<int64_t>& ptr,
                     std::vector<int32_t>& inc);
void build_pattern(int64_t n, int k, const int32_t* tets, const std::vector<int64_t>& ptr,
                   const std::vector<int32_t>& inc, std::vector<int64_t>& rowptr,
                   std::vector<int32_t>& col);
void rcm_order(int64_t n, const std::vector<int64_t>& rowptr, const std::vector<int32_t>& col,
               std::vector<int32_t>& perm);
void permute_csr(int64_t n, const std::vector<int64_t>& rowptr, const std::vector<int32_t>& col,
                 const std::vector<int32_t>& perm, const std::vector<int32_t>& inv,
                 std::vector<int64_t>& rowptr2, std::vector<int32_t>& col2);
void csr_to_sell(int32_t n, const int64_t* rowptr, const int32_t* col, HostSell& s,
                 std::vector<int64_t>* csr_slot = nullptr);
void compress_sell(HostSell& s);

// ---- device-side setup (setup_dev.cu): single-partition pattern, RCM, SELL, incidence
struct DevPattern {         // device arrays, cudaMalloc'ed by dev_setup (dev_setup_free)
  int64_t n = 0, nnz = 0, nnz_pad = 0;
  int32_t nslices = 0;
  int32_t* perm = nullptr;      // [n] internal -> original
  int32_t* inv = nullptr;       // [n] original -> internal
  int64_t* slice_ptr = nullptr; // [nslices + 1]
  int32_t* col = nullptr;       // [nnz_pad] SELL columns (internal numbering)
  int32_t* rowlen = nullptr;    // [n]
  int64_t* iptr = nullptr;      // [n + 1] incidence of the permuted elements
  int32_t* inc = nullptr;       // [k E] 4 e + a, ascending e per node
  int32_t* tets2 = nullptr;     // [k E] element nodes in internal numbering
  // partitioned systems (nparts > 1): the permuted CSR instead of SELL
  int64_t* rowptr = nullptr;    // [n + 1]
  int32_t* colidx = nullptr;    // [nnz]
  std::vector<int64_t> n_int;   // interior rows of each block (interior-first order)
};
cudaError_t dev_setup(int64_t n, int64_t E, int k, const int32_t* d_tets, int use_rcm, int nparts,
                      bool reorder_parts, bool csr_out, DevPattern& out, cudaStream_t s);
void dev_setup_free(DevPattern& p);
cudaError_t dev_gather3(int64_t n, const int32_t* perm, const double* in, double* out, cudaStream_t s);

// Row-block partition of a system in internal (RCM) order: part p owns the
// contiguous rows [g0, g1); ghosts = columns of owned rows outside the block.
struct PartPlan {
  int64_t g0 = 0, g1 = 0;
  int64_t n_interior = 0;          // leading owned rows with no ghost column (interior-first order)
  std::vector<int32_t> ghosts;     // sorted internal indices
  std::vector<int32_t> nbr;        // neighbour parts, ascending
  std::vector<int64_t> recv_off;   // nbr.size()+1 offsets into ghosts (ghosts of one owner are contiguous)
  std::vector<int64_t> send_off;   // nbr.size()+1 offsets into send_g
  std::vector<int32_t> send_g;     // owned internal indices each neighbour needs, grouped by neighbour
};
void plan_partitions(int64_t n, const int64_t* rowptr, const int32_t* col, int nparts,
                     std::vector<PartPlan>& plans);
int64_t block_start(int64_t n, int nparts, int p);
PartPlan plan_from_rows(int64_t n, int nparts, int p, const int64_t* lrp, const int32_t* lcol);
void interior_first(int64_t n, const int64_t* rowptr, const int32_t* col, int nparts,
                    std::vector<int32_t>& order, std::vector<int64_t>& n_int);

}  // namespace tcb
