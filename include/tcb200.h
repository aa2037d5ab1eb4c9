/*
 * tcb200.h -- C ABI of the B200-native TorchCor monodomain step
 * (arXiv 2510.12011).  Plain C types only; no C++ / torch types cross it.
 *
 * What one time step computes (tc_step):
 *   Eq. (2) row 1:  u^{k+1} = u^k + dt g(V^k, u^k)
 *       (TT2006: Rush-Larsen gates, reading I1)
 *   Eq. (3):  (chi Cm M + theta dt K) V^{k+1} = b,
 *       b = chi M (Cm V^k - dt I_ion(V^k,u^{k+1}) + dt I_stim) - (1-theta) dt K V^k
 *       (sign reading S1, unit reading U1)
 *   Algorithm 1: Jacobi PCG from x0 = 2V^k - V^{k-1}
 *   LAT / LRT.
 *
 * Conventions (apply to every entry point):
 *  - Units: mm, ms, mV, S/m (== mS/mm), uF/mm^2, volumetric stimulus uA/mm^3.
 *  - Ownership: every pointer argument is a HOST pointer owned by the caller;
 *    the library copies what it needs during the call and never retains it.
 *    Output buffers are caller-allocated with the documented length.  Device
 *    memory is allocated and freed by the library (tc_destroy frees all),
 *    through the caller's allocator when one is set (tc_set_allocator).
 *  - Node order: all per-node inputs/outputs use the caller's ORIGINAL node
 *    numbering; the RCM permutation is internal.
 *  - Errors: return codes only, no exception crosses the ABI; tc_last_error()
 *    returns a message (owned by the context, valid until the next call on it).
 *  - Threading: a context is used by one host thread at a time; independent
 *    contexts are independent (cohort mode) -- no launch state or
 *    flag is shared between them (the exp / log tables of the ionic kernels
 *    are one read-only copy per device).
 *  - All arithmetic of the step is IEEE fp64 on the GPU; there is no
 *    CPU fallback: without a CUDA device tc_create returns TC_ECUDA.
 */
#ifndef TCB200_H
#define TCB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tc_ctx tc_ctx;

/* Device allocator callbacks (the torch caching allocator).
 * alloc(bytes, cuda_stream, user) returns device memory of at least `bytes`
 * on the context's device, usable on cuda_stream, or NULL; release(ptr,
 * cuda_stream, user) gives it back.  Called from the thread that calls the
 * library, during setup (tc_assemble, first tc_step_io / tc_set_state) and
 * tc_destroy; never inside tc_step. */
typedef void* (*tc_alloc_fn)(size_t bytes, void* cuda_stream, void* user);
typedef void (*tc_free_fn)(void* ptr, void* cuda_stream, void* user);

typedef enum {
  TC_OK = 0,
  TC_EINVAL = 1,   /* bad argument (index out of range, bad size, zero fibre ...) */
  TC_ENOMEM = 2,   /* host or device allocation failed */
  TC_ECUDA = 3,    /* CUDA runtime error / no device */
  TC_ENCCL = 4,    /* communicator error (multi-GPU) */
  TC_ESOLVER = 5,  /* PCG failed fail_budget consecutive steps */
  TC_ENAN = 6,     /* NaN in a PCG inner product or in V */
  TC_ESTATE = 7,   /* call out of order (e.g. tc_step before tc_assemble) */
  TC_EDEGEN = 8,   /* zero-volume tetrahedron */
  TC_EREGION = 9   /* region tag without conductivity, or sigma <= 0 */
} tc_status;

typedef enum {
  TC_ION_TT2006_EPI = 0, /* ten Tusscher-Panfilov 2006, epicardial */
  TC_ION_MS = 1,         /* Mitchell-Schaeffer 2003 (reading I5) */
  TC_ION_MMS = 2,        /* no ionic model: manufactured source r of Eq. 8 */
  TC_ION_CRN = 3         /* Courtemanche-Ramirez-Nattel 1998 human atrial cell (
                            DESIGN.md reading I6), 20 states */
} tc_ionic;

/* Execution engine of tc_step for a single-partition context (DESIGN.md
 * "Cluster engine").  Both compute the same step; they differ in how the work
 * is laid out on the GPU. */
typedef enum {
  TC_ENGINE_AUTO = 0,    /* cluster engine for small systems, grid engine otherwise */
  TC_ENGINE_GRID = 1,    /* per step: ionic kernel + RHS kernel + one cooperative PCG
                            kernel over all SMs (grid barriers) */
  TC_ENGINE_CLUSTER = 2, /* every step of the tc_step call in ONE launch on one
                            thread-block cluster (<= 16 CTAs; cluster barriers, DSMEM
                            reductions); matrix and own-row vectors resident in shared
                            memory when they fit.  TT2006 / MS only. */
  TC_ENGINE_CLUSTER_STREAMING = 3 /* the cluster engine with everything streamed from
                            global memory (measurement; what large systems get) */
} tc_engine;

typedef enum {
  TC_REL_CONSECUTIVE = 0, /* ||z_{k+1}|| / ||z_k||  (Alg. 1 literal, reading C1) */
  TC_REL_INITIAL = 1      /* ||z_{k+1}|| / ||z_0|| */
} tc_relmode;

/* Simulation settings. */
typedef struct {
  double theta;          /* 0 FE, 0.5 CN (default), 2/3, 1 BE (Table 2) */
  double dt;             /* ms */
  double chi;            /* surface-to-volume ratio, mm^-1 (Table 3: 140) */
  double cm;             /* membrane capacitance, uF/mm^2 (Table 3: 0.01) */
  double abs_tol;        /* eps_a of Alg. 1 (1e-5) */
  double rel_tol;        /* eps_r of Alg. 1 */
  int32_t max_iters;     /* m of Alg. 1 (100) */
  int32_t rel_mode;      /* tc_relmode */
  int32_t model;         /* tc_ionic */
  int32_t fail_budget;   /* consecutive non-converged steps before TC_ESOLVER (3) */
  double lat_threshold;  /* LAT: first V > this (0 mV) */
  double lrt_threshold;  /* LRT: first later V < this with dV/dt < 0 (-70 mV) */
  int32_t use_rcm;       /* 1: Reverse Cuthill-McKee reordering */
  int32_t pcg_variant;   /* PCG kernel memory pipeline: 0 direct
                            loads at full occupancy (default), 1 TMA-staged matrix stream,
                            2 direct loads with 16-bit column offsets, 3 direct loads with
                            the matrix held in L2 (evict-last policy; for systems whose
                            values + indices fit in L2), 4 every slot of a row in flight
                            at once (latency-bound mid-size systems), 5 the solve as a CUDA
                            graph with a device-driven WHILE node (init, S, U, final
                            kernels; tc_step only), 6 the single-reduction (Chronopoulos-Gear)
                            recurrence: Algorithm 1's iterates in exact arithmetic with one
                            grid reduction per iteration (not the paper's order
                            of operations, so opt-in; single-part grid path only -- partitioned
                            paths run Algorithm 1); -1 (default):
                            automatic, 4 when the system has at most 4 slices per
                            resident warp of variant 0, else 0 */
  int32_t partitions;    /* row-block partitions of the RCM order held by this context on
                            its GPU (1 = persistent single-kernel PCG; >1 = split-phase PCG
                            with device-copy halos).  Ignored after tc_comm_init (one
                            partition per rank). */
  int32_t check_every;   /* split-phase PCG: iterations enqueued between host checks of the
                            device convergence flag (4) */
  int32_t peer;          /* partitioned systems: 1 (default) = one persistent kernel per GPU
                            doing halos and reductions itself over peer memory (NVLink via
                            CUDA IPC between ranks, plain device memory between the parts of
                            one GPU); 0 = split-phase kernels + NCCL / device copies */
  int32_t engine;        /* tc_engine (TC_ENGINE_AUTO) */
  int32_t device_setup;  /* 1 (default): single-partition systems build their pattern, RCM,
                            SELL layout and element incidence on the GPU (
                            identical result to the host path); 0: host setup */
  int32_t peer_timeout_s; /* multi-GPU peer kernels: wall-clock bound (seconds, %globaltimer)
                            of every wait for another rank (halo flags, reduction slots,
                            group barriers); a rank that does not answer within it turns
                            the step into TC_ENCCL instead of a hang.  0 = default 300 s
                            (a collective-style timeout: rank skew from host-side work such
                            as checkpoint writes stays far below it) */
} tc_config;

/* Per-step PCG report. */
typedef struct {
  int32_t iters;     /* iterations of Alg. 1's loop executed */
  int32_t converged; /* 1 if the stopping test fired (incl. ||z_0|| < eps_a) */
  double znorm;      /* last ||z|| */
} tc_step_stat;

/* Fills the defaults: theta 0.5, dt 0.01, chi 140, cm 0.01, tolerances 1e-5,
 * max_iters 100, consecutive rel-mode, TT2006 epi, fail_budget 3,
 * thresholds 0 / -70 mV, use_rcm 1, pcg_variant -1, partitions 1, check_every 4, peer 1,
 * engine auto, device_setup 1, peer_timeout_s 0 (= 300 s). */
void tc_config_default(tc_config* cfg);

/* Create a context on CUDA device `device`.  `cuda_stream` is a cudaStream_t
 * (NULL = the library creates its own non-blocking stream); all device work
 * of the context is ordered on it.  TC_ECUDA if no device is usable. */
tc_status tc_create(const tc_config* cfg, int device, void* cuda_stream, tc_ctx** out);

/* Frees every host and device resource of the context. NULL is accepted. */
tc_status tc_destroy(tc_ctx* ctx);

/* Message describing the last error on ctx ("" if none). */
const char* tc_last_error(const tc_ctx* ctx);
/* Route the context's persistent device memory (matrix, vectors, cell state,
 * I/O staging) through the caller's allocator (both callbacks, or both NULL
 * for cudaMalloc).  Call right after tc_create, before anything allocates
 * (TC_ESTATE otherwise).  Ignored for multi-process contexts (tc_comm_init),
 * whose buffers are shared over CUDA IPC and need whole cudaMalloc blocks.
 * Setup scratch memory is always cudaMalloc'ed and freed within the call.
 * The callbacks and `user` must stay valid until tc_destroy returns. */
tc_status tc_set_allocator(tc_ctx* ctx, tc_alloc_fn alloc, tc_free_fn release, void* user);

/* Mesh.  xyz: n_nodes*3 doubles (mm).  tets: n_tets*4
 * zero-based node indices (any orientation; negatively oriented tets get two
 * indices swapped).  region: n_tets tags (NULL = all 0).  fibre:
 * n_tets*3 doubles, any non-zero length, normalised here (NULL = (1,0,0)).
 * Errors: TC_EINVAL index out of range / zero fibre; TC_EDEGEN zero volume.
 * Must precede tc_assemble; may be called once per context. */
tc_status tc_set_mesh(tc_ctx* ctx, int64_t n_nodes, const double* xyz, int64_t n_tets,
                      const int32_t* tets, const int32_t* region, const double* fibre);

/* Mesh with `nodes_per_elem` nodes per element ("triangular or tetrahedral
 * elements"): 4 = tetrahedra (exactly tc_set_mesh), 3 = P1 triangles embedded in
 * 3-D (surface meshes, e.g. atria or the paper's MMS unit square).  elems:
 * n_elems*nodes_per_elem node indices.  For triangles the gradients are taken in
 * the element plane, so a fibre component normal to it does not act;
 * M_e = |e|/12 (1 + delta_ab).  Same ownership and errors as tc_set_mesh, plus
 * TC_EINVAL for nodes_per_elem not in {3, 4} and TC_EDEGEN for zero area. */
tc_status tc_set_mesh_elems(tc_ctx* ctx, int64_t n_nodes, const double* xyz, int64_t n_elems,
                            int32_t nodes_per_elem, const int32_t* elems, const int32_t* region,
                            const double* fibre);

/* Region conductivities: sigma = sigma_t I + (sigma_l - sigma_t) f f^T
 * (reading A13).  S/m, both > 0.  Replaces any previous table. */
tc_status tc_set_conductivity(tc_ctx* ctx, int32_t n_regions, const int32_t* ids,
                              const double* sigma_l, const double* sigma_t);

/* Ionic-model parameter by name ("parameters ... programmatically
 * reset"); TT2006 names: R T F CAP Vc Vsr Vss Ko Nao Cao GNa GK1 Gto GKr GKs pKNa
 * GCaL GbNa GbCa GpCa KpCa GpK PNaK KmK KmNa kNaCa KmNai KmCa ksat gamma alpha
 * Bufc Kbufc Bufsr Kbufsr Bufss Kbufss Vmaxup Kup Vrel k1p k2p k3 k4 EC maxsr
 * minsr Vleak Vxfer;  MS: tau_in tau_out tau_open tau_close v_gate V_min V_max.
 * TC_EINVAL for an unknown name.  Takes effect at the next tc_step. */
tc_status tc_set_ionic_param(tc_ctx* ctx, const char* name, double value);
tc_status tc_get_ionic_param(const tc_ctx* ctx, const char* name, double* value);

/* Add a stimulus: nodes (original numbering) receive the
 * volumetric current `amplitude` (uA/mm^3) for steps k with
 * round(t_start/dt) <= k < round((t_start+duration)/dt) (reading T1);
 * overlapping stimuli add.  Must precede tc_assemble. */
tc_status tc_add_stimulus(tc_ctx* ctx, int64_t n_idx, const int32_t* nodes, double t_start,
                          double duration, double amplitude);

/* Manufactured-solution configuration (model TC_ION_MMS):
 * source r(x,y,t) of Eq. 8 evaluated at t_k + theta dt, Dirichlet V = w(x,y,t_{k+1})
 * on `nodes` (reading M3), initial V = w(x,y,0).  Must precede tc_assemble. */
tc_status tc_set_mms(tc_ctx* ctx, double k, double w1, double w2, double lambda,
                     int64_t n_dirichlet, const int32_t* nodes);
/* The two halves of tc_set_mms: the Dirichlet node set (values
 * w(x,y,t_{k+1}), reading M3) and the source constants k, w1, w2, lambda of
 * Eq. 5 / Eq. 8 (default 1, pi, pi, pi: reading M2).  Same preconditions and
 * errors as tc_set_mms; each keeps the other half. */
tc_status tc_set_dirichlet(tc_ctx* ctx, int64_t n_idx, const int32_t* nodes);
tc_status tc_set_mms_source(tc_ctx* ctx, double k, double w1, double w2, double lambda);

/* Build the system (boundary, not timed per step): pattern, RCM, GPU
 * assembly of M, K into A = chi Cm M + theta dt K and diag(A)^-1,
 * initial state (model initial conditions, V^{-1} := V^0, step 0, LAT/LRT unset). */
tc_status tc_assemble(tc_ctx* ctx);

/* Advance n_steps time steps on the GPU.  stats (nullable) receives n_steps
 * reports.  Non-convergence of a step is not an error; TC_ESOLVER after
 * fail_budget consecutive failures, TC_ENAN on NaN (the context then refuses
 * further steps).  Synchronises the stream once at the end. */
tc_status tc_step(tc_ctx* ctx, int64_t n_steps, tc_step_stat* stats);

/* Number of nodes, current step index k (t = k dt), state length. */
int64_t tc_num_nodes(const tc_ctx* ctx);
int64_t tc_current_step(const tc_ctx* ctx);

/* V^k (n_nodes doubles, original order). */
tc_status tc_get_v(tc_ctx* ctx, double* v_out);

/* y = A x (which = 0; A = chi Cm M + theta dt K, Eq. 3) or y = K x (which = 1)
 * with the assembled matrices; x, y: n_nodes doubles in the original order.
 * Single-partition contexts (TC_ESTATE otherwise).  Inspection / parity. */
tc_status tc_apply(tc_ctx* ctx, int32_t which, const double* x, double* y);

/* LAT and LRT (n_nodes doubles each, original order; -1.0 = unset). */
tc_status tc_get_activation(tc_ctx* ctx, double* lat, double* lrt);

/* Full cell state for checkpoint / state injection:
 * [V^k (n) | V^{k-1} (n) | u_0 (n) ... u_{S-1} (n) | k | has_prev], original order,
 * S = 18 (TT2006, state order Ki Nai Cai CaSS CaSR Rbar m h j xr1 xr2 xs r s d f
 * f2 fCass), 1 (MS: h), 0 (MMS).  has_prev = 0 means V^{k-1} := V^k.
 * Both calls return once buf has been read / written (the caller owns buf;
 * tc_set_state is one host->device copy and one synchronisation in a
 * single-process context, staging in the tc_step_io buffers, or one copy per
 * field when those buffers cannot be allocated).  tc_set_state also clears a
 * sticky abort of the context (NaN, fail budget, peer timeout): the new state
 * is a fresh start. */
int64_t tc_state_len(const tc_ctx* ctx);
tc_status tc_get_state(tc_ctx* ctx, double* buf, int64_t len);
tc_status tc_set_state(tc_ctx* ctx, const double* buf, int64_t len);

/* Pipelined host I/O: n_steps independent one-step problems.  For j = 0 ..
 * n_steps-1: the state states[j*stride .. j*stride + tc_state_len) (host, the
 * tc_set_state layout; pinned memory lets the copies overlap) is loaded, one
 * step is taken (Eq. 2-3 and Algorithm 1, as tc_step), and V^{k+1}
 * (n_nodes doubles, original order) is written to v_out[j*n_nodes ..].  The
 * host->device copy of input j+1 and the device->host copy of output j-1 run
 * on two copy streams while step j computes -- the result equals
 * tc_set_state + tc_step(1) + tc_get_v for every j.  stats: nullable,
 * n_steps entries.  After the call the context holds the state after the last
 * problem.  stride = 0: every problem reads the same host state (one
 * tc_state_len buffer, still copied host -> device once per problem) and
 * writes its V^{k+1} to the same n_nodes output (copied back once per problem;
 * the last one remains) -- a stream of n_steps identical problems in bounded
 * host memory.  Errors: TC_EINVAL (null pointers, 0 < stride < tc_state_len,
 * a bad step index in an input), TC_ESTATE (before tc_assemble, or a
 * multi-process context), and tc_step's errors.  Host buffers stay owned by
 * the caller. */
tc_status tc_step_io(tc_ctx* ctx, int64_t n_steps, const double* states, int64_t stride, double* v_out,
                     tc_step_stat* stats);

/* Device time (ms) spent per phase since the last reset, measured with CUDA
 * events on the context stream when profiling is enabled:
 * out[0] ionic + stimulus kernels, out[1] PCG kernel (RHS + Alg. 1),
 * out[2] LAT epilogue; out[3] total PCG iterations; out[4] steps;
 * out[5] kernel launches issued by tc_step (counted whether or not profiling). */
tc_status tc_profile(tc_ctx* ctx, int enable);
tc_status tc_profile_read(tc_ctx* ctx, double out[6], int reset);

/* Sizes of the assembled system: out[0] n, out[1] nnz (stored entries of A,
 * CSR count), out[2] padded SELL-32 slots of the parts held here, out[3] their
 * slices, out[4] PCG grid (CTAs) of the first part, out[5] slices kept at int32
 * indices (variant 2), out[6] partitions, out[7] ghost columns of the parts held,
 * out[8] PCG path (0 persistent single part, 1 split-phase, 2 persistent peer),
 * out[9] CTAs per partition of the peer kernel, out[10] PCG kernel variant
 * launched for the first part (tc_config.pcg_variant, or the automatic choice).
 * TC_ESTATE before tc_assemble/tc_csr_upload. */
tc_status tc_matrix_info(const tc_ctx* ctx, int64_t out[11]);

/* ---- Minimum-slice operators on an uploaded CSR (no mesh needed) ---------- */
/* Upload an n x n CSR (rowptr n+1, col/val nnz, columns sorted per row, the
 * diagonal present for tc_pcg).  Replaces any previous matrix of the context. */
tc_status tc_csr_upload(tc_ctx* ctx, int32_t n, int64_t nnz, const int32_t* rowptr,
                        const int32_t* col, const double* val);
/* y = A x, x and y host arrays of length n. */
tc_status tc_spmv(tc_ctx* ctx, const double* x, double* y);
/* Algorithm 1 with Jacobi preconditioner on the uploaded matrix; tolerances,
 * max_iters and rel_mode from the context config.  Host arrays of length n. */
tc_status tc_pcg(tc_ctx* ctx, const double* b, const double* x0, double* x_out,
                 tc_step_stat* report);

/* ---- Multi-GPU (row partition + halo) ---
 * One process per GPU.  Rank 0 creates an NCCL unique id (128 bytes) and
 * broadcasts it (e.g. with torch.distributed); every rank then calls
 * tc_comm_init before tc_set_mesh and passes the SAME global mesh, stimuli and
 * conductivities.  The system in RCM order is cut into `world` contiguous row
 * blocks; rank r owns block r.  Each PCG iteration exchanges the halo of p
 * with ncclSend/ncclRecv (neighbouring blocks only) and all-reduces the two CG
 * scalars (ncclAllReduce, identical bits on every rank -> identical stopping
 * decisions).  Outputs (tc_get_v, tc_get_activation, tc_get_state) are
 * all-gathered: every rank receives the full field.  TC_ENCCL on NCCL errors
 * (NCCL is loaded at run time; without it tc_comm_init fails with TC_ENCCL). */
tc_status tc_nccl_unique_id(uint8_t id[128]);
tc_status tc_comm_init(tc_ctx* ctx, int rank, int world, const uint8_t id[128]);

/* Internal row order of the assembled system: perm[i] = original index of
 * internal row i (n_nodes entries; the RCM order of P:135 when use_rcm, the
 * identity otherwise).  Host and device setup give the same order. */
tc_status tc_node_order(const tc_ctx* ctx, int32_t* perm);

/* Engine tc_step uses for this context: out[0] TC_ENGINE_GRID or
 * TC_ENGINE_CLUSTER, out[1] CTAs per cluster, out[2] dynamic shared memory per
 * CTA (0 = streaming), out[3] clusters of that shape resident at once. */
tc_status tc_engine_info(tc_ctx* ctx, int64_t out[4]);

/* ---- Cohorts: many independent simulations per GPU ------------
 * A cohort batches assembled single-partition contexts ("members": different
 * meshes, conductivities, stimuli, ionic parameters, time steps, tolerances)
 * that share the device and the ionic model (TT2006, MS or CRN).  tc_cohort_step
 * advances EVERY member by n_steps: the small members (those TC_ENGINE_AUTO
 * would give the cluster engine) in ONE launch, one thread-block cluster per
 * member, each with its own PCG stopping test (per-replica stopping); larger
 * members with their own grid-engine tc_step while that launch runs.  Each member's results equal what
 * tc_step(member, n_steps) gives (same arithmetic; inner-product partial sums
 * grouped per cluster), and afterwards every tc_get_* call on a member works as
 * usual.  The members stay owned by the caller and must outlive the cohort;
 * members must not be stepped concurrently with tc_cohort_step. */
typedef struct tc_cohort tc_cohort;
/* members: host array of `count` context pointers (copied).  cluster_size: CTAs
 * per member cluster (1, 2, 4, 8, 16) or 0 = automatic: at most one SELL slice
 * per warp for the largest member, at least 2, chosen with the mode (below).
 * resident: 0 = stream from global memory; 2 = "full": keep each CTA's matrix
 * block (values, column indices) and own-row vectors in shared memory for the
 * whole launch when the largest member's block fits; 3 = "compact": keep only
 * the column indices and the vectors there (the matrix values are read through
 * L2), a smaller footprint; 4 = "dense" streaming: the kernel built for two
 * CTAs per SM (128 registers, some spills), twice the resident clusters;
 * 1 = automatic: the cluster size (when cluster_size is 0) and the mode
 * (full / compact by footprint, streaming, dense) with the lowest modelled
 * time = ceil(members / resident clusters) x the measured time of one round
 * (DESIGN.md "Cohorts").  A resident mode whose footprint does not fit
 * streams (tc_cohort_info reports what was chosen).
 * TC_EINVAL if resident is outside 0..4.
 * TC_ESTATE if a member is not assembled or is partitioned / multi-GPU;
 * TC_EINVAL on mixed devices or models, MMS members, or a bad cluster size. */
tc_status tc_cohort_create(tc_ctx* const* members, int32_t count, int32_t cluster_size,
                           int32_t resident, tc_cohort** out);
/* Advance every member n_steps.  stats (nullable): count * n_steps reports,
 * member-major (member m's step s at [m * n_steps + s]).  The work runs on
 * member 0's stream, ordered after and before the other members' streams.
 * A member that exceeds its fail budget or hits a NaN stops (its context
 * reports the error on its next tc_step); the call then returns TC_ESOLVER /
 * TC_ENAN naming the first such member, after all members were advanced. */
tc_status tc_cohort_step(tc_cohort* cohort, int64_t n_steps, tc_step_stat* stats);
/* Batched member I/O (the per-member tc_set_state / tc_get_v, one
 * synchronisation per call instead of one per member).  count: the number of
 * members (must equal the cohort's); bufs[i]: host state of member i in the
 * tc_set_state layout, lens[i] its length in doubles (must equal
 * tc_state_len(member i)); v_out[i]: host array of lens[i] == n_nodes(member i)
 * doubles, filled with the member's V^k in the original order.  Arrays of
 * `count` pointers / lengths, member order of tc_cohort_create; the caller owns
 * every buffer (pinned memory lets the copies run at full rate).  Both return
 * after every copy completed.  TC_EINVAL: a null pointer, a count or length
 * mismatch, or a bad step index -- every input is validated, and every
 * member's staging allocated (TC_ENOMEM / TC_ECUDA), before any member
 * changes.  A TC_ECUDA from a copy or kernel launch after that point leaves
 * the members' states undefined (the device context is then unusable). */
tc_status tc_cohort_set_states(tc_cohort* cohort, int64_t count, const double* const* bufs, const int64_t* lens);
tc_status tc_cohort_get_v(tc_cohort* cohort, int64_t count, double* const* v_out, const int64_t* lens);
/* out[0] members, out[1] CTAs per cluster, out[2] clusters resident at once,
 * out[3] dynamic shared memory per CTA (0 = streaming), out[4] 1 when the
 * resident launch keeps only the column indices (and vectors) in shared
 * memory and reads the matrix values through L2 (chosen when that keeps more
 * clusters resident and the members outnumber the full-resident clusters),
 * out[5] 1 for the dense (two CTAs per SM) streaming kernel. */
tc_status tc_cohort_info(const tc_cohort* cohort, int32_t out[6]);
const char* tc_cohort_last_error(const tc_cohort* cohort);
tc_status tc_cohort_destroy(tc_cohort* cohort);

/* Ionic || RHS pipeline of the grid engine:
 * out[0] = row chunks (0: the kernels run one after the other), out[1] = rows
 * per chunk.  With chunks, tc_profile_read's out[0] covers the overlapped ionic
 * and RHS kernels and out[1] the PCG kernel alone. */
tc_status tc_pipeline_info(tc_ctx* ctx, int64_t out[2]);
/* Index audit of an assembled context: downloads
 * every device index array the step kernels address memory through and checks
 * it against its allocation -- node permutation, SELL slice pointers and column
 * indices (owned rows and ghost region, padding, diagonal slot, interior slices
 * free of ghosts), halo send / receive lists, stimulus lists -- plus finite
 * matrix values and diag(A)^-1.  checked (nullable): number of indices checked.
 * TC_EINVAL with the first violation in tc_last_error.  Debug / test use. */
tc_status tc_validate(tc_ctx* ctx, int64_t* checked);

/* ---- Host-only helpers (no GPU needed; used by the CPU tests) ------------- */
/* CSR pattern of a tet mesh: (i,j) iff an element holds both.  Call
 * with col = NULL to get rowptr (n+1) first, then again with col (rowptr[n]). */
tc_status tc_mesh_pattern(int64_t n, int64_t n_tets, const int32_t* tets, int64_t* rowptr,
                          int32_t* col);
/* Reverse Cuthill-McKee of a symmetric pattern (SPEC S:146 tie rules);
 * perm[new] = old. */
tc_status tc_rcm(int64_t n, const int64_t* rowptr, const int32_t* col, int32_t* perm);
/* Interior-first order of the nparts row blocks of a pattern in internal order
 * (what tc_assemble applies to partitioned systems):
 * order[new] = old, n_interior[p] (nparts entries) = leading rows of block p
 * with no column outside the block; the multi-GPU PCG computes those while
 * the halo is in flight.  Blocks and ghost sets are unchanged. */
tc_status tc_interior_first(int64_t n, const int64_t* rowptr, const int32_t* col, int32_t nparts,
                            int32_t* order, int64_t* n_interior);
/* The row-block partition plan of part `part` (of nparts) for a pattern in
 * internal order: sizes = {ghosts, neighbours, send entries, owned rows};
 * bounds (nparts+1), ghosts (sorted), nbr, recv_off (nbr+1), send_off (nbr+1),
 * send_g (internal indices) -- each nullable. */
tc_status tc_partition_plan(int64_t n, const int64_t* rowptr, const int32_t* col, int32_t nparts,
                            int32_t part, int64_t sizes[4], int64_t* bounds, int32_t* ghosts,
                            int32_t* nbr, int64_t* recv_off, int64_t* send_off, int32_t* send_g);

/* Version of this ABI. */
int32_t tc_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TCB200_H */
