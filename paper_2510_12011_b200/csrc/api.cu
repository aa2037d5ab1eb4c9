// api.cu -- the C ABI of libtcb200 (include/tcb200.h): context, setup, the
// per-step launch sequence and state I/O.  Every step of the path runs in the
// CUDA kernels of ionic.cu / pcg.cu; this file only orchestrates.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "internal.h"

using namespace tcb;

struct Stim {
  std::vector<int32_t> nodes;
  double t0, dur, amp;
};
struct Epoch {
  int64_t k0, k1;  // [k0, k1)
  int32_t off, m;  // slice of the concatenated (node, s) list
};

struct tc_ctx {
  tc_config cfg;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  // host mesh
  int64_t n = 0, E = 0;
  bool have_mesh = false;
  std::vector<double> xyz, fibre;
  std::vector<int32_t> tets, region;
  std::vector<int32_t> reg_ids;
  std::vector<double> sig_l, sig_t;
  TTParams tt;
  double tt_V0;
  double tt_u0[kTTStates];
  MSParams ms;
  MMSParams mms{1.0, M_PI, M_PI, M_PI};
  std::vector<Stim> stims;
  std::vector<int32_t> dirichlet_nodes;
  // assembled system
  bool assembled = false;
  bool csr_mode = false;
  bool has_diag_zero = false;
  std::vector<int32_t> perm, inv;  // perm[new] = old, inv[old] = new
  int32_t nslices = 0;
  int64_t n_pad = 0, nnz_pad = 0;
  int nstates = 0;
  // device
  int64_t* d_sp = nullptr;
  int32_t* d_col = nullptr;
  uint16_t* d_col16 = nullptr;
  int32_t* d_kbase = nullptr;
  uint8_t* d_fmt = nullptr;
  int64_t n_wide = 0;
  double *d_A = nullptr, *d_K = nullptr, *d_dinv = nullptr;
  double* d_V[3] = {nullptr, nullptr, nullptr};
  int iVk = 0, iVkm1 = 1, iX = 2;
  double* d_U = nullptr;
  double *d_r = nullptr, *d_z = nullptr, *d_q = nullptr, *d_p0 = nullptr, *d_p1 = nullptr;
  double *d_up = nullptr, *d_vp = nullptr, *d_b = nullptr, *d_tmp = nullptr;
  uint8_t* d_act = nullptr;
  double *d_lat = nullptr, *d_lrt = nullptr;
  int32_t *d_perm = nullptr, *d_inv = nullptr;
  double2* d_part = nullptr;
  int32_t* d_flags = nullptr;
  tc_step_stat* d_stats = nullptr;
  int64_t stats_cap = 0;
  double* d_xyz = nullptr;
  uint8_t* d_dir = nullptr;
  std::vector<Epoch> epochs;
  int32_t* d_stim_idx = nullptr;
  double* d_stim_s = nullptr;
  int64_t k = 0;
  bool has_prev = false;
  int cg_grid = 1;
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> evs;
  double t_ion = 0, t_cg = 0, t_other = 0, prof_iters = 0, prof_steps = 0, launches = 0;
  int64_t nnz = 0;
  std::vector<void*> allocs;
};

// ------------------------------------------------------------------ helpers
static tc_status fail(tc_ctx* c, tc_status st, const std::string& msg) {
  if (c) c->err = msg;
  return st;
}
#define CUDA_TRY(c, expr)                                                           \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail((c), TC_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
static cudaError_t dalloc(tc_ctx* c, T** p, int64_t count) {
  size_t bytes = (size_t)std::max<int64_t>(count, 1) * sizeof(T);
  void* v = nullptr;
  cudaError_t e = cudaMalloc(&v, bytes);
  if (e != cudaSuccess) return e;
  c->allocs.push_back(v);
  *p = (T*)v;
  return cudaMemsetAsync(v, 0, bytes, c->stream);
}

static void free_all(tc_ctx* c) {
  for (void* p : c->allocs) cudaFree(p);
  c->allocs.clear();
  for (auto e : c->evs) cudaEventDestroy(e);
  c->evs.clear();
}

extern "C" {

int32_t tc_abi_version(void) { return 1; }

void tc_config_default(tc_config* c) {
  c->theta = 0.5;
  c->dt = 0.01;
  c->chi = 140.0;
  c->cm = 0.01;
  c->abs_tol = 1e-5;
  c->rel_tol = 1e-5;
  c->max_iters = 100;
  c->rel_mode = TC_REL_CONSECUTIVE;
  c->model = TC_ION_TT2006_EPI;
  c->fail_budget = 3;
  c->lat_threshold = 0.0;
  c->lrt_threshold = -70.0;
  c->use_rcm = 1;
  c->pcg_variant = 0;
}

tc_status tc_create(const tc_config* cfg, int device, void* cuda_stream, tc_ctx** out) {
  if (!cfg || !out) return TC_EINVAL;
  *out = nullptr;
  if (!(cfg->dt > 0) || !(cfg->theta >= 0 && cfg->theta <= 1) || !(cfg->chi > 0) || !(cfg->cm > 0) ||
      cfg->max_iters < 0 || !(cfg->abs_tol >= 0) || !(cfg->rel_tol >= 0) || cfg->model < 0 || cfg->model > 2 || cfg->pcg_variant < 0 || cfg->pcg_variant > 2)
    return TC_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device || device < 0) return TC_ECUDA;
  if (cudaSetDevice(device) != cudaSuccess) return TC_ECUDA;
  tc_ctx* c = new tc_ctx();
  c->cfg = *cfg;
  c->device = device;
  tt_defaults(&c->tt, &c->tt_V0, c->tt_u0);
  ms_defaults(&c->ms);
  if (cuda_stream) {
    c->stream = (cudaStream_t)cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete c;
      return TC_ECUDA;
    }
    c->own_stream = true;
  }
  if (dalloc(c, &c->d_flags, 8) != cudaSuccess) {
    delete c;
    return TC_ECUDA;
  }
  *out = c;
  return TC_OK;
}

tc_status tc_destroy(tc_ctx* c) {
  if (!c) return TC_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  free_all(c);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return TC_OK;
}

const char* tc_last_error(const tc_ctx* c) { return c ? c->err.c_str() : "null context"; }

int64_t tc_num_nodes(const tc_ctx* c) { return c ? c->n : 0; }
int64_t tc_current_step(const tc_ctx* c) { return c ? c->k : 0; }

tc_status tc_set_mesh(tc_ctx* c, int64_t n, const double* xyz, int64_t E, const int32_t* tets,
                      const int32_t* region, const double* fibre) {
  if (!c) return TC_EINVAL;
  if (c->have_mesh || c->csr_mode) return fail(c, TC_ESTATE, "tc_set_mesh: mesh already set");
  if (n <= 0 || E <= 0 || !xyz || !tets) return fail(c, TC_EINVAL, "tc_set_mesh: empty mesh");
  if (n >= (1ll << 31) - 64 || 4 * E >= (1ll << 31)) return fail(c, TC_EINVAL, "tc_set_mesh: mesh too large for int32 indices");
  c->n = n;
  c->E = E;
  c->xyz.assign(xyz, xyz + 3 * n);
  c->tets.assign(tets, tets + 4 * E);
  if (region) c->region.assign(region, region + E); else c->region.assign(E, 0);
  if (fibre) {
    c->fibre.assign(fibre, fibre + 3 * E);
    for (int64_t e = 0; e < E; ++e) {
      const double* f = fibre + 3 * e;
      double nn = f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
      if (!(nn > 0) || !std::isfinite(nn))
        return fail(c, TC_EINVAL, "tc_set_mesh: zero or non-finite fibre at tet " + std::to_string(e));
    }
  } else {
    c->fibre.assign(3 * E, 0.0);
    for (int64_t e = 0; e < E; ++e) c->fibre[3 * e] = 1.0;
  }
  std::string m = orient_and_validate(n, E, c->tets.data(), c->xyz.data());
  if (!m.empty()) {
    tc_status st = m.rfind("EDEGEN", 0) == 0 ? TC_EDEGEN : TC_EINVAL;
    c->tets.clear();
    return fail(c, st, "tc_set_mesh: " + m.substr(m.find(':') + 1));
  }
  c->have_mesh = true;
  return TC_OK;
}

tc_status tc_set_conductivity(tc_ctx* c, int32_t nr, const int32_t* ids, const double* sl,
                              const double* st) {
  if (!c) return TC_EINVAL;
  if (nr <= 0 || !ids || !sl || !st) return fail(c, TC_EINVAL, "tc_set_conductivity: empty table");
  for (int32_t r = 0; r < nr; ++r)
    if (!(sl[r] >= 0) || !(st[r] >= 0) || !std::isfinite(sl[r]) || !std::isfinite(st[r]))
      return fail(c, TC_EREGION, "tc_set_conductivity: sigma must be finite and >= 0 (region " +
                                     std::to_string(ids[r]) + ")");
  c->reg_ids.assign(ids, ids + nr);
  c->sig_l.assign(sl, sl + nr);
  c->sig_t.assign(st, st + nr);
  return TC_OK;
}

tc_status tc_set_ionic_param(tc_ctx* c, const char* name, double v) {
  if (!c || !name) return TC_EINVAL;
  double* p = nullptr;
  if (c->cfg.model == TC_ION_TT2006_EPI) p = tt_param_slot(&c->tt, name);
  if (c->cfg.model == TC_ION_MS) p = ms_param_slot(&c->ms, name);
  if (!p) return fail(c, TC_EINVAL, std::string("unknown ionic parameter ") + name);
  *p = v;
  return TC_OK;
}

tc_status tc_get_ionic_param(const tc_ctx* c, const char* name, double* v) {
  if (!c || !name || !v) return TC_EINVAL;
  tc_ctx* m = const_cast<tc_ctx*>(c);
  double* p = nullptr;
  if (c->cfg.model == TC_ION_TT2006_EPI) p = tt_param_slot(&m->tt, name);
  if (c->cfg.model == TC_ION_MS) p = ms_param_slot(&m->ms, name);
  if (!p) return TC_EINVAL;
  *v = *p;
  return TC_OK;
}

tc_status tc_add_stimulus(tc_ctx* c, int64_t m, const int32_t* nodes, double t0, double dur,
                          double amp) {
  if (!c) return TC_EINVAL;
  if (c->assembled) return fail(c, TC_ESTATE, "tc_add_stimulus after tc_assemble");
  if (!c->have_mesh) return fail(c, TC_ESTATE, "tc_add_stimulus before tc_set_mesh");
  if (m < 0 || (m > 0 && !nodes) || !(dur > 0) || !std::isfinite(amp) || !std::isfinite(t0))
    return fail(c, TC_EINVAL, "tc_add_stimulus: bad arguments");
  for (int64_t t = 0; t < m; ++t)
    if (nodes[t] < 0 || nodes[t] >= c->n)
      return fail(c, TC_EINVAL, "tc_add_stimulus: node index out of range at " + std::to_string(t));
  c->stims.push_back(Stim{std::vector<int32_t>(nodes, nodes + m), t0, dur, amp});
  return TC_OK;
}

tc_status tc_set_mms(tc_ctx* c, double k, double w1, double w2, double lam, int64_t m,
                     const int32_t* nodes) {
  if (!c) return TC_EINVAL;
  if (c->cfg.model != TC_ION_MMS) return fail(c, TC_ESTATE, "tc_set_mms needs model TC_ION_MMS");
  if (c->assembled || !c->have_mesh) return fail(c, TC_ESTATE, "tc_set_mms: call after tc_set_mesh, before tc_assemble");
  for (int64_t t = 0; t < m; ++t)
    if (nodes[t] < 0 || nodes[t] >= c->n) return fail(c, TC_EINVAL, "tc_set_mms: node out of range");
  c->mms = MMSParams{k, w1, w2, lam};
  c->dirichlet_nodes.assign(nodes, nodes + m);
  return TC_OK;
}

static double mms_w_host(const MMSParams& p, double x, double y, double t) {
  return std::exp(-p.k * t) * std::cos(p.w1 * x + p.w2 * y - p.lam * t);
}

// (re)initialise the cell state: model initial conditions everywhere
static tc_status init_state(tc_ctx* c) {
  const int64_t n = c->n, np = c->n_pad;
  std::vector<double> v(np, 0.0);
  if (c->cfg.model == TC_ION_TT2006_EPI) {
    for (int64_t i = 0; i < n; ++i) v[i] = c->tt_V0;
    std::vector<double> u((size_t)kTTStates * np, 0.0);
    for (int s = 0; s < kTTStates; ++s)
      for (int64_t i = 0; i < n; ++i) u[s * np + i] = c->tt_u0[s];
    CUDA_TRY(c, cudaMemcpyAsync(c->d_U, u.data(), u.size() * 8, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  } else if (c->cfg.model == TC_ION_MS) {
    for (int64_t i = 0; i < n; ++i) v[i] = c->ms.V_min;
    std::vector<double> u(np, 0.0);
    for (int64_t i = 0; i < n; ++i) u[i] = 1.0;
    CUDA_TRY(c, cudaMemcpyAsync(c->d_U, u.data(), u.size() * 8, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  } else {
    for (int64_t i = 0; i < n; ++i) {
      int64_t o = c->perm[i];
      v[i] = mms_w_host(c->mms, c->xyz[3 * o], c->xyz[3 * o + 1], 0.0);
    }
  }
  for (int b = 0; b < 3; ++b)
    CUDA_TRY(c, cudaMemcpyAsync(c->d_V[b], v.data(), np * 8, cudaMemcpyHostToDevice, c->stream));
  std::vector<double> unset(np, -1.0);
  CUDA_TRY(c, cudaMemcpyAsync(c->d_lat, unset.data(), np * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_lrt, unset.data(), np * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->d_act, 0, np, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->iVk = 0; c->iVkm1 = 1; c->iX = 2;
  c->k = 0;
  c->has_prev = false;
  return TC_OK;
}

// 16-bit index compression for the direct PCG pipeline
static tc_status upload_compressed(tc_ctx* c, HostSell& hs) {
  if (c->cfg.pcg_variant != 2) return TC_OK;  // variants 0 (default) and 1 (TMA) stream int32 indices
  compress_sell(hs);
  c->n_wide = hs.n_wide;
  CUDA_TRY(c, dalloc(c, &c->d_col16, (int64_t)hs.col16.size()));
  CUDA_TRY(c, dalloc(c, &c->d_kbase, (int64_t)hs.kbase.size()));
  CUDA_TRY(c, dalloc(c, &c->d_fmt, (int64_t)hs.fmt.size()));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_col16, hs.col16.data(), hs.col16.size() * 2, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_kbase, hs.kbase.data(), hs.kbase.size() * 4, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_fmt, hs.fmt.data(), hs.fmt.size(), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TC_OK;
}

static tc_status alloc_vectors(tc_ctx* c) {
  const int64_t np = c->n_pad;
  for (int b = 0; b < 3; ++b) CUDA_TRY(c, dalloc(c, &c->d_V[b], np));
  for (double** p : {&c->d_r, &c->d_z, &c->d_q, &c->d_p0, &c->d_p1, &c->d_up, &c->d_vp, &c->d_b,
                     &c->d_tmp})
    CUDA_TRY(c, dalloc(c, p, np));
  CUDA_TRY(c, dalloc(c, &c->d_dinv, np));
  return TC_OK;
}

static tc_status ensure_stats(tc_ctx* c, int64_t m) {
  if (m <= c->stats_cap) return TC_OK;
  int64_t cap = std::max<int64_t>(m, 1024);
  CUDA_TRY(c, dalloc(c, &c->d_stats, cap));
  c->stats_cap = cap;
  return TC_OK;
}

tc_status tc_assemble(tc_ctx* c) {
  if (!c) return TC_EINVAL;
  if (!c->have_mesh) return fail(c, TC_ESTATE, "tc_assemble before tc_set_mesh");
  if (c->assembled) return fail(c, TC_ESTATE, "tc_assemble called twice");
  if (c->reg_ids.empty()) return fail(c, TC_EREGION, "tc_assemble: no conductivity table");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int64_t n = c->n, E = c->E;
  // region tag -> table index
  std::map<int32_t, int32_t> rmap;
  for (size_t r = 0; r < c->reg_ids.size(); ++r) rmap[c->reg_ids[r]] = (int32_t)r;
  std::vector<int32_t> ereg(E);
  for (int64_t e = 0; e < E; ++e) {
    auto it = rmap.find(c->region[e]);
    if (it == rmap.end())
      return fail(c, TC_EREGION, "tet " + std::to_string(e) + " has region " +
                                     std::to_string(c->region[e]) + " without conductivity");
    ereg[e] = it->second;
  }
  // pattern and RCM
  std::vector<int64_t> iptr, rp;
  std::vector<int32_t> inc, col;
  build_incidence(n, E, c->tets.data(), iptr, inc);
  build_pattern(n, c->tets.data(), iptr, inc, rp, col);
  c->perm.resize(n);
  if (c->cfg.use_rcm) {
    rcm_order(n, rp, col, c->perm);
  } else {
    for (int64_t i = 0; i < n; ++i) c->perm[i] = (int32_t)i;
  }
  c->inv.resize(n);
  for (int64_t i = 0; i < n; ++i) c->inv[c->perm[i]] = (int32_t)i;
  std::vector<int64_t> rp2;
  std::vector<int32_t> col2;
  permute_csr(n, rp, col, c->perm, c->inv, rp2, col2);
  rp.clear(); rp.shrink_to_fit(); col.clear(); col.shrink_to_fit();
  std::vector<int32_t> tets2(4 * E);
  for (int64_t t = 0; t < 4 * E; ++t) tets2[t] = c->inv[c->tets[t]];
  std::vector<double> xyz2(3 * n);
  for (int64_t i = 0; i < n; ++i)
    for (int q = 0; q < 3; ++q) xyz2[3 * i + q] = c->xyz[3 * (int64_t)c->perm[i] + q];
  build_incidence(n, E, tets2.data(), iptr, inc);
  HostSell hs;
  c->nnz = rp2[n];
  csr_to_sell((int32_t)n, rp2.data(), col2.data(), hs);
  rp2.clear(); rp2.shrink_to_fit(); col2.clear(); col2.shrink_to_fit();
  c->nslices = hs.nslices;
  c->n_pad = hs.n_pad;
  c->nnz_pad = hs.slice_ptr[hs.nslices];
  // device upload
  const int64_t np = c->n_pad;
  CUDA_TRY(c, dalloc(c, &c->d_sp, (int64_t)hs.slice_ptr.size()));
  CUDA_TRY(c, dalloc(c, &c->d_col, c->nnz_pad));
  CUDA_TRY(c, dalloc(c, &c->d_A, c->nnz_pad));
  CUDA_TRY(c, dalloc(c, &c->d_K, c->nnz_pad));
  if (alloc_vectors(c) != TC_OK) return TC_ECUDA;
  c->nstates = c->cfg.model == TC_ION_TT2006_EPI ? kTTStates : (c->cfg.model == TC_ION_MS ? 1 : 0);
  CUDA_TRY(c, dalloc(c, &c->d_U, (int64_t)std::max(c->nstates, 1) * np));
  CUDA_TRY(c, dalloc(c, &c->d_act, np));
  CUDA_TRY(c, dalloc(c, &c->d_lat, np));
  CUDA_TRY(c, dalloc(c, &c->d_lrt, np));
  CUDA_TRY(c, dalloc(c, &c->d_perm, n));
  CUDA_TRY(c, dalloc(c, &c->d_inv, n));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_sp, hs.slice_ptr.data(), hs.slice_ptr.size() * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_col, hs.col.data(), hs.col.size() * 4, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_perm, c->perm.data(), n * 4, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_inv, c->inv.data(), n * 4, cudaMemcpyHostToDevice, c->stream));
  // setup-only buffers
  double *d_xyz = nullptr, *d_fib = nullptr, *d_sl = nullptr, *d_st = nullptr;
  int32_t *d_tets = nullptr, *d_ereg = nullptr, *d_inc = nullptr, *d_rowlen = nullptr, *d_err = nullptr;
  int64_t* d_iptr = nullptr;
  const size_t nr = c->reg_ids.size();
  bool ok = cudaMalloc(&d_xyz, 3 * n * 8) == cudaSuccess && cudaMalloc(&d_fib, 3 * E * 8) == cudaSuccess &&
            cudaMalloc(&d_sl, nr * 8) == cudaSuccess && cudaMalloc(&d_st, nr * 8) == cudaSuccess &&
            cudaMalloc(&d_tets, 4 * E * 4) == cudaSuccess && cudaMalloc(&d_ereg, E * 4) == cudaSuccess &&
            cudaMalloc(&d_inc, 4 * E * 4) == cudaSuccess && cudaMalloc(&d_rowlen, n * 4) == cudaSuccess &&
            cudaMalloc(&d_err, 4) == cudaSuccess && cudaMalloc(&d_iptr, (n + 1) * 8) == cudaSuccess;
  auto free_setup = [&]() {
    cudaFree(d_xyz); cudaFree(d_fib); cudaFree(d_sl); cudaFree(d_st); cudaFree(d_tets);
    cudaFree(d_ereg); cudaFree(d_inc); cudaFree(d_rowlen); cudaFree(d_err); cudaFree(d_iptr);
  };
  if (!ok) {
    free_setup();
    return fail(c, TC_ENOMEM, "tc_assemble: device allocation failed");
  }
  // fibre in the element order is unchanged by the node permutation
  cudaMemcpyAsync(d_xyz, xyz2.data(), 3 * n * 8, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(d_fib, c->fibre.data(), 3 * E * 8, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(d_sl, c->sig_l.data(), nr * 8, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(d_st, c->sig_t.data(), nr * 8, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(d_tets, tets2.data(), 4 * E * 4, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(d_ereg, ereg.data(), E * 4, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(d_inc, inc.data(), 4 * E * 4, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(d_rowlen, hs.rowlen.data(), n * 4, cudaMemcpyHostToDevice, c->stream);
  cudaMemcpyAsync(d_iptr, iptr.data(), (n + 1) * 8, cudaMemcpyHostToDevice, c->stream);
  cudaMemsetAsync(d_err, 0, 4, c->stream);
  // Dirichlet mask (MMS)
  if (c->cfg.model == TC_ION_MMS) {
    std::vector<uint8_t> dir(np, 0);
    for (int32_t o : c->dirichlet_nodes) dir[c->inv[o]] = 1;
    CUDA_TRY(c, dalloc(c, &c->d_dir, np));
    CUDA_TRY(c, dalloc(c, &c->d_xyz, 3 * np));
    CUDA_TRY(c, cudaMemcpyAsync(c->d_dir, dir.data(), np, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->d_xyz, xyz2.data(), 3 * n * 8, cudaMemcpyHostToDevice, c->stream));
  }
  AsmArgs a{};
  a.n = (int32_t)n; a.xyz = d_xyz; a.tets = d_tets; a.ereg = d_ereg; a.fibre = d_fib;
  a.sig_l = d_sl; a.sig_t = d_st; a.inc_ptr = d_iptr; a.inc = d_inc;
  a.slice_ptr = c->d_sp; a.col = c->d_col; a.rowlen = d_rowlen;
  a.A = c->d_A; a.K = c->d_K; a.dinv = c->d_dinv; a.dirichlet = c->d_dir;
  a.c_mass = c->cfg.chi * c->cfg.cm; a.c_stiff = c->cfg.theta * c->cfg.dt; a.err = d_err;
  cudaError_t le = launch_assemble(a, c->stream);
  int32_t herr = 0;
  cudaError_t se = cudaMemcpyAsync(&herr, d_err, 4, cudaMemcpyDeviceToHost, c->stream);
  cudaError_t ss = cudaStreamSynchronize(c->stream);
  free_setup();
  if (le != cudaSuccess || se != cudaSuccess || ss != cudaSuccess)
    return fail(c, TC_ECUDA, std::string("assembly kernel: ") + cudaGetErrorString(le != cudaSuccess ? le : (se != cudaSuccess ? se : ss)));
  if (herr == 1) return fail(c, TC_EDEGEN, "assembly: zero-volume element");
  if (herr == 2) return fail(c, TC_EINVAL, "assembly: pattern slot missing (internal)");
  // stimulus epochs: step windows [round(t0/dt), round((t0+dur)/dt)) (reading T1)
  {
    std::set<int64_t> cuts;
    std::vector<std::pair<int64_t, int64_t>> win;
    for (auto& s : c->stims) {
      int64_t k0 = (int64_t)std::llround(s.t0 / c->cfg.dt), k1 = (int64_t)std::llround((s.t0 + s.dur) / c->cfg.dt);
      win.push_back({k0, k1});
      cuts.insert(k0);
      cuts.insert(k1);
    }
    std::vector<int64_t> cv(cuts.begin(), cuts.end());
    std::vector<int32_t> idx;
    std::vector<double> sv;
    const double inv_chicm = 1.0 / (c->cfg.chi * c->cfg.cm);
    for (size_t q = 0; q + 1 < cv.size(); ++q) {
      std::map<int32_t, double> acc;  // new index -> summed amplitude
      for (size_t s = 0; s < c->stims.size(); ++s)
        if (win[s].first <= cv[q] && cv[q] < win[s].second)
          for (int32_t o : c->stims[s].nodes) acc[c->inv[o]] += c->stims[s].amp;
      if (acc.empty()) continue;
      Epoch ep{cv[q], cv[q + 1], (int32_t)idx.size(), (int32_t)acc.size()};
      for (auto& kv : acc) {
        idx.push_back(kv.first);
        sv.push_back(kv.second * inv_chicm);
      }
      c->epochs.push_back(ep);
    }
    if (!idx.empty()) {
      CUDA_TRY(c, dalloc(c, &c->d_stim_idx, (int64_t)idx.size()));
      CUDA_TRY(c, dalloc(c, &c->d_stim_s, (int64_t)sv.size()));
      CUDA_TRY(c, cudaMemcpyAsync(c->d_stim_idx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(c, cudaMemcpyAsync(c->d_stim_s, sv.data(), sv.size() * 8, cudaMemcpyHostToDevice, c->stream));
    }
  }
  if (upload_compressed(c, hs) != TC_OK) return TC_ECUDA;
  c->cg_grid = cg_grid_size(1, c->cfg.pcg_variant, c->nslices, c->device);
  CUDA_TRY(c, dalloc(c, &c->d_part, 2 * (int64_t)c->cg_grid));
  int32_t flags[8] = {0, 0, 0, c->cfg.fail_budget, -1, 0, 0, 0};
  CUDA_TRY(c, cudaMemcpyAsync(c->d_flags, flags, sizeof(flags), cudaMemcpyHostToDevice, c->stream));
  if (ensure_stats(c, 1024) != TC_OK) return TC_ECUDA;
  // free the big host copies no longer needed
  c->tets.clear(); c->tets.shrink_to_fit();
  c->fibre.clear(); c->fibre.shrink_to_fit();
  c->region.clear(); c->region.shrink_to_fit();
  tc_status st = init_state(c);
  if (st != TC_OK) return st;
  c->assembled = true;
  return TC_OK;
}

static IonArgs ion_args(tc_ctx* c, int do_lat) {
  IonArgs a{};
  a.n = (int32_t)c->n;
  a.stride = c->n_pad;
  a.Vk = c->d_V[c->iVk];
  a.Vkm1 = c->d_V[c->iVkm1];
  a.U = c->d_U;
  a.x0 = c->d_V[c->iX];
  a.up = c->d_up;
  a.vp = c->d_vp;
  a.act = c->d_act;
  a.lat = c->d_lat;
  a.lrt = c->d_lrt;
  a.do_lat = do_lat;
  a.has_prev = c->has_prev ? 1 : 0;
  a.t_k = c->k * c->cfg.dt;
  a.lat_thr = c->cfg.lat_threshold;
  a.lrt_thr = c->cfg.lrt_threshold;
  a.dt = c->cfg.dt;
  a.theta = c->cfg.theta;
  a.flags = c->d_flags;
  a.xyz = c->d_xyz;
  a.dirichlet = c->d_dir;
  a.t_src = c->k * c->cfg.dt + c->cfg.theta * c->cfg.dt;
  a.t_next = (c->k + 1) * c->cfg.dt;
  return a;
}

static CgArgs cg_args(tc_ctx* c) {
  CgArgs a{};
  a.slice_ptr = c->d_sp;
  a.col = c->d_col;
  a.col16 = c->d_col16;
  a.kbase = c->d_kbase;
  a.fmt = c->d_fmt;
  a.A = c->d_A;
  a.K = c->d_K;
  a.dinv = c->d_dinv;
  a.nslices = c->nslices;
  a.x = c->csr_mode ? c->d_V[0] : c->d_V[c->iX];
  a.r = c->d_r;
  a.z = c->d_z;
  a.q = c->d_q;
  a.p0 = c->d_p0;
  a.p1 = c->d_p1;
  a.up = c->d_up;
  a.vp = c->d_vp;
  a.b = c->d_b;
  a.part = c->d_part;
  a.eps_a = c->cfg.abs_tol;
  a.eps_r = c->cfg.rel_tol;
  a.max_iters = c->cfg.max_iters;
  a.rel_mode = c->cfg.rel_mode;
  a.flags = c->d_flags;
  a.step_tag = (int32_t)c->k;
  return a;
}

static cudaEvent_t ev(tc_ctx* c, size_t i) {
  while (c->evs.size() <= i) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->evs.push_back(e);
  }
  return c->evs[i];
}

tc_status tc_step(tc_ctx* c, int64_t nsteps, tc_step_stat* stats) {
  if (!c) return TC_EINVAL;
  if (!c->assembled || c->csr_mode) return fail(c, TC_ESTATE, "tc_step before tc_assemble");
  if (nsteps < 0) return fail(c, TC_EINVAL, "tc_step: negative step count");
  if (nsteps == 0) return TC_OK;
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (ensure_stats(c, nsteps) != TC_OK) return TC_ECUDA;
  const int model = c->cfg.model;
  size_t evi = 0;
  for (int64_t s = 0; s < nsteps; ++s) {
    if (c->prof) CUDA_TRY(c, cudaEventRecord(ev(c, evi++), c->stream));
    // (1) ionic step + LAT/LRT of V^k + x0, u', v'
    IonArgs ia = ion_args(c, (s > 0 && c->has_prev) ? 1 : 0);
    cudaError_t e;
    if (model == TC_ION_TT2006_EPI) e = launch_ionic_tt(ia, c->tt, c->stream);
    else if (model == TC_ION_MS) e = launch_ionic_ms(ia, c->ms, c->stream);
    else e = launch_ionic_mms(ia, c->mms, c->stream);
    CUDA_TRY(c, e);
    c->launches += 1;
    // (2) stimulus of the epoch containing step k
    for (const Epoch& ep : c->epochs)
      if (ep.k0 <= c->k && c->k < ep.k1) {
        CUDA_TRY(c, launch_stimulus(ep.m, c->d_stim_idx + ep.off, c->d_stim_s + ep.off, c->d_up,
                                    c->d_vp, c->cfg.dt, c->cfg.theta, c->d_flags, c->stream));
        c->launches += 1;
      }
    if (c->prof) CUDA_TRY(c, cudaEventRecord(ev(c, evi++), c->stream));
    // (3) RHS + Algorithm 1 in one cooperative kernel
    CgArgs ca = cg_args(c);
    ca.stat = c->d_stats + s;
    CUDA_TRY(c, launch_pcg(1, c->cfg.pcg_variant, ca, c->cg_grid, c->stream));
    c->launches += 2;  // RHS kernel + cooperative PCG kernel
    if (c->prof) CUDA_TRY(c, cudaEventRecord(ev(c, evi++), c->stream));
    // (4) V^{k-1} <- V^k <- x
    int old = c->iVkm1;
    c->iVkm1 = c->iVk;
    c->iVk = c->iX;
    c->iX = old;
    c->k += 1;
    c->has_prev = true;
  }
  // LAT/LRT of the last V (time t_k)
  if (model != TC_ION_MMS) {
    CUDA_TRY(c, launch_lat_epilogue(ion_args(c, 1), c->stream));
    c->launches += 1;
  }
  if (c->prof) CUDA_TRY(c, cudaEventRecord(ev(c, evi++), c->stream));
  std::vector<tc_step_stat> hst(nsteps);
  int32_t flags[8];
  CUDA_TRY(c, cudaMemcpyAsync(hst.data(), c->d_stats, nsteps * sizeof(tc_step_stat), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(flags, c->d_flags, sizeof(flags), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (stats) std::memcpy(stats, hst.data(), nsteps * sizeof(tc_step_stat));
  if (c->prof) {
    for (int64_t s = 0; s < nsteps; ++s) {
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, c->evs[3 * s], c->evs[3 * s + 1]);
      cudaEventElapsedTime(&b, c->evs[3 * s + 1], c->evs[3 * s + 2]);
      c->t_ion += a;
      c->t_cg += b;
      c->prof_iters += hst[s].iters;
    }
    float o = 0;
    cudaEventElapsedTime(&o, c->evs[3 * nsteps - 1], c->evs[3 * nsteps]);
    c->t_other += o;
    c->prof_steps += nsteps;
  }
  if (flags[0]) {
    if (flags[1]) return fail(c, TC_ENAN, "NaN in a PCG inner product at step " + std::to_string(flags[4]));
    return fail(c, TC_ESOLVER, "PCG did not converge for " + std::to_string(flags[3]) +
                                   " consecutive steps (last at step " + std::to_string(flags[4]) + ")");
  }
  return TC_OK;
}

tc_status tc_profile(tc_ctx* c, int enable) {
  if (!c) return TC_EINVAL;
  c->prof = enable != 0;
  return TC_OK;
}

tc_status tc_profile_read(tc_ctx* c, double out[6], int reset) {
  if (!c || !out) return TC_EINVAL;
  out[0] = c->t_ion;
  out[1] = c->t_cg;
  out[2] = c->t_other;
  out[3] = c->prof_iters;
  out[4] = c->prof_steps;
  out[5] = c->launches;
  if (reset) c->t_ion = c->t_cg = c->t_other = c->prof_iters = c->prof_steps = c->launches = 0;
  return TC_OK;
}

tc_status tc_matrix_info(const tc_ctx* c, int64_t out[6]) {
  if (!c || !out) return TC_EINVAL;
  if (!c->assembled && !c->csr_mode) return TC_ESTATE;
  out[0] = c->n;
  out[1] = c->nnz;
  out[2] = c->nnz_pad;
  out[3] = c->nslices;
  out[4] = c->cg_grid;
  out[5] = c->n_wide;
  return TC_OK;
}

// ------------------------------------------------------------------ outputs / state
static tc_status to_host_orig(tc_ctx* c, const double* dvec, double* out) {
  CUDA_TRY(c, launch_gather(c->n, c->d_inv, dvec, c->d_tmp, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(out, c->d_tmp, c->n * 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TC_OK;
}
static tc_status from_host_orig(tc_ctx* c, const double* in, double* dvec) {
  CUDA_TRY(c, cudaMemcpyAsync(c->d_tmp, in, c->n * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, launch_gather(c->n, c->d_perm, c->d_tmp, dvec, c->stream));
  return TC_OK;
}

tc_status tc_get_v(tc_ctx* c, double* v) {
  if (!c || !v) return TC_EINVAL;
  if (!c->assembled) return fail(c, TC_ESTATE, "tc_get_v before tc_assemble");
  return to_host_orig(c, c->d_V[c->iVk], v);
}

tc_status tc_get_activation(tc_ctx* c, double* lat, double* lrt) {
  if (!c) return TC_EINVAL;
  if (!c->assembled) return fail(c, TC_ESTATE, "tc_get_activation before tc_assemble");
  if (lat) { tc_status s = to_host_orig(c, c->d_lat, lat); if (s) return s; }
  if (lrt) { tc_status s = to_host_orig(c, c->d_lrt, lrt); if (s) return s; }
  return TC_OK;
}

int64_t tc_state_len(const tc_ctx* c) {
  if (!c || !c->assembled) return 0;
  return (2 + c->nstates) * c->n + 2;
}

tc_status tc_get_state(tc_ctx* c, double* buf, int64_t len) {
  if (!c || !buf) return TC_EINVAL;
  if (!c->assembled) return fail(c, TC_ESTATE, "tc_get_state before tc_assemble");
  if (len != tc_state_len(c)) return fail(c, TC_EINVAL, "tc_get_state: wrong length");
  const int64_t n = c->n;
  tc_status s;
  if ((s = to_host_orig(c, c->d_V[c->iVk], buf))) return s;
  if ((s = to_host_orig(c, c->has_prev ? c->d_V[c->iVkm1] : c->d_V[c->iVk], buf + n))) return s;
  for (int q = 0; q < c->nstates; ++q)
    if ((s = to_host_orig(c, c->d_U + q * c->n_pad, buf + (2 + q) * n))) return s;
  buf[(2 + c->nstates) * n] = (double)c->k;
  buf[(2 + c->nstates) * n + 1] = c->has_prev ? 1.0 : 0.0;
  return TC_OK;
}

tc_status tc_set_state(tc_ctx* c, const double* buf, int64_t len) {
  if (!c || !buf) return TC_EINVAL;
  if (!c->assembled) return fail(c, TC_ESTATE, "tc_set_state before tc_assemble");
  if (len != tc_state_len(c)) return fail(c, TC_EINVAL, "tc_set_state: wrong length");
  const int64_t n = c->n;
  const double kk = buf[(2 + c->nstates) * n], hp = buf[(2 + c->nstates) * n + 1];
  if (!(kk >= 0) || kk != std::floor(kk)) return fail(c, TC_EINVAL, "tc_set_state: bad step index");
  tc_status s;
  if ((s = from_host_orig(c, buf, c->d_V[c->iVk]))) return s;
  if ((s = from_host_orig(c, buf + n, c->d_V[c->iVkm1]))) return s;
  for (int q = 0; q < c->nstates; ++q)
    if ((s = from_host_orig(c, buf + (2 + q) * n, c->d_U + q * c->n_pad))) return s;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->k = (int64_t)kk;
  c->has_prev = hp != 0.0;
  return TC_OK;
}

// ------------------------------------------------------------------ minimum slice (CSR)
tc_status tc_csr_upload(tc_ctx* c, int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* col,
                        const double* val) {
  if (!c) return TC_EINVAL;
  if (c->have_mesh || c->csr_mode) return fail(c, TC_ESTATE, "tc_csr_upload: context already holds a system");
  if (n <= 0 || nnz < 0 || !rowptr || (nnz > 0 && (!col || !val))) return fail(c, TC_EINVAL, "tc_csr_upload: bad arguments");
  if (rowptr[0] != 0 || rowptr[n] != nnz) return fail(c, TC_EINVAL, "tc_csr_upload: rowptr inconsistent with nnz");
  std::vector<int64_t> rp(n + 1);
  std::vector<double> diag(n, 0.0);
  for (int32_t i = 0; i <= n; ++i) rp[i] = rowptr[i];
  for (int32_t i = 0; i < n; ++i) {
    if (rp[i + 1] < rp[i]) return fail(c, TC_EINVAL, "tc_csr_upload: rowptr decreasing at row " + std::to_string(i));
    for (int64_t t = rp[i]; t < rp[i + 1]; ++t) {
      if (col[t] < 0 || col[t] >= n) return fail(c, TC_EINVAL, "tc_csr_upload: column out of range in row " + std::to_string(i));
      if (t > rp[i] && col[t] <= col[t - 1]) return fail(c, TC_EINVAL, "tc_csr_upload: columns not strictly increasing in row " + std::to_string(i));
      if (col[t] == i) diag[i] = val[t];
    }
  }
  CUDA_TRY(c, cudaSetDevice(c->device));
  HostSell hs;
  std::vector<int64_t> slot;
  csr_to_sell(n, rp.data(), col, hs, &slot);
  std::vector<double> sv(hs.slice_ptr[hs.nslices], 0.0);
  for (int64_t t = 0; t < nnz; ++t) sv[slot[t]] = val[t];
  c->n = n;
  c->nnz = nnz;
  c->nslices = hs.nslices;
  c->n_pad = hs.n_pad;
  c->nnz_pad = hs.slice_ptr[hs.nslices];
  CUDA_TRY(c, dalloc(c, &c->d_sp, (int64_t)hs.slice_ptr.size()));
  CUDA_TRY(c, dalloc(c, &c->d_col, c->nnz_pad));
  CUDA_TRY(c, dalloc(c, &c->d_A, c->nnz_pad));
  if (alloc_vectors(c) != TC_OK) return TC_ECUDA;
  std::vector<double> dinv(c->n_pad, 0.0);
  for (int32_t i = 0; i < n; ++i) dinv[i] = diag[i] != 0.0 ? 1.0 / diag[i] : 0.0;
  CUDA_TRY(c, cudaMemcpyAsync(c->d_sp, hs.slice_ptr.data(), hs.slice_ptr.size() * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_col, hs.col.data(), hs.col.size() * 4, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_A, sv.data(), sv.size() * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_dinv, dinv.data(), dinv.size() * 8, cudaMemcpyHostToDevice, c->stream));
  if (upload_compressed(c, hs) != TC_OK) return TC_ECUDA;
  c->cg_grid = cg_grid_size(0, c->cfg.pcg_variant, c->nslices, c->device);
  CUDA_TRY(c, dalloc(c, &c->d_part, 2 * (int64_t)c->cg_grid));
  if (ensure_stats(c, 1) != TC_OK) return TC_ECUDA;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->csr_mode = true;
  c->has_diag_zero = false;
  for (int32_t i = 0; i < n; ++i) if (diag[i] == 0.0) c->has_diag_zero = true;
  return TC_OK;
}

tc_status tc_spmv(tc_ctx* c, const double* x, double* y) {
  if (!c || !x || !y) return TC_EINVAL;
  if (!c->csr_mode) return fail(c, TC_ESTATE, "tc_spmv before tc_csr_upload");
  CUDA_TRY(c, cudaMemcpyAsync(c->d_r, x, c->n * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, launch_spmv(c->d_sp, c->d_col, c->d_A, c->nslices, c->d_r, c->d_q, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(y, c->d_q, c->n * 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TC_OK;
}

tc_status tc_pcg(tc_ctx* c, const double* b, const double* x0, double* x, tc_step_stat* rep) {
  if (!c || !b || !x0 || !x) return TC_EINVAL;
  if (!c->csr_mode) return fail(c, TC_ESTATE, "tc_pcg before tc_csr_upload");
  if (c->has_diag_zero) return fail(c, TC_EINVAL, "tc_pcg: zero diagonal entry (Jacobi undefined, S:216)");
  int32_t flags[8] = {0, 0, 0, 0, -1, 0, 0, 0};
  CUDA_TRY(c, cudaMemcpyAsync(c->d_flags, flags, sizeof(flags), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_b, b, c->n * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_V[0], x0, c->n * 8, cudaMemcpyHostToDevice, c->stream));
  CgArgs ca = cg_args(c);
  ca.stat = c->d_stats;
  CUDA_TRY(c, launch_pcg(0, c->cfg.pcg_variant, ca, c->cg_grid, c->stream));
  tc_step_stat h;
  CUDA_TRY(c, cudaMemcpyAsync(&h, c->d_stats, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(x, c->d_V[0], c->n * 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(flags, c->d_flags, sizeof(flags), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (rep) *rep = h;
  if (flags[1]) return fail(c, TC_ENAN, "tc_pcg: NaN in an inner product");
  return TC_OK;
}

}  // extern "C"
