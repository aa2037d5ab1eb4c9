"""CPU ORACLE of the TorchCor monodomain step (arXiv 2510.12011) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_2510_12011_b200``) and never imports it.

Heavy loops (assembly, RCM, SpMV, PCG, ionic models) are plain C in
``oracle.c`` (fp64, ``-O2 -ffp-contract=off``); the per-step vector algebra of
Eq. (2)/(3) is written out below with numpy so that it can be read against the
paper line by line.  Citations: ``P:n`` = PAPER.md line n, ``S:n`` = SPEC.md line
n; the readings of ambiguous passages (S1, U1, I1-I5, C1-C5, T1, M2, N2 ...) are
listed in DESIGN.md.

Parity pins: tests/test_oracle_*.py.  "parity unpinned": the biological
constants / initial conditions of TT2006 (the paper prints none; only the
qualitative behaviour of S:293-294 and mathematical invariants are pinned).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_EINVAL, OR_EDEGEN, OR_ENAN, OR_ENOMEM, OR_EREGION, OR_EFIBRE = range(7)


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, no FMA contraction, no fast-math;
    -fopenmp for the independent per-row / per-node loops)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math",
                               "-fopenmp", "-fPIC", "-shared", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_L = None


def _lib():
    global _L
    if _L is None:
        L = C.CDLL(build())
        P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.or_conductivity_tensor.argtypes = [P, D, D, P]
        L.or_tet_local.argtypes = [P, P, P, P, P]
        L.or_pattern.argtypes = [I64, I64, P, P, P]
        L.or_pattern.restype = I64
        L.or_pattern_k.argtypes = [I64, I64, C.c_int, P, P, P]
        L.or_pattern_k.restype = I64
        L.or_assemble_k.argtypes = [I64, P, I64, C.c_int, P, P, P, I32, P, P, P, P, P, P, P]
        L.or_tri_local.argtypes = [P, P, P, P, P]
        L.or_assemble.argtypes = [I64, P, I64, P, P, P, I32, P, P, P, P, P, P, P]
        L.or_rcm.argtypes = [I32, P, P, P]
        L.or_set_threads.argtypes = [I32]
        L.or_set_threads.restype = None
        L.or_max_threads.restype = I32
        L.or_spmv.argtypes = [I32, P, P, P, P, P]
        L.or_spmv.restype = None
        L.or_pcg.argtypes = [I32, P, P, P, P, P, I32, D, D, I32, I32, P, P, P, P, P]
        L.or_ms_default_params.argtypes = [P]
        L.or_ms_default_params.restype = None
        L.or_ms_step.argtypes = [I64, P, P, D, P, P]
        L.or_ms_step.restype = None
        L.or_tt_default_params.argtypes = [P]
        L.or_tt_default_params.restype = None
        L.or_tt_initial_state.argtypes = [P]
        L.or_tt_initial_state.restype = D
        L.or_tt_step.argtypes = [I64, P, P, D, P, P]
        L.or_tt_step.restype = None
        L.or_tt_current.argtypes = [D, P, P]
        L.or_tt_current.restype = D
        L.or_tt_buffer.argtypes = [D, D, D, D]
        L.or_tt_buffer.restype = D
        L.or_rush_larsen.argtypes = [D, D, D, D]
        L.or_rush_larsen.restype = D
        L.or_tt_nparams.restype = I32
        L.or_tt_nstates.restype = I32
        L.or_tt_param_name.argtypes = [I32]
        L.or_tt_param_name.restype = C.c_char_p
        L.or_tt_state_name.argtypes = [I32]
        L.or_tt_state_name.restype = C.c_char_p
        L.or_crn_default_params.argtypes = [P]
        L.or_crn_default_params.restype = None
        L.or_crn_initial_state.argtypes = [P]
        L.or_crn_initial_state.restype = D
        L.or_crn_step.argtypes = [I64, P, P, D, P, P]
        L.or_crn_step.restype = None
        L.or_crn_current.argtypes = [D, P, P]
        L.or_crn_current.restype = D
        L.or_crn_nparams.restype = I32
        L.or_crn_nstates.restype = I32
        L.or_crn_param_name.argtypes = [I32]
        L.or_crn_param_name.restype = C.c_char_p
        L.or_crn_state_name.argtypes = [I32]
        L.or_crn_state_name.restype = C.c_char_p
        _L = L
    return _L


def set_threads(k: int) -> None:
    """Threads for the oracle's per-row / per-node loops (results are bitwise
    independent of k; 1 = sequential)."""
    max_threads()
    _lib().or_set_threads(int(k))


_DEFAULT_THREADS = None


def max_threads() -> int:
    """The OpenMP default (all host cores unless OMP_NUM_THREADS says otherwise),
    captured before any set_threads call."""
    global _DEFAULT_THREADS
    if _DEFAULT_THREADS is None:
        _DEFAULT_THREADS = int(_lib().or_max_threads())
    return _DEFAULT_THREADS


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class OracleError(RuntimeError):
    pass


def _check(st: int, what: str):
    if st != OR_OK:
        raise OracleError(f"{what}: oracle status {st}")


# --------------------------------------------------------------------------
# FEM building blocks
# --------------------------------------------------------------------------
def conductivity_tensor(f, sigma_l: float, sigma_t: float) -> np.ndarray:
    """sigma_t I + (sigma_l - sigma_t) f f^T, f normalised (DESIGN A13)."""
    f = _f64(f)
    out = np.zeros(9)
    _check(_lib().or_conductivity_tensor(_p(f), sigma_l, sigma_t, _p(out)), "conductivity")
    return out.reshape(3, 3)


def tet_local(x, sigma):
    """Local P1 mass / stiffness matrices of one tet; returns (Me, Ke, |e|)."""
    x = _f64(x).reshape(12)
    s = _f64(sigma).reshape(9)
    Me, Ke, vol = np.zeros(16), np.zeros(16), np.zeros(1)
    _check(_lib().or_tet_local(_p(x), _p(s), _p(Me), _p(Ke), _p(vol)), "tet_local")
    return Me.reshape(4, 4), Ke.reshape(4, 4), float(vol[0])


def tri_local(x, sigma):
    """Local P1 mass / stiffness matrices of one triangle in 3-D; returns (Me, Ke, |e|)."""
    x = _f64(x).reshape(9)
    s = _f64(sigma).reshape(9)
    Me, Ke, area = np.zeros(9), np.zeros(9), np.zeros(1)
    _check(_lib().or_tri_local(_p(x), _p(s), _p(Me), _p(Ke), _p(area)), "tri_local")
    return Me.reshape(3, 3), Ke.reshape(3, 3), float(area[0])


def pattern(n: int, tets):
    """CSR pattern of M u K: (i,j) iff an element holds both.
    tets: (E, 4) tetrahedra or (E, 3) surface triangles."""
    tets = _i32(tets)
    E, k = tets.shape
    rowptr = np.zeros(n + 1, np.int32)
    nnz = _lib().or_pattern_k(n, E, k, _p(tets), _p(rowptr), None)
    if nnz < 0:
        raise OracleError("pattern: connectivity index out of range")
    col = np.zeros(nnz, np.int32)
    _lib().or_pattern_k(n, E, k, _p(tets), _p(rowptr), _p(col))
    return rowptr, col


def assemble(xyz, tets, region, fibre, conductivities: dict):
    """Global (rowptr, col, M, K) by element-order scatter-add;
    tets (E,4) tetrahedra or (E,3) triangles embedded in 3-D.

    ``conductivities`` maps region tag -> (sigma_l, sigma_t) in S/m."""
    xyz, tets, region, fibre = _f64(xyz), _i32(tets), _i32(region), _f64(fibre)
    n = xyz.shape[0]
    rowptr, col = pattern(n, tets)
    ids = _i32(sorted(conductivities))
    sl = _f64([conductivities[int(i)][0] for i in ids])
    st = _f64([conductivities[int(i)][1] for i in ids])
    M = np.zeros(col.shape[0])
    K = np.zeros(col.shape[0])
    _check(_lib().or_assemble_k(n, _p(xyz), tets.shape[0], tets.shape[1], _p(tets), _p(region),
                                _p(fibre), len(ids), _p(ids), _p(sl), _p(st), _p(rowptr),
                                _p(col), _p(M), _p(K)), "assemble")
    return rowptr, col, M, K


def rcm(rowptr, col) -> np.ndarray:
    """Reverse Cuthill-McKee permutation, perm[new] = old (S:146 ties)."""
    rowptr, col = _i32(rowptr), _i32(col)
    n = rowptr.shape[0] - 1
    perm = np.zeros(n, np.int32)
    _check(_lib().or_rcm(n, _p(rowptr), _p(col), _p(perm)), "rcm")
    return perm


def spmv(rowptr, col, val, x) -> np.ndarray:
    """y = A x, CSR row-wise in fp64."""
    rowptr, col, val, x = _i32(rowptr), _i32(col), _f64(val), _f64(x)
    y = np.zeros(rowptr.shape[0] - 1)
    _lib().or_spmv(rowptr.shape[0] - 1, _p(rowptr), _p(col), _p(val), _p(x), _p(y))
    return y


@dataclass
class SolveReport:
    iters: int
    znorm: float
    converged: bool
    trace: np.ndarray | None = None


def pcg(rowptr, col, val, b, x0, eps_a: float, eps_r: float, max_iters: int,
        rel_mode: int = 0, jacobi: bool = True, trace: bool = False):
    """Algorithm 1 with Jacobi preconditioner. -> (x, SolveReport)."""
    rowptr, col, val, b, x0 = _i32(rowptr), _i32(col), _f64(val), _f64(b), _f64(x0)
    n = rowptr.shape[0] - 1
    x = np.zeros(n)
    it, zn, cv = C.c_int32(0), C.c_double(0.0), C.c_int32(0)
    tr = np.zeros(max_iters + 1) if trace else None
    st = _lib().or_pcg(n, _p(rowptr), _p(col), _p(val), _p(b), _p(x0), int(jacobi),
                       eps_a, eps_r, max_iters, rel_mode, _p(x), C.byref(it), C.byref(zn),
                       C.byref(cv), _p(tr) if trace else None)
    _check(st, "pcg")
    rep = SolveReport(it.value, zn.value, bool(cv.value),
                      tr[: it.value + 1].copy() if trace else None)
    return x, rep


# --------------------------------------------------------------------------
# Ionic models (readings I1-I5 in DESIGN.md)
# --------------------------------------------------------------------------
MS_PARAM_NAMES = ["tau_in", "tau_out", "tau_open", "tau_close", "v_gate", "V_min", "V_max"]


def ms_default_params() -> np.ndarray:
    p = np.zeros(7)
    _lib().or_ms_default_params(_p(p))
    return p


def ms_initial_state(n: int, params=None):
    """Rest: v = 0 (V = V_min), h = 1."""
    p = ms_default_params() if params is None else _f64(params)
    return np.full(n, p[5]), np.ones((1, n))


def ms_step(V, U, dt: float, params=None) -> np.ndarray:
    """Forward-Euler gate step at (V^k, h^k); returns I_n(V^k, h^{k+1}) (mV/ms).

    U is (1, n) and updated in place."""
    p = ms_default_params() if params is None else _f64(params)
    V = _f64(V)
    assert U.dtype == np.float64 and U.flags.c_contiguous
    In = np.zeros(V.shape[0])
    _lib().or_ms_step(V.shape[0], _p(V), _p(U), dt, _p(p), _p(In))
    return In


def tt_param_names() -> list[str]:
    L = _lib()
    return [L.or_tt_param_name(k).decode() for k in range(L.or_tt_nparams())]


def tt_state_names() -> list[str]:
    L = _lib()
    return [L.or_tt_state_name(k).decode() for k in range(L.or_tt_nstates())]


def tt_default_params() -> np.ndarray:
    p = np.zeros(_lib().or_tt_nparams())
    _lib().or_tt_default_params(_p(p))
    return p


def tt_initial_state(n: int):
    """(V0 (n,), U (18, n)) -- epicardial initial conditions (reading I4)."""
    u = np.zeros(_lib().or_tt_nstates())
    v0 = _lib().or_tt_initial_state(_p(u))
    return np.full(n, v0), np.ascontiguousarray(np.repeat(u[:, None], n, axis=1))


def tt_step(V, U, dt: float, params=None) -> np.ndarray:
    """TT2006 step: U (18, n) updated in place; returns I_n(V^k, u^{k+1}) (mV/ms)."""
    p = tt_default_params() if params is None else _f64(params)
    V = _f64(V)
    assert U.dtype == np.float64 and U.flags.c_contiguous and U.shape[0] == 18
    In = np.zeros(V.shape[0])
    _lib().or_tt_step(V.shape[0], _p(V), _p(U), dt, _p(p), _p(In))
    return In


def tt_current(V: float, u, params=None) -> float:
    p = tt_default_params() if params is None else _f64(params)
    return _lib().or_tt_current(V, _p(_f64(u)), _p(p))


def crn_param_names() -> list[str]:
    """Courtemanche-Ramirez-Nattel 1998 (reading I6)."""
    L = _lib()
    return [L.or_crn_param_name(k).decode() for k in range(L.or_crn_nparams())]


def crn_state_names() -> list[str]:
    L = _lib()
    return [L.or_crn_state_name(k).decode() for k in range(L.or_crn_nstates())]


def crn_default_params() -> np.ndarray:
    p = np.zeros(_lib().or_crn_nparams())
    _lib().or_crn_default_params(_p(p))
    return p


def crn_initial_state(n: int):
    """-> V0 (n,), U0 (20, n) state-major."""
    u = np.zeros(_lib().or_crn_nstates())
    v0 = _lib().or_crn_initial_state(_p(u))
    return np.full(n, v0), np.repeat(u[:, None], n, axis=1).copy()


def crn_step(V, U, dt: float, params=None) -> np.ndarray:
    """Advance U (20, n) in place (RL gates, FE concentrations); -> I_n(V, U^{k+1})."""
    V = _f64(V)
    p = crn_default_params() if params is None else _f64(params)
    In = np.zeros(V.shape[0])
    _lib().or_crn_step(V.shape[0], _p(V), _p(U), dt, _p(p), _p(In))
    return In


def crn_current(V: float, u, params=None) -> float:
    p = crn_default_params() if params is None else _f64(params)
    return _lib().or_crn_current(V, _p(_f64(u)), _p(p))


def tt_buffer(c_old, delta, B, K) -> float:
    return _lib().or_tt_buffer(c_old, delta, B, K)


def rush_larsen(y, yinf, tau, dt) -> float:
    return _lib().or_rush_larsen(y, yinf, tau, dt)


# --------------------------------------------------------------------------
# The time step, Eq. (2)/(3) and P:200-203
# --------------------------------------------------------------------------
def system_matrix(M, K, chi, cm, theta, dt):
    """A = chi C_m M + theta dt K (Eq. 3), on the shared pattern."""
    return chi * cm * _f64(M) + theta * dt * _f64(K)


def assemble_rhs(rowptr, col, M, K, Vk, In, Isv, chi, cm, theta, dt):
    """b = chi M (C_m V^k - dt I_ion + dt I_stim) - (1-theta) dt K V^k  (Eq. 3).

    Units reading U1: the ionic model returns I_n per capacitance (mV/ms), so the
    per-area current is I_ion = C_m I_n; the stimulus is volumetric (uA/mm^3,
    P:280) and enters as dt M Isv (i.e. chi I_stim = Isv).  Sign reading S1:
    minus, as printed in Eq. (3)."""
    Vk, In, Isv = _f64(Vk), _f64(In), _f64(Isv)
    MV = spmv(rowptr, col, M, chi * (cm * Vk - dt * cm * In) + dt * Isv)
    KV = spmv(rowptr, col, K, Vk)
    return MV - (1.0 - theta) * dt * KV


def extrapolated_guess(Vk, Vkm1):
    """x0 = 2 V^k - V^{k-1}; at the first step V^{-1} := V^k."""
    Vk = _f64(Vk)
    if Vkm1 is None:
        return Vk.copy()
    return 2.0 * Vk - _f64(Vkm1)


@dataclass
class Stimulus:
    """P:72 / S:327-330: node set, start (ms), duration (ms), intensity (uA/mm^3)."""
    nodes: np.ndarray
    start: float
    duration: float
    amplitude: float


def stimulus_window(s: Stimulus, dt: float):
    """Integer step window [k_start, k_end): k_start = round(start/dt),
    k_end = round((start+duration)/dt) (reading T1)."""
    return int(round(s.start / dt)), int(round((s.start + s.duration) / dt))


def stimulus_vector(stims, k: int, dt: float, n: int):
    """Isv_i = sum of intensities of stimuli active at step k."""
    Isv = np.zeros(n)
    for s in stims:
        k0, k1 = stimulus_window(s, dt)
        if k0 <= k < k1:
            np.add.at(Isv, np.asarray(s.nodes, np.int64), s.amplitude)
    return Isv


UNSET = -1.0


def update_activation(lat, lrt, Vprev, Vnow, t, lat_thr=0.0, lrt_thr=-70.0):
    """LAT: first time V > 0; LRT: first later time V < -70 with dV/dt < 0."""
    new_lat = (lat == UNSET) & (Vnow > lat_thr)
    new_lrt = (lat != UNSET) & (lrt == UNSET) & (Vnow < lrt_thr) & (Vnow - Vprev < 0)
    lat[new_lat] = t
    lrt[new_lrt] = t


@dataclass
class Config:
    """Simulation settings."""
    dt: float
    theta: float = 0.5
    chi: float = 140.0        # mm^-1 (Table 3)
    cm: float = 0.01          # uF/mm^2 (Table 3; unit reading U1)
    abs_tol: float = 1e-5
    rel_tol: float = 1e-5
    max_iters: int = 100
    rel_mode: int = 0         # reading C1: 0 literal consecutive, 1 initial
    fail_budget: int = 3
    model: str = "tt2006"     # "tt2006" | "ms" | "crn"
    params: np.ndarray | None = None


class SolverAbort(RuntimeError):
    pass


class Monodomain:
    """Oracle simulator: Eq. (2) operator split + Eq. (3) + Algorithm 1.

    The order of one step is S:390 / P:139: (1) ionic step, (2) stimulus,
    (3) right-hand side, (4) extrapolated guess + PCG, (5) LAT/LRT."""

    def __init__(self, xyz, tets, region, fibre, conductivities, cfg: Config,
                 stimuli=(), V0=None, U0=None):
        self.cfg = cfg
        self.rowptr, self.col, self.M, self.K = assemble(xyz, tets, region, fibre, conductivities)
        self.n = xyz.shape[0]
        self.A = system_matrix(self.M, self.K, cfg.chi, cfg.cm, cfg.theta, cfg.dt)
        self.stimuli = list(stimuli)
        if cfg.model == "tt2006":
            self.params = tt_default_params() if cfg.params is None else _f64(cfg.params)
            v, u = tt_initial_state(self.n)
        elif cfg.model == "ms":
            self.params = ms_default_params() if cfg.params is None else _f64(cfg.params)
            v, u = ms_initial_state(self.n, self.params)
        elif cfg.model == "crn":
            self.params = crn_default_params() if cfg.params is None else _f64(cfg.params)
            v, u = crn_initial_state(self.n)
        else:
            raise ValueError(cfg.model)
        self.Vk = v if V0 is None else _f64(V0).copy()
        self.U = u if U0 is None else np.ascontiguousarray(U0, dtype=np.float64).copy()
        self.Vkm1 = None
        self.k = 0
        self.lat = np.full(self.n, UNSET)
        self.lrt = np.full(self.n, UNSET)
        self.reports: list[SolveReport] = []
        self._fails = 0

    def ionic(self, V, U):
        if self.cfg.model == "tt2006":
            return tt_step(V, U, self.cfg.dt, self.params)
        if self.cfg.model == "crn":
            return crn_step(V, U, self.cfg.dt, self.params)
        return ms_step(V, U, self.cfg.dt, self.params)

    def step(self) -> SolveReport:
        c = self.cfg
        In = self.ionic(self.Vk, self.U)                              # Eq. (2) row 1
        Isv = stimulus_vector(self.stimuli, self.k, c.dt, self.n)
        b = assemble_rhs(self.rowptr, self.col, self.M, self.K, self.Vk, In, Isv,
                         c.chi, c.cm, c.theta, c.dt)                   # Eq. (3)
        x0 = extrapolated_guess(self.Vk, self.Vkm1)
        x, rep = pcg(self.rowptr, self.col, self.A, b, x0, c.abs_tol, c.rel_tol,
                     c.max_iters, c.rel_mode)                          # Alg. 1
        self.Vkm1, self.Vk = self.Vk, x
        self.k += 1
        update_activation(self.lat, self.lrt, self.Vkm1, self.Vk, self.k * c.dt)
        self.reports.append(rep)
        if not np.all(np.isfinite(self.Vk)):
            raise SolverAbort(f"NaN in V at step {self.k}")
        self._fails = 0 if rep.converged else self._fails + 1
        if self._fails >= c.fail_budget:
            raise SolverAbort(f"PCG failed {self._fails} consecutive steps at step {self.k}")
        return rep

    def run(self, nsteps: int):
        for _ in range(nsteps):
            self.step()
        return self

    # state injection (one-step parity at any size)
    def set_state(self, Vk, Vkm1, U, k: int):
        self.Vk = _f64(Vk).copy()
        self.Vkm1 = None if Vkm1 is None else _f64(Vkm1).copy()
        self.U = np.ascontiguousarray(U, dtype=np.float64).copy()
        self.k = int(k)


# --------------------------------------------------------------------------
# Manufactured solution (readings M2, T1, M3)
# --------------------------------------------------------------------------
def mms_w(x, y, t, k=1.0, w1=math.pi, w2=math.pi, lam=math.pi):
    """w = e^{-kt} cos(w1 x + w2 y - lambda t)  (Eq. 5)."""
    return np.exp(-k * t) * np.cos(w1 * x + w2 * y - lam * t)


def mms_r(x, y, t, k=1.0, w1=math.pi, w2=math.pi, lam=math.pi):
    """r = e^{-kt}[-k cos(.) + lambda sin(.)] + (w1^2 + w2^2) w   (Eq. 8)."""
    ph = w1 * x + w2 * y - lam * t
    return (np.exp(-k * t) * (-k * np.cos(ph) + lam * np.sin(ph))
            + (w1 * w1 + w2 * w2) * mms_w(x, y, t, k, w1, w2, lam))


def csr_submatrix(rowptr, col, val, keep):
    """Rows/columns of the CSR matrix where keep is True, renumbered (plain indexing)."""
    keep = np.asarray(keep, bool)
    n = keep.shape[0]
    newidx = -np.ones(n, np.int64)
    newidx[keep] = np.arange(int(keep.sum()))
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    m = keep[rows] & keep[col]
    r2, c2, v2 = newidx[rows[m]], newidx[col[m]], val[m]
    rp = np.zeros(int(keep.sum()) + 1, np.int64)
    np.add.at(rp, r2 + 1, 1)
    return np.cumsum(rp).astype(np.int32), c2.astype(np.int32), v2.astype(np.float64)


def run_mms(xyz, tets, boundary, dt, T, theta=0.5, tol=1e-10, max_iters=1000,
            mms=dict(), return_history=False):
    """Diffusion with source on [0,1]^3, chi = C_m = 1, sigma = I.

    Per step: b = M (V^k + dt r(., t_k + theta dt)) - (1-theta) dt K V^k (reading T1);
    Dirichlet V_B = w(t_{k+1}) by elimination: the PCG of Algorithm 1 runs on the
    reduced interior system A_II V_I = b_I - A_IB w_B (reading M3).
    Returns V at T, and the M-norm and max-norm errors vs w(., T)."""
    n = xyz.shape[0]
    E = tets.shape[0]
    rowptr, col, M, K = assemble(xyz, tets, np.zeros(E, np.int32),
                                 np.tile([1.0, 0.0, 0.0], (E, 1)), {0: (1.0, 1.0)})
    A = system_matrix(M, K, 1.0, 1.0, theta, dt)
    B = np.zeros(n, bool)
    B[np.asarray(boundary)] = True
    I = ~B
    rpI, cI, AII = csr_submatrix(rowptr, col, A, I)
    # A_IB as a (rows I, cols B) product: zero the interior columns.
    X, Y = xyz[:, 0], xyz[:, 1]
    nsteps = int(round(T / dt))
    V = mms_w(X, Y, 0.0, **mms)
    Vprev = None
    iters = []
    hist = []
    for k in range(nsteps):
        tk = k * dt
        src = mms_r(X, Y, tk + theta * dt, **mms)
        b = spmv(rowptr, col, M, V + dt * src) - (1.0 - theta) * dt * spmv(rowptr, col, K, V)
        wB = np.where(B, mms_w(X, Y, tk + dt, **mms), 0.0)
        bI = (b - spmv(rowptr, col, A, wB))[I]
        x0 = extrapolated_guess(V, Vprev)[I]
        xI, rep = pcg(rpI, cI, AII, bI, x0, tol, tol, max_iters, 0)
        Vnew = wB.copy()
        Vnew[I] = xI
        Vprev, V = V, Vnew
        iters.append(rep.iters)
        if return_history:
            hist.append(V.copy())
    e = V - mms_w(X, Y, nsteps * dt, **mms)
    errM = math.sqrt(float(e @ spmv(rowptr, col, M, e)))
    out = dict(V=V, err_M=errM, err_inf=float(np.abs(e).max()), iters=iters)
    if return_history:
        out["history"] = hist
    return out
