"""Pins of the oracle's ionic models.  The paper prints no ionic equations
(P:98 cites them), so TT2006's biological constants are "parity unpinned";
what is pinned: closed forms of the integrators (forward Euler gate, Rush-Larsen,
rapid-buffer conservation), reversal potentials (Nernst, from R, T, F only), the
Mitchell-Schaeffer threshold/fixed point, and the qualitative single-cell
behaviour of S:293-294 / S:284."""
import math

import numpy as np
import pytest
from scipy.integrate import solve_ivp

import oracle as O


# ---------------------------------------------------------------- Mitchell-Schaeffer
def test_ms_rest_fixed_point_and_dt0():
    V, U = O.ms_initial_state(4)
    In = O.ms_step(V, U, 0.05)
    assert np.array_equal(U, np.ones((1, 4))) and np.array_equal(In, np.zeros(4))
    V = np.array([-80.0, -60.0, 0.0, 15.0])
    U = np.array([[0.3, 0.5, 0.7, 0.9]])
    U0 = U.copy()
    O.ms_step(V, U, 0.0)
    assert np.array_equal(U, U0)


def test_ms_gate_closed_form():
    """v >= v_gate -> h (1 - dt/tau_close); v < v_gate -> h + dt (1-h)/tau_open."""
    p = O.ms_default_params()
    dt = 0.01
    V = np.array([-80 + 100 * 0.5, -80 + 100 * 0.05])
    U = np.array([[0.8, 0.3]])
    O.ms_step(V, U, dt, p)
    assert U[0, 0] == pytest.approx(0.8 * (1 - dt / 150.0), rel=1e-15)
    assert U[0, 1] == pytest.approx(0.3 + dt * 0.7 / 120.0, rel=1e-15)


def test_ms_threshold_is_the_unstable_fixed_point():
    """With h = 1 the reaction dv/dt = v^2(1-v)/tau_in - v/tau_out has an unstable
    fixed point at v(1-v) = tau_in/tau_out (MS 2003).  Just above it the cell
    depolarises, just below it relaxes -- pins sign and terms of I_n."""
    tin, tout = 0.3, 6.0
    vth = (1 - math.sqrt(1 - 4 * tin / tout)) / 2
    for dv, up in ((+5e-3, True), (-5e-3, False)):
        V = np.array([-80 + 100 * (vth + dv)])
        U = np.ones((1, 1))
        dt = 1e-2
        for _ in range(6000):
            In = O.ms_step(V, U, dt)
            V = V - dt * In
        assert (V[0] > -80 + 100 * 0.5) == up


def test_ms_single_cell_action_potential():
    """a suprathreshold stimulus -> v exceeds v_gate then returns below it;
    APD ~ tau_close ln(1/h_min), h_min = 4 tau_in/tau_out (MS 2003 asymptotics)."""
    dt = 0.01
    V, U = O.ms_initial_state(1)
    vs = []
    for k in range(int(600 / dt)):
        In = O.ms_step(V, U, dt)
        s = 50.0 / 1.4 if k * dt < 2.0 else 0.0
        V = V - dt * In + dt * s
        vs.append((V[0] + 80) / 100)
    vs = np.array(vs)
    t = (np.arange(len(vs)) + 1) * dt
    up = np.argmax(vs > 0.13)
    assert vs.max() > 0.9
    down = up + np.argmax(vs[up:] < 0.13)
    assert down > up
    apd = t[down] - t[up]
    assert 0.8 * 150 * math.log(1 / 0.2) < apd < 1.2 * 150 * math.log(1 / 0.2)


# ---------------------------------------------------------------- TT2006 integrator pieces
def test_rush_larsen_is_exact_linear_ode_solution():
    """dy/dt = (yinf - y)/tau solved by a library ODE integrator at 1e-12."""
    for y0, yinf, tau, dt in ((0.1, 0.9, 3.0, 0.5), (0.99, 0.01, 0.2, 0.05), (0.5, 0.5, 1.0, 1.0)):
        sol = solve_ivp(lambda t, y: (yinf - y) / tau, (0, dt), [y0], rtol=1e-12, atol=1e-14)
        assert O.rush_larsen(y0, yinf, tau, dt) == pytest.approx(sol.y[0, -1], rel=1e-10, abs=1e-13)
        assert O.rush_larsen(y0, yinf, tau, 0.0) == pytest.approx(y0, rel=1e-15)


def test_rapid_buffer_conserves_total_calcium():
    """c + B c/(c+K) increases by exactly delta (free + buffered calcium balance)."""
    rng = np.random.default_rng(0)
    for _ in range(100):
        c0 = 10 ** rng.uniform(-5, 0.7)
        B, K = 10 ** rng.uniform(-1, 1), 10 ** rng.uniform(-4, 0)
        tot0 = c0 + B * c0 / (c0 + K)
        delta = rng.uniform(-0.5, 0.5) * tot0
        c1 = O.tt_buffer(c0, delta, B, K)
        assert c1 > 0
        assert c1 + B * c1 / (c1 + K) - tot0 == pytest.approx(delta, rel=1e-9, abs=1e-15 * tot0)
    assert O.tt_buffer(3.64, 0.0, 10.0, 0.3) == pytest.approx(3.64, rel=1e-14)


def _only(names_on, p=None):
    """TT2006 parameter vector with every conductance zero except names_on."""
    p = O.tt_default_params() if p is None else p.copy()
    names = O.tt_param_names()
    for g in ("GNa", "GK1", "Gto", "GKr", "GKs", "GCaL", "GbNa", "GbCa", "GpCa", "GpK", "PNaK", "kNaCa"):
        if g not in names_on:
            p[names.index(g)] = 0.0
    return p


def test_tt_reversal_potentials_nernst():
    """Background currents are linear in V and vanish at the Nernst potential
    computed here from R, T, F and the concentrations alone."""
    _, U = O.tt_initial_state(1)
    u = U[:, 0]
    sn = O.tt_state_names()
    R, T, F = 8314.472, 310.0, 96485.3415
    RTF = R * T / F
    ENa = RTF * math.log(140.0 / u[sn.index("Nai")])
    ECa = 0.5 * RTF * math.log(2.0 / u[sn.index("Cai")])
    EKs = RTF * math.log((5.4 + 0.03 * 140.0) / (u[sn.index("Ki")] + 0.03 * u[sn.index("Nai")]))
    for g, E, slope in (("GbNa", ENa, 2.9e-4), ("GbCa", ECa, 5.92e-4)):
        p = _only({g})
        assert O.tt_current(E, u, p) == pytest.approx(0.0, abs=1e-12)
        assert O.tt_current(E + 10.0, u, p) == pytest.approx(10.0 * slope, rel=1e-12)
    p = _only({"GKs"})
    assert O.tt_current(EKs, u, p) == pytest.approx(0.0, abs=1e-12)
    EK = RTF * math.log(5.4 / u[sn.index("Ki")])
    for g in ("GK1", "Gto", "GKr", "GpK"):
        p = _only({g})
        assert O.tt_current(EK, u, p) == pytest.approx(0.0, abs=1e-12)
        assert O.tt_current(EK + 5.0, u, p) > 0 > O.tt_current(EK - 5.0, u, p)


def test_tt_dt0_identity_and_independence():
    V, U = O.tt_initial_state(6)
    rng = np.random.default_rng(1)
    V = V + rng.uniform(-5, 60, 6)
    U0 = U.copy()
    In = O.tt_step(V, U, 0.0)
    assert np.allclose(U, U0, rtol=1e-11, atol=0)   # quadratic buffer solve: cancellation ~1e-13
    for i in range(6):
        assert In[i] == pytest.approx(O.tt_current(V[i], U0[:, i]), rel=1e-14)
    # per-node independence, bit-exact and determinism
    V2, U2 = O.tt_initial_state(6)
    V2 = V2 + rng.uniform(-5, 60, 6)
    Ua, Ub, Uab = U0.copy(), U0.copy(), np.ascontiguousarray(np.hstack([U0, U0]))
    Ia = O.tt_step(V, Ua, 0.02)
    Ib = O.tt_step(V2, Ub, 0.02)
    Iab = O.tt_step(np.concatenate([V, V2]), Uab, 0.02)
    assert np.array_equal(Iab, np.concatenate([Ia, Ib]))
    assert np.array_equal(Uab, np.hstack([Ua, Ub]))


def _single_cell(dt, T, stim_amp=0.0, stim_dur=1.0):
    V, U = O.tt_initial_state(1)
    Vs = np.empty(int(round(T / dt)))
    for k in range(Vs.shape[0]):
        In = O.tt_step(V, U, dt)
        s = stim_amp if k * dt < stim_dur else 0.0
        V = V - dt * In + dt * s
        Vs[k] = V[0]
    return Vs


def test_tt_quiescence():
    """no stimulus -> V within 1 mV of rest over 500 ms."""
    Vs = _single_cell(0.02, 500.0)
    assert np.abs(Vs + 85.23).max() < 1.0


def test_tt_stimulated_action_potential():
    """stimulated -> V > 0 mV, later < -70 mV, within 500 ms."""
    dt = 0.02
    Vs = _single_cell(dt, 500.0, stim_amp=52.0, stim_dur=1.0)
    up = np.argmax(Vs > 0)
    assert Vs[up] > 0
    assert (Vs[up:] < -70).any()
    down = up + np.argmax(Vs[up:] < -70)
    assert 150 < (down - up) * dt < 450     # a ventricular-length action potential


# ---------------------------------------------------------------- CRN 1998
def _crn_only(keep):
    """CRN parameters with every membrane conductance / pump maximum zeroed except `keep`."""
    names = O.crn_param_names()
    p = O.crn_default_params()
    for g in ("gNa", "gK1", "gto", "gKr", "gKs", "gCaL", "gbNa", "gbCa", "INaKmax", "INaCamax",
              "IpCamax"):
        if g not in keep:
            p[names.index(g)] = 0.0
    return p, names


def test_crn_reversal_potentials_nernst():
    """I_Kur has no conductance parameter; with every other current off, the
    model current is I_Kur alone: zero at E_K.  Each K, Na, Ca channel current
    vanishes at its Nernst potential computed here from R, T, F and the
    concentrations only, and is linear in V with the conductance as slope."""
    _, U = O.crn_initial_state(1)
    u = U[:, 0].copy()
    sn = O.crn_state_names()
    R, T, F = 8.3143, 310.0, 96.4867
    RTF = R * T / F
    EK = RTF * math.log(5.4 / u[sn.index("Ki")])
    ENa = RTF * math.log(140.0 / u[sn.index("Nai")])
    ECa = 0.5 * RTF * math.log(1.8 / u[sn.index("Cai")])
    assert EK == pytest.approx(-86.765, abs=2e-3) and ENa == pytest.approx(67.5, abs=0.2)
    # I_Kur alone (every parameterised current off)
    p, _ = _crn_only(set())
    assert O.crn_current(EK, u, p) == pytest.approx(0.0, abs=1e-14)
    assert O.crn_current(EK + 5.0, u, p) > 0 > O.crn_current(EK - 5.0, u, p)
    # open every gate fully so that each channel current is g (V - E) x rectification
    for g in ("m", "h", "j", "oa", "oi", "xr", "xs", "d", "f", "fCa"):
        u[sn.index(g)] = 1.0
    u[sn.index("ua")] = 0.0                       # I_Kur off
    for g, E in (("gK1", EK), ("gto", EK), ("gKr", EK), ("gKs", EK), ("gNa", ENa), ("gbNa", ENa),
                 ("gbCa", ECa)):
        p, _ = _crn_only({g})
        assert O.crn_current(E, u, p) == pytest.approx(0.0, abs=1e-12), g
        assert O.crn_current(E + 5.0, u, p) > 0 > O.crn_current(E - 5.0, u, p), g
    for g, slope in (("gNa", 7.8), ("gbNa", 6.744375e-4), ("gbCa", 1.131e-3), ("gto", 0.1652),
                     ("gKs", 0.12941176)):
        p, _ = _crn_only({g})
        E = ENa if g in ("gNa", "gbNa") else (ECa if g == "gbCa" else EK)
        assert O.crn_current(E + 10.0, u, p) == pytest.approx(10.0 * slope, rel=1e-12), g


def test_crn_rush_larsen_gates_and_dt0():
    """dt = 0 leaves the state unchanged and returns I_ion(V, u); at a held V a
    gate follows the exact solution of its linear ODE: two half steps == one
    full step (Rush-Larsen is exact for frozen V and frozen other states)."""
    V, U = O.crn_initial_state(5)
    rng = np.random.default_rng(3)
    V = V + rng.uniform(-10, 80, 5)
    U0 = U.copy()
    In = O.crn_step(V, U, 0.0)
    assert np.allclose(U, U0, rtol=1e-14, atol=1e-15)   # RL: yinf - (yinf - y) rounds (gates in [0, 1])
    for i in range(5):
        assert In[i] == pytest.approx(O.crn_current(V[i], U0[:, i]), rel=1e-14)
    sn = O.crn_state_names()
    voltage_only = ["m", "h", "j", "oa", "oi", "ua", "ui", "xr", "xs", "d", "f", "w"]
    Ua, Ub = U0.copy(), U0.copy()
    O.crn_step(V, Ua, 0.2)
    O.crn_step(V, Ub, 0.1)
    O.crn_step(V, Ub, 0.1)
    for g in voltage_only:
        k = sn.index(g)
        assert np.allclose(Ua[k], Ub[k], rtol=1e-12, atol=1e-15), g


def _crn_single_cell(dt, T, stim_amp=0.0, stim_dur=2.0):
    V, U = O.crn_initial_state(1)
    Vs = np.empty(int(round(T / dt)))
    for k in range(Vs.shape[0]):
        In = O.crn_step(V, U, dt)
        s = stim_amp if k * dt < stim_dur else 0.0
        V = V - dt * In + dt * s
        Vs[k] = V[0]
    return Vs, U


def test_crn_quiescence():
    """No stimulus: the published resting state stays within 0.1 mV for 300 ms."""
    Vs, U = _crn_single_cell(0.02, 300.0)
    assert np.abs(Vs + 81.18).max() < 0.1


def test_crn_stimulated_action_potential():
    """A 2 ms, 20 pA/pF stimulus: overshoot, then repolarisation to rest with an
    atrial-length APD90 (the model's published ~300 ms at this pacing)."""
    dt = 0.02
    Vs, U = _crn_single_cell(dt, 700.0, stim_amp=20.0, stim_dur=2.0)
    pk = int(np.argmax(Vs))
    assert 10.0 < Vs[pk] < 40.0
    up = int(np.argmax(Vs > -40.0))
    v90 = Vs[pk] - 0.9 * (Vs[pk] + 81.18)
    down = pk + int(np.argmax(Vs[pk:] < v90))
    assert 250.0 < (down - up) * dt < 360.0
    assert abs(Vs[-1] + 81.18) < 1.5
    sn = O.crn_state_names()
    assert U[sn.index("Cai"), 0] > 0 and U[sn.index("Carel"), 0] > 0
