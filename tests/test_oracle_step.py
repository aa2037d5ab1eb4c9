"""Pins of the oracle's time step (Eq. 2/3)
and of the two verification problems of the paper (MMS P:214-250, N-version
P:261-289)."""
import math

import numpy as np
import pytest

import meshgen as G
import oracle as O


def _csr(Adense):
    rows, cols = np.nonzero(np.ones_like(Adense))
    rp = np.arange(0, Adense.size + 1, Adense.shape[1]).astype(np.int32)
    return rp, cols.astype(np.int32), Adense.reshape(-1).astype(float)


def test_system_matrix_examples(golden):
    w = golden["worked_examples"]
    e = w["system_matrix_1x1"]
    assert O.system_matrix(np.array([e["M"]]), np.array([e["K"]]), e["chi"], e["cm"], e["theta"],
                           e["dt"])[0] == pytest.approx(e["A"], rel=1e-15)
    e = w["system_matrix_2x2"]
    A = O.system_matrix(np.array(e["M"]).ravel(), np.array(e["K"]).ravel(), e["chi"], e["cm"],
                        e["theta"], e["dt"])
    assert np.allclose(A, np.array(e["A"]).ravel(), rtol=1e-14, atol=1e-17)
    # theta = 0 -> A = chi Cm M exactly
    assert np.array_equal(O.system_matrix(np.array([2.0]), np.array([3.0]), 140, 0.01, 0.0, 0.1),
                          np.array([140 * 0.01 * 2.0]))


def test_rhs_examples(golden):
    e = golden["worked_examples"]["rhs_1x1"]
    rp, col, M = _csr(np.array([[e["M"]]]))
    b = O.assemble_rhs(rp, col, M, np.array([e["K"]]), [e["V"]], [e["I_ion"] / e["cm"]],
                       [e["I_stim"]], e["chi"], e["cm"], e["theta"], e["dt"])
    assert b[0] == pytest.approx(e["b"], rel=1e-14)
    # V=0, currents 0 -> b = 0; theta=1, currents 0 -> b = chi Cm M V
    Md = np.array([[2.0, 1.0], [1.0, 2.0]]) / 6
    Kd = np.array([[1.0, -1.0], [-1.0, 1.0]])
    rp, col, M = _csr(Md)
    K = Kd.ravel()
    assert np.array_equal(O.assemble_rhs(rp, col, M, K, [0, 0], [0, 0], [0, 0], 140, .01, .5, .1), [0, 0])
    V = np.array([-80.0, 10.0])
    b = O.assemble_rhs(rp, col, M, K, V, [0, 0], [0, 0], 140, 0.01, 1.0, 0.1)
    assert np.allclose(b, 140 * 0.01 * Md @ V, rtol=1e-14)


def test_extrapolation_examples(golden):
    for vk, vkm1, ref in golden["worked_examples"]["extrapolation"]["cases"]:
        assert np.array_equal(O.extrapolated_guess(vk, vkm1), ref)
    assert np.array_equal(O.extrapolated_guess([1.0, 2.0], None), [1.0, 2.0])   # first step
    assert np.array_equal(O.extrapolated_guess([4.0], [4.0]), [4.0])


def test_stimulus_vector():
    s = O.Stimulus(np.array([0]), 0.0, 2.0, 50.0)
    assert np.array_equal(O.stimulus_vector([s], 20, 0.05, 3), [50.0, 0, 0])       # t = 1
    assert np.array_equal(O.stimulus_vector([s], 40, 0.05, 3), [0, 0, 0])          # t = 2 (end excl.)
    late = O.Stimulus(np.array([1]), 5.0, 1.0, 7.0)
    assert not O.stimulus_vector([late], 10, 0.05, 3).any()                         # before start
    a = O.Stimulus(np.array([2, 1]), 0.0, 1.0, 3.0)
    b = O.Stimulus(np.array([2]), 0.0, 1.0, 4.0)
    assert np.array_equal(O.stimulus_vector([a, b], 0, 0.1, 3), [0, 3.0, 7.0])     # overlaps add
    assert O.stimulus_window(O.Stimulus(np.array([0]), 0.1, 0.2, 1.0), 0.1) == (1, 3)


def test_activation_examples(golden):
    e = golden["worked_examples"]["lat_lrt"]
    lat, lrt = np.full(1, O.UNSET), np.full(1, O.UNSET)
    c = e["lat_cross"]
    O.update_activation(lat, lrt, np.array([c["Vprev"]]), np.array([c["Vnow"]]), c["t"])
    assert lat[0] == c["t"] and lrt[0] == O.UNSET
    c = e["lrt_fall"]
    O.update_activation(lat, lrt, np.array([c["Vprev"]]), np.array([c["Vnow"]]), c["t"])
    assert lrt[0] == c["t"]
    # rising through -70 does not set LRT; exactly 0 is not "positive"
    lat, lrt = np.array([5.0]), np.full(1, O.UNSET)
    O.update_activation(lat, lrt, np.array([-75.0]), np.array([-71.0]), 9.0)
    assert lrt[0] == O.UNSET
    lat = np.full(1, O.UNSET)
    O.update_activation(lat, lrt, np.array([-1.0]), np.array([0.0]), 9.0)
    assert lat[0] == O.UNSET


def _mesh(nx=6, ny=4, nz=3, dx=0.5):
    xyz, tets = G.kuhn_box(nx, ny, nz, dx)
    E = tets.shape[0]
    return xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E)


@pytest.mark.parametrize("model", ["ms", "tt2006"])
def test_zero_diffusion_reduces_to_single_cell(model):
    """sigma = 0 -> K = 0 and M cancels: every node follows
    V^{k+1} = V^k - dt I_n + dt Isv/(chi Cm) (pins U1 and the RHS algebra)."""
    xyz, tets, reg, fib = _mesh()
    n = xyz.shape[0]
    stim = O.Stimulus(np.arange(0, n, 3), 0.0, 1.0, 50.0)
    cfg = O.Config(dt=0.02, model=model, abs_tol=1e-13, rel_tol=0.0, max_iters=200)
    sim = O.Monodomain(xyz, tets, reg, fib, {0: (0.0, 0.0)}, cfg, [stim])
    V = sim.Vk.copy()
    U = sim.U.copy()
    for k in range(60):
        In = (O.tt_step if model == "tt2006" else O.ms_step)(V, U, cfg.dt)
        V = V - cfg.dt * In + cfg.dt * O.stimulus_vector([stim], k, cfg.dt, n) / (cfg.chi * cfg.cm)
        sim.step()
        assert np.abs(sim.Vk - V).max() < 1e-9
    assert sim.Vk[0] > sim.Vk[1] + 5   # stimulated nodes depolarised


def test_residual_reformulation_equals_eq3():
    """b - A x0 == A u' - K v' with u' = y - x0,
    v' = dt (V^k + theta (y - V^k)), y = V^k - dt I_n + dt Isv/(chi Cm)."""
    xyz, tets, reg, fib = _mesh(7, 5, 4, 0.3)
    rp, col, M, K = O.assemble(xyz, tets, reg, fib, {0: (0.1334177, 0.0173515)})
    n = xyz.shape[0]
    chi, cm, th, dt = 140.0, 0.01, 0.5, 0.05
    A = O.system_matrix(M, K, chi, cm, th, dt)
    Vk = G.random_vector(n, 1, -85, 30)
    Vkm1 = G.random_vector(n, 2, -85, 30)
    In = G.random_vector(n, 3, -50, 50)
    Isv = np.where(np.arange(n) % 5 == 0, 50.0, 0.0)
    b = O.assemble_rhs(rp, col, M, K, Vk, In, Isv, chi, cm, th, dt)
    x0 = O.extrapolated_guess(Vk, Vkm1)
    y = Vk - dt * In + dt * Isv / (chi * cm)
    r_ref = b - O.spmv(rp, col, A, x0)
    r_new = O.spmv(rp, col, A, y - x0) - O.spmv(rp, col, K, dt * (Vk + th * (y - Vk)))
    assert np.abs(r_new - r_ref).max() <= 1e-12 * np.abs(b).max()


def test_tissue_quiescence_and_rcm_invariance():
    """no stimulus -> |V - V_rest| < 0.5 mV over 100 ms (10+ node mesh);
    S:490: relabelling nodes (RCM order) changes nothing but the order."""
    xyz, tets, reg, fib = _mesh(4, 3, 2, 0.5)
    cfg = O.Config(dt=0.05, model="tt2006", abs_tol=1e-10, rel_tol=0.0)
    sim = O.Monodomain(xyz, tets, reg, fib, {0: (0.1334177, 0.0173515)}, cfg).run(2000)
    assert np.abs(sim.Vk + 85.23).max() < 0.5
    # RCM relabelling
    xyz, tets, reg, fib = _mesh(8, 5, 3, 0.5)
    n = xyz.shape[0]
    rp, col = O.pattern(n, tets)
    perm = O.rcm(rp, col)
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    stim = O.Stimulus(G.nodes_in_box(xyz, (0, 0, 0), (1, 1, 1)), 0.0, 2.0, 50.0)
    cfg = O.Config(dt=0.05, model="tt2006", abs_tol=1e-11, rel_tol=0.0)
    a = O.Monodomain(xyz, tets, reg, fib, {0: (0.1334177, 0.0173515)}, cfg, [stim]).run(100)
    stim_p = O.Stimulus(inv[stim.nodes], 0.0, 2.0, 50.0)
    b = O.Monodomain(xyz[perm], inv[tets].astype(np.int32), reg, fib,
                     {0: (0.1334177, 0.0173515)}, cfg, [stim_p]).run(100)
    assert np.abs(b.Vk - a.Vk[perm]).max() < 1e-8
    assert np.abs(b.lat - a.lat[perm]).max() < 1e-6


def test_mms_constant_solution_exact():
    """k = w = lambda = 0 -> w == 1, r == 0: V stays 1 to solver tolerance."""
    xyz, tets = G.unit_cube(6)
    out = O.run_mms(xyz, tets, G.box_boundary(xyz), dt=0.01, T=0.1, tol=1e-12,
                    mms=dict(k=0.0, w1=0.0, w2=0.0, lam=0.0))
    assert out["err_inf"] < 1e-10


def test_mms_matches_dense_direct_solve():
    """Brute force on a tiny input: each step's reduced system solved by numpy's
    dense LU (no PCG) reproduces the oracle trajectory (reading M3)."""
    N = 6
    xyz, tets = G.unit_cube(N)
    B = G.box_boundary(xyz)
    dt, T, th = 0.02, 0.2, 0.5
    out = O.run_mms(xyz, tets, B, dt=dt, T=T, tol=1e-13, max_iters=500)
    n = xyz.shape[0]
    E = tets.shape[0]
    rp, col, M, K = O.assemble(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E), {0: (1.0, 1.0)})
    rows = np.repeat(np.arange(n), np.diff(rp))
    Md = np.zeros((n, n)); Kd = np.zeros((n, n))
    Md[rows, col] = M; Kd[rows, col] = K
    A = Md + th * dt * Kd
    bd = np.zeros(n, bool); bd[B] = True
    I = ~bd
    X, Y = xyz[:, 0], xyz[:, 1]
    V = O.mms_w(X, Y, 0.0)
    for k in range(int(round(T / dt))):
        b = Md @ (V + dt * O.mms_r(X, Y, k * dt + th * dt)) - (1 - th) * dt * Kd @ V
        Vn = np.where(bd, O.mms_w(X, Y, (k + 1) * dt), 0.0)
        Vn[I] = np.linalg.solve(A[np.ix_(I, I)], (b - A @ Vn)[I])
        V = Vn
    assert np.abs(out["V"] - V).max() < 1e-10


def test_mms_convergence_order(golden):
    """BASELINE config 2 / S:487: L2 (M-norm) error order in [1.7, 2.3] under
    h-refinement with dt proportional to h (readings M2, T1); the errors
    themselves equal the independent direct-solve values of SURVEY 8(c) M2
    (tests/golden/mms_reference_errors.json) to their printed precision."""
    g = golden["mms_reference_errors"]
    errs = []
    for i, N in enumerate(g["N"]):
        xyz, tets = G.unit_cube(N)
        out = O.run_mms(xyz, tets, G.box_boundary(xyz), dt=0.01 * 8 / N, T=0.5, tol=1e-10)
        errs.append(out["err_M"])
        assert out["err_M"] == pytest.approx(g["err_M"][i], rel=g["rel_tol"]), (N, out["err_M"])
        assert out["err_inf"] == pytest.approx(g["err_inf"][i], rel=g["rel_tol"]), (N, out["err_inf"])
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all((orders > 1.7) & (orders < 2.3)), orders


def test_mms_source_golden_and_pde_residual(golden):
    """The source r of Eq. 8: (i) the worked value at the origin
    (tests/golden/worked_examples.json 'mms_r_origin'); (ii) r is the
    residual of the PDE it manufactures, r = dw/dt - (w_xx + w_yy) (monodomain
    with chi = C_m = 1, sigma = I, I_ion = 0), checked with central
    differences of Eq. 5's w at random points -- independent of r's formula."""
    g = golden["worked_examples"]["mms_r_origin"]
    r0 = O.mms_r(0.0, 0.0, 0.0, k=g["k"], w1=g["w1"], w2=g["w2"], lam=g["lam"])
    assert r0 == pytest.approx(g["r"], rel=1e-14)
    rng = np.random.default_rng(3)
    x, y, t = rng.uniform(0, 1, 50), rng.uniform(0, 1, 50), rng.uniform(0, 0.5, 50)
    h = 1e-4
    w = O.mms_w
    wt = (w(x, y, t + h) - w(x, y, t - h)) / (2 * h)
    lap = (w(x + h, y, t) + w(x - h, y, t) + w(x, y + h, t) + w(x, y - h, t) - 4 * w(x, y, t)) / (h * h)
    assert np.allclose(O.mms_r(x, y, t), wt - lap, rtol=0, atol=2e-5)


def test_mms_wrong_sign_breaks_order():
    """The S1 sign reading is what the MMS check pins: flipping the (1-theta) K
    sign (Eq. 2's '+') destroys convergence."""
    errs = []
    for N in (8, 16):
        xyz, tets = G.unit_cube(N)
        n, E = xyz.shape[0], tets.shape[0]
        rp, col, M, K = O.assemble(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E), {0: (1.0, 1.0)})
        dt, th = 0.01 * 8 / N, 0.5
        A = O.system_matrix(M, K, 1, 1, th, dt)
        bd = np.zeros(n, bool); bd[G.box_boundary(xyz)] = True
        rpI, cI, AII = O.csr_submatrix(rp, col, A, ~bd)
        X, Y = xyz[:, 0], xyz[:, 1]
        V = O.mms_w(X, Y, 0.0)
        for k in range(int(round(0.5 / dt))):
            b = O.spmv(rp, col, M, V + dt * O.mms_r(X, Y, k * dt + th * dt)) \
                + (1 - th) * dt * O.spmv(rp, col, K, V)          # '+' as printed in Eq. 2
            wB = np.where(bd, O.mms_w(X, Y, (k + 1) * dt), 0.0)
            xI, _ = O.pcg(rpI, cI, AII, (b - O.spmv(rp, col, A, wB))[~bd], V[~bd], 1e-10, 1e-10, 500)
            V = wB.copy(); V[~bd] = xI
        e = V - O.mms_w(X, Y, 0.5)
        errs.append(math.sqrt(e @ O.spmv(rp, col, M, e)))
    assert errs[1] > 0.5 * errs[0]      # no O(h^2) decrease


def test_nversion_qualitative(golden):
    """P:265 / S:482-489 on the Delta x = 0.5 slab (BASELINE config 1 parameters,
    run to 80 ms so the far corner activates): every node activates,
    LAT(P1) < LAT(P8), and LAT is monotone along the P1-P8 diagonal."""
    t3 = golden["table3_nversion"]
    xyz, tets = G.slab(*t3["domain_mm"], 0.5)
    E = tets.shape[0]
    stim = O.Stimulus(G.nodes_in_box(xyz, (0, 0, 0), (1.5, 1.5, 1.5)), 0.0, 2.0,
                      t3["I_stim_uA_per_mm3"])
    cfg = O.Config(dt=0.05, chi=t3["chi_per_mm"], cm=t3["Cm_uF_per_mm2"])
    sim = O.Monodomain(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E, t3["fibre"]),
                       {0: (t3["sigma_l_S_per_m"], t3["sigma_t_S_per_m"])}, cfg, [stim])
    sim.run(1600)
    assert (sim.lat >= 0).all()
    diag = [G.nearest_node(xyz, s * np.array(t3["domain_mm"])) for s in np.linspace(0, 1, 21)]
    lats = sim.lat[diag]
    assert lats[0] < lats[-1]
    assert np.all(np.diff(lats) >= 0)
    # extrapolated guess helps: iterations mostly small
    assert np.mean([r.iters for r in sim.reports]) < 20


def test_extrapolated_guess_beats_zero_guess():
    """S:590 / P:200-203: with x0 = 2V^k - V^{k-1} Algorithm 1 needs no more
    iterations than from a zero guess on >= 90 % of the steps of a propagating
    TT2006 front (same system and right-hand side, solved both ways each step)."""
    xyz, tets = G.kuhn_box(25, 9, 5, 0.5)
    E = tets.shape[0]
    stim = O.Stimulus(G.nodes_in_box(xyz, (0, 0, 0), (1.5, 1.5, 1.5)), 0.0, 2.0, 50.0)
    cfg = O.Config(dt=0.05)
    sim = O.Monodomain(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E),
                       {0: (0.1334177, 0.0173515)}, cfg, [stim])
    better = total = 0
    for _ in range(240):
        In = sim.ionic(sim.Vk, sim.U.copy())   # updates the copy in place; sim.step redoes it
        Isv = O.stimulus_vector(sim.stimuli, sim.k, cfg.dt, sim.n)
        b = O.assemble_rhs(sim.rowptr, sim.col, sim.M, sim.K, sim.Vk, In, Isv, cfg.chi, cfg.cm, cfg.theta, cfg.dt)
        _, rz = O.pcg(sim.rowptr, sim.col, sim.A, b, np.zeros(sim.n), cfg.abs_tol, cfg.rel_tol, cfg.max_iters)
        rep = sim.step()
        if sim.k > 1:                 # step 0 has no V^{k-1}: x0 = V^0
            total += 1
            better += rep.iters <= rz.iters
    assert total > 200 and better >= 0.9 * total, (better, total)
