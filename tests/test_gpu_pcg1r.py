"""GPU parity of PCG variant 6, the single-reduction (Chronopoulos-Gear) form of
the Jacobi PCG (optional, "not the paper's algorithm, so it sits
behind a flag and is parity-checked").

It computes Algorithm 1's iterates in exact arithmetic with both
inner products of an iteration in one grid reduction, so it is compared with
the oracle's literal Algorithm 1 (oracle.pcg / oracle.Monodomain) at the same
tolerances as the other variants, except that the iteration count may differ
by one where rounding moves ||z|| across the stopping threshold."""
import numpy as np
import pytest

import meshgen as G
import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2510_12011_b200 as T
    return T


def _fem_matrix(nx=41, ny=15, nz=7, dx=0.5, permute=False):
    xyz, tets = G.kuhn_box(nx, ny, nz, dx)
    if permute:
        xyz, tets, _ = G.permute_nodes(xyz, tets)
    E = tets.shape[0]
    rp, col, M, K = O.assemble(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E),
                               {0: (0.1334177, 0.0173515)})
    return rp, col, O.system_matrix(M, K, 140.0, 0.01, 0.5, 0.05)


@pytest.mark.parametrize("case,rel_mode", [("fem", 0), ("fem_perm", 1), ("spd", 0), ("big", 0), ("tiny", 0)])
def test_pcg1r_solve_parity(T, case, rel_mode):
    if case == "fem":
        rp, col, A = _fem_matrix()
    elif case == "fem_perm":
        rp, col, A = _fem_matrix(permute=True)
    elif case == "big":
        rp, col, A = _fem_matrix(101, 36, 16, 0.2)   # 58k rows, many CTAs, ragged tail
    elif case == "tiny":
        rp, col, A, _ = G.random_spd_csr(33, density=0.2, seed=4)   # one slice + 1 row
    else:
        rp, col, A, _ = G.random_spd_csr(777, density=0.03, seed=8)
    n = rp.shape[0] - 1
    b = G.random_vector(n, seed=1)
    x0 = G.random_vector(n, seed=2, lo=-0.1, hi=0.1)
    cfg = T.tc_config_default(abs_tol=1e-12, rel_tol=1e-3 if rel_mode else 0.0, rel_mode=rel_mode,
                              max_iters=500, pcg_variant=6)
    ctx = T.tc_create(cfg)
    try:
        T.tc_csr_upload(ctx, rp, col, A)
        x, rep = T.tc_pcg(ctx, b, x0)
        xe, rep0 = T.tc_pcg(ctx, O.spmv(rp, col, A, x0), x0)   # zero residual: x0, <= 1 iteration
    finally:
        T.tc_destroy(ctx)
    xr, rr = O.pcg(rp, col, A, b, x0, 1e-12, 1e-3 if rel_mode else 0.0, 500, rel_mode)
    assert abs(rep["iters"] - rr.iters) <= 1 and rep["converged"] == rr.converged
    assert np.abs(x - xr).max() <= 1e-10 * np.abs(xr).max()
    assert rep0["iters"] <= 1 and np.abs(xe - x0).max() <= 1e-10


def test_pcg1r_max_iters_zero_and_budget(T):
    """max_iters = 0: x = x0, not converged (Alg. 1 with an empty loop)."""
    rp, col, A = _fem_matrix(21, 8, 5)
    n = rp.shape[0] - 1
    b = G.random_vector(n, seed=3)
    x0 = G.random_vector(n, seed=4)
    ctx = T.tc_create(T.tc_config_default(abs_tol=1e-12, rel_tol=0.0, max_iters=0, pcg_variant=6))
    try:
        T.tc_csr_upload(ctx, rp, col, A)
        x, rep = T.tc_pcg(ctx, b, x0)
    finally:
        T.tc_destroy(ctx)
    assert rep["iters"] == 0 and not rep["converged"]
    assert np.array_equal(x, x0)


def _slab_case(model, nx=21, ny=8, nz=5, dx=0.5, permute=False, seed=0):
    xyz, tets = G.kuhn_box(nx, ny, nz, dx)
    if permute:
        xyz, tets, _ = G.permute_nodes(xyz, tets, seed=seed + 1)
    E = tets.shape[0]
    fib = G.random_fibres(E, seed) if seed else G.uniform_fibres(E)
    stim = O.Stimulus(G.nodes_in_box(xyz, (0, 0, 0), (1.5, 1.5, 1.5)), 0.0, 2.0, 50.0)
    return xyz, tets, np.zeros(E, np.int32), fib, {0: (0.1334177, 0.0173515)}, [stim]


@pytest.mark.parametrize("model,permute", [("tt2006", True), ("ms", False), ("crn", True)])
def test_pcg1r_step_trajectory_parity(T, model, permute):
    """120 steps through the stimulus window: V per step within rel-L2 1e-8 of the
    oracle's Algorithm 1, LAT within one dt (the same bar as the other variants)."""
    xyz, tets, region, fib, cond, stims = _slab_case(model, permute=permute, seed=3 if permute else 0)
    dt = 0.05
    ref = O.Monodomain(xyz, tets, region, fib, cond, O.Config(dt=dt, model=model, abs_tol=1e-8, rel_tol=0.0), stims)
    cfg = T.tc_config_default(dt=dt, model=model, abs_tol=1e-8, rel_tol=0.0, pcg_variant=6, engine="grid")
    sim = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims)
    try:
        assert T.tc_matrix_info(sim.ctx)["pcg_variant"] == 6
        for k in range(120):
            st = sim.step(1)
            rep = ref.step()
            rel = np.linalg.norm(sim.V - ref.Vk) / np.linalg.norm(ref.Vk)
            assert rel <= 1e-8, (k, rel)
            assert abs(int(st["iters"][0]) - rep.iters) <= 1
        lat, _ = sim.activation()
        assert np.all((lat < 0) == (ref.lat < 0))
        assert np.abs(lat - ref.lat).max() <= dt + 1e-12
    finally:
        sim.close()


def test_pcg1r_mms_dirichlet_matches_oracle(T):
    """Dirichlet rows (D^-1 = 0, u = t = sigma = 0 there) on the manufactured
    solution (readings M2/M3): V at T equals the oracle's to 1e-8."""
    for N in (8, 16):
        xyz, tets = G.unit_cube(N)
        B = G.box_boundary(xyz)
        dt = 0.01 * 8 / N
        E = tets.shape[0]
        cfg = T.tc_config_default(dt=dt, model="mms", chi=1.0, cm=1.0, abs_tol=1e-10, rel_tol=1e-10,
                                  max_iters=1000, pcg_variant=6, engine="grid")
        sim = T.Monodomain(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E), {0: (1.0, 1.0)}, cfg,
                           mms=(1.0, np.pi, np.pi, np.pi, B))
        try:
            st = sim.step(int(round(0.5 / dt)))
            v = sim.V
        finally:
            sim.close()
        assert st["converged"].all()
        out = O.run_mms(xyz, tets, B, dt=dt, T=0.5, tol=1e-10)
        assert np.abs(v - out["V"]).max() <= 1e-8, N


def test_pcg1r_cohort_large_members(T):
    """Variant 6 on the shared-GPU cohort path (each large member's RHS + single-
    reduction kernel shaped for its share of the GPU, on its own stream): every
    member against its own oracle run (Algorithm 1), 30 steps through the upstroke."""
    members, refs = [], []
    try:
        for dims, seed in (((61, 23, 9), 3), ((57, 25, 10), 5)):
            xyz, tets, region, fib, cond, stims = _slab_case("tt2006", *dims, 0.5, permute=True, seed=seed)
            refs.append(O.Monodomain(xyz, tets, region, fib, cond,
                                     O.Config(dt=0.05, model="tt2006", abs_tol=1e-8, rel_tol=0.0), stims))
            cfg = T.tc_config_default(dt=0.05, model="tt2006", abs_tol=1e-8, rel_tol=0.0, pcg_variant=6,
                                      engine="grid")
            members.append(T.Monodomain(xyz, tets, region, fib, cond, cfg, stims))
        co = T.Cohort(members)
        try:
            for c in range(3):
                stats = co.step(10)
                for m, (sim, ref) in enumerate(zip(members, refs)):
                    reps = [ref.step() for _ in range(10)]
                    rel = np.linalg.norm(sim.V - ref.Vk) / np.linalg.norm(ref.Vk)
                    assert rel <= 1e-8, (m, c, rel)
                    for a, b in zip(stats[m], reps):
                        assert abs(int(a["iters"]) - b.iters) <= 1
        finally:
            co.close()
    finally:
        for s in members:
            s.close()
