"""The N-version benchmark at PAPER.md Table 3's own settings:
20 x 7 x 3 mm slab, fibres along x, TT2006 epi, chi = 140 /mm, C_m = 0.01
uF/mm^2, sigma = (0.1334177, 0.0173515) S/m, 50 uA/mm^3 corner stimulus for
2 ms, dt = 0.005 ms, dx in {0.5, 0.2, 0.1} mm, run to 100 ms (the far corner P8
activates at ~45-50 ms).

* dx = 0.5: the GPU against the oracle over the WHOLE 20 000-step trajectory,
  V compared every step (rel-L2), LAT of every node within one dt.
* dx = 0.2 and 0.1 (58 k and 442 k nodes): GPU only, with the pins of SURVEY
  8(c) / S:482-489: every node activates, LAT monotone along the P1 -> P8
  diagonal, and the refinement gap at P8 shrinks, |LAT_0.5 - LAT_0.2| >
  |LAT_0.2 - LAT_0.1|.

`run_gpu` is shared with tools/nversion_table3.py, which writes the diagonal
LAT table to profiles/ (DESIGN.md "N-version").  Tolerances: PCG eps_a = 1e-8
(reading C5, the verification setting)."""
import numpy as np
import pytest

import meshgen as G
import oracle as O

pytestmark = pytest.mark.gpu

DT, T_END = 0.005, 100.0
STEPS = int(round(T_END / DT))
TOL = 1e-8


def table3(golden_t3, dx):
    """Mesh and inputs of the Table 3 N-version case at spacing dx."""
    t3 = golden_t3
    xyz, tets = G.slab(*t3["domain_mm"], dx)
    E = tets.shape[0]
    region = np.zeros(E, np.int32)
    fib = G.uniform_fibres(E, t3["fibre"])
    cond = {0: (t3["sigma_l_S_per_m"], t3["sigma_t_S_per_m"])}
    stim = O.Stimulus(G.nodes_in_box(xyz, (0, 0, 0), (1.5, 1.5, 1.5)), 0.0, 2.0, t3["I_stim_uA_per_mm3"])
    diag = [G.nearest_node(xyz, s * np.array(t3["domain_mm"])) for s in np.linspace(0, 1, 21)]
    return xyz, tets, region, fib, cond, [stim], diag


def run_gpu(T, golden_t3, dx, steps=STEPS):
    """Run the library to T_END; returns (lat, lrt, per-step iterations, diag, xyz)."""
    xyz, tets, region, fib, cond, stims, diag = table3(golden_t3, dx)
    t3 = golden_t3
    cfg = T.tc_config_default(dt=DT, chi=t3["chi_per_mm"], cm=t3["Cm_uF_per_mm2"], abs_tol=TOL, rel_tol=0.0,
                              max_iters=200)
    sim = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims)
    try:
        st = sim.step(steps)
        lat, lrt = sim.activation()
        return lat, lrt, st["iters"], diag, xyz
    finally:
        sim.close()


@pytest.fixture(scope="module")
def T():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2510_12011_b200 as T
    return T


def test_table3_dx05_full_trajectory_vs_oracle(T, golden):
    t3 = golden["table3_nversion"]
    xyz, tets, region, fib, cond, stims, diag = table3(t3, 0.5)
    ref = O.Monodomain(xyz, tets, region, fib, cond,
                       O.Config(dt=DT, chi=t3["chi_per_mm"], cm=t3["Cm_uF_per_mm2"], abs_tol=TOL, rel_tol=0.0,
                                max_iters=200), stims)
    cfg = T.tc_config_default(dt=DT, chi=t3["chi_per_mm"], cm=t3["Cm_uF_per_mm2"], abs_tol=TOL, rel_tol=0.0,
                              max_iters=200)
    sim = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims)
    worst, worst_k, iters_off = 0.0, -1, 0
    try:
        for k in range(STEPS):
            st = sim.step(1)
            rep = ref.step()
            v = sim.V
            rel = np.linalg.norm(v - ref.Vk) / np.linalg.norm(ref.Vk)
            if rel > worst:
                worst, worst_k = rel, k
            iters_off = max(iters_off, abs(int(st["iters"][0]) - rep.iters))
        lat, lrt = sim.activation()
    finally:
        sim.close()
    print(f"dx 0.5, {STEPS} steps: worst per-step rel-L2(V) {worst:.2e} at step {worst_k}, "
          f"max |iters diff| {iters_off}, LAT(P8) gpu {lat[diag[-1]]:.3f} oracle {ref.lat[diag[-1]]:.3f} ms")
    assert worst <= 1e-8, (worst, worst_k)
    assert iters_off <= 1
    assert (lat >= 0).all() and (ref.lat >= 0).all()            # every node activates by 100 ms
    assert np.abs(lat - ref.lat).max() <= DT + 1e-12            # LAT within one dt (north_star)
    assert np.all((lrt < 0) == (ref.lrt < 0))
    assert np.abs(lrt - ref.lrt).max() <= DT + 1e-12


def test_table3_refinement_pins(T, golden):
    t3 = golden["table3_nversion"]
    p8 = {}
    for dx in t3["dx_mm"]:
        lat, lrt, iters, diag, xyz = run_gpu(T, t3, dx)
        assert (lat >= 0).all(), dx                              # every node activates
        d = lat[diag]
        assert np.all(np.diff(d) >= 0), (dx, d)                  # monotone along P1 -> P8
        assert d[0] < d[-1]
        assert np.allclose(xyz[diag[-1]], t3["domain_mm"])       # P8 is the far corner node
        p8[dx] = d[-1]
        print(f"dx {dx}: LAT(P8) = {d[-1]:.3f} ms, mean PCG iterations {np.mean(iters):.2f}")
    g1 = abs(p8[0.5] - p8[0.2])
    g2 = abs(p8[0.2] - p8[0.1])
    assert g1 > g2, (p8, g1, g2)                                 # the refinement gap shrinks
