"""Parity at BASELINE.json's FULL sizes, in the launch configuration bench.py
times (same inputs, config, engine and preroll):

* sampled outputs the oracle computes one by one: rows of the assembled
  A = chi Cm M + theta dt K and K (element by element, oracle `tet_local`),
  and the per-node ionic update u^{k+1} (oracle `tt_step` / `ms_step` /
  `crn_step` on the sampled nodes);
* a property that holds at any size: the V^{k+1} the GPU returns solves
  Eq. 3 to Algorithm 1's tolerance, with b built on the host from
  the literal Eq. 3 formula and the oracle's ionic currents;
* configs[2] (442 k nodes), a 1.28 M-node TT2006 slab and a 416 k-node BiV
  against the whole oracle step from injected GPU states, on the multi-slice
  PCG kernels (variants 0, 1 and the automatic choice).
"""
import math

import numpy as np
import pytest

import bench
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


def _bench_sim(T, name, preroll=None):
    """The context exactly as bench.py builds and prerolls it."""
    w = bench.WORKLOADS[name]
    xyz, tets, stims, region, fibre = bench.make_inputs(w)
    cfg = T.tc_config_default(dt=w["dt"], model=w["model"], chi=bench.CHI, cm=bench.CM, abs_tol=1e-5,
                              rel_tol=1e-5, max_iters=100, use_rcm=1, pcg_variant=-1, partitions=1)
    sim = T.Monodomain(xyz, tets, region, fibre, {0: bench.SIGMA, 1: bench.SIGMA}, cfg, stims)
    sim.step(w["preroll"] if preroll is None else preroll)
    return w, sim, xyz, tets, region, fibre


def _split_state(s, n, ns):
    return s[:n].copy(), s[n:2 * n].copy(), s[2 * n:(2 + ns) * n].reshape(ns, n).copy()


@pytest.mark.parametrize("name", ["slab20M_ms", "biv3M_tt", "sphere2.6M_ms"])
def test_fullsize_assembly_rows_sampled(T, name):
    w, sim, xyz, tets, region, fibre = _bench_sim(T, name, preroll=0)
    try:
        n = xyz.shape[0]
        rng = np.random.default_rng(11)
        sample = np.unique(np.concatenate([rng.choice(n, 48, replace=False), [0, n - 1]]))
        x = rng.uniform(-1.0, 1.0, n)
        yA = T.tc_apply(sim.ctx, 0, x)
        yK = T.tc_apply(sim.ctx, 1, x)
        hit = np.nonzero(np.isin(tets, sample).any(axis=1))[0]
        accA = {int(i): [0.0, 0.0] for i in sample}      # value, sum of |terms|
        accK = {int(i): [0.0, 0.0] for i in sample}
        cm, st = w.get("chi", bench.CHI) * bench.CM, 0.5 * w["dt"]
        for e in hit:
            nodes = tets[e]
            f = (1.0, 0.0, 0.0) if fibre is None else fibre[e]
            sig = O.conductivity_tensor(f, *bench.SIGMA)
            Me, Ke, _ = (O.tri_local if tets.shape[1] == 3 else O.tet_local)(xyz[nodes], sig)
            for a, i in enumerate(nodes):
                if int(i) in accA:
                    ta = (cm * Me[a] + st * Ke[a]) * x[nodes]
                    tk = Ke[a] * x[nodes]
                    accA[int(i)][0] += ta.sum()
                    accA[int(i)][1] += np.abs(ta).sum()
                    accK[int(i)][0] += tk.sum()
                    accK[int(i)][1] += np.abs(tk).sum()
        for i in sample:
            a, sa = accA[int(i)]
            k, sk = accK[int(i)]
            assert abs(yA[i] - a) <= 1e-12 * sa + 1e-300, (i, yA[i], a)
            assert abs(yK[i] - k) <= 1e-12 * sk + 1e-300, (i, yK[i], k)
    finally:
        sim.close()


@pytest.mark.parametrize("name", ["slab10M_tt", "slab10M_crn", "slab20M_ms", "biv3M_tt", "sphere2.6M_ms"])
def test_fullsize_ionic_update_sampled(T, name):
    """u^{k+1} at sampled nodes after one full-size step equals the oracle's
    per-node update of (V^k, u^k) read back from the GPU."""
    w, sim, xyz, tets, region, fibre = _bench_sim(T, name)
    try:
        n = xyz.shape[0]
        ns = {"tt2006": 18, "crn": 20, "ms": 1}[w["model"]]
        Vk, _, U0 = _split_state(sim.get_state(), n, ns)
        sim.step(1)
        _, _, U1 = _split_state(sim.get_state(), n, ns)
        rng = np.random.default_rng(5)
        # sampled nodes, biased to the propagating front (largest |dV| states)
        front = np.argsort(-np.abs(Vk - np.median(Vk)))[:256]
        sample = np.unique(np.concatenate([rng.choice(n, 256, replace=False), front]))
        u = np.ascontiguousarray(U0[:, sample])
        step = {"tt2006": O.tt_step, "crn": O.crn_step, "ms": O.ms_step}[w["model"]]
        step(Vk[sample], u, w["dt"])
        assert np.allclose(U1[:, sample], u, rtol=1e-10, atol=1e-14)
    finally:
        sim.close()


def _kuhn_diag(T, sim, dims):
    """diag(A) of a Kuhn-grid system with 8 probes: nodes coloured by the parity
    of their grid indices never share a row (every stencil offset changes some
    index by one)."""
    nx, ny, nz = dims
    idx = np.arange(nx * ny * nz)
    i, j, k = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    colour = (i % 2) + 2 * (j % 2) + 4 * (k % 2)
    d = np.zeros(idx.shape[0])
    for c in range(8):
        e = (colour == c).astype(np.float64)
        y = T.tc_apply(sim.ctx, 0, e)
        d[colour == c] = y[colour == c]
    return d


def test_fullsize_step_solves_eq3_to_tolerance(T):
    """20 M-node MS slab, one step in the timing window: with b from the literal
    Eq. 3 (oracle ionic currents, M x = (A x - theta dt K x)/(chi Cm)) and
    z = D^-1 (b - A V^{k+1}), ||z|| meets Algorithm 1's absolute test and agrees
    with the norm the GPU reported."""
    name = "slab20M_ms"
    w, sim, xyz, tets, region, fibre = _bench_sim(T, name)
    try:
        n = xyz.shape[0]
        Vk, _, U0 = _split_state(sim.get_state(), n, 1)
        st = sim.step(1)
        Vn = sim.V
        dt, th, chicm = w["dt"], 0.5, bench.CHI * bench.CM
        In = O.ms_step(Vk, np.ascontiguousarray(U0), dt)
        y = Vk - dt * In                                     # stimulus has ended (t > 2 ms)
        b = (T.tc_apply(sim.ctx, 0, y) - th * dt * T.tc_apply(sim.ctx, 1, y)
             - (1.0 - th) * dt * T.tc_apply(sim.ctx, 1, Vk))
        r = b - T.tc_apply(sim.ctx, 0, Vn)
        d = _kuhn_diag(T, sim, w["dims"])
        z = np.linalg.norm(r / d)
        assert bool(st["converged"][0])
        assert z < 1e-5 * 1.01, z
        assert z == pytest.approx(float(st["znorm"][0]), rel=1e-3, abs=1e-9)
    finally:
        sim.close()


def _warps_per_cta():
    return 16            # kCgWarps (csrc/internal.h: 512-thread PCG CTAs)


# Whole-oracle-step parity on the grid engine's multi-slice paths (VERDICT r01
# item 1): the automatic variant and the forced direct (0) and TMA-staged (1)
# kernels at sizes where every warp walks several SELL slices (variant 0's
# grid-stride slice loop, variant 1's TMA ring wrapping), on
#   * configs[2] (N-version dx 0.1 mm, 442 401 nodes, the bench's preroll),
#   * a 1.28 M-node TT2006 slab (160 x 100 x 80, planar front; the automatic
#     choice is variant 0 at > 4 slices per resident warp -- the kernel the
#     north-star / configs[4] bench lines time),
#   * the BiV recipe at h = 0.65 mm (416 k nodes, permuted numbering, rotating
#     fibres, two regions).
# One step from the GPU's own state, injected into the oracle (SURVEY 8c "one-
# step parity from injected states at all sizes"): rel-L2(V) <= 1e-8
# (north_star), every cell state to 1e-9, PCG iterations within 1.
_MULTI = {
    "configs2": dict(w="nversion_dx0.1_tt", dims=None, preroll=500),
    "slab1.28M_tt": dict(w="slab10M_tt", dims=(160, 100, 80), preroll=300),
    "biv416k_tt": dict(w="biv3M_tt", dims=0.65, preroll=300),
}


@pytest.mark.parametrize("name", ["slab10M_tt", "slab20M_ms", "slab10M_crn", "biv3M_tt", "sphere2.6M_ms"])
def test_fullsize_whole_oracle_step(T, name):
    """The bench's own configurations at FULL size -- the north-star 10 M-node
    TT2006 slab, the default 20 M-node MS slab (configs[4]), the 10 M CRN slab
    (f4), the 3 M BiV (configs[3]) and the 2.6 M-node triangle sphere (f2) -- built and
    prerolled exactly as bench.py times them: one step from the GPU's state
    against the WHOLE oracle step (assembly, ionic update, Eq. 3 RHS,
    Algorithm 1) on the same state: rel-L2(V) <= 1e-8 (north_star), every cell
    state to 1e-9, PCG iterations within 1."""
    w, sim, xyz, tets, region, fibre = _bench_sim(T, name)
    try:
        n = xyz.shape[0]
        ns = {"tt2006": 18, "crn": 20, "ms": 1}[w["model"]]
        s = sim.get_state()
        Vk, Vkm1, U = _split_state(s, n, ns)
        k = int(round(s[-2]))
        stg = sim.step(1)
        v = sim.V
        _, _, U1 = _split_state(sim.get_state(), n, ns)
        sim.close()
        sim = None
        del s
        E = tets.shape[0]
        stims = bench.make_inputs(w)[2]
        ref = O.Monodomain(xyz, tets, np.zeros(E, np.int32) if region is None else region,
                           G.uniform_fibres(E) if fibre is None else fibre, {0: bench.SIGMA, 1: bench.SIGMA},
                           O.Config(dt=w["dt"], model=w["model"], chi=bench.CHI, cm=bench.CM, abs_tol=1e-5,
                                    rel_tol=1e-5, max_iters=100),
                           [O.Stimulus(*st_) for st_ in stims])
        ref.set_state(Vk, Vkm1, U, k)
        rep = ref.step()
        rel = np.linalg.norm(v - ref.Vk) / np.linalg.norm(ref.Vk)
        print(f"{name}: {n} nodes, step {k}, iters {int(stg['iters'][0])} vs {rep.iters}, rel-L2 {rel:.2e}")
        assert abs(int(stg["iters"][0]) - rep.iters) <= 1
        assert rel <= 1e-8, rel
        assert np.allclose(U1, ref.U, rtol=1e-9, atol=1e-14)
    finally:
        if sim is not None:
            sim.close()


@pytest.mark.parametrize("case,variant,parts,peer", [("configs2", -1, 1, 1), ("configs2", 0, 1, 1),
                                                     ("configs2", 1, 1, 1), ("slab1.28M_tt", -1, 1, 1),
                                                     ("slab1.28M_tt", 1, 1, 1), ("biv416k_tt", -1, 1, 1),
                                                     ("biv416k_tt", 0, 1, 1), ("configs2", 6, 1, 1),
                                                     ("slab1.28M_tt", -1, 4, 1), ("slab1.28M_tt", -1, 3, 0),
                                                     ("biv416k_tt", -1, 4, 1)])
def test_multislice_full_oracle_step(T, case, variant, parts, peer):
    """(parts > 1: the multi-GPU PCG emulated on one GPU -- interior-first row
    blocks, halos overlapped with the interior slices, peer kernels or split
    phases -- at a size where every part is still multi-slice.)"""
    c = _MULTI[case]
    w = bench.WORKLOADS[c["w"]]
    xyz, tets, stims, region, fibre = bench.make_inputs(w, c["dims"])
    E = tets.shape[0]
    cfg = T.tc_config_default(dt=w["dt"], model=w["model"], chi=bench.CHI, cm=bench.CM, abs_tol=1e-5,
                              rel_tol=1e-5, max_iters=100, use_rcm=1, pcg_variant=variant, partitions=parts,
                              peer=peer)
    sim = T.Monodomain(xyz, tets, region, fibre, {0: bench.SIGMA, 1: bench.SIGMA}, cfg, stims)
    try:
        info = T.tc_matrix_info(sim.ctx)
        assert T.tc_engine_info(sim.ctx)["engine"] == "grid"
        used = info["pcg_variant"]
        if parts > 1:
            assert info["partitions"] == parts and info["path"] == ("peer" if peer else "split")
            assert T.tc_validate(sim.ctx) > 0
        if variant >= 0:
            assert used == variant
        spw = info["nslices"] / (info["pcg_grid"] * _warps_per_cta())
        if used in (0, 1) and parts == 1:
            assert spw > 1.0, spw          # the multi-slice loop / ring wrap is exercised
        sim.step(c["preroll"])
        n = xyz.shape[0]
        ns = {"tt2006": 18, "crn": 20, "ms": 1}[w["model"]]
        s = sim.get_state()
        Vk, Vkm1, U = _split_state(s, n, ns)
        k = int(round(s[-2]))
        assert k == c["preroll"]
        assert (Vk > 0).any() and (Vk < -80).any()       # a front is in the domain
        ref = O.Monodomain(xyz, tets, np.zeros(E, np.int32) if region is None else region,
                           G.uniform_fibres(E) if fibre is None else fibre,
                           {0: bench.SIGMA, 1: bench.SIGMA},
                           O.Config(dt=w["dt"], model=w["model"], chi=bench.CHI, cm=bench.CM,
                                    abs_tol=1e-5, rel_tol=1e-5, max_iters=100),
                           [O.Stimulus(*st_) for st_ in stims])
        ref.set_state(Vk, Vkm1, U, k)
        rep = ref.step()
        stg = sim.step(1)
        v = sim.V
        assert abs(int(stg["iters"][0]) - rep.iters) <= 1, (int(stg["iters"][0]), rep.iters)
        rel = np.linalg.norm(v - ref.Vk) / np.linalg.norm(ref.Vk)
        assert rel <= 1e-8, rel
        _, _, U1 = _split_state(sim.get_state(), n, ns)
        assert np.allclose(U1, ref.U, rtol=1e-9, atol=1e-14)
        print(f"{case} variant {used} parts {parts} ({info['path']}): {n} nodes, {spw:.2f} slices/warp, iters {int(stg['iters'][0])} "
              f"vs {rep.iters}, rel-L2 {rel:.2e}")
    finally:
        sim.close()


@pytest.mark.parametrize("name", ["slab20M_ms", "slab10M_tt"])
def test_fullsize_activation_front_is_planar_and_ordered(T, name):
    """The bench's planar stimulus (x <= 0.3 mm) on a fibre-aligned slab drives a
    front along x: every activated node's LAT is non-decreasing in x
    along each grid line, the activated region is a prefix of every line, the
    front position varies by at most one node across (y, z), and the front
    moves (LAT grows along x).  (LAT at one x is NOT equal across (y, z): the
    boundary nodes' smaller mass rows bend the front by ~0.1 ms.)"""
    w, sim, xyz, tets, region, fibre = _bench_sim(T, name, preroll=0)
    try:
        sim.step(700)                                   # 7 ms: the front is well inside the slab
        lat, _ = sim.activation()
        nx, ny, nz = w["dims"]
        L = lat.reshape(nz, ny, nx)
        act = L >= 0
        assert act[:, :, 0].all() and not act[:, :, -1].any()
        first_off = act.argmin(axis=2)                  # first non-activated x index on every line
        assert np.all(act.sum(axis=2) == first_off)     # activated set is a prefix along x
        assert first_off.max() - first_off.min() <= 1   # planar front (within one node)
        dt = w["dt"]
        m = int(first_off.min())
        sub = L[:, :, :m]
        assert np.all(np.diff(sub, axis=2) >= -1e-12)   # ordered along x
        assert sub[:, :, m - 1].min() > sub[:, :, 0].max() + 10 * dt   # the front travelled
    finally:
        sim.close()
