"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element, on seeded synthetic inputs.

Tolerances: SpMV 1e-13 relative to the row's |A||x| sum
(FMA contraction + summation order); PCG x to 1e-10 relative at tight tolerance
and identical iteration counts; one monodomain step V to rel-L2 <= 1e-8
(north_star); LAT within one dt."""
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
    A = O.system_matrix(M, K, 140.0, 0.01, 0.5, 0.05)
    return rp, col, A


@pytest.mark.parametrize("case", ["fem", "fem_perm", "spd_ragged", "one_row", "33_rows"])
def test_spmv_parity(T, case):
    if case.startswith("fem"):
        rp, col, A = _fem_matrix(permute=case == "fem_perm")
    elif case == "spd_ragged":
        rp, col, A, _ = G.random_spd_csr(1000, density=0.02, seed=3)
    elif case == "one_row":
        rp, col, A = np.array([0, 1], np.int32), np.array([0], np.int32), np.array([2.5])
    else:
        rp, col, A, _ = G.random_spd_csr(33, density=0.3, seed=4)
    n = rp.shape[0] - 1
    x = G.random_vector(n, seed=7, lo=-90, hi=40)
    ctx = T.tc_create(T.tc_config_default())
    try:
        T.tc_csr_upload(ctx, rp, col, A)
        y = T.tc_spmv(ctx, x)
    finally:
        T.tc_destroy(ctx)
    yref = O.spmv(rp, col, A, x)
    scale = O.spmv(rp, col, np.abs(A), np.abs(x)) + 1e-300
    assert np.all(np.abs(y - yref) <= 1e-13 * scale)


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 5, -1])
@pytest.mark.parametrize("case,rel_mode", [("fem", 0), ("fem_perm", 1), ("spd", 0), ("big", 0)])
def test_pcg_parity(T, case, rel_mode, variant):
    if case == "fem":
        rp, col, A = _fem_matrix()
    elif case == "fem_perm":
        rp, col, A = _fem_matrix(permute=True)
    elif case == "big":
        rp, col, A = _fem_matrix(101, 36, 16, 0.2)   # 58k rows, many CTAs, ragged tail
    else:
        rp, col, A, _ = G.random_spd_csr(777, density=0.03, seed=8)
    n = rp.shape[0] - 1
    b = G.random_vector(n, seed=1)
    x0 = G.random_vector(n, seed=2, lo=-0.1, hi=0.1)
    cfg = T.tc_config_default(abs_tol=1e-12, rel_tol=1e-3 if rel_mode else 0.0, rel_mode=rel_mode,
                              max_iters=500, pcg_variant=variant)
    ctx = T.tc_create(cfg)
    try:
        T.tc_csr_upload(ctx, rp, col, A)
        x, rep = T.tc_pcg(ctx, b, x0)
        # zero initial residual -> 0 iterations, x = x0 (reading C4)
        xe, rep0 = T.tc_pcg(ctx, O.spmv(rp, col, A, x0), x0)
    finally:
        T.tc_destroy(ctx)
    xr, rr = O.pcg(rp, col, A, b, x0, 1e-12, 1e-3 if rel_mode else 0.0, 500, rel_mode)
    assert rep["iters"] == rr.iters and rep["converged"] == rr.converged
    assert np.abs(x - xr).max() <= 1e-10 * np.abs(xr).max()
    assert rep0["iters"] <= 1 and np.abs(xe - x0).max() <= 1e-10


def _slab_case(model, nx=21, ny=8, nz=5, dx=0.5, permute=False, seed=0):
    xyz, tets = G.kuhn_box(nx, ny, nz, dx)
    if permute:
        xyz, tets, _ = G.permute_nodes(xyz, tets, seed=seed + 1)
    E = tets.shape[0]
    region = np.zeros(E, np.int32)
    fib = G.random_fibres(E, seed) if seed else G.uniform_fibres(E)
    cond = {0: (0.1334177, 0.0173515)}
    stim = O.Stimulus(G.nodes_in_box(xyz, (0, 0, 0), (1.5, 1.5, 1.5)), 0.0, 2.0, 50.0)
    return xyz, tets, region, fib, cond, [stim]


@pytest.mark.parametrize("model,permute,rcm,variant", [("ms", False, 1, 0), ("tt2006", False, 1, 0),
                                                        ("tt2006", True, 1, 0), ("tt2006", True, 0, 1),
                                                        ("ms", True, 0, 1), ("tt2006", False, 1, 1),
                                                        ("tt2006", True, 1, 2), ("crn", False, 1, 0),
                                                        ("crn", True, 1, 1), ("tt2006", True, 1, 3),
                                                        ("tt2006", True, 1, 4), ("crn", False, 1, 4),
                                                        ("tt2006", True, 1, 5), ("ms", False, 0, 5), ("crn", True, 1, 5)])
def test_step_trajectory_parity(T, model, permute, rcm, variant):
    """Multi-step trajectory through the real stimulus window (upstroke), V per
    step within rel-L2 1e-8, LAT within one dt, per-step iteration counts equal."""
    xyz, tets, region, fib, cond, stims = _slab_case(model, permute=permute, seed=3 if permute else 0)
    dt = 0.05
    ref = O.Monodomain(xyz, tets, region, fib, cond, O.Config(dt=dt, model=model, abs_tol=1e-8, rel_tol=0.0), stims)
    cfg = T.tc_config_default(dt=dt, model=model, abs_tol=1e-8, rel_tol=0.0, use_rcm=rcm,
                              pcg_variant=variant, engine="grid")
    sim = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims)
    try:
        for k in range(120):
            st = sim.step(1)
            rep = ref.step()
            v = sim.V
            rel = np.linalg.norm(v - ref.Vk) / np.linalg.norm(ref.Vk)
            assert rel <= 1e-8, (k, rel)
            assert abs(int(st["iters"][0]) - rep.iters) <= 1
        lat, lrt = sim.activation()
        assert np.all((lat < 0) == (ref.lat < 0))
        assert np.abs(lat - ref.lat).max() <= dt + 1e-12
        # state vector round trip (original order)
        s = sim.get_state()
        n = xyz.shape[0]
        assert np.allclose(s[:n], ref.Vk, rtol=0, atol=1e-8 * np.abs(ref.Vk).max())
        U = s[2 * n:-2].reshape(-1, n)
        assert np.allclose(U, ref.U, rtol=1e-8, atol=1e-14)
    finally:
        sim.close()


@pytest.mark.parametrize("peer,variant", [(1, -1), (1, 4), (0, -1)])
@pytest.mark.parametrize("model,nparts,permute", [("ms", 2, False), ("tt2006", 3, True), ("tt2006", 2, False),
                                                  ("ms", 5, True)])
def test_partitioned_trajectory_parity(T, model, nparts, permute, peer, variant):
    """Row-block partitions on one GPU (split-phase PCG, device-copy halos,
    in-order scalar sums; or the peer-memory kernels with the latency (auto, 4)
    or direct (0) row product): same trajectory as the oracle and as 1 partition."""
    xyz, tets, region, fib, cond, stims = _slab_case(model, 25, 9, 5, permute=permute, seed=2 if permute else 0)
    dt = 0.05
    ref = O.Monodomain(xyz, tets, region, fib, cond, O.Config(dt=dt, model=model, abs_tol=1e-8, rel_tol=0.0), stims)
    cfg = T.tc_config_default(dt=dt, model=model, abs_tol=1e-8, rel_tol=0.0, partitions=nparts, check_every=3,
                              peer=peer, pcg_variant=variant)
    sim = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims)
    try:
        info = T.tc_matrix_info(sim.ctx)
        assert info["partitions"] == nparts and info["ghosts"] > 0
        assert info["path"] == ("peer" if peer else "split")
        if peer:   # emulated partitions: direct kernel unless the latency variant is asked for
            assert info["pcg_variant"] == (0 if variant < 0 else variant)
        for k in range(80):
            st = sim.step(1)
            rep = ref.step()
            rel = np.linalg.norm(sim.V - ref.Vk) / np.linalg.norm(ref.Vk)
            assert rel <= 1e-8, (k, rel)
            assert abs(int(st["iters"][0]) - rep.iters) <= 1
        lat, _ = sim.activation()
        assert np.abs(lat - ref.lat).max() <= dt + 1e-12
        s = sim.get_state()
        n = xyz.shape[0]
        assert np.allclose(s[2 * n:-2].reshape(-1, n), ref.U, rtol=1e-8, atol=1e-14)
    finally:
        sim.close()


@pytest.mark.parametrize("peer", [1, 0])
def test_nccl_path_world1_parity(T, peer):
    """The NCCL paths (communicator of one rank; peer kernel or split phases) against the oracle."""
    xyz, tets, region, fib, cond, stims = _slab_case("tt2006", 21, 8, 5)
    dt = 0.05
    ref = O.Monodomain(xyz, tets, region, fib, cond, O.Config(dt=dt, abs_tol=1e-8, rel_tol=0.0), stims)
    cfg = T.tc_config_default(dt=dt, abs_tol=1e-8, rel_tol=0.0, peer=peer)
    try:
        uid = T.tc_nccl_unique_id()
    except T.TcError:
        pytest.skip("NCCL not loadable")
    sim = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims, comm=(0, 1, uid))
    try:
        if peer:   # one partition per process: the automatic choice takes the latency variant
            assert T.tc_matrix_info(sim.ctx)["pcg_variant"] == 4
        for k in range(60):
            sim.step(1)
            ref.step()
            assert np.linalg.norm(sim.V - ref.Vk) / np.linalg.norm(ref.Vk) <= 1e-8
        lat, _ = sim.activation()
        assert np.abs(lat - ref.lat).max() <= dt + 1e-12
    finally:
        sim.close()


@pytest.mark.parametrize("peer_parts,engine", [(1, "grid"), (1, "cluster"), (3, "auto")])
def test_biv_mesh_trajectory_parity(T, peer_parts, engine):
    """Synthetic BiV recipe (configs[3]) at coarse h: unstructured (jittered, randomly
    relabelled) mesh, two regions, rule-based rotating fibres, five stimulus spheres."""
    m = G.biv(2.5)
    stims = [O.Stimulus(nodes, 0.0, 2.0, 50.0) for nodes in G.biv_stimuli(m, radius=3.0)]
    cond = {0: (0.1334177, 0.0173515), 1: (0.1334177, 0.0173515)}
    dt = 0.05
    ref = O.Monodomain(m["xyz"], m["tets"], m["region"], m["fibre"], cond,
                       O.Config(dt=dt, abs_tol=1e-8, rel_tol=0.0), stims)
    cfg = T.tc_config_default(dt=dt, abs_tol=1e-8, rel_tol=0.0, partitions=peer_parts, engine=engine)
    sim = T.Monodomain(m["xyz"], m["tets"], m["region"], m["fibre"], cond, cfg, stims)
    try:
        for k in range(60):
            sim.step(1)
            ref.step()
            assert np.linalg.norm(sim.V - ref.Vk) / np.linalg.norm(ref.Vk) <= 1e-8, k
        lat, _ = sim.activation()
        assert np.abs(lat - ref.lat).max() <= dt + 1e-12
    finally:
        sim.close()


@pytest.mark.parametrize("engine", ["grid", "cluster"])
def test_state_injection_one_step(T, engine):
    """One step from an injected mid-upstroke state: GPU == oracle (any size path)."""
    xyz, tets, region, fib, cond, stims = _slab_case("tt2006", 31, 12, 7, 0.5, permute=True, seed=5)
    dt = 0.02
    ref = O.Monodomain(xyz, tets, region, fib, cond, O.Config(dt=dt, abs_tol=1e-9, rel_tol=0.0), stims)
    ref.run(300)                       # 6 ms: front is propagating
    n = xyz.shape[0]
    buf = np.concatenate([ref.Vk, ref.Vkm1, ref.U.reshape(-1), [ref.k, 1.0]])
    cfg = T.tc_config_default(dt=dt, abs_tol=1e-9, rel_tol=0.0, engine=engine)
    sim = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims)
    try:
        sim.set_state(buf)
        assert np.array_equal(sim.get_state(), buf)
        sim.step(1)
        ref.step()
        v = sim.V
        assert np.linalg.norm(v - ref.Vk) / np.linalg.norm(ref.Vk) <= 1e-8
    finally:
        sim.close()


@pytest.mark.parametrize("model,engine,dt", [("tt2006", "grid", 0.05), ("tt2006", "cluster", 0.1),
                                             ("crn", "grid", 0.05), ("crn", "cluster", 0.1),
                                             ("ms", "grid", 0.05)])
def test_ionic_voltage_range_one_step(T, model, engine, dt):
    """One step from an injected state whose V^k spans -130 .. +70 mV node by node
    (plus exact points around the TT2006 m-gate underflow, V ~ -99 mV at dt 0.05,
    where the Rush-Larsen factor e^{-dt/tau_m} drops below e^{-708}): every gate
    and concentration equals the oracle's libm-exp update, V^{k+1} the oracle's.
    A cohort member reached V = -98.9 mV after 394 steps and the fast exp wrapped
    there (regression)."""
    xyz, tets, region, fib, cond, stims = _slab_case(model, 21, 8, 5, 0.5, permute=True, seed=3)
    n = xyz.shape[0]
    rng = np.random.default_rng(11)
    V = rng.uniform(-130.0, 70.0, n)
    V[:8] = [-99.0, -98.93, -100.0, -105.0, -110.0, -120.0, -130.0, -150.0]
    init = {"tt2006": O.tt_initial_state, "crn": O.crn_initial_state,
            "ms": lambda m: O.ms_initial_state(m)}[model]
    _, U = init(n)
    U = np.ascontiguousarray(U, dtype=np.float64).reshape(-1, n)
    ref = O.Monodomain(xyz, tets, region, fib, cond, O.Config(dt=dt, model=model, abs_tol=1e-9, rel_tol=0.0),
                       stims)
    ref.set_state(V, V, U, 60)
    buf = np.concatenate([V, V, U.reshape(-1), [60, 1.0]])
    cfg = T.tc_config_default(dt=dt, model=model, abs_tol=1e-9, rel_tol=0.0, engine=engine)
    sim = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims)
    try:
        sim.set_state(buf)
        sim.step(1)
        ref.step()
        ns = U.shape[0]
        s = sim.get_state()
        U1 = s[2 * n:(2 + ns) * n].reshape(ns, n)
        assert np.all(np.isfinite(s))
        assert np.allclose(U1, ref.U.reshape(ns, n), rtol=1e-10, atol=1e-14)
        v = sim.V
        assert np.linalg.norm(v - ref.Vk) / np.linalg.norm(ref.Vk) <= 1e-8
    finally:
        sim.close()


@pytest.mark.parametrize("engine,where", [("grid", "V"), ("cluster", "V"), ("grid", "gate"), ("cluster", "gate")])
def test_blow_up_is_reported(T, engine, where):
    """A non-finite value in V^k or in one gate of one node makes tc_step fail
    with TC_ENAN ("NaN detected in any inner product"), and the context then
    refuses further steps."""
    xyz, tets, region, fib, cond, stims = _slab_case("tt2006", 13, 6, 4, 0.5)
    n = xyz.shape[0]
    cfg = T.tc_config_default(dt=0.05, engine=engine)
    sim = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims)
    try:
        sim.step(2)
        buf = sim.get_state()
        buf[n // 2 if where == "V" else 2 * n + 6 * n + n // 3] = np.nan   # V or the m gate
        sim.set_state(buf)
        with pytest.raises(T.TcError) as ei:
            sim.step(3)
        assert ei.value.status == T.TC_ENAN
        with pytest.raises(T.TcError):
            sim.step(1)
    finally:
        sim.close()


@pytest.mark.parametrize("engine,nparts", [("grid", 1), ("cluster", 1), ("auto", 2)])
def test_step_io_equals_serial_calls(T, engine, nparts):
    """tc_step_io (pipelined H2D / step / D2H over copy streams) returns, for every
    input state, exactly what tc_set_state + tc_step(1) + tc_get_v return; and
    the first problem matches the oracle's step from the same state."""
    xyz, tets, region, fib, cond, stims = _slab_case("tt2006", 31, 12, 7, 0.5, permute=True, seed=5)
    dt = 0.02
    ref = O.Monodomain(xyz, tets, region, fib, cond, O.Config(dt=dt, abs_tol=1e-9, rel_tol=0.0), stims)
    states = []
    for k in (100, 150, 200, 250, 300):          # distinct states along an upstroke, has_prev 1
        ref.run(k - ref.k)
        states.append(np.concatenate([ref.Vk, ref.Vkm1, ref.U.reshape(-1), [ref.k, 1.0]]))
    states.append(states[0].copy())
    states[-1][-1] = 0.0                         # has_prev 0: V^{k-1} := V^k
    n = xyz.shape[0]
    cfg = T.tc_config_default(dt=dt, abs_tol=1e-9, rel_tol=0.0, engine=engine, partitions=nparts)
    sim = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims)
    try:
        serial = []
        for b in states:
            sim.set_state(b)
            sim.step(1)
            serial.append(sim.V.copy())
        pad = np.zeros((len(states), len(states[0]) + 3))   # stride > state length
        pad[:, :len(states[0])] = np.array(states)
        out = np.zeros((len(states), n))
        st = T.tc_step_io(sim.ctx, pad, out, want_stats=True)
        for j in range(len(states)):
            assert np.array_equal(out[j], serial[j]), j
        assert (st["iters"] > 0).all()
        assert np.array_equal(sim.V, serial[-1])     # the context holds the last problem's result
        ref2 = O.Monodomain(xyz, tets, region, fib, cond, O.Config(dt=dt, abs_tol=1e-9, rel_tol=0.0), stims)
        ref2.run(100)
        ref2.step()
        assert np.linalg.norm(out[0] - ref2.Vk) / np.linalg.norm(ref2.Vk) <= 1e-8
        # stride 0: the same state for every problem, one output buffer (the last result)
        one = np.zeros(n)
        st0 = T.tc_step_io_repeat(sim.ctx, np.ascontiguousarray(pad[1]), one, 5, want_stats=True)
        assert np.array_equal(one, serial[1]) and len(set(st0["iters"].tolist())) == 1
        with pytest.raises(ValueError):
            T.tc_step_io(sim.ctx, pad, np.zeros((len(states), n + 1)))
        bad = pad.copy()
        bad[2, len(states[0]) - 2] = 1.5             # non-integer step index
        with pytest.raises(T.TcError):
            T.tc_step_io(sim.ctx, bad, out)
    finally:
        sim.close()


def test_ionic_params_match_oracle_transcription(T):
    """Two independent transcriptions of TT2006 / MS constants agree."""
    for model, names, vals in (("tt2006", O.tt_param_names(), O.tt_default_params()),
                               ("ms", O.MS_PARAM_NAMES, O.ms_default_params()),
                               ("crn", O.crn_param_names(), O.crn_default_params())):
        ctx = T.tc_create(T.tc_config_default(model=model))
        try:
            for nme, v in zip(names, vals):
                assert T.tc_get_ionic_param(ctx, nme) == v, nme
            with pytest.raises(T.TcError):
                T.tc_get_ionic_param(ctx, "no_such_parameter")
        finally:
            T.tc_destroy(ctx)


def test_mms_on_gpu_matches_oracle_and_converges(T, golden):
    """configs[1] (readings M2/M3/T1): h-refinement N = 8, 16, 32, 64
    on the GPU.  N <= 32: V at T equals the oracle's to 1e-8 and the M-norm
    errors equal the independent direct-solve values of SURVEY 8(c)
    (tests/golden/mms_reference_errors.json); every ratio N -> 2N has observed
    L2 order in [1.7, 2.3], including 32 -> 64."""
    g = golden["mms_reference_errors"]
    errs = []
    for N in (8, 16, 32, 64):
        xyz, tets = G.unit_cube(N)
        B = G.box_boundary(xyz)
        dt = 0.01 * 8 / N
        E = tets.shape[0]
        cfg = T.tc_config_default(dt=dt, model="mms", chi=1.0, cm=1.0, abs_tol=1e-10, rel_tol=1e-10,
                                  max_iters=1000)
        sim = T.Monodomain(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E), {0: (1.0, 1.0)}, cfg,
                           mms=(1.0, np.pi, np.pi, np.pi, B))
        try:
            st = sim.step(int(round(0.5 / dt)))
            v = sim.V
        finally:
            sim.close()
        assert st["converged"].all()
        e = v - O.mms_w(xyz[:, 0], xyz[:, 1], 0.5)
        rp, col, M, _ = O.assemble(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E), {0: (1.0, 1.0)})
        errs.append(np.sqrt(e @ O.spmv(rp, col, M, e)))
        if N <= 32:
            out = O.run_mms(xyz, tets, B, dt=dt, T=0.5, tol=1e-10)
            assert np.abs(v - out["V"]).max() <= 1e-8, N
            i = g["N"].index(N)
            assert errs[-1] == pytest.approx(g["err_M"][i], rel=g["rel_tol"]), (N, errs[-1])
        print(f"MMS N={N}: ||e||_M = {errs[-1]:.4e}, mean PCG iterations {np.mean(st['iters']):.1f}")
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    print("observed orders", orders)
    assert np.all((orders > 1.7) & (orders < 2.3)), orders


@pytest.mark.parametrize("model,parts,rot,engine,variant", [("ms", 1, False, "grid", -1), ("tt2006", 1, True, "cluster", -1),
                                                            ("tt2006", 3, False, "auto", -1), ("ms", 2, True, "auto", -1),
                                                            ("ms", 1, True, "cluster", -1), ("ms", 2, False, "auto", 4),
                                                            ("tt2006", 1, False, "grid", 0)])
def test_surface_sphere_trajectory_parity(T, model, parts, rot, engine, variant):
    """Surface (triangle) meshes: an icosphere with tangent
    fibres, two regions, stimulus at one pole; V per step within rel-L2 1e-8,
    LAT within one dt, also under a rigid rotation and on row-block partitions."""
    xyz, tris = G.sphere(3)
    xyz, tris, _ = G.permute_nodes(xyz, tris, seed=11)
    if rot:
        xyz, _ = G.rotate(xyz)
    E = tris.shape[0]
    fib = G.sphere_fibres(xyz, tris)
    c = xyz[tris].mean(1)
    region = (c[:, 0] > 3.0).astype(np.int32)
    cond = {0: (0.1334177, 0.0173515), 1: (0.3, 0.05)}
    top = np.argmax(xyz @ np.array([0.3, 0.2, 0.93]))
    d = np.linalg.norm(xyz - xyz[top], axis=1)
    stims = [O.Stimulus(np.nonzero(d < 2.5)[0], 0.0, 2.0, 50.0)]
    dt = 0.05
    ref = O.Monodomain(xyz, tris, region, fib, cond, O.Config(dt=dt, model=model, abs_tol=1e-8, rel_tol=0.0),
                       stims)
    cfg = T.tc_config_default(dt=dt, model=model, abs_tol=1e-8, rel_tol=0.0, partitions=parts, engine=engine,
                              pcg_variant=variant)
    sim = T.Monodomain(xyz, tris, region, fib, cond, cfg, stims)
    try:
        for k in range(150):
            st = sim.step(1)
            rep = ref.step()
            rel = np.linalg.norm(sim.V - ref.Vk) / np.linalg.norm(ref.Vk)
            assert rel <= 1e-8, (k, rel)
            assert abs(int(st["iters"][0]) - rep.iters) <= 1
        lat, _ = sim.activation()
        assert np.all((lat < 0) == (ref.lat < 0))
        assert np.abs(lat - ref.lat).max() <= dt + 1e-12
        assert (ref.lat >= 0).sum() > 10      # the wave actually propagated
    finally:
        sim.close()


def test_surface_mms_unit_square_on_gpu(T):
    """The paper's own MMS setup: [0,1]^2 triangulated, Dirichlet w on the
    perimeter, Crank-Nicolson; GPU V equals the oracle's, L2 order ~2."""
    errs = []
    for N in (8, 16):
        xyz, tris = G.unit_square(N)
        B = G.box_boundary(xyz[:, :2])
        dt = 0.01 * 8 / N
        out = O.run_mms(xyz, tris, B, dt=dt, T=0.5, tol=1e-10)
        E = tris.shape[0]
        cfg = T.tc_config_default(dt=dt, model="mms", chi=1.0, cm=1.0, abs_tol=1e-10, rel_tol=1e-10,
                                  max_iters=1000)
        sim = T.Monodomain(xyz, tris, np.zeros(E, np.int32), G.uniform_fibres(E), {0: (1.0, 1.0)}, cfg,
                           mms=(1.0, np.pi, np.pi, np.pi, B))
        try:
            sim.step(int(round(0.5 / dt)))
            v = sim.V
        finally:
            sim.close()
        assert np.abs(v - out["V"]).max() <= 1e-8
        errs.append(out["err_M"])
    order = np.log2(errs[0] / errs[1])
    assert 1.7 < order < 2.3


def test_surface_mesh_errors(T):
    xyz, tris = G.unit_square(2)
    ctx = T.tc_create(T.tc_config_default())
    try:
        bad = tris.copy()
        bad[0] = [0, 1, 2]          # collinear nodes on the bottom edge -> zero area
        with pytest.raises(T.TcError) as ei:
            T.tc_set_mesh_elems(ctx, xyz, bad)
        assert ei.value.status == T.TC_EDEGEN
        with pytest.raises(T.TcError):
            T.tc_set_mesh_elems(ctx, xyz, np.zeros((2, 5), np.int32))
    finally:
        T.tc_destroy(ctx)


def test_errors_are_reported(T):
    xyz, tets = G.kuhn_box(3, 3, 3, 1.0)
    ctx = T.tc_create(T.tc_config_default())
    try:
        bad = tets.copy()
        bad[0, 0] = 10_000
        with pytest.raises(T.TcError) as ei:
            T.tc_set_mesh(ctx, xyz, bad)
        assert ei.value.status == T.TC_EINVAL
        flat = xyz.copy()
        flat[:, 2] = 0.0
        with pytest.raises(T.TcError) as ei:
            T.tc_set_mesh(ctx, flat, tets)
        assert ei.value.status == T.TC_EDEGEN
        with pytest.raises(T.TcError) as ei:
            T.tc_step(ctx, 1)
        assert ei.value.status == T.TC_ESTATE
    finally:
        T.tc_destroy(ctx)


def test_torch_allocator_hook(T):
    """tc_set_allocator: with torch's caching allocator the
    context's device memory comes from torch (memory_allocated grows, every block
    is returned by tc_destroy) and the trajectory is bitwise the default one."""
    import torch
    xyz, tets, region, fib, cond, stims = _slab_case("tt2006")
    cfg = T.tc_config_default(dt=0.05, engine="grid")
    ref = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims)
    before = torch.cuda.memory_allocated()
    al = T.TorchAllocator(0)
    sim = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims, allocator=al)
    try:
        assert len(al.live) > 10 and torch.cuda.memory_allocated() > before
        a = ref.step(40)
        b = sim.step(40)
        assert np.array_equal(ref.V, sim.V) and np.array_equal(a["iters"], b["iters"])
        st = sim.get_state()
        sim.set_state(st)                       # staging buffers through the hook too
        assert np.array_equal(sim.get_state(), st)
    finally:
        sim.close()
        ref.close()
    assert not al.live and torch.cuda.memory_allocated() == before
    ctx = T.tc_create(T.tc_config_default())
    try:                                        # too late once the context has allocated
        T.tc_set_mesh(ctx, xyz, tets)
        T.tc_set_conductivity(ctx, [0], [0.13], [0.02])
        T.tc_assemble(ctx)
        with pytest.raises(T.TcError) as ei:
            T.tc_set_allocator(ctx, T.TorchAllocator(0))
        assert ei.value.status == T.TC_ESTATE
    finally:
        T.tc_destroy(ctx)


@pytest.mark.parametrize("case", ["grid_v0", "grid_v1", "grid_v2", "grid_v4", "grid_v5", "grid_v6", "parts2_peer",
                                  "parts3_split", "parts5_peer_host", "sphere_parts3", "biv_parts4", "mms_parts2",
                                  "cluster"])
def test_index_audit(T, case):
    """Memory safety without compute-sanitizer (closed on the GPU pool): every
    device index array the step kernels address memory through is inside its
    allocation (tc_validate, include/tcb200.h), for every layout and path;
    then 10 steps run and the audit still holds."""
    kw = dict(dt=0.05, abs_tol=1e-8, rel_tol=0.0)
    mms = None
    if case.startswith("sphere"):
        xyz, el = G.sphere(4)
        region, fib = np.zeros(el.shape[0], np.int32), G.sphere_fibres(xyz, el)
        cond = {0: (0.1334177, 0.0173515)}
        stims = [(np.nonzero(xyz[:, 2] > 0.9 * xyz[:, 2].max())[0].astype(np.int32), 0.0, 2.0, 50.0)]
        kw.update(model="ms", partitions=3)
    elif case.startswith("biv"):
        m = G.biv(2.5)
        xyz, el, region, fib = m["xyz"], m["tets"], m["region"], m["fibre"]
        cond = {0: (0.1334177, 0.0173515), 1: (0.1334177, 0.0173515)}
        stims = [(nodes, 0.0, 2.0, 50.0) for nodes in G.biv_stimuli(m, radius=3.0)]
        kw.update(partitions=4)
    elif case.startswith("mms"):
        xyz, el = G.unit_cube(12)
        region, fib = np.zeros(el.shape[0], np.int32), G.uniform_fibres(el.shape[0])
        cond = {0: (1.0, 1.0)}
        stims = []
        mms = (1.0, np.pi, np.pi, np.pi, G.box_boundary(xyz))
        kw.update(model="mms", chi=1.0, cm=1.0, dt=0.01, partitions=2)
    else:
        xyz, el, region, fib, cond, stims = _slab_case("tt2006", permute=True, seed=3)
        if case.startswith("grid_v"):
            kw.update(engine="grid", pcg_variant=int(case[6:]))
        elif case == "parts2_peer":
            kw.update(partitions=2, peer=1)
        elif case == "parts3_split":
            kw.update(partitions=3, peer=0)
        elif case == "parts5_peer_host":
            kw.update(partitions=5, peer=1, device_setup=0)
        elif case == "cluster":
            kw.update(engine="cluster")
    sim = T.Monodomain(xyz, el, region, fib, cond, T.tc_config_default(**kw), stims, mms=mms)
    try:
        n0 = T.tc_validate(sim.ctx)
        assert n0 >= xyz.shape[0]
        sim.step(10)
        assert T.tc_validate(sim.ctx) == n0
    finally:
        sim.close()


def test_mms_split_setters_equal_tc_set_mms(T):
    """tc_set_dirichlet + tc_set_mms_source (SURVEY 8(b) names) configure the
    same manufactured problem as tc_set_mms: bitwise-equal trajectories."""
    xyz, tets = G.unit_cube(8)
    B = G.box_boundary(xyz)
    E = tets.shape[0]
    vs = []
    for split in (False, True):
        ctx = T.tc_create(T.tc_config_default(dt=0.01, model="mms", chi=1.0, cm=1.0, abs_tol=1e-10, rel_tol=1e-10,
                                              max_iters=500))
        try:
            T.tc_set_mesh(ctx, xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E))
            T.tc_set_conductivity(ctx, [0], [1.0], [1.0])
            if split:
                T.tc_set_mms_source(ctx, 1.0, np.pi, np.pi, np.pi)
                T.tc_set_dirichlet(ctx, B)
            else:
                T.tc_set_mms(ctx, 1.0, np.pi, np.pi, np.pi, B)
            T.tc_assemble(ctx)
            T.tc_step(ctx, 20)
            vs.append(T.tc_get_v(ctx))
        finally:
            T.tc_destroy(ctx)
    assert np.array_equal(vs[0], vs[1])


@pytest.mark.parametrize("nparts", [2, 3])
def test_split_path_overlapped_launches(T, nparts):
    """The split path as a real communicator runs it -- the interior slices of
    every S / RHS pass as one launch while the halo is in flight, the boundary
    slices as a second launch that adds the first one's per-CTA partials before
    the deterministic reduction (reduce_phase) -- forced on one GPU with
    TCB_SPLIT_OVERLAP=1 (read at tc_assemble): a trajectory against the oracle."""
    import os
    xyz, tets, region, fib, cond, stims = _slab_case("tt2006", 61, 23, 9, permute=True, seed=4)
    dt = 0.05
    ref = O.Monodomain(xyz, tets, region, fib, cond, O.Config(dt=dt, abs_tol=1e-8, rel_tol=0.0), stims)
    os.environ["TCB_SPLIT_OVERLAP"] = "1"
    try:
        cfg = T.tc_config_default(dt=dt, abs_tol=1e-8, rel_tol=0.0, partitions=nparts, peer=0)
        sim = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims)
    finally:
        os.environ.pop("TCB_SPLIT_OVERLAP", None)
    try:
        info = T.tc_matrix_info(sim.ctx)
        assert info["path"] == "split" and info["ghosts"] > 0
        T.tc_validate(sim.ctx)    # includes: interior slices read no ghost column
        for k in range(60):
            st = sim.step(1)
            rep = ref.step()
            rel = np.linalg.norm(sim.V - ref.Vk) / np.linalg.norm(ref.Vk)
            assert rel <= 1e-8, (k, rel)
            assert abs(int(st["iters"][0]) - rep.iters) <= 1
        lat, _ = sim.activation()
        assert np.abs(lat - ref.lat).max() <= dt + 1e-12
    finally:
        sim.close()
