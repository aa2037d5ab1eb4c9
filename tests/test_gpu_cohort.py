"""GPU parity of the cluster engine and of cohorts.

The cluster engine runs every step of a tc_step call inside one thread-block
cluster; a cohort runs many independent members
in one launch, one cluster each, with per-member PCG stopping.  Each member is
checked against its own CPU oracle run (same seeded inputs) with the
north_star tolerances: V per step within rel-L2 1e-8, LAT within one dt,
per-step PCG iteration counts within 1."""
import numpy as np
import pytest

import meshgen as G
import oracle as O

pytestmark = pytest.mark.gpu

SIG = (0.1334177, 0.0173515)   # Table 3


@pytest.fixture(scope="module")
def T():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2510_12011_b200 as T
    return T


def _member(spec):
    """spec -> (xyz, tets, region, fibre, cond, stimuli, oracle Config kwargs, params dict)."""
    kind = spec.get("mesh", "slab")
    if kind == "biv":
        m = G.biv(spec.get("h", 2.5))
        xyz, tets, region, fib = m["xyz"], m["tets"], m["region"], m["fibre"]
        stims = [O.Stimulus(nodes, 0.0, 2.0, 50.0) for nodes in G.biv_stimuli(m, radius=3.0)]
        cond = {0: SIG, 1: SIG}
    else:
        nx, ny, nz = spec["dims"]
        dx = spec.get("dx", 0.5)
        xyz, tets = G.kuhn_box(nx, ny, nz, dx)
        if spec.get("permute"):
            xyz, tets, _ = G.permute_nodes(xyz, tets, seed=spec["permute"])
        E = tets.shape[0]
        region = np.zeros(E, np.int32)
        fib = G.random_fibres(E, spec["fib_seed"]) if spec.get("fib_seed") else G.uniform_fibres(E)
        sl, st = SIG
        s = spec.get("sigma_scale", 1.0)
        cond = {0: (sl * s, st * s)}
        hi = spec.get("stim_box", 1.5)
        stims = [O.Stimulus(G.nodes_in_box(xyz, (0, 0, 0), (hi, hi, hi)), spec.get("t0", 0.0),
                            2.0, spec.get("amp", 50.0))]
    return xyz, tets, region, fib, cond, stims


def _oracle(spec, xyz, tets, region, fib, cond, stims):
    model = spec.get("model", "tt2006")
    params = None
    if spec.get("params"):
        if model == "tt2006":
            names, params = O.tt_param_names(), O.tt_default_params().copy()
        elif model == "crn":
            names, params = O.crn_param_names(), O.crn_default_params().copy()
        else:
            names, params = list(O.MS_PARAM_NAMES), O.ms_default_params().copy()
        for k, v in spec["params"].items():
            params[names.index(k)] = v
    cfg = O.Config(dt=spec.get("dt", 0.05), model=model, abs_tol=spec.get("tol", 1e-8), rel_tol=0.0,
                   max_iters=spec.get("max_iters", 100), fail_budget=spec.get("fail_budget", 3),
                   params=params)
    return O.Monodomain(xyz, tets, region, fib, cond, cfg, stims)


def _gpu(T, spec, xyz, tets, region, fib, cond, stims, engine="cluster"):
    cfg = T.tc_config_default(dt=spec.get("dt", 0.05), model=spec.get("model", "tt2006"),
                              abs_tol=spec.get("tol", 1e-8), rel_tol=0.0,
                              max_iters=spec.get("max_iters", 100),
                              fail_budget=spec.get("fail_budget", 3), engine=engine)
    return T.Monodomain(xyz, tets, region, fib, cond, cfg, stims, params=spec.get("params"))


def _check(sim, ref, stats_row, reps, dt, what):
    v = sim.V
    rel = np.linalg.norm(v - ref.Vk) / np.linalg.norm(ref.Vk)
    assert rel <= 1e-8, (what, rel)
    if stats_row is not None:
        for a, b in zip(stats_row, reps):
            assert abs(int(a["iters"]) - b.iters) <= 1, (what, int(a["iters"]), b.iters)
    lat, _ = sim.activation()
    assert np.all((lat < 0) == (ref.lat < 0)), what
    assert np.abs(lat - ref.lat).max() <= dt + 1e-12, what


@pytest.mark.parametrize("model,permute,chunk,engine", [("tt2006", 0, 1, "cluster"), ("tt2006", 7, 9, "cluster"),
                                                        ("ms", 0, 5, "cluster"), ("ms", 3, 1, "cluster"),
                                                        ("tt2006", 7, 9, "cluster_streaming"),
                                                        ("ms", 3, 4, "cluster_streaming"),
                                                        ("crn", 0, 6, "cluster"), ("crn", 5, 3, "cluster_streaming")])
def test_cluster_engine_trajectory_parity(T, model, permute, chunk, engine):
    """One context on the cluster engine (shared-memory resident or streaming),
    `chunk` steps per tc_step call (the in-kernel rotation, the V write-back and
    the LAT epilogue across call boundaries)."""
    spec = dict(dims=(21, 8, 5), model=model, permute=permute, fib_seed=3 if permute else 0)
    args = _member(spec)
    ref = _oracle(spec, *args)
    sim = _gpu(T, spec, *args, engine=engine)
    try:
        info = T.tc_engine_info(sim.ctx)
        assert info["engine"] == "cluster"
        assert (info["smem_per_cta"] > 0) == (engine == "cluster")
        for c in range(120 // chunk):
            st = sim.step(chunk)
            reps = [ref.step() for _ in range(chunk)]
            _check(sim, ref, st, reps, 0.05, f"chunk {c}")
        s = sim.get_state()
        n = args[0].shape[0]
        U = s[2 * n:-2].reshape(-1, n)
        assert np.allclose(U, ref.U, rtol=1e-8, atol=1e-14)
    finally:
        sim.close()


def test_cluster_engine_equals_grid_engine(T):
    """Both engines compute the same step (only inner-product grouping differs)."""
    spec = dict(dims=(41, 15, 7), model="tt2006", permute=11, fib_seed=2)
    args = _member(spec)
    a = _gpu(T, spec, *args, engine="cluster")
    b = _gpu(T, spec, *args, engine="grid")
    try:
        for _ in range(8):
            sa = a.step(10)
            sb = b.step(10)
            assert np.abs(sa["iters"] - sb["iters"]).max() <= 1
            va, vb = a.V, b.V
            assert np.linalg.norm(va - vb) / np.linalg.norm(vb) <= 1e-10
        la, _ = a.activation()
        lb, _ = b.activation()
        assert np.array_equal(la, lb)
    finally:
        a.close()
        b.close()


COHORT = [
    dict(dims=(21, 8, 5)),                                                  # small slab
    dict(dims=(41, 15, 7), permute=5, fib_seed=4),                          # configs[0] mesh, relabelled
    dict(dims=(13, 6, 4), sigma_scale=2.0, params={"GKr": 0.0765, "GNa": 11.0}),  # parameter reset
    dict(dims=(2, 2, 2), stim_box=0.6),                                     # 8 nodes, 6 tets, one slice
    dict(mesh="biv", h=2.5, dt=0.02),                                       # unstructured, 2 regions, other dt
    dict(dims=(17, 9, 6), tol=1e-10, t0=1.0, amp=80.0),                     # other tolerance / stimulus
]


@pytest.mark.parametrize("cluster_size,resident", [(0, 1), (1, 0), (4, 1), (4, 0), (16, 1), (4, 2), (4, 3), (8, 3),
                                                    (2, 4), (4, 4), (0, 4)])
def test_cohort_parity(T, cluster_size, resident):
    """A heterogeneous cohort (meshes of 8 .. ~5k nodes, structured and BiV, other
    dt / tolerances / conductivities / ionic parameters / stimuli) advanced in
    chunks of 10 steps per launch; every member against its own oracle run."""
    members, refs, dts = [], [], []
    try:
        for spec in COHORT:
            args = _member(spec)
            refs.append(_oracle(spec, *args))
            members.append(_gpu(T, spec, *args))
            dts.append(spec.get("dt", 0.05))
        co = T.Cohort(members, cluster_size, resident)
        try:
            info = co.info()
            assert info["members"] == len(COHORT)
            if not resident:
                assert info["smem_per_cta"] == 0
            if resident == 2:
                assert not info["compact"]
            if resident == 3:   # indices-only residency fits every member of this cohort
                assert info["compact"] and info["smem_per_cta"] > 0
            assert info["dense"] == (resident == 4)
            if cluster_size:
                assert info["cluster_size"] == cluster_size
            assert info["resident_clusters"] >= 1
            for c in range(6):
                stats = co.step(10)
                assert stats.shape == (len(COHORT), 10)
                for m, (sim, ref) in enumerate(zip(members, refs)):
                    reps = [ref.step() for _ in range(10)]
                    _check(sim, ref, stats[m], reps, dts[m], f"member {m} chunk {c}")
                    assert T.tc_current_step(sim.ctx) == 10 * (c + 1)
        finally:
            co.close()
        # members stay usable on their own after the cohort
        for sim, ref in zip(members, refs):
            st = sim.step(3)
            reps = [ref.step() for _ in range(3)]
            _check(sim, ref, st, reps, 0.05, "after cohort")
    finally:
        for s in members:
            s.close()


def test_cohort_crn_members(T):
    """CRN atrial members in one cohort, each against its oracle."""
    specs = [dict(dims=(21, 8, 5), model="crn"), dict(dims=(13, 6, 4), model="crn", params={"gto": 0.08}),
             dict(dims=(17, 9, 6), model="crn", permute=2, fib_seed=5)]
    members, refs = [], []
    try:
        for spec in specs:
            args = _member(spec)
            refs.append(_oracle(spec, *args))
            members.append(_gpu(T, spec, *args))
        co = T.Cohort(members)
        try:
            for c in range(4):
                stats = co.step(15)
                for m, (sim, ref) in enumerate(zip(members, refs)):
                    reps = [ref.step() for _ in range(15)]
                    _check(sim, ref, stats[m], reps, 0.05, f"crn member {m} chunk {c}")
        finally:
            co.close()
    finally:
        for s in members:
            s.close()


def test_cohort_of_identical_members_is_bitwise_uniform(T):
    """Identical members give bitwise-identical results (no cross-member coupling)."""
    spec = dict(dims=(21, 8, 5), model="ms")
    members = [_gpu(T, spec, *_member(spec)) for _ in range(40)]
    try:
        co = T.Cohort(members)
        st = co.step(50)
        co.close()
        v0 = members[0].V
        for s in members[1:]:
            assert np.array_equal(s.V, v0)
        assert np.all(st["iters"] == st["iters"][0])
    finally:
        for s in members:
            s.close()


def test_cohort_per_member_failure(T):
    """A member that exhausts its fail budget stops alone; the call reports it by
    index; the other members advance exactly as their oracle runs."""
    good = dict(dims=(21, 8, 5))
    bad = dict(dims=(21, 8, 5), max_iters=1, fail_budget=2, tol=1e-14)
    ga, ba = _member(good), _member(bad)
    ref = _oracle(good, *ga)
    members = [_gpu(T, good, *ga), _gpu(T, bad, *ba)]
    try:
        co = T.Cohort(members)
        with pytest.raises(T.TcError) as ei:
            co.step(5)
        assert ei.value.status == T.TC_ESOLVER and "member 1" in str(ei.value)
        reps = [ref.step() for _ in range(5)]
        _check(members[0], ref, None, reps, 0.05, "good member")
        with pytest.raises(T.TcError):   # the failed member's context stays failed
            members[1].step(1)
        co.close()
    finally:
        for s in members:
            s.close()


def test_cohort_errors(T):
    spec = dict(dims=(9, 5, 4))
    a = _gpu(T, spec, *_member(spec))
    b = _gpu(T, dict(spec, model="ms"), *_member(spec))
    cfg = T.tc_config_default(dt=0.05, partitions=2)
    xyz, tets, region, fib, cond, stims = _member(spec)
    p = T.Monodomain(xyz, tets, region, fib, cond, cfg, stims)
    try:
        with pytest.raises(T.TcError) as ei:
            T.Cohort([a, b])                       # mixed ionic models
        assert ei.value.status == T.TC_EINVAL
        with pytest.raises(T.TcError) as ei:
            T.Cohort([a, p])                       # partitioned member
        assert ei.value.status == T.TC_ESTATE
        with pytest.raises(T.TcError):
            T.Cohort([a, a])                       # repeated member
        with pytest.raises(T.TcError):
            T.Cohort([a], cluster_size=3)          # not a power of two
        with pytest.raises(T.TcError) as ei:
            T.Cohort([a], resident=5)              # no such residency mode
        assert ei.value.status == T.TC_EINVAL
    finally:
        for s in (a, b, p):
            s.close()


def test_cohort_mixes_small_and_large_members(T):
    """A member above the cluster engine's size runs on the grid engine inside the
    same tc_cohort_step; every member still matches its oracle run."""
    specs = [dict(dims=(21, 8, 5)), dict(dims=(61, 23, 9), permute=3, fib_seed=2), dict(dims=(13, 6, 4))]
    members, refs = [], []
    try:
        for spec in specs:
            args = _member(spec)
            refs.append(_oracle(spec, *args))
            members.append(_gpu(T, spec, *args, engine="auto"))
        assert T.tc_matrix_info(members[1].ctx)["nslices"] > 256     # grid-engine size
        co = T.Cohort(members)
        try:
            for c in range(3):
                stats = co.step(10)
                for m, (sim, ref) in enumerate(zip(members, refs)):
                    reps = [ref.step() for _ in range(10)]
                    _check(sim, ref, stats[m], reps, 0.05, f"member {m} chunk {c}")
        finally:
            co.close()
    finally:
        for s in members:
            s.close()


def test_cohort_large_members_share_the_gpu(T):
    """Three grid-engine-sized members (plus a small one) in one cohort: the large
    ones run side by side, each on its own stream with the PCG variant and
    cooperative grid chosen for a third of the GPU (DESIGN.md "Cohorts of large
    members"); every member matches its own oracle run, and the shared-GPU shape
    gives the same trajectory as the member stepped alone up to rounding."""
    specs = [dict(dims=(61, 23, 9), permute=3, fib_seed=2), dict(dims=(21, 8, 5)),
             dict(dims=(57, 25, 10), permute=5, sigma_scale=0.9),
             dict(dims=(65, 21, 9), permute=7, fib_seed=4)]
    members, refs = [], []
    try:
        for spec in specs:
            args = _member(spec)
            refs.append(_oracle(spec, *args))
            members.append(_gpu(T, spec, *args, engine="auto"))
        big = [m for m in members if T.tc_matrix_info(m.ctx)["nslices"] > 256]
        assert len(big) == 3
        co = T.Cohort(members)
        try:
            for c in range(3):
                stats = co.step(10)
                for m, (sim, ref) in enumerate(zip(members, refs)):
                    reps = [ref.step() for _ in range(10)]
                    _check(sim, ref, stats[m], reps, 0.05, f"member {m} chunk {c}")
        finally:
            co.close()
    finally:
        for s in members:
            s.close()


def test_cohort_long_horizon_bench_members(T):
    """The bench's cohort members 8 and 1 (meshgen.cohort_members, seeded; the
    ones whose trajectories undershoot to V ~ -99 mV, where the fast exp once
    wrapped: DESIGN.md "Exp range") advanced 450 steps (22.5 ms, past the
    first repolarisation undershoot) in one cohort, each against its own oracle
    run every 50 steps with the north_star tolerances."""
    ms = G.cohort_members(100, seed=G.SEED)
    members, refs = [], []
    try:
        for i in (8, 1):
            m = ms[i]
            E = m["tets"].shape[0]
            cond = {0: (SIG[0] * m["sigma_scale"], SIG[1] * m["sigma_scale"])}
            stims = [O.Stimulus(m["stim_nodes"], 0.0, 2.0, 50.0)]
            names, params = O.tt_param_names(), O.tt_default_params().copy()
            for k, f in m["param_factors"].items():
                params[names.index(k)] *= f
            spec = dict(params={k: params[names.index(k)] for k in m["param_factors"]})
            region = np.zeros(E, np.int32)
            refs.append(O.Monodomain(m["xyz"], m["tets"], region, m["fibre"], cond,
                                     O.Config(dt=0.05, abs_tol=1e-8, rel_tol=0.0, params=params), stims))
            members.append(_gpu(T, spec, m["xyz"], m["tets"], region, m["fibre"], cond, stims))
        co = T.Cohort(members)
        vmin = np.inf
        try:
            for c in range(9):
                stats = co.step(50)
                for j, (sim, ref) in enumerate(zip(members, refs)):
                    reps = []
                    for _ in range(50):
                        reps.append(ref.step())
                        vmin = min(vmin, float(ref.Vk.min()))
                    _check(sim, ref, stats[j], reps, 0.05, f"member {j} chunk {c}")
            assert vmin < -98.0   # member 8 reaches -98.93 mV at step 394
        finally:
            co.close()
    finally:
        for s in members:
            s.close()


def test_cohort_batched_io_equals_serial_calls(T):
    """tc_cohort_set_states / tc_cohort_get_v give bitwise what the per-member
    tc_set_state / tc_get_v give (include/tcb200.h); a bad state is rejected
    before any member changes."""
    specs = [dict(dims=(21, 8, 5)), dict(dims=(17, 9, 6), permute=5), dict(dims=(25, 7, 5), permute=9)]
    members = [_gpu(T, sp, *_member(sp)) for sp in specs]
    try:
        co = T.Cohort(members)
        co.step(20, want_stats=False)
        states = [s.get_state() for s in members]
        for s, st in zip(members, states):
            T.tc_set_state(s.ctx, st)
        co.step(3, want_stats=False)
        v_serial = [T.tc_get_v(s.ctx) for s in members]
        full_serial = [s.get_state() for s in members]
        co.set_states(states)
        co.step(3, want_stats=False)
        outs = [np.full(T.tc_num_nodes(s.ctx), np.nan) for s in members]
        co.get_v(outs)
        for i, s in enumerate(members):
            assert np.array_equal(outs[i], v_serial[i]), i
            assert np.array_equal(s.get_state(), full_serial[i]), i
        bad = [st.copy() for st in states]
        bad[2][-2] = -1.0                      # step index of member 2
        before = [s.get_state() for s in members]
        with pytest.raises(T.TcError) as ei:
            co.set_states(bad)
        assert ei.value.status == T.TC_EINVAL and "member 2" in str(ei.value)
        for s, b in zip(members, before):
            assert np.array_equal(s.get_state(), b)
        # count and length mismatches are rejected in C before any member changes
        for args, what in (([st.copy() for st in states[:2]], "2 states for 3 members"),
                           ([states[0], states[1][:-3].copy(), states[2]], "member 1 state has")):
            with pytest.raises(T.TcError) as ei:
                co.set_states(args)
            assert ei.value.status == T.TC_EINVAL and what in str(ei.value), str(ei.value)
        with pytest.raises(T.TcError) as ei:
            co.get_v([np.zeros(T.tc_num_nodes(s.ctx) + (1 if i == 1 else 0)) for i, s in enumerate(members)])
        assert ei.value.status == T.TC_EINVAL and "member 1 output" in str(ei.value)
        for s, b in zip(members, before):
            assert np.array_equal(s.get_state(), b)
        co.close()
    finally:
        for s in members:
            s.close()
