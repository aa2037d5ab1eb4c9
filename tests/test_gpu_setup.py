"""Device-side setup: the pattern, RCM, SELL layout
and element incidence built on the GPU must equal the host path's, which the
CPU tests pin against the oracle (tests/test_host_logic.py: pattern and RCM vs
oracle / brute force).  Equal order + equal layout + equal assembly order =>
bitwise-identical trajectories."""
import numpy as np
import pytest

import meshgen as G
import oracle as O

pytestmark = pytest.mark.gpu
SIG = (0.1334177, 0.0173515)


@pytest.fixture(scope="module")
def T():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2510_12011_b200 as T
    return T


def _mesh(kind):
    if kind == "slab_perm":
        xyz, el = G.kuhn_box(21, 8, 5, 0.5)
        xyz, el, _ = G.permute_nodes(xyz, el, seed=7)
    elif kind == "two_components":          # two disjoint slabs: RCM restarts per component
        a, ea = G.kuhn_box(9, 5, 4, 0.5)
        b, eb = G.kuhn_box(7, 6, 3, 0.5, origin=(20.0, 0.0, 0.0))
        xyz = np.concatenate([a, b])
        el = np.concatenate([ea, eb + a.shape[0]]).astype(np.int32)
        xyz, el, _ = G.permute_nodes(xyz, el, seed=3)
    elif kind == "biv":
        m = G.biv(2.5)
        return m["xyz"], m["tets"], m["region"], m["fibre"]
    elif kind == "sphere":
        xyz, el = G.sphere(3)
        xyz, el, _ = G.permute_nodes(xyz, el, seed=11)
        return xyz, el, np.zeros(el.shape[0], np.int32), G.sphere_fibres(xyz, el)
    elif kind == "slab58k":
        xyz, el = G.kuhn_box(101, 36, 16, 0.2)
        xyz, el, _ = G.permute_nodes(xyz, el, seed=5)
    E = el.shape[0]
    return xyz, el, np.zeros(E, np.int32), G.random_fibres(E, 2)


@pytest.mark.parametrize("kind,rcm", [("slab_perm", 1), ("slab_perm", 0), ("two_components", 1),
                                      ("biv", 1), ("sphere", 1), ("slab58k", 1)])
def test_device_setup_equals_host_setup(T, kind, rcm):
    xyz, el, region, fib = _mesh(kind)
    cond = {0: SIG, 1: SIG}
    stim = [(G.nodes_in_box(xyz, xyz.min(0), xyz.min(0) + 1.5), 0.0, 2.0, 50.0)]
    sims = []
    try:
        for dev in (1, 0):
            cfg = T.tc_config_default(dt=0.05, abs_tol=1e-8, rel_tol=0.0, use_rcm=rcm, device_setup=dev)
            sims.append(T.Monodomain(xyz, el, region, fib, cond, cfg, stim))
        d, h = sims
        pd, ph = T.tc_node_order(d.ctx), T.tc_node_order(h.ctx)
        assert np.array_equal(pd, ph)
        if rcm and el.shape[1] == 4:   # the library's host RCM (pinned to the oracle's by the CPU tests)
            rp, col = T.tc_mesh_pattern(xyz.shape[0], el)
            assert np.array_equal(pd, T.tc_rcm(rp, col))
        elif not rcm:
            assert np.array_equal(pd, np.arange(xyz.shape[0]))
        mi, mh = T.tc_matrix_info(d.ctx), T.tc_matrix_info(h.ctx)
        for key in ("n", "nnz", "nnz_pad", "nslices"):
            assert mi[key] == mh[key], key
        steps = 5 if kind == "slab58k" else 20
        for _ in range(steps):
            sd, sh = d.step(1), h.step(1)
            assert np.array_equal(d.V, h.V)
            assert sd["iters"][0] == sh["iters"][0]
    finally:
        for s in sims:
            s.close()


def test_device_setup_trajectory_matches_oracle(T):
    """The device-setup path against the oracle directly (rel-L2 <= 1e-8 per step)."""
    xyz, el, region, fib = _mesh("biv")
    cond = {0: SIG, 1: SIG}
    m = G.biv(2.5)
    stims = [O.Stimulus(nodes, 0.0, 2.0, 50.0) for nodes in G.biv_stimuli(m, radius=3.0)]
    ref = O.Monodomain(xyz, el, region, fib, cond, O.Config(dt=0.05, abs_tol=1e-8, rel_tol=0.0), stims)
    cfg = T.tc_config_default(dt=0.05, abs_tol=1e-8, rel_tol=0.0, device_setup=1, engine="grid")
    sim = T.Monodomain(xyz, el, region, fib, cond, cfg, stims)
    try:
        for k in range(40):
            sim.step(1)
            ref.step()
            assert np.linalg.norm(sim.V - ref.Vk) / np.linalg.norm(ref.Vk) <= 1e-8, k
    finally:
        sim.close()


@pytest.mark.parametrize("kind,parts,peer", [("slab_perm", 2, 1), ("slab_perm", 3, 0), ("two_components", 3, 1),
                                             ("biv", 4, 1), ("slab58k", 5, 0)])
def test_partitioned_device_setup_equals_host_setup(T, kind, parts, peer):
    """SURVEY 8f f3 "RCM/partition on device": a partitioned context set up on the
    GPU (global pattern + RCM + interior-first order there, each part planned
    from its own rows) equals the host path -- same node order, same blocks,
    ghosts and layout, bitwise-identical trajectories."""
    xyz, el, region, fib = _mesh(kind)
    cond = {0: SIG, 1: SIG}
    stim = [(G.nodes_in_box(xyz, xyz.min(0), xyz.min(0) + 1.5), 0.0, 2.0, 50.0)]
    sims = []
    try:
        for dev in (1, 0):
            cfg = T.tc_config_default(dt=0.05, abs_tol=1e-8, rel_tol=0.0, device_setup=dev, partitions=parts,
                                      peer=peer)
            sims.append(T.Monodomain(xyz, el, region, fib, cond, cfg, stim))
        d, h = sims
        assert np.array_equal(T.tc_node_order(d.ctx), T.tc_node_order(h.ctx))
        mi, mh = T.tc_matrix_info(d.ctx), T.tc_matrix_info(h.ctx)
        for key in ("n", "nnz", "nnz_pad", "nslices", "partitions", "ghosts", "path"):
            assert mi[key] == mh[key], key
        for _ in range(5 if kind == "slab58k" else 15):
            sd, sh = d.step(1), h.step(1)
            assert np.array_equal(d.V, h.V)
            assert sd["iters"][0] == sh["iters"][0]
    finally:
        for s in sims:
            s.close()
