"""Pins of the oracle's FEM assembly against closed forms,
an independent gradient computation and global invariants -- not against itself."""
import itertools

import numpy as np
import pytest

import meshgen as G
import oracle as O


def _grads_independent(x):
    """Barycentric gradients by solving [1 x y z] c = e_a (a different derivation
    from the oracle's adjugate formula)."""
    Aff = np.hstack([np.ones((4, 1)), x])
    C = np.linalg.solve(Aff, np.eye(4))   # column a = coefficients of phi_a
    return C[1:, :].T                      # (4,3)


def test_reference_tet_closed_form():
    # reference tet (0,e1,e2,e3), sigma = I: M_e = (1/120)(1+delta), K_e closed form
    x = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]])
    Me, Ke, vol = O.tet_local(x, np.eye(3))
    assert vol == pytest.approx(1 / 6, rel=1e-15)
    assert np.allclose(Me, (np.ones((4, 4)) + np.eye(4)) / 120, rtol=0, atol=1e-16)
    Kref = np.array([[3, -1, -1, -1], [-1, 1, 0, 0], [-1, 0, 1, 0], [-1, 0, 0, 1]]) / 6
    assert np.allclose(Ke, Kref, rtol=0, atol=1e-15)
    assert Me.sum() == pytest.approx(1 / 6, rel=1e-14)


def test_random_tets_vs_independent_gradients():
    rng = np.random.default_rng(7)
    for _ in range(50):
        x = rng.normal(size=(4, 3))
        f = rng.normal(size=3)
        sl, st = rng.uniform(0.05, 2, 2)
        sig = O.conductivity_tensor(f, sl, st)
        Me, Ke, vol = O.tet_local(x, sig)
        vref = abs(np.linalg.det(x[1:] - x[0])) / 6
        assert vol == pytest.approx(vref, rel=1e-12)
        Gr = _grads_independent(x)
        fn = f / np.linalg.norm(f)
        sref = st * np.eye(3) + (sl - st) * np.outer(fn, fn)
        Kref = vref * Gr @ sref @ Gr.T
        assert np.allclose(Ke, Kref, rtol=1e-10, atol=1e-12 * np.abs(Kref).max())
        assert np.allclose(Ke.sum(1), 0, atol=1e-12 * np.abs(Ke).max())
        assert Me.sum() == pytest.approx(vref, rel=1e-12)
        # a P1 function reproduced exactly: K_e applied to a linear field = boundary flux form
        Me2, Ke2, _ = O.tet_local(x, 2 * sig)
        assert np.allclose(Ke2, 2 * Ke, rtol=1e-14, atol=0)


def test_conductivity_examples(golden):
    w = golden["worked_examples"]
    for key in ("conductivity_diag", "conductivity_rot"):
        e = w[key]
        assert np.allclose(O.conductivity_tensor(e["f"], e["sl"], e["st"]), e["sigma"], atol=1e-15)
    # isotropy: sl == st -> s I for any fibre
    assert np.allclose(O.conductivity_tensor([0.3, -2, 1], 0.7, 0.7), 0.7 * np.eye(3), atol=1e-15)
    with pytest.raises(O.OracleError):
        O.conductivity_tensor([0, 0, 0], 1, 1)


def test_degenerate_tet_rejected():
    x = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0], [0, 0, 1.0]])
    with pytest.raises(O.OracleError):
        O.tet_local(x, np.eye(3))


def _kuhn(nx=7, ny=6, nz=5, h=0.5, sl=0.1334177, st=0.0173515):
    xyz, tets = G.kuhn_box(nx, ny, nz, h)
    E = tets.shape[0]
    rp, col, M, K = O.assemble(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E), {0: (sl, st)})
    return xyz, tets, rp, col, M, K


def test_kuhn_interior_stencils():
    """Interior rows on the Kuhn grid (closed form):
    M/h^3: diag 0.4, axis and body-diagonal offsets 1/20, face diagonals 1/30;
    K/h: the 7-point FD stencil (2 sl + 4 st; -sl on +-x; -st on +-y,+-z; 0 elsewhere)."""
    h, sl, st = 0.5, 0.1334177, 0.0173515
    xyz, tets, rp, col, M, K = _kuhn(h=h, sl=sl, st=st)
    nx, ny = 7, 6
    i = 3 + nx * (2 + ny * 2)
    assert rp[i + 1] - rp[i] == 15
    for t in range(rp[i], rp[i + 1]):
        d = tuple(np.round((xyz[col[t]] - xyz[i]) / h).astype(int))
        nzc = sum(abs(c) for c in d)
        if d == (0, 0, 0):
            mref, kref = 0.4, 2 * sl + 4 * st
        elif nzc == 1:
            mref = 1 / 20
            kref = -sl if d[0] != 0 else -st
        elif nzc == 3:
            mref, kref = 1 / 20, 0.0
        else:
            mref, kref = 1 / 30, 0.0
        assert M[t] / h**3 == pytest.approx(mref, rel=1e-13)
        assert K[t] / h == pytest.approx(kref, abs=1e-15)


def test_global_invariants():
    xyz, tets, rp, col, M, K = _kuhn()
    n = xyz.shape[0]
    vol = 3 * 2.5 * 2.0
    assert M.sum() == pytest.approx(vol, rel=1e-12)
    assert np.abs(O.spmv(rp, col, K, np.ones(n))).max() <= 1e-12 * np.abs(K).max()
    D = np.zeros((n, n))
    Kd = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(rp))
    D[rows, col] = M
    Kd[rows, col] = K
    assert np.array_equal(D, D.T)                                       # S:164 exact
    assert np.abs(Kd - Kd.T).max() <= 1e-12 * np.abs(Kd).max()
    ev = np.linalg.eigvalsh((Kd + Kd.T) / 2)
    assert ev.min() > -1e-12                                            # S:167 PSD
    assert np.linalg.eigvalsh(D).min() > 0                              # M SPD
    assert (M >= 0).all()
    # doubling sigma doubles K, M unchanged
    _, _, _, _, M2, K2 = _kuhn(sl=2 * 0.1334177, st=2 * 0.0173515)
    assert np.array_equal(M2, M)
    assert np.allclose(K2, 2 * K, rtol=1e-14, atol=1e-18)


def test_pattern_is_mesh_graph():
    xyz, tets = G.kuhn_box(4, 3, 3, 1.0)
    n = xyz.shape[0]
    rp, col = O.pattern(n, tets)
    ref = [set([i]) for i in range(n)]
    for t in tets:
        for a, b in itertools.product(t, t):
            ref[a].add(int(b))
    for i in range(n):
        assert list(col[rp[i]:rp[i + 1]]) == sorted(ref[i])


def test_orientation_and_relabel_invariance():
    """Flipped tets (negative orientation) and a node relabelling give the same
    matrices up to the permutation (S:71 orientation fix; assembly is geometric)."""
    xyz, tets = G.kuhn_box(5, 4, 3, 0.3)
    E = tets.shape[0]
    f = G.random_fibres(E)
    cond = {0: (0.2, 0.05)}
    rp, col, M, K = O.assemble(xyz, tets, np.zeros(E, np.int32), f, cond)
    rp2, col2, M2, K2 = O.assemble(xyz, G.flip_some(tets), np.zeros(E, np.int32), f, cond)
    assert np.array_equal(col, col2)
    assert np.allclose(M2, M, rtol=1e-14) and np.allclose(K2, K, rtol=1e-12, atol=1e-15)
    xyzp, tetsp, perm = G.permute_nodes(xyz, tets)
    rp3, col3, M3, K3 = O.assemble(xyzp, tetsp, np.zeros(E, np.int32), f, cond)
    n = xyz.shape[0]
    Dk = np.zeros((n, n)); Dk3 = np.zeros((n, n))
    Dk[np.repeat(np.arange(n), np.diff(rp)), col] = K
    Dk3[np.repeat(np.arange(n), np.diff(rp3)), col3] = K3
    assert np.allclose(Dk3, Dk[np.ix_(perm, perm)], rtol=1e-12, atol=1e-15)


def test_regions_and_missing_region():
    xyz, tets = G.kuhn_box(4, 4, 4, 1.0)
    E = tets.shape[0]
    reg = (np.arange(E) % 2).astype(np.int32)
    rp, col, M, K = O.assemble(xyz, tets, reg, G.uniform_fibres(E), {0: (1.0, 1.0), 1: (1.0, 1.0)})
    rp1, col1, M1, K1 = O.assemble(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E), {0: (1.0, 1.0)})
    assert np.allclose(K, K1, rtol=1e-14, atol=1e-16)
    with pytest.raises(O.OracleError):
        O.assemble(xyz, tets, reg, G.uniform_fibres(E), {0: (1.0, 1.0)})


def test_cuboid_counts(golden):
    e = golden["worked_examples"]["cuboid_counts"]
    t3 = golden["table3_nversion"]
    xyz, tets = G.slab(*t3["domain_mm"], e["dx"])
    assert xyz.shape[0] == e["nodes"]
    xyz, tets = G.slab(1, 1, 1, 1.0)
    assert xyz.shape[0] == 8
    _, _, _, _, M, _ = (None, None, *O.assemble(xyz, tets, np.zeros(len(tets), np.int32),
                                                  G.uniform_fibres(len(tets)), {0: (1, 1)}))
    assert M.sum() == pytest.approx(1.0, rel=1e-14)
    xyz, _ = G.slab(2, 1, 1, 0.5)
    assert xyz.shape[0] == 45
