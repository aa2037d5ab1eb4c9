"""Pins of the oracle's surface (triangle-in-3-D) elements ("triangular or
tetrahedral elements") and of the paper's own MMS setup,
a triangulated unit square with Dirichlet data on the perimeter."""
import numpy as np
import pytest

import meshgen as G
import oracle as O


def test_unit_right_triangle_closed_form(golden):
    x = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0.0]])
    Me, Ke, area = O.tri_local(x, np.eye(3))
    assert area == pytest.approx(0.5, rel=1e-15)
    assert np.allclose(Me, (np.ones((3, 3)) + np.eye(3)) / 24, rtol=0, atol=1e-16)
    assert np.allclose(Ke, [[1, -0.5, -0.5], [-0.5, 0.5, 0], [-0.5, 0, 0.5]], atol=1e-15)
    Me2, Ke2, _ = O.tri_local(x, 2 * np.eye(3))
    assert np.allclose(Ke2, 2 * Ke, rtol=1e-15)


def _grads_lsq(x):
    """In-plane gradients from E (E^T E)^{-1} (independent of the oracle's cross products)."""
    E = np.stack([x[1] - x[0], x[2] - x[0]], 1)          # 3x2
    Gr = E @ np.linalg.inv(E.T @ E)                       # columns: grad phi_1, grad phi_2
    g1, g2 = Gr[:, 0], Gr[:, 1]
    return np.stack([-(g1 + g2), g1, g2])


def test_random_triangles_vs_independent_gradients():
    rng = np.random.default_rng(17)
    for _ in range(50):
        x = rng.normal(size=(3, 3))
        f = rng.normal(size=3)
        sl, st = rng.uniform(0.05, 2, 2)
        sig = O.conductivity_tensor(f, sl, st)
        Me, Ke, area = O.tri_local(x, sig)
        aref = 0.5 * np.linalg.norm(np.cross(x[1] - x[0], x[2] - x[0]))
        assert area == pytest.approx(aref, rel=1e-12)
        Gr = _grads_lsq(x)
        Kref = aref * Gr @ sig @ Gr.T
        assert np.allclose(Ke, Kref, rtol=1e-10, atol=1e-12 * np.abs(Kref).max())
        assert np.allclose(Ke.sum(1), 0.0, atol=1e-12 * np.abs(Ke).max())
        assert Me.sum() == pytest.approx(aref, rel=1e-12)


def test_surface_assembly_is_rotation_invariant():
    """A planar mesh and the same mesh rigidly rotated in 3-D (fibres rotated too)
    give identical M and K."""
    xyz, tris = G.tri_grid(7, 5, 0.4)
    E = tris.shape[0]
    fib = np.tile([0.6, 0.8, 0.0], (E, 1))
    cond = {0: (0.1334177, 0.0173515)}
    rp, col, M, K = O.assemble(xyz, tris, np.zeros(E, np.int32), fib, cond)
    xr, Q = G.rotate(xyz)
    rp2, col2, M2, K2 = O.assemble(xr, tris, np.zeros(E, np.int32), fib @ Q.T, cond)
    assert np.array_equal(col, col2)
    assert np.allclose(M2, M, rtol=1e-12) and np.allclose(K2, K, rtol=1e-10, atol=1e-14)
    # a fibre component normal to the plane does not act (tangent-plane restriction)
    fn = fib + np.array([0.0, 0.0, 5.0])
    _, _, _, Kn = O.assemble(xyz, tris, np.zeros(E, np.int32), fn / np.linalg.norm(fn, axis=1, keepdims=True),
                             {0: (0.1334177, 0.0173515)})
    f_in = fib * (1.0 / np.linalg.norm(fn, axis=1, keepdims=True))     # in-plane part of the unit fibre
    s_eff = 0.0173515 + (0.1334177 - 0.0173515) * np.sum(f_in ** 2, axis=1)
    assert not np.allclose(Kn, K)   # the longitudinal weight shrinks with the in-plane fibre length
    assert np.all(s_eff < 0.1334177)


def test_sphere_invariants():
    v, f = G.sphere(3)
    E = f.shape[0]
    rp, col, M, K = O.assemble(v, f, np.zeros(E, np.int32), G.sphere_fibres(v, f), {0: (1.0, 0.3)})
    area = sum(0.5 * np.linalg.norm(np.cross(v[t[1]] - v[t[0]], v[t[2]] - v[t[0]])) for t in f)
    assert M.sum() == pytest.approx(area, rel=1e-12)
    assert np.abs(O.spmv(rp, col, K, np.ones(len(v)))).max() < 1e-12 * np.abs(K).max()
    n = len(v)
    Kd = np.zeros((n, n))
    Kd[np.repeat(np.arange(n), np.diff(rp)), col] = K
    assert np.abs(Kd - Kd.T).max() <= 1e-12 * np.abs(Kd).max()
    assert np.linalg.eigvalsh((Kd + Kd.T) / 2).min() > -1e-10


def test_mms_unit_square_order():
    """The paper's own MMS geometry: [0,1]^2 triangulated, Dirichlet w on the
    perimeter, Crank-Nicolson; observed L2 order in [1.7, 2.3]."""
    errs = []
    for N in (8, 16, 32):
        xyz, tris = G.unit_square(N)
        out = O.run_mms(xyz, tris, G.box_boundary(xyz[:, :2]), dt=0.01 * 8 / N, T=0.5, tol=1e-11)
        errs.append(out["err_M"])
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all((orders > 1.7) & (orders < 2.3)), orders
