"""Pins of the oracle's SpMV, PCG (Algorithm 1) and RCM
against textbook results, library solves and brute force."""
import itertools

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.csgraph as csg
import scipy.sparse.linalg as spla

import meshgen as G
import oracle as O


def _csr(Adense):
    rows, cols = np.nonzero(Adense)
    rp = np.zeros(Adense.shape[0] + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    return np.cumsum(rp).astype(np.int32), cols.astype(np.int32), Adense[rows, cols].astype(float)


def test_spmv_examples(golden):
    e = golden["worked_examples"]["spmv_2x2"]
    rp, col, val = _csr(np.array(e["A"]))
    assert np.array_equal(O.spmv(rp, col, val, e["x"]), e["y"])
    rp, col, val = _csr(np.eye(4))
    x = np.array([1.5, -2, 3, 0.25])
    assert np.array_equal(O.spmv(rp, col, val, x), x)
    rp, col, val = _csr(np.diag([1.0, 2, 3]))
    assert np.array_equal(O.spmv(rp, col, val, np.ones(3)), [1, 2, 3])


def test_spmv_dense_random():
    rng = np.random.default_rng(3)
    for n in (1, 7, 40):
        A = rng.normal(size=(n, n)) * (rng.random((n, n)) < 0.3)
        x = rng.normal(size=n)
        rp, col, val = _csr(A)
        assert np.allclose(O.spmv(rp, col, val, x), A @ x, rtol=1e-13, atol=1e-13)


def test_pcg_2x2(golden):
    e = golden["worked_examples"]["pcg_2x2"]
    rp, col, val = _csr(np.array(e["A"]))
    x, rep = O.pcg(rp, col, val, e["b"], np.zeros(2), 1e-12, 0.0, 50)
    assert np.allclose(x, e["x"], atol=1e-10)
    assert rep.converged and rep.iters <= 2


def test_jacobi_example(golden):
    """z = r / diag(A): the first z of PCG equals S:220's example."""
    e = golden["worked_examples"]["jacobi_2x2"]
    rp, col, val = _csr(np.array(e["A"]))
    x, rep = O.pcg(rp, col, val, e["r"], np.zeros(2), 0.0, 0.0, 1, trace=True)
    assert rep.trace[0] == pytest.approx(np.linalg.norm(e["z"]), rel=1e-15)


def test_pcg_identity_and_exact_guess():
    rp, col, val = _csr(np.eye(5))
    b = np.arange(5.0)
    x, rep = O.pcg(rp, col, val, b, np.zeros(5), 1e-12, 0.0, 10)
    assert np.allclose(x, b) and rep.iters <= 1
    rp, col, val, A = G.random_spd_csr(20, seed=1)
    xs = np.linalg.solve(A, np.ones(20))
    x, rep = O.pcg(rp, col, val, A @ xs, xs, 1e-8, 0.0, 10)
    assert rep.iters == 0 and rep.converged and np.array_equal(x, xs)   # reading C4


def test_pcg_random_spd_vs_direct():
    """random SPD (A = B^T B + n I), eps_a = 1e-12 -> within 1e-8 of a dense solve."""
    rng = np.random.default_rng(11)
    for trial in range(200):
        n = int(rng.integers(1, 51))
        Bm = rng.normal(size=(n, n))
        A = Bm.T @ Bm + n * np.eye(n)
        b = rng.normal(size=n)
        rp, col, val = _csr(A)
        x, rep = O.pcg(rp, col, val, b, np.zeros(n), 1e-12, 0.0, 10 * n + 10)
        assert np.abs(x - np.linalg.solve(A, b)).max() <= 1e-8
        # unpreconditioned CG terminates in <= n+2 iterations
        x2, rep2 = O.pcg(rp, col, val, b, np.zeros(n), 1e-12, 0.0, 10 * n + 10, jacobi=False)
        assert rep2.iters <= n + 2
        assert np.abs(x2 - x).max() <= 1e-8


def test_pcg_stopping_trace_fidelity():
    """Acceptance 8: the reported stop is the FIRST k with ||z_{k+1}|| < eps_a
    or ||z_{k+1}||/||z_k|| < eps_r (consecutive reading C1), or ||z_{k+1}||/||z_0||
    in rel_mode 1; the trace is the ||z|| sequence independently recomputed here."""
    rp, col, val, A = G.random_spd_csr(60, density=0.1, seed=5)
    d = np.diag(A)
    b = G.random_vector(60, seed=9)
    for rel_mode, eps_a, eps_r in ((0, 1e-9, 0.3), (0, 1e-6, 0.0), (1, 1e-12, 1e-4)):
        x, rep = O.pcg(rp, col, val, b, np.zeros(60), eps_a, eps_r, 200, rel_mode, trace=True)
        tr = rep.trace
        # independent textbook PCG in numpy, same stopping rule
        r = b.copy(); z = r / d; p = z.copy(); rho = r @ z; zs = [np.linalg.norm(z)]
        xx = np.zeros(60)
        for k in range(200):
            q = A @ p; al = rho / (p @ q); xx += al * p; r -= al * q; z = r / d
            zs.append(np.linalg.norm(z))
            ref = zs[-2] if rel_mode == 0 else zs[0]
            if zs[-1] < eps_a or zs[-1] / ref < eps_r:
                break
            rn = r @ z; p = z + (rn / rho) * p; rho = rn
        assert rep.iters == len(zs) - 1
        assert np.allclose(tr, zs, rtol=1e-9)
        assert np.allclose(x, xx, rtol=1e-9, atol=1e-12)
        for k in range(1, len(tr) - 1):      # no earlier k satisfied the rule
            ref = tr[k - 1] if rel_mode == 0 else tr[0]
            assert not (tr[k] < eps_a or tr[k] / ref < eps_r)


def test_pcg_max_iters_not_converged_and_residual_recurrence():
    rp, col, val, A = G.random_spd_csr(50, density=0.2, seed=2)
    b = G.random_vector(50, seed=4)
    x, rep = O.pcg(rp, col, val, b, np.zeros(50), 1e-14, 0.0, 3)
    assert rep.iters == 3 and not rep.converged
    x, rep = O.pcg(rp, col, val, b, np.zeros(50), 1e-12, 0.0, 500)
    # ||(b - A x) / d|| equals the reported ||z|| up to rounding (S:235 recurrence)
    zt = (b - A @ x) / np.diag(A)
    assert abs(np.linalg.norm(zt) - rep.znorm) <= 1e-8 * np.linalg.norm(b)


def test_pcg_fem_system_vs_spsolve():
    """Tight tolerance on an assembled monodomain matrix vs scipy's direct solve."""
    xyz, tets = G.kuhn_box(9, 7, 5, 0.5)
    E = tets.shape[0]
    rp, col, M, K = O.assemble(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E),
                               {0: (0.1334177, 0.0173515)})
    A = O.system_matrix(M, K, 140.0, 0.01, 0.5, 0.05)
    n = xyz.shape[0]
    b = G.random_vector(n, seed=12)
    x, rep = O.pcg(rp, col, A, b, np.zeros(n), 1e-13, 0.0, 500)
    xs = spla.spsolve(sp.csr_matrix((A, col, rp), shape=(n, n)).tocsc(), b)
    assert np.abs(x - xs).max() <= 1e-10 * np.abs(xs).max()
    assert rep.iters < 60   # kappa(D^-1 A) ~ 4 -> fast convergence


def _bandwidth(rp, col, perm=None):
    n = len(rp) - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    if perm is None:
        return int(np.abs(rows - col).max()) if len(col) else 0
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    return int(np.abs(inv[rows] - inv[col]).max())


def test_rcm_basic_cases():
    # tridiagonal: bandwidth 1 preserved
    n = 9
    A = np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1)
    rp, col, _ = _csr(A)
    perm = O.rcm(rp, col)
    assert sorted(perm) == list(range(n))
    assert _bandwidth(rp, col, perm) == 1
    # diagonal only: bandwidth 0
    rp, col, _ = _csr(np.eye(5))
    perm = O.rcm(rp, col)
    assert sorted(perm) == list(range(5)) and _bandwidth(rp, col, perm) == 0
    # 5-node star centred at 4: RCM < original 4 and >= the brute-force optimum 2
    A = np.eye(5)
    A[4, :] = A[:, 4] = 1
    rp, col, _ = _csr(A)
    perm = O.rcm(rp, col)
    best = min(_bandwidth(rp, col, np.array(p)) for p in itertools.permutations(range(5)))
    assert best == 2 and best <= _bandwidth(rp, col, perm) < 4


def test_rcm_tie_rules_match_textbook():
    """S:146 tie rules reproduce the plain textbook RCM written independently here."""
    xyz, tets = G.kuhn_box(5, 4, 3, 1.0)
    xyz, tets, _ = G.permute_nodes(xyz, tets, seed=3)
    rp, col = O.pattern(xyz.shape[0], tets)
    n = xyz.shape[0]
    adj = [set(col[rp[i]:rp[i + 1]]) - {i} for i in range(n)]
    deg = [len(a) for a in adj]
    seen = [False] * n
    order = []
    for s in sorted(range(n), key=lambda v: (deg[v], v)):
        if seen[s]:
            continue
        seen[s] = True
        q = [s]
        while q:
            v = q.pop(0)
            order.append(v)
            nb = sorted([w for w in adj[v] if not seen[w]], key=lambda w: (deg[w], w))
            for w in nb:
                seen[w] = True
            q.extend(nb)
    assert list(O.rcm(rp, col)) == order[::-1]


def test_rcm_reduces_bandwidth_on_permuted_mesh():
    xyz, tets = G.kuhn_box(12, 8, 6, 1.0)
    n0 = _bandwidth(*O.pattern(xyz.shape[0], tets))
    xyz, tets, _ = G.permute_nodes(xyz, tets)
    rp, col = O.pattern(xyz.shape[0], tets)
    perm = O.rcm(rp, col)
    assert _bandwidth(rp, col, perm) < _bandwidth(rp, col)
    assert _bandwidth(rp, col, perm) <= 2 * n0
    # same bandwidth class as scipy's RCM (a library routine, different ties)
    sperm = csg.reverse_cuthill_mckee(sp.csr_matrix((np.ones(len(col)), col, rp)), symmetric_mode=True)
    assert _bandwidth(rp, col, perm) <= 1.5 * _bandwidth(rp, col, np.asarray(sperm))


@pytest.mark.parametrize("model", ["tt2006", "ms", "crn"])
def test_oracle_threads_bitwise(model):
    """The OpenMP pragmas sit only on independent per-row / per-node loops
    (oracle.c header): a trajectory at 1 thread and at 4 threads is bitwise
    identical (V, every cell state, LAT, iteration counts)."""
    import meshgen as G
    xyz, tets = G.kuhn_box(23, 9, 6, 0.5)
    E = tets.shape[0]
    stim = O.Stimulus(G.nodes_in_box(xyz, (0, 0, 0), (1.5, 1.5, 1.5)), 0.0, 2.0, 50.0)
    runs = []
    try:
        for k in (1, 4):
            O.set_threads(k)
            sim = O.Monodomain(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E),
                               {0: (0.1334177, 0.0173515)}, O.Config(dt=0.05, model=model), [stim]).run(60)
            runs.append(sim)
    finally:
        O.set_threads(O.max_threads())
    a, b = runs
    assert np.array_equal(a.Vk, b.Vk) and np.array_equal(a.U, b.U) and np.array_equal(a.lat, b.lat)
    assert [r.iters for r in a.reports] == [r.iters for r in b.reports]
    assert (a.lat >= 0).any()
