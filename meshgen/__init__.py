"""Seeded synthetic INPUT generators shared by the oracle tests and the CUDA path.

This module holds none of the method's arithmetic (no FEM, no ionic model, no
solver): it only produces meshes (node coordinates, tetrahedra, region tags,
fibre vectors), node selections (stimulus boxes, Dirichlet boundaries) and
seeded random vectors / permutations.  Recipes are stated in DESIGN.md
("Inputs").
"""
from __future__ import annotations

import itertools

import numpy as np

SEED = 2510012011

# The six path-simplices of the unit cube around the (0,0,0)-(1,1,1) diagonal
# (Kuhn / Freudenthal split; "fixed 6-tet split, consistent diagonal").
_KUHN = []
for perm in itertools.permutations(range(3)):
    v = [0, 0, 0]
    verts = [tuple(v)]
    for ax in perm:
        v[ax] = 1
        verts.append(tuple(v))
    _KUHN.append(verts)
_KUHN = np.array(_KUHN, dtype=np.int64)  # (6, 4, 3) corner offsets


def _positive(corners: np.ndarray) -> np.ndarray:
    """Reorder the 4 corners of each template tet to positive orientation."""
    out = corners.copy()
    for t in range(out.shape[0]):
        d = out[t, 1:] - out[t, 0]
        if np.linalg.det(d.astype(float)) < 0:
            out[t, [1, 2]] = out[t, [2, 1]]
    return out


_KUHN_POS = _positive(_KUHN)


def kuhn_box(nx: int, ny: int, nz: int, dx: float, origin=(0.0, 0.0, 0.0)):
    """Structured nx*ny*nz-node grid with spacing dx, each cube cut into 6 tets.

    Node (i,j,k) -> index i + nx*(j + ny*k), coordinates origin + dx*(i,j,k).
    Returns xyz (n,3) float64 and tets (E,4) int32 (positively oriented)."""
    i = np.arange(nx, dtype=np.float64)
    j = np.arange(ny, dtype=np.float64)
    k = np.arange(nz, dtype=np.float64)
    X, Y, Z = np.meshgrid(i, j, k, indexing="ij")
    xyz = np.empty((nx * ny * nz, 3))
    # index i + nx*(j + ny*k): i fastest
    xyz[:, 0] = X.transpose(2, 1, 0).reshape(-1) * dx + origin[0]
    xyz[:, 1] = Y.transpose(2, 1, 0).reshape(-1) * dx + origin[1]
    xyz[:, 2] = Z.transpose(2, 1, 0).reshape(-1) * dx + origin[2]
    ci = np.arange(nx - 1, dtype=np.int64)
    cj = np.arange(ny - 1, dtype=np.int64)
    ck = np.arange(nz - 1, dtype=np.int64)
    base = (ci[None, None, :] + nx * (cj[None, :, None] + ny * ck[:, None, None])).reshape(-1)
    offs = _KUHN_POS[..., 0] + nx * (_KUHN_POS[..., 1] + ny * _KUHN_POS[..., 2])  # (6,4)
    tets = (base[:, None, None] + offs[None, :, :]).reshape(-1, 4).astype(np.int32)
    return xyz, tets


def slab(lx: float, ly: float, lz: float, dx: float):
    """Cuboid [0,lx]x[0,ly]x[0,lz] meshed with Kuhn tets."""
    n = [int(round(L / dx)) + 1 for L in (lx, ly, lz)]
    for L, m in zip((lx, ly, lz), n):
        if abs((m - 1) * dx - L) > 1e-9 * max(1.0, L):
            raise ValueError("dimensions must be multiples of dx")
    return kuhn_box(n[0], n[1], n[2], dx)


def unit_cube(N: int):
    """[0,1]^3 with N cells per side (MMS config)."""
    return kuhn_box(N + 1, N + 1, N + 1, 1.0 / N)


def uniform_fibres(E: int, f=(1.0, 0.0, 0.0)) -> np.ndarray:
    return np.tile(np.asarray(f, np.float64), (E, 1))


def nodes_in_box(xyz, lo, hi, tol=1e-9) -> np.ndarray:
    """Indices of nodes with lo <= x <= hi componentwise (inclusive, +-tol)."""
    lo = np.asarray(lo, float) - tol
    hi = np.asarray(hi, float) + tol
    m = np.all((xyz >= lo) & (xyz <= hi), axis=1)
    return np.nonzero(m)[0].astype(np.int32)


def box_boundary(xyz, tol=1e-9) -> np.ndarray:
    """Nodes on any face of the bounding box (MMS Dirichlet set)."""
    lo, hi = xyz.min(0), xyz.max(0)
    m = np.any((np.abs(xyz - lo) <= tol) | (np.abs(xyz - hi) <= tol), axis=1)
    return np.nonzero(m)[0].astype(np.int32)


def nearest_node(xyz, p) -> int:
    """Nearest node to p; ties -> lowest index."""
    d = np.sum((xyz - np.asarray(p, float)) ** 2, axis=1)
    return int(np.argmin(d))


def permute_nodes(xyz, tets, seed=SEED):
    """Random relabelling of nodes (so RCM / partitioning do real work)."""
    rng = np.random.default_rng(seed)
    n = xyz.shape[0]
    perm = rng.permutation(n)            # new -> old
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    return xyz[perm].copy(), inv[tets].astype(np.int32), perm


def flip_some(tets, frac=0.3, seed=SEED):
    """Swap two vertices of a random subset of tets (negative orientation)."""
    rng = np.random.default_rng(seed)
    t = tets.copy()
    m = rng.random(t.shape[0]) < frac
    t[m, 1], t[m, 2] = tets[m, 2], tets[m, 1]
    return t


def jitter(xyz, h, amount=0.15, seed=SEED, fixed=None):
    """Uniform +-amount*h perturbation of node coordinates (fixed nodes untouched)."""
    rng = np.random.default_rng(seed)
    d = rng.uniform(-amount * h, amount * h, size=xyz.shape)
    if fixed is not None:
        d[np.asarray(fixed)] = 0.0
    return xyz + d


def random_fibres(E: int, seed=SEED) -> np.ndarray:
    rng = np.random.default_rng(seed)
    f = rng.normal(size=(E, 3))
    return f / np.linalg.norm(f, axis=1, keepdims=True)


def random_vector(n: int, seed=SEED, lo=-1.0, hi=1.0) -> np.ndarray:
    return np.random.default_rng(seed).uniform(lo, hi, n)


def random_spd_csr(n: int, density=0.2, seed=SEED):
    """Random sparse symmetric pattern with diagonal dominance -> SPD (CSR, sorted)."""
    rng = np.random.default_rng(seed)
    Adense = np.zeros((n, n))
    mask = rng.random((n, n)) < density
    mask = mask | mask.T
    vals = rng.uniform(-1, 1, (n, n))
    vals = (vals + vals.T) / 2
    Adense[mask] = vals[mask]
    np.fill_diagonal(Adense, 0.0)
    np.fill_diagonal(Adense, np.abs(Adense).sum(1) + rng.uniform(0.5, 2.0, n))
    rows, cols = np.nonzero(Adense)
    rowptr = np.zeros(n + 1, np.int64)
    np.add.at(rowptr, rows + 1, 1)
    return np.cumsum(rowptr).astype(np.int32), cols.astype(np.int32), Adense[rows, cols].copy(), Adense
