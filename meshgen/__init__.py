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


# --------------------------------------------------------------------------
# Synthetic biventricular-sized mesh (BASELINE configs[3]; recipe in DESIGN.md)
# --------------------------------------------------------------------------
LV_ENDO, LV_EPI = (25.0, 25.0, 45.0), (35.0, 35.0, 52.0)
RV_ENDO, RV_EPI = (40.0, 28.0, 40.0), (46.0, 33.0, 46.0)
RV_SHIFT = 18.0


def _inside(p, ax, cx=0.0):
    return ((p[..., 0] - cx) / ax[0]) ** 2 + (p[..., 1] / ax[1]) ** 2 + (p[..., 2] / ax[2]) ** 2 <= 1.0


def _radial(p, ax, cx=0.0):
    return np.sqrt(((p[..., 0] - cx) / ax[0]) ** 2 + (p[..., 1] / ax[1]) ** 2 + (p[..., 2] / ax[2]) ** 2)


def biv(h: float, seed=SEED, jitter_frac=0.15, permute=True):
    """Voxelised union of two truncated ellipsoidal shells (z <= 0), Kuhn-split.

    Returns dict(xyz, tets, region (0 LV, 1 RV), fibre, endo_nodes).  Fibres:
    helix angle 60 deg (endo) -> -60 deg (epi) about the local circumferential
    direction, rotated towards the apex-base axis (rule-based, per element)."""
    lo = np.array([-36.0, -36.0, -53.0])
    hi = np.array([RV_SHIFT + 47.0, 36.0, 0.0])
    nc = np.ceil((hi - lo) / h).astype(int)
    ci = np.stack(np.meshgrid(*(np.arange(m) for m in nc), indexing="ij"), -1).reshape(-1, 3)
    cen = lo + (ci + 0.5) * h
    lv = _inside(cen, LV_EPI) & ~_inside(cen, LV_ENDO)
    rv = _inside(cen, RV_EPI, RV_SHIFT) & ~_inside(cen, RV_ENDO, RV_SHIFT) & ~_inside(cen, LV_ENDO)
    keep = (lv | rv) & (cen[:, 2] <= 0.0)
    cells = ci[keep]
    cell_rv = (rv & ~lv)[keep]
    # nodes: corners of kept cells, compact numbering
    nx, ny, nz = nc + 1
    gid = lambda ijk: ijk[..., 0] + nx * (ijk[..., 1] + ny * ijk[..., 2])
    corners = cells[:, None, :] + _KUHN_POS.reshape(-1, 3)[None, :, :]          # (C, 24, 3)
    g = gid(corners).reshape(-1)
    uniq, inv = np.unique(g, return_inverse=True)
    tets = inv.reshape(-1, 6, 4).reshape(-1, 4).astype(np.int32)
    region = np.repeat(cell_rv.astype(np.int32), 6)
    k = uniq // (nx * ny)
    j = (uniq // nx) % ny
    i = uniq % nx
    xyz = lo + np.stack([i, j, k], 1) * h
    # jitter nodes, rejecting moves that flatten a tet below 0.2 of its volume
    rng = np.random.default_rng(seed)
    d = rng.uniform(-jitter_frac * h, jitter_frac * h, size=xyz.shape)
    v0 = h ** 3 / 6.0
    for _ in range(20):
        x = xyz + d
        p = x[tets]
        vol = np.abs(np.einsum("ij,ij->i", p[:, 1] - p[:, 0], np.cross(p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]))) / 6
        bad = vol < 0.2 * v0
        if not bad.any():
            break
        d[np.unique(tets[bad])] = 0.0
    xyz = xyz + d
    # rule-based fibres from the element centroid
    c = xyz[tets].mean(1)
    isr = region == 1
    cx = np.where(isr, RV_SHIFT, 0.0)
    rad = np.where(isr, _radial(c, RV_ENDO, RV_SHIFT), _radial(c, LV_ENDO))
    rad_epi = np.where(isr, _radial(c, RV_EPI, RV_SHIFT), _radial(c, LV_EPI))
    # transmural coordinate: 0 on the endo ellipsoid, 1 on the epi ellipsoid
    e = np.clip((rad - 1.0) / np.maximum(rad - rad_epi, 1e-12), 0.0, 1.0)
    ang = np.deg2rad(60.0 - 120.0 * e)
    circ = np.stack([-c[:, 1], c[:, 0] - cx, np.zeros(len(c))], 1)
    circ /= np.maximum(np.linalg.norm(circ, axis=1, keepdims=True), 1e-12)
    fib = np.cos(ang)[:, None] * circ + np.sin(ang)[:, None] * np.array([0.0, 0.0, 1.0])
    # endocardial nodes of the LV (for stimulus sites)
    endo = np.nonzero(_radial(xyz, LV_ENDO) < 1.0 + 1.5 * h / LV_ENDO[0])[0].astype(np.int32)
    out = dict(xyz=xyz, tets=tets, region=region, fibre=fib, endo_nodes=endo)
    if permute:
        xyz2, tets2, perm = permute_nodes(xyz, tets, seed=seed + 1)
        invp = np.empty(len(perm), np.int64)
        invp[perm] = np.arange(len(perm))
        out.update(xyz=xyz2, tets=tets2, endo_nodes=invp[endo].astype(np.int32))
    return out


def biv_stimuli(mesh, n_sites=5, radius=1.5, seed=SEED):
    """Five spheres of radius 1.5 mm around seeded LV endocardial nodes (P:320 'five initial stimuli')."""
    rng = np.random.default_rng(seed + 7)
    xyz = mesh["xyz"]
    sites = rng.choice(mesh["endo_nodes"], size=n_sites, replace=False)
    out = []
    for s in sites:
        nodes = np.nonzero(np.sum((xyz - xyz[s]) ** 2, axis=1) <= radius ** 2)[0].astype(np.int32)
        out.append(nodes)
    return out


# --------------------------------------------------------------------------
# Surface (triangle) meshes embedded in 3-D ("surface meshes")
# --------------------------------------------------------------------------
def tri_grid(nx: int, ny: int, dx: float, origin=(0.0, 0.0, 0.0)):
    """nx*ny-node planar grid in z = origin[2], each square cut into 2 triangles
    along its (0,0)-(1,1) diagonal.  Returns xyz (n,3), tris (E,3)."""
    i = np.arange(nx)
    j = np.arange(ny)
    J, I = np.meshgrid(j, i, indexing="ij")
    xyz = np.zeros((nx * ny, 3))
    xyz[:, 0] = I.reshape(-1) * dx + origin[0]
    xyz[:, 1] = J.reshape(-1) * dx + origin[1]
    xyz[:, 2] = origin[2]
    ci, cj = np.meshgrid(np.arange(nx - 1), np.arange(ny - 1), indexing="xy")
    v00 = (ci + nx * cj).reshape(-1)
    v10, v01, v11 = v00 + 1, v00 + nx, v00 + nx + 1
    tris = np.concatenate([np.stack([v00, v10, v11], 1), np.stack([v00, v11, v01], 1)])
    return xyz, tris.astype(np.int32)


def unit_square(N: int):
    """[0,1]^2 (z = 0) with N cells per side, 2 triangles per cell (the MMS domain of P:250)."""
    return tri_grid(N + 1, N + 1, 1.0 / N)


def rotate(xyz, seed=SEED):
    """A seeded rigid rotation of the coordinates (surface meshes must not care)."""
    q, _ = np.linalg.qr(np.random.default_rng(seed).normal(size=(3, 3)))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return xyz @ q.T, q


def sphere(level: int, radius: float = 10.0):
    """Icosphere surface (subdivided icosahedron, `level` 2x refinements) of the
    given radius (a closed surface: no boundary)."""
    t = (1.0 + 5 ** 0.5) / 2.0
    v = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t], [0, -1, -t],
                  [0, 1, -t], [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], float)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4],
                  [11, 10, 2], [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8],
                  [3, 8, 9], [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]])
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    for _ in range(level):
        e = np.sort(np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]]), axis=1)
        ue, inv = np.unique(e, axis=0, return_inverse=True)
        mid = v[ue[:, 0]] + v[ue[:, 1]]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        m = len(v) + inv.reshape(3, -1).T            # midpoints of edges 01, 12, 20
        v = np.concatenate([v, mid])
        a, b, c = f[:, 0], f[:, 1], f[:, 2]
        m01, m12, m20 = m[:, 0], m[:, 1], m[:, 2]
        f = np.concatenate([np.stack([a, m01, m20], 1), np.stack([b, m12, m01], 1),
                            np.stack([c, m20, m12], 1), np.stack([m01, m12, m20], 1)])
    return v * radius, f.astype(np.int32)


def sphere_fibres(xyz, tris):
    """Per-triangle fibre along the local 'latitude' direction (tangent, rule-based)."""
    c = xyz[tris].mean(1)
    f = np.stack([-c[:, 1], c[:, 0], np.zeros(len(c))], 1)
    bad = np.linalg.norm(f, axis=1) < 1e-9 * np.linalg.norm(c, axis=1)
    f[bad] = [1.0, 0.0, 0.0]
    return f / np.linalg.norm(f, axis=1, keepdims=True)


def cohort_members(count: int, seed=SEED, base=(41, 15, 7), dx=0.5):
    """Seeded cohort of `count` N-version-like slabs (SURVEY 8f f1, P:349-353:
    many patient meshes with per-patient settings).  Member m: Kuhn slab of
    (nx, ny, nz) = base + (U{-6..6}, U{-3..3}, U{-2..2}) nodes at spacing dx,
    node numbering randomly permuted, one fibre direction in the x-y plane at
    U[-30, 30] degrees, conductivity scale U[0.8, 1.2], TT2006 parameter resets
    GKr, GKs x U[0.7, 1.3] and GCaL x U[0.8, 1.2] (factors, applied by the
    caller to its defaults), corner stimulus box <= 1.5 mm.  Returns a list of
    dicts: xyz, tets, fibre, sigma_scale, param_factors, stim_nodes."""
    rng = np.random.default_rng(seed)
    out = []
    for m in range(count):
        nx = base[0] + int(rng.integers(-6, 7))
        ny = base[1] + int(rng.integers(-3, 4))
        nz = base[2] + int(rng.integers(-2, 3))
        xyz, tets = kuhn_box(nx, ny, nz, dx)
        stim = nodes_in_box(xyz, (0, 0, 0), (1.5, 1.5, 1.5))
        perm_seed = int(rng.integers(1 << 31))
        xyz, tets, perm = permute_nodes(xyz, tets, seed=perm_seed)   # perm: new -> old
        inv = np.empty(perm.shape[0], np.int64)
        inv[perm] = np.arange(perm.shape[0])
        stim = np.sort(inv[stim]).astype(np.int32)
        ang = np.deg2rad(rng.uniform(-30.0, 30.0))
        fib = uniform_fibres(tets.shape[0], (np.cos(ang), np.sin(ang), 0.0))
        out.append(dict(xyz=xyz, tets=tets, fibre=fib, sigma_scale=float(rng.uniform(0.8, 1.2)),
                        param_factors={"GKr": float(rng.uniform(0.7, 1.3)),
                                       "GKs": float(rng.uniform(0.7, 1.3)),
                                       "GCaL": float(rng.uniform(0.8, 1.2))},
                        stim_nodes=stim))
    return out


def sphere_cohort_members(count: int, seed=SEED, level: int = 8, radius: float = 28.0):
    """Seeded cohort of `count` atrium-surface-sized icospheres (SURVEY 8f f1 with
    P:349-353's 660 k-node left-atrium surface meshes, Mitchell-Schaeffer):
    member m: radius x U[0.9, 1.1], tangent fibres rotated about the local normal
    by U[-30, 30] degrees, conductivity scale U[0.8, 1.2], MS tau_close x
    U[0.8, 1.2] and tau_in x U[0.9, 1.1] (factors applied by the caller), a polar
    cap stimulus (the 2 mm cap of the bench's sphere workloads, scaled).  Same
    dict keys as cohort_members; "tets" holds the triangles."""
    rng = np.random.default_rng(seed)
    base_xyz, tris = sphere(level, 1.0)
    out = []
    for m in range(count):
        r = radius * float(rng.uniform(0.9, 1.1))
        xyz = base_xyz * r
        f = sphere_fibres(xyz, tris)
        ang = np.deg2rad(rng.uniform(-30.0, 30.0))
        c = xyz[tris].mean(1)
        nrm = c / np.linalg.norm(c, axis=1, keepdims=True)
        f = np.cos(ang) * f + np.sin(ang) * np.cross(nrm, f)      # rotate in the tangent plane
        stim = np.nonzero(xyz[:, 2] >= r - 2.0 * r / radius)[0].astype(np.int32)
        out.append(dict(xyz=xyz, tets=tris, fibre=f, sigma_scale=float(rng.uniform(0.8, 1.2)),
                        param_factors={"tau_close": float(rng.uniform(0.8, 1.2)),
                                       "tau_in": float(rng.uniform(0.9, 1.1))},
                        stim_nodes=stim))
    return out
