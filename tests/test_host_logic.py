"""Host-side logic of the library, checked on CPU (no GPU): the sparsity
pattern and RCM (bit-exact against the oracle: integer work), the row-block
partition / halo plan of the multi-GPU path, and -- with world_size 2 over
gloo -- the split-phase distributed PCG schedule that the CUDA kernels of
pcg_split.cu implement, driven by the library's own partition plan."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import meshgen as G
import oracle as O


@pytest.fixture(scope="module")
def T():
    import paper_2510_12011_b200 as T
    return T


@pytest.mark.parametrize("dims,perm", [((5, 4, 3), False), ((9, 6, 4), True), ((2, 2, 2), False)])
def test_pattern_matches_oracle(T, dims, perm):
    xyz, tets = G.kuhn_box(*dims, 0.5)
    if perm:
        xyz, tets, _ = G.permute_nodes(xyz, tets, seed=4)
    rp, col = T.tc_mesh_pattern(xyz.shape[0], tets)
    orp, ocol = O.pattern(xyz.shape[0], tets)
    assert np.array_equal(rp, orp) and np.array_equal(col, ocol)


@pytest.mark.parametrize("dims,seed", [((7, 5, 4), 1), ((12, 3, 3), 2), ((6, 6, 6), 3)])
def test_rcm_matches_oracle(T, dims, seed):
    xyz, tets = G.kuhn_box(*dims, 1.0)
    xyz, tets, _ = G.permute_nodes(xyz, tets, seed=seed)
    rp, col = O.pattern(xyz.shape[0], tets)
    assert np.array_equal(T.tc_rcm(rp.astype(np.int64), col), O.rcm(rp, col))


def _internal_pattern(dims, seed=7, nparts=None):
    """RCM internal order (oracle RCM == library RCM); with nparts, followed by
    the library's interior-first order of the nparts row blocks."""
    xyz, tets = G.kuhn_box(*dims, 1.0)
    xyz, tets, _ = G.permute_nodes(xyz, tets, seed=seed)
    n = xyz.shape[0]
    rp, col = O.pattern(n, tets)
    perm = O.rcm(rp, col)
    if nparts:
        import paper_2510_12011_b200 as T
        inv = np.empty(n, np.int64)
        inv[perm] = np.arange(n)
        rpi, coli = O.pattern(n, inv[tets].astype(np.int32))
        order, _ = T.tc_interior_first(rpi.astype(np.int64), coli, nparts)
        perm = perm[order]
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    tets_i = inv[tets].astype(np.int32)
    rpi, coli = O.pattern(n, tets_i)
    return xyz[perm], tets_i, rpi, coli


@pytest.mark.parametrize("dims,nparts", [((11, 6, 5), 2), ((9, 7, 4), 3), ((14, 5, 5), 5)])
def test_interior_first_order(T, dims, nparts):
    """tc_interior_first: a permutation inside each row block of the plan;
    the first n_interior rows of a block read no column outside it, every
    later row reads at least one; ghost sets and block bounds are unchanged."""
    xyz, tets, rp, col = _internal_pattern(dims)
    n = rp.shape[0] - 1
    order, nint = T.tc_interior_first(rp.astype(np.int64), col, nparts)
    assert np.array_equal(np.sort(order), np.arange(n))
    b = T.tc_partition_plan(rp, col, nparts, 0)["bounds"]
    inv = np.empty(n, np.int64)
    inv[order] = np.arange(n)
    for p in range(nparts):
        g0, g1 = b[p], b[p + 1]
        assert np.all((order[g0:g1] >= g0) & (order[g0:g1] < g1))          # block preserved
        outside = [np.any((col[rp[i]:rp[i + 1]] < g0) | (col[rp[i]:rp[i + 1]] >= g1)) for i in order[g0:g1]]
        k = int(nint[p])
        assert 0 < k < g1 - g0 and not any(outside[:k]) and all(outside[k:])
        assert np.all(np.diff(order[g0:g0 + k]) > 0) and np.all(np.diff(order[g0 + k:g1]) > 0)   # stable
    # the plan of the reordered pattern has the same ghost sets (as sets of old indices)
    rows = np.repeat(np.arange(n), np.diff(rp))
    m = np.zeros(n + 1, np.int64)
    np.add.at(m, inv[rows] + 1, 1)
    rp2 = np.cumsum(m)
    col2 = np.empty_like(col)
    fill = rp2[:-1].copy()
    for r, c in zip(inv[rows], inv[col]):
        col2[fill[r]] = c
        fill[r] += 1
    for r in range(n):
        col2[rp2[r]:rp2[r + 1]] = np.sort(col2[rp2[r]:rp2[r + 1]])
    for p in range(nparts):
        g_old = T.tc_partition_plan(rp, col, nparts, p)["ghosts"]
        g_new = T.tc_partition_plan(rp2, col2, nparts, p)["ghosts"]
        assert np.array_equal(np.sort(order[g_new]), g_old)


@pytest.mark.parametrize("nparts", [2, 3, 5])
def test_partition_plan_invariants(T, nparts):
    xyz, tets, rp, col = _internal_pattern((11, 6, 5))
    n = rp.shape[0] - 1
    plans = [T.tc_partition_plan(rp, col, nparts, p) for p in range(nparts)]
    b = plans[0]["bounds"]
    assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) > 0)
    for p, pl in enumerate(plans):
        g0, g1 = b[p], b[p + 1]
        cols = col[rp[g0]:rp[g1]]
        expect = np.unique(cols[(cols < g0) | (cols >= g1)])
        assert np.array_equal(pl["ghosts"], expect)
        owners = np.searchsorted(b, pl["ghosts"], side="right") - 1
        assert np.array_equal(np.unique(owners), pl["nbr"])
        for j, q in enumerate(pl["nbr"]):
            gq = pl["ghosts"][pl["recv_off"][j]:pl["recv_off"][j + 1]]
            assert np.all(owners[pl["recv_off"][j]:pl["recv_off"][j + 1]] == q)
            # what q sends to p is exactly what p receives from q, same order
            ql = plans[q]
            jq = list(ql["nbr"]).index(p)
            sent = ql["send_g"][ql["send_off"][jq]:ql["send_off"][jq + 1]]
            assert np.array_equal(sent, gq)


# ---------------------------------------------------------------- gloo, world_size 2
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    """Split-phase PCG of pcg_split.cu, rank-local rows, halos and all-reduces over gloo."""
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_12011_b200 as T
        xyz, tets, rp, col = _internal_pattern((10, 6, 5), nparts=world)
        n = rp.shape[0] - 1
        E = tets.shape[0]
        rpA, colA, M, K = O.assemble(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E), {0: (0.13, 0.02)})
        A = O.system_matrix(M, K, 140.0, 0.01, 0.5, 0.05)
        b = G.random_vector(n, seed=21)
        x0 = G.random_vector(n, seed=22, lo=-0.01, hi=0.01)
        pl = T.tc_partition_plan(rp, col, world, rank)
        g0, g1 = pl["bounds"][rank], pl["bounds"][rank + 1]
        nl, ng = g1 - g0, len(pl["ghosts"])
        ghost_pos = {int(g): nl + t for t, g in enumerate(pl["ghosts"])}
        loc = lambda g: g - g0 if g0 <= g < g1 else ghost_pos[int(g)]
        rows = [(np.array([loc(c) for c in colA[rpA[i]:rpA[i + 1]]]), A[rpA[i]:rpA[i + 1]])
                for i in range(g0, g1)]
        dinv = np.array([1.0 / A[rpA[i]:rpA[i + 1]][colA[rpA[i]:rpA[i + 1]] == i][0] for i in range(g0, g1)])
        send_loc = pl["send_g"] - g0

        def allreduce(v):
            t = torch.tensor(v, dtype=torch.float64)
            dist.all_reduce(t)
            return t.numpy()

        # the pattern is already interior-first; the library finds the same split
        order, nints = T.tc_interior_first(rp.astype(np.int64), col, world)
        assert np.array_equal(order, np.arange(n))
        nint = int(nints[rank])

        def halo_start(values):  # values: owned vector -> nonblocking sends and receives
            reqs, recvs = [], []
            for j, qn in enumerate(pl["nbr"]):
                buf = torch.tensor(values[send_loc[pl["send_off"][j]:pl["send_off"][j + 1]]])
                reqs.append(dist.isend(buf, int(qn)))
            for j, qn in enumerate(pl["nbr"]):
                r = torch.zeros(int(pl["recv_off"][j + 1] - pl["recv_off"][j]), dtype=torch.float64)
                recvs.append((j, r, dist.irecv(r, int(qn))))
            return reqs, recvs

        def halo_finish(h, dst):  # dst: ghost region of a length nl+ng vector
            reqs, recvs = h
            for j, r, rq in recvs:
                rq.wait()
                dst[nl + pl["recv_off"][j]: nl + pl["recv_off"][j + 1]] = r.numpy()
            for rq in reqs:
                rq.wait()

        def halo(values, dst):
            halo_finish(halo_start(values), dst)

        spmv = lambda v, lo=0, hi=None: np.array([a @ v[c] for c, a in rows[lo:hi]])

        # the block is interior-first: rows [0, nint) read no ghost (the plan of the
        # reordered pattern), so they are computed while the halo is in flight --
        # with the ghost region still holding the previous iteration's values
        assert 0 < nint < nl
        for c, _ in rows[:nint]:
            assert np.all(c < nl)
        # r0 = b - A x0 (x0 halo), z0, rho0, ||z0||
        xv = np.zeros(nl + ng); xv[:nl] = x0[g0:g1]; halo(xv[:nl], xv)
        r = b[g0:g1] - spmv(xv)
        z = np.zeros(nl + ng); z[:nl] = dinv * r
        rho, zz = allreduce([r @ z[:nl], z[:nl] @ z[:nl]])
        zeta = zref = np.sqrt(zz)
        x = x0[g0:g1].copy()
        p = [np.zeros(nl + ng), np.zeros(nl + ng)]   # ghost regions stay 0
        it, beta, alpha, eps_a, conv = 0, 0.0, 0.0, 1e-11, False
        while not conv and it < 500:
            pold, pnew = p[(it + 1) % 2], p[it % 2]
            # pack + halo of p into the ghost region of z
            pb = z[:nl] + (beta * pold[:nl] if it else 0.0)
            h = halo_start(pb)                      # halo in flight ...
            if it:
                x += alpha * pold[:nl]
            pnew[:nl] = pb
            zp = z.copy()
            zp[:nl] = pb                            # ghost region: still the last halo
            q_int = spmv(zp, 0, nint)               # ... interior rows meanwhile
            halo_finish(h, z)
            q_ = np.concatenate([q_int, spmv(z + (beta * pold if it else 0.0), nint, None)])
            pq = allreduce([pnew[:nl] @ q_, 0.0])[0]
            alpha = rho / pq
            r -= alpha * q_
            z[:nl] = dinv * r
            rz, zz = allreduce([r @ z[:nl], z[:nl] @ z[:nl]])
            it += 1
            zeta = np.sqrt(zz)
            if zeta < eps_a:
                conv = True
                break
            beta = rz / rho
            rho = rz
        x += alpha * pnew[:nl]
        q.put((rank, g0, g1, x, it))
    finally:
        dist.destroy_process_group()


def test_distributed_pcg_gloo_world2():
    """world_size 2 over gloo: the partitioned schedule (library plan and
    interior-first order, ghost-p trick, interior rows computed while the halo is
    in flight, two all-reduces per iteration) reproduces the oracle's PCG."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    xyz, tets, rp, col = _internal_pattern((10, 6, 5), nparts=2)
    n = rp.shape[0] - 1
    E = tets.shape[0]
    rpA, colA, M, K = O.assemble(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E), {0: (0.13, 0.02)})
    A = O.system_matrix(M, K, 140.0, 0.01, 0.5, 0.05)
    xr, rep = O.pcg(rpA, colA, A, G.random_vector(n, seed=21), G.random_vector(n, seed=22, lo=-0.01, hi=0.01),
                    1e-11, 0.0, 500)
    x = np.zeros(n)
    for rank, g0, g1, xl, it in res:
        x[g0:g1] = xl
        assert it == rep.iters
    assert np.abs(x - xr).max() <= 1e-10 * np.abs(xr).max()


def test_rcm_blocks_partition_the_biv_like_slabs(T):
    """contiguous blocks of the RCM order cut the unstructured BiV
    (permuted numbering) into bands with at most two neighbours each and a ghost
    set of a small fraction of the part."""
    m = G.biv(1.2)
    xyz, tets = m["xyz"], m["tets"]
    n = xyz.shape[0]
    rp, col = T.tc_mesh_pattern(n, tets)
    perm = T.tc_rcm(rp, col)
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    rp2, col2 = T.tc_mesh_pattern(n, inv[tets].astype(np.int32))
    for P in (2, 4):
        plans = [T.tc_partition_plan(rp2, col2, P, p) for p in range(P)]
        assert max(len(pl["nbr"]) for pl in plans) <= 2
        assert max(len(pl["ghosts"]) for pl in plans) < 0.2 * n / P


def test_interior_first_edge_cases(T):
    """One block: every row is interior and the order is the identity; a block
    count above the row count is rejected by the plan (bounds must grow)."""
    xyz, tets, rp, col = _internal_pattern((5, 4, 3))
    n = rp.shape[0] - 1
    order, nint = T.tc_interior_first(rp.astype(np.int64), col, 1)
    assert np.array_equal(order, np.arange(n)) and nint.tolist() == [n]
    with pytest.raises(T.TcError):
        T.tc_interior_first(rp.astype(np.int64), col, 0)
