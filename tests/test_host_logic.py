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


def _internal_pattern(dims, seed=7):
    xyz, tets = G.kuhn_box(*dims, 1.0)
    xyz, tets, _ = G.permute_nodes(xyz, tets, seed=seed)
    n = xyz.shape[0]
    rp, col = O.pattern(n, tets)
    perm = O.rcm(rp, col)
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    tets_i = inv[tets].astype(np.int32)
    rpi, coli = O.pattern(n, tets_i)
    return xyz[perm], tets_i, rpi, coli


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
        xyz, tets, rp, col = _internal_pattern((10, 6, 5))
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

        def halo(values, dst):  # values: owned vector; dst: ghost region of a length nl+ng vector
            reqs = []
            for j, qn in enumerate(pl["nbr"]):
                buf = torch.tensor(values[send_loc[pl["send_off"][j]:pl["send_off"][j + 1]]])
                reqs.append(dist.isend(buf, int(qn)))
            for j, qn in enumerate(pl["nbr"]):
                r = torch.zeros(int(pl["recv_off"][j + 1] - pl["recv_off"][j]), dtype=torch.float64)
                dist.recv(r, int(qn))
                dst[nl + pl["recv_off"][j]: nl + pl["recv_off"][j + 1]] = r.numpy()
            for rq in reqs:
                rq.wait()

        spmv = lambda v: np.array([a @ v[c] for c, a in rows])
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
            halo(pb, z)
            if it:
                x += alpha * pold[:nl]
            pnew[:nl] = pb
            q_ = spmv(z + (beta * pold if it else 0.0))
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
    """world_size 2 over gloo: the partitioned schedule (library plan, ghost-p
    trick, two all-reduces per iteration) reproduces the oracle's PCG."""
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
    xyz, tets, rp, col = _internal_pattern((10, 6, 5))
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
