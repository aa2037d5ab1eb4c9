"""Experiment: the peer-memory PCG kernel with the direct (0) and the latency
(auto -> 4) row product on configs[2]-sized systems: one rank (NCCL comm of 1)
and 2 / 4 emulated partitions on one GPU (each partition = one rank's share at
N GPUs).  Prints PCG ms per iteration.
  python tools/exp_peer_batch.py [nx,ny,nz]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import meshgen as G  # noqa: E402
import paper_2510_12011_b200 as T  # noqa: E402

dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "201,71,31").split(","))
xyz, tets = G.kuhn_box(*dims, 0.1)
stim = (G.nodes_in_box(xyz, (0, -1, -1), (0.3, 1e9, 1e9)), 0.0, 2.0, 50.0)
for parts, comm in [(1, "nccl"), (2, None), (4, None), (8, None)]:
    for variant in (0, -1):
        c = (0, 1, T.tc_nccl_unique_id()) if comm else None
        cfg = T.tc_config_default(dt=0.01, model="ms", partitions=parts, peer=1, pcg_variant=variant)
        sim = T.Monodomain(xyz, tets, None, None, {0: (0.1334177, 0.0173515)}, cfg, [stim], comm=c)
        info = T.tc_matrix_info(sim.ctx)
        sim.step(200)
        T.tc_profile(sim.ctx, True)
        T.tc_profile_read(sim.ctx, True)
        st = sim.step(20)
        p = T.tc_profile_read(sim.ctx, True)
        print(f"{dims} parts={parts}{' comm' if comm else ''} path={info['path']} variant={info['pcg_variant']}: "
              f"pcg {p['pcg_ms'] / p['iters']:.4f} ms/iter, {p['pcg_ms'] / 20:.3f} ms/step, "
              f"iters {st['iters'].mean():.1f}", flush=True)
        sim.close()
