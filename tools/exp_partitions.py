"""Experiment: per-step time of the split-phase (partitioned) PCG vs the persistent kernel."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import meshgen as G
import paper_2510_12011_b200 as T
dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "200,125,100").split(","))
xyz, tets = G.kuhn_box(*dims, 0.1)
stim = (G.nodes_in_box(xyz, (0, -1, -1), (0.3, 1e9, 1e9)), 0.0, 2.0, 50.0)
E = len(tets)
for parts, chk, peer, comm in [(1, 4, 1, None), (1, 4, 1, "nccl"), (1, 4, 0, "nccl"), (2, 4, 1, None),
                               (2, 4, 0, None), (4, 4, 1, None)]:
    if comm:
        comm = (0, 1, T.tc_nccl_unique_id())
    cfg = T.tc_config_default(dt=0.01, model="ms", partitions=parts, check_every=chk, peer=peer)
    sim = T.Monodomain(xyz, tets, None, None, {0: (0.1334177, 0.0173515)}, cfg, [stim], comm=comm)
    print(T.tc_matrix_info(sim.ctx)["path"], "comm" if comm else "", end=" ")
    sim.step(300)
    torch.cuda.synchronize()
    T.tc_profile(sim.ctx, True); T.tc_profile_read(sim.ctx, True)
    t0 = time.perf_counter(); st = sim.step(10); t1 = time.perf_counter()
    p = T.tc_profile_read(sim.ctx, True)
    print(f"parts={parts} check_every={chk}: {1e3*(t1-t0)/10:.3f} ms/step wall, pcg {p['pcg_ms']/10:.3f} ms/step, "
          f"ionic {p['ionic_ms']/10:.3f}, iters {st['iters'].mean():.1f}, launches {p['launches']}", flush=True)
    sim.close()
