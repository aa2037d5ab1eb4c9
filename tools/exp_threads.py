"""Experiment: persistent PCG per-step time for a given library build (TCB200_LIB)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import meshgen as G
import paper_2510_12011_b200 as T
for dims in [(41, 15, 7), (201, 71, 31), (200, 125, 100), (400, 250, 200)]:
    dx = 0.5 if dims[0] == 41 else 0.1
    xyz, tets = G.kuhn_box(*dims, dx)
    stim = (G.nodes_in_box(xyz, (0, -1, -1), (0.3 if dx == 0.1 else 1.5, 1e9, 1e9)), 0.0, 2.0, 50.0)
    cfg = T.tc_config_default(dt=0.01, model="ms")
    sim = T.Monodomain(xyz, tets, None, None, {0: (0.1334177, 0.0173515)}, cfg, [stim])
    sim.step(300)
    torch.cuda.synchronize()
    T.tc_profile(sim.ctx, True); T.tc_profile_read(sim.ctx, True)
    st = sim.step(20)
    p = T.tc_profile_read(sim.ctx, True)
    print(f"{os.path.basename(os.environ.get('TCB200_LIB','default'))} n={len(xyz)}: pcg {p['pcg_ms']/20:.4f} ms/step, "
          f"{p['pcg_ms']/p['iters']*1e3:.1f} us/iter (incl RHS), iters {st['iters'].mean():.1f}", flush=True)
    sim.close()
