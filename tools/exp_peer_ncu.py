"""Small driver for an ncu comparison of the persistent and peer PCG kernels."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import meshgen as G
import paper_2510_12011_b200 as T
xyz, tets = G.kuhn_box(200, 125, 100, 0.1)
stim = (G.nodes_in_box(xyz, (0, -1, -1), (0.3, 1e9, 1e9)), 0.0, 2.0, 50.0)
for mode in sys.argv[1:]:
    comm = (0, 1, T.tc_nccl_unique_id()) if mode == "peer" else None
    cfg = T.tc_config_default(dt=0.01, model="ms")
    sim = T.Monodomain(xyz, tets, None, None, {0: (0.1334177, 0.0173515)}, cfg, [stim], comm=comm)
    sim.step(30)
    torch.cuda.synchronize()
    sim.close()
