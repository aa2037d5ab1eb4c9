#!/usr/bin/env python
"""Halo / interior overlap, before and after: PCG
ms per iteration of the partitioned paths emulated on one GPU, with the
interior-first row order (default; interior slices run while the halo is in
flight) and without it (TCB_NO_INTERIOR_FIRST=1: every row waits for the halo).
Mesh: 2.5 M nodes per part, (100 P) x 250 x 100 Kuhn slab, MS, dt 0.01, the
bench's planar stimulus, 300 steps of preroll, 20 timed steps."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import meshgen as G  # noqa: E402
import paper_2510_12011_b200 as T  # noqa: E402

for P in (2, 4):
    xyz, tets = G.kuhn_box(100 * P, 250, 100, 0.1)
    stim = (G.nodes_in_box(xyz, (0, -1, -1), (0.3, 1e9, 1e9)), 0.0, 2.0, 50.0)
    for peer in (1, 0):
        for nif in ("1", "0"):
            os.environ["TCB_NO_INTERIOR_FIRST"] = nif
            cfg = T.tc_config_default(dt=0.01, model="ms", partitions=P, peer=peer)
            sim = T.Monodomain(xyz, tets, None, None, {0: (0.1334177, 0.0173515)}, cfg, [stim])
            info = T.tc_matrix_info(sim.ctx)
            sim.step(300)
            torch.cuda.synchronize()
            T.tc_profile(sim.ctx, True)
            T.tc_profile_read(sim.ctx, True)
            t0 = time.perf_counter()
            st = sim.step(20)
            t1 = time.perf_counter()
            p = T.tc_profile_read(sim.ctx, True)
            it = int(st["iters"].sum())
            print(f"parts={P} path={info['path']} interior_first={'no' if nif == '1' else 'yes'}: "
                  f"{p['pcg_ms'] / it:.4f} ms/iteration, pcg {p['pcg_ms'] / 20:.3f} ms/step, "
                  f"{1e3 * (t1 - t0) / 20:.3f} ms/step wall, iters/step {it / 20:.2f}, ghosts {info['ghosts']}",
                  flush=True)
            sim.close()
os.environ.pop("TCB_NO_INTERIOR_FIRST", None)
