#!/usr/bin/env python
"""One small run of a library code path, for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck):  python tools/sanitize_case.py CASE
CASE: grid_v0 grid_v1 grid_v4 grid_v5 cluster_res cluster_stream cohort peer3 split3 split3_ms crn_grid
Every case: a 21x8x5 TT2006 slab (840 nodes) with the corner stimulus, 4 steps."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import meshgen as G  # noqa: E402
import paper_2510_12011_b200 as T  # noqa: E402

case = sys.argv[1]
xyz, tets = G.kuhn_box(21, 8, 5, 0.5)
E = tets.shape[0]
stim = [(G.nodes_in_box(xyz, (0, 0, 0), (1.5, 1.5, 1.5)), 0.0, 2.0, 50.0)]
cond = {0: (0.1334177, 0.0173515)}
model = "crn" if case.startswith("crn") else ("ms" if case.endswith("_ms") else "tt2006")
kw = dict(dt=0.05, model=model, abs_tol=1e-8, rel_tol=0.0)
if case.startswith("grid_v"):
    kw.update(engine="grid", pcg_variant=int(case[6:]))
elif case == "crn_grid":
    kw.update(engine="grid")
elif case == "cluster_res":
    kw.update(engine="cluster")
elif case == "cluster_stream":
    kw.update(engine="cluster_streaming")
elif case == "peer3":
    kw.update(partitions=3, peer=1)
elif case.startswith("split3"):
    kw.update(partitions=3, peer=0)
if case == "cohort":
    sims = [T.Monodomain(xyz, tets, None, None, cond, T.tc_config_default(**kw), stim) for _ in range(3)]
    co = T.Cohort(sims)
    co.step(4)
    outs = [np.zeros(xyz.shape[0]) for _ in sims]
    co.get_v(outs)
    co.close()
    for s in sims:
        s.close()
    print(case, "ok", float(outs[0].max()))
else:
    sim = T.Monodomain(xyz, tets, None, None, cond, T.tc_config_default(**kw), stim)
    st = sim.step(4)
    v = sim.V
    print(case, "ok", T.tc_engine_info(sim.ctx), T.tc_matrix_info(sim.ctx)["pcg_variant"], int(st["iters"].sum()),
          float(v.max()))
    sim.close()
