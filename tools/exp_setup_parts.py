#!/usr/bin/env python
"""Setup time of a PARTITIONED context ("setup_s for 8-part
emulation at 20 M nodes"): device setup (global pattern + RCM + interior-first
order on the GPU, each part planned from its own rows) vs the host path, same
node order.  python tools/exp_setup_parts.py [parts] [nx ny nz]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import meshgen as G  # noqa: E402


def main():
    import torch
    import paper_2510_12011_b200 as T
    parts = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    dims = tuple(int(v) for v in sys.argv[2:5]) if len(sys.argv) > 4 else (400, 250, 200)
    xyz, tets = G.kuhn_box(*dims, 0.1)
    st = [(G.nodes_in_box(xyz, (0, -1, -1), (0.3, 1e9, 1e9)), 0.0, 2.0, 50.0)]
    out = {"nodes": int(xyz.shape[0]), "tets": int(tets.shape[0]), "parts": parts}
    perms, vs = [], []
    for dev in (1, 0):
        cfg = T.tc_config_default(dt=0.01, model="ms", device_setup=dev, partitions=parts, peer=1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim = T.Monodomain(xyz, tets, None, None, {0: (0.1334177, 0.0173515)}, cfg, st)
        torch.cuda.synchronize()
        out["device_setup_s" if dev else "host_setup_s"] = time.perf_counter() - t0
        info = T.tc_matrix_info(sim.ctx)
        out["path" if dev else "path_host"] = info["path"]
        out["ghosts"] = info["ghosts"]
        perms.append(T.tc_node_order(sim.ctx))
        sim.step(3)
        vs.append(sim.V)
        sim.close()
    out["same_order"] = bool(np.array_equal(perms[0], perms[1]))
    out["same_V_after_3_steps"] = bool(np.array_equal(vs[0], vs[1]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
