#!/usr/bin/env python
"""Setup time (mesh upload + pattern + RCM + SELL + assembly) of the default
workload, device setup vs host setup.
  python tools/exp_setup.py [--dims 400 250 200]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import meshgen as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs=3, default=[400, 250, 200])
    a = ap.parse_args()
    import torch
    import paper_2510_12011_b200 as T
    xyz, tets = G.kuhn_box(*a.dims, 0.1)
    E = tets.shape[0]
    st = [(G.nodes_in_box(xyz, (0, -1, -1), (0.3, 1e9, 1e9)), 0.0, 2.0, 50.0)]
    out = {"nodes": int(xyz.shape[0]), "tets": int(E)}
    perms = []
    for dev in (1, 0):
        cfg = T.tc_config_default(dt=0.01, model="ms", device_setup=dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim = T.Monodomain(xyz, tets, None, None, {0: (0.1334177, 0.0173515)}, cfg, st)
        torch.cuda.synchronize()
        out["device_setup_s" if dev else "host_setup_s"] = time.perf_counter() - t0
        perms.append(T.tc_node_order(sim.ctx))
        sim.close()
    out["same_order"] = bool(np.array_equal(perms[0], perms[1]))
    # phases of the device path through the C ABI
    cfg = T.tc_config_default(dt=0.01, model="ms", device_setup=1)
    ph = {}
    t0 = time.perf_counter()
    ctx = T.tc_create(cfg)
    ph["create"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    T.tc_set_mesh(ctx, xyz, tets, None, None)
    ph["set_mesh"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    T.tc_set_conductivity(ctx, [0], [0.1334177], [0.0173515])
    T.tc_add_stimulus(ctx, *st[0])
    ph["cond_stim"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    T.tc_assemble(ctx)
    torch.cuda.synchronize()
    ph["assemble"] = time.perf_counter() - t0
    T.tc_destroy(ctx)
    out["device_phases_s"] = ph
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
