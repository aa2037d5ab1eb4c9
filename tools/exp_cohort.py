#!/usr/bin/env python
"""Cluster engine / cohort measurements.

  python tools/exp_cohort.py [--quick]

(1) one context, grid vs cluster engine, ms per step at several mesh sizes;
(2) cohorts of configs[0]-sized members (4 305 nodes, TT2006, dt 0.05) at
    several member counts and cluster sizes: node-steps/s of the whole cohort.
Times are CUDA-event times on the context stream around tc_step / tc_cohort_step."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import meshgen as G  # noqa: E402

SIG = (0.1334177, 0.0173515)


def make(T, dims, dx, model, dt, engine, stream):
    xyz, tets = G.kuhn_box(*dims, dx)
    E = tets.shape[0]
    cfg = T.tc_config_default(dt=dt, model=model, engine=engine)
    st = [(G.nodes_in_box(xyz, (0, 0, 0), (1.5, 1.5, 1.5)), 0.0, 2.0, 50.0)]
    return T.Monodomain(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E), {0: SIG}, cfg, st,
                        stream=stream), xyz.shape[0]


def timed(torch, stream, fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    import torch
    import paper_2510_12011_b200 as T
    stream = torch.cuda.current_stream()
    sid = stream.cuda_stream
    res = {"single": [], "cohort": []}
    sizes = [((41, 15, 7), 0.5, "tt2006", 0.05), ((81, 29, 13), 0.25, "tt2006", 0.02),
             ((101, 36, 16), 0.2, "tt2006", 0.01), ((161, 57, 25), 0.125, "tt2006", 0.01)]
    if args.quick:
        sizes = sizes[:2]
    for dims, dx, model, dt in sizes:
        row = {"dims": dims, "model": model}
        for engine in ("grid", "cluster", "cluster_streaming"):
            sim, n = make(T, dims, dx, model, dt, engine, sid)
            sim.step(200)                      # through the stimulus: propagating front
            ms, st = timed(torch, stream, lambda: sim.step(200))
            row[engine] = {"ms_per_step": ms / 200, "iters": float(st["iters"].mean())}
            row["n"] = n
            row[engine]["info"] = T.tc_engine_info(sim.ctx)
            sim.close()
        print(json.dumps(row), flush=True)
        res["single"].append(row)
    counts = [1, 9, 18, 37, 74, 148, 296] if not args.quick else [1, 18, 74]
    for cs, resident in ((4, False), (8, True), (8, False), (16, True)):
        for cnt in counts:
            mem = [make(T, (41, 15, 7), 0.5, "tt2006", 0.05, "cluster", sid)[0] for _ in range(cnt)]
            co = T.Cohort(mem, cs, resident)
            co.step(100, want_stats=False)
            ms, st = timed(torch, stream, lambda: co.step(200))
            info = co.info()
            row = {"cluster_size": cs, "members": cnt, "resident_clusters": info["resident_clusters"],
                   "smem_per_cta": info["smem_per_cta"],
                   "ms_per_step": ms / 200, "node_steps_per_s": cnt * 4305 * 200 / (ms / 1e3),
                   "iters": float(st["iters"].mean())}
            print(json.dumps(row), flush=True)
            res["cohort"].append(row)
            co.close()
            for m in mem:
                m.close()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "exp_cohort.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
