#!/usr/bin/env python
"""One small-mesh run for profiling: configs[0] (41x15x7, TT2006, dt 0.05) on the
given engine, `--pre` untimed steps in one call, then `--steps` steps in one call.
  python tools/run_small.py [--engine cluster|grid|cluster_streaming] [--model tt2006|ms]"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import meshgen as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--engine", default="cluster")
    ap.add_argument("--model", default="tt2006")
    ap.add_argument("--pre", type=int, default=60)
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    import paper_2510_12011_b200 as T
    xyz, tets = G.kuhn_box(41, 15, 7, 0.5)
    E = tets.shape[0]
    cfg = T.tc_config_default(dt=0.05, model=a.model, engine=a.engine)
    st = [(G.nodes_in_box(xyz, (0, 0, 0), (1.5, 1.5, 1.5)), 0.0, 2.0, 50.0)]
    sim = T.Monodomain(xyz, tets, np.zeros(E, np.int32), G.uniform_fibres(E), {0: (0.1334177, 0.0173515)},
                       cfg, st)
    sim.step(a.pre)
    s = sim.step(a.steps)
    print("engine", T.tc_engine_info(sim.ctx), "iters/step", s["iters"].mean())
    sim.close()


if __name__ == "__main__":
    main()
