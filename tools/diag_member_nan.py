#!/usr/bin/env python
"""Diagnose the NaN seen in cohort100 member 8 after a few hundred steps:
the member alone on the grid and cluster engines, stepped one call of 20 steps
at a time; prints the first chunk whose result holds a NaN (or none), and the
oracle over the same steps when asked (--oracle N steps)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import meshgen as G  # noqa: E402

SIG = (0.1334177, 0.0173515)


def build(T, m, engine):
    cfg = T.tc_config_default(dt=0.05, model="tt2006", abs_tol=1e-5, rel_tol=1e-5, max_iters=100, engine=engine)
    s = T.Monodomain(m["xyz"], m["tets"], None, m["fibre"],
                     {0: (SIG[0] * m["sigma_scale"], SIG[1] * m["sigma_scale"])}, cfg,
                     [(m["stim_nodes"], 0.0, 2.0, 50.0)])
    for name, f in m["param_factors"].items():
        T.tc_set_ionic_param(s.ctx, name, T.tc_get_ionic_param(s.ctx, name) * f)
    return s


def main():
    import paper_2510_12011_b200 as T
    ms = G.cohort_members(100, seed=G.SEED)
    idx = [int(a) for a in sys.argv[1:]] or [8]
    for i in idx:
        m = ms[i]
        for engine in ("grid", "cluster"):
            s = build(T, m, engine)
            row = {"member": i, "n": int(m["xyz"].shape[0]), "engine": engine, "first_bad_step": None}
            vmax = []
            for c in range(60):
                try:
                    st = s.step(20)
                except T.TcError as ex:
                    row["first_bad_step"] = 20 * c
                    row["error"] = str(ex)
                    break
                V = s.V
                vmax.append([float(np.min(V)), float(np.max(V)), float(np.mean(st["iters"]))])
                if not np.all(np.isfinite(V)):
                    row["first_bad_step"] = 20 * c
                    break
            row["trace_min_max_iters"] = vmax[::5] + vmax[-3:]
            print(json.dumps(row), flush=True)
            s.close()


if __name__ == "__main__":
    main()
