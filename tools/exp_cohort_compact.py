#!/usr/bin/env python
"""Cohort residency modes (tc_cohort_create resident 0 streaming, 2 full, 3
compact = column indices only in shared memory) at cluster sizes 2 / 4 / 8 / 16:
(a) configs[0]-sized TT2006 members (74 and 148 of them); (b) the bench's
cohort100 members (meshgen.cohort_members, 2 160 .. 7 191 nodes)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import exp_cohort as E  # noqa: E402
import meshgen as G  # noqa: E402

SIG = (0.1334177, 0.0173515)


def bench_members(T, sid):
    sims = []
    for m in G.cohort_members(100, seed=G.SEED):
        cfg = T.tc_config_default(dt=0.05, model="tt2006", abs_tol=1e-5, rel_tol=1e-5, max_iters=100)
        sims.append(T.Monodomain(m["xyz"], m["tets"], None, m["fibre"],
                                 {0: (SIG[0] * m["sigma_scale"], SIG[1] * m["sigma_scale"])}, cfg,
                                 [(m["stim_nodes"], 0.0, 2.0, 50.0)], stream=sid))
        for name, f in m["param_factors"].items():
            T.tc_set_ionic_param(sims[-1].ctx, name, T.tc_get_ionic_param(sims[-1].ctx, name) * f)
    return sims


def run(T, torch, stream, label, make_members, grid=((2, 4, 8, 16), (0, 2, 3))):
    """Fresh members for every (cluster size, mode): the same simulated interval."""
    for cs in grid[0]:
        for res in grid[1]:
            mem = make_members()
            nodes = sum(T.tc_num_nodes(m.ctx) for m in mem)
            try:
                co = T.Cohort(mem, cs, res)
            except Exception as ex:
                print(json.dumps({"set": label, "cluster_size": cs, "resident": res, "error": str(ex)}), flush=True)
                for m in mem:
                    m.close()
                continue
            co.step(60, want_stats=False)
            ms, st = E.timed(torch, stream, lambda: co.step(200, want_stats=False))
            info = co.info()
            print(json.dumps({"set": label, "resident": res, **info, "ms_per_step": ms / 200,
                              "node_steps_per_s": nodes * 200 / (ms / 1e3)}), flush=True)
            co.close()
            for m in mem:
                m.close()


def main():
    import torch
    import paper_2510_12011_b200 as T
    stream = torch.cuda.current_stream()
    sid = stream.cuda_stream
    grid = ((0, 1, 2, 4, 8, 16), (1,)) if "--small" in sys.argv else ((2, 4, 8, 16), (0, 2, 3))
    if "--dense" in sys.argv:   # resident 4: the two-CTA-per-SM streaming kernel, beside auto
        grid = ((0, 2, 4, 8), (1, 4))
    for cnt in ((16, 74, 148) if ("--small" in sys.argv or "--dense" in sys.argv) else (74, 148)):
        run(T, torch, stream, f"configs0 x{cnt}",
            lambda: [E.make(T, (41, 15, 7), 0.5, "tt2006", 0.05, "cluster", sid)[0] for _ in range(cnt)], grid)
    run(T, torch, stream, "cohort100", lambda: bench_members(T, sid), grid)


if __name__ == "__main__":
    main()
