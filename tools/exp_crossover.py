#!/usr/bin/env python
"""Crossover of the PCG kernel variants 0 (direct, 64 warps/SM) and 4 (every slot
of a row in flight, 16 warps/SM) over system size: MS slabs (dx 0.1 mm, dt 0.01,
planar stimulus) of growing y-z cross-section, PCG ms per iteration after a
preroll.  Prints slices per resident warp of variant 0 beside the timings.
  python tools/exp_crossover.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def run(T, dims, variant, steps=40, preroll=200):
    w = dict(bench.WORKLOADS["slab20M_ms"])
    xyz, tets, stims, region, fibre = bench.make_inputs(w, dims)
    E = tets.shape[0]
    cfg = T.tc_config_default(dt=w["dt"], model="ms", chi=bench.CHI, cm=bench.CM, pcg_variant=variant)
    sim = T.Monodomain(xyz, tets, np.zeros(E, np.int32), None, {0: bench.SIGMA}, cfg, stims)
    sim.step(preroll)
    T.tc_profile(sim.ctx, True)
    T.tc_profile_read(sim.ctx, reset=True)
    sim.step(steps)
    p = T.tc_profile_read(sim.ctx, reset=True)
    info = T.tc_matrix_info(sim.ctx)
    sim.close()
    return xyz.shape[0], info["nslices"], info["pcg_variant"], p["pcg_ms"] / p["iters"]


def main():
    import paper_2510_12011_b200 as T
    warps = 148 * 64
    for dims in [(201, 71, 31), (201, 81, 41), (201, 101, 51), (201, 121, 61), (201, 141, 71), (201, 161, 81)]:
        res = [run(T, dims, v) for v in (0, 4, -1)]
        n, ns = res[0][0], res[0][1]
        print(f"dims {dims} n {n} slices/warp {ns / warps:.2f}  v0 {res[0][3]:.5f}  v4 {res[1][3]:.5f}  "
              f"auto->v{res[2][2]} {res[2][3]:.5f} ms/iter", flush=True)


if __name__ == "__main__":
    main()
