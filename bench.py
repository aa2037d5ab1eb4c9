#!/usr/bin/env python
"""bench.py -- throughput of the B200-native TorchCor monodomain step.

One "step" = one full time step of the hot path: ionic update
(+ LAT/LRT, x0, u', v'), RHS + Jacobi-PCG (Algorithm 1) to tolerance, on one
batch of synthetic input (a Kuhn-split tetrahedral slab).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

Prints ONE JSON line (rank 0).  metric = node-steps/s (BASELINE.json metric);
sim-ms per wall-s, PCG iterations, the roofline of the dominant kernel (the
cooperative PCG kernel) and the oracle's CPU rate ride along.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import meshgen as G  # noqa: E402  (input generator: no method arithmetic)

SIGMA = (0.1334177, 0.0173515)  # Table 3
CHI, CM = 140.0, 0.01           # Table 3

# BASELINE.json configs -> synthetic workloads
WORKLOADS = {
    # configs[4]: large synthetic slab ~20M nodes, Mitchell-Schaeffer (default at N=1)
    "slab20M_ms": dict(cfg=4, dims=(400, 250, 200), dx=0.1, model="ms", dt=0.01,
                       stim="face", preroll=500, sample_dims=(64, 64, 64), cpu_dims=(128, 128, 128)),
    # north-star target: ~10M-node TT2006 slab
    "slab10M_tt": dict(cfg="north_star", dims=(250, 200, 200), dx=0.1, model="tt2006", dt=0.01,
                       stim="face", preroll=500, sample_dims=(48, 48, 48), cpu_dims=(64, 64, 64)),
    # the north-star slab with the CRN atrial model
    "slab10M_crn": dict(cfg="f4 (north-star slab, CRN)", dims=(250, 200, 200), dx=0.1, model="crn", dt=0.01,
                        stim="face", preroll=500, sample_dims=(48, 48, 48), cpu_dims=(64, 64, 64)),
    # configs[2]: N-version dx = 0.1 mm (~442k nodes), TT2006 epi, dt 0.01
    "nversion_dx0.1_tt": dict(cfg=2, dims=(201, 71, 31), dx=0.1, model="tt2006", dt=0.01,
                              stim="corner", preroll=500, sample_dims=(48, 48, 31), cpu_dims=(201, 71, 31)),
    # configs[3]: synthetic biventricular-sized tet mesh (~3M nodes), rotating fibres, TT2006
    "biv3M_tt": dict(cfg=3, dims=None, h=0.33, dx=0.33, model="tt2006", dt=0.01, stim="biv",
                     preroll=500, sample_h=1.2, cpu_dims=1.0),
    # configs[0]: N-version dx = 0.5 mm (4305 nodes), TT2006 epi, dt 0.05, 40 ms
    "nversion_dx0.5_tt": dict(cfg=0, dims=(41, 15, 7), dx=0.5, model="tt2006", dt=0.05,
                              stim="corner", preroll=0, sample_dims=(41, 15, 7), cpu_dims=(41, 15, 7)),
    # SURVEY 8f row f2 (Fig. 8c/d): surface meshes (P1 triangles in 3-D) with
    # Mitchell-Schaeffer -- an icosphere of the left-atrium surface's size (660,557 nodes)
    # and one of the largest cube-surface size (~2 M nodes, Fig. 8c); tangent fibres, cap stimulus
    "sphere655k_ms": dict(cfg="f2 surface (LA-surface-sized, P:389)", dims=None, level=8, radius=28.0,
                          dx=0.13, model="ms", dt=0.01, stim="sphere", preroll=500, sample_level=7, cpu_dims=7),
    "sphere2.6M_ms": dict(cfg="f2 surface (Fig. 8c-sized)", dims=None, level=9, radius=56.0,
                          dx=0.13, model="ms", dt=0.01, stim="sphere", preroll=500, sample_level=7, cpu_dims=7),
    # a cohort of 100 configs[0]-sized slabs (seeded sizes,
    # numbering, fibres, conductivities, TT2006 parameter resets), one cluster each
    "cohort100_nversion05_tt": dict(cfg="f1 cohort", cohort=100, dims=None, dx=0.5, model="tt2006",
                                    dt=0.05, stim="corner", preroll=40),
    # SURVEY 8f row f1 with members of configs[2]'s size (P:349-353's cohort members are 660 k-node
    # meshes): 8 seeded N-version slabs at dx 0.1 mm (~440 k nodes each), the members sharing the GPU
    "cohort8_nversion01_tt": dict(cfg="f1 cohort (configs[2]-sized members)", cohort=8, dims=None, dx=0.1,
                                  member_base=(201, 71, 31), model="tt2006", dt=0.01, stim="corner",
                                  preroll=500),
    # SURVEY 8f f1 at the paper's member kind: 8 left-atrium-surface-sized icospheres (655 k nodes,
    # P1 triangles, MS; P:349-353 runs 100 LA surface meshes of 660,557 nodes), sharing the GPU
    "cohort8_sphere655k_ms": dict(cfg="f1 cohort (LA-surface-sized members, P:349)", cohort=8, dims=None,
                                  dx=0.13, model="ms", dt=0.01, stim="sphere", level=8, radius=28.0,
                                  preroll=500),
    # the paper's second workflow at its own size: 100 left-atrium-sized surface
    # meshes (100 LA meshes of 660,557 nodes, modified MS)
    "cohort100_sphere655k_ms": dict(cfg="f1 cohort (100 LA-surface-sized members, P:349-353)", cohort=100,
                                    dims=None, dx=0.13, model="ms", dt=0.01, stim="sphere", level=8,
                                    radius=28.0, preroll=500),
}
DEFAULT_WORKLOAD = "slab20M_ms"


def mesh_desc(w):
    if w.get("dims"):
        return list(w["dims"])
    if w["stim"] == "sphere":
        return f"icosphere level {w['level']} r={w['radius']} mm (P1 triangles)"
    return f"BiV h={w['h']} mm"


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def make_inputs(w, dims=None):
    """-> xyz, tets, stimuli, region, fibre (region/fibre None = single region, (1,0,0))."""
    if w["stim"] == "biv":
        m = G.biv(dims if dims is not None else w["h"])
        stims = [(nodes, 0.0, 2.0, 50.0) for nodes in G.biv_stimuli(m)]
        return m["xyz"], m["tets"], stims, m["region"], m["fibre"]
    if w["stim"] == "sphere":    # surface mesh: icosphere triangles, stimulus on a 2 mm polar cap
        level = dims if dims is not None else w["level"]
        r = w["radius"] * 2.0 ** (level - w["level"])       # samples keep the edge length
        xyz, tris = G.sphere(level, r)
        nodes = np.nonzero(xyz[:, 2] >= r - 2.0 * r / w["radius"])[0].astype(np.int32)
        return xyz, tris, [(nodes, 0.0, 2.0, 50.0)], None, G.sphere_fibres(xyz, tris)
    nx, ny, nz = dims or w["dims"]
    xyz, tets = G.kuhn_box(nx, ny, nz, w["dx"])
    if w["stim"] == "face":      # planar stimulus on x <= 0.3 mm (SURVEY 8d, C5 / C*)
        nodes = G.nodes_in_box(xyz, (0, -1, -1), (0.3, 1e9, 1e9))
    else:                        # N-version corner box <= 1.5 mm (reading N2)
        nodes = G.nodes_in_box(xyz, (0, 0, 0), (1.5, 1.5, 1.5))
    return xyz, tets, [(nodes, 0.0, 2.0, 50.0)], None, None


def kuhn_nnz(nx, ny, nz):
    """Stored entries of A on a Kuhn grid: n + 2 x edges (7 edge directions)."""
    n = nx * ny * nz
    axis = (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1)
    face = (nx - 1) * (ny - 1) * nz + (nx - 1) * ny * (nz - 1) + nx * (ny - 1) * (nz - 1)
    body = (nx - 1) * (ny - 1) * (nz - 1)
    return n + 2 * (axis + face + body)


def bytes_per_step(n, nnz, iters, model, steps):
    """Algorithmic bytes: B_rhs + iters B_it per PCG launch; ionic per node."""
    b_it = 12 * nnz + 4 * (n + 1) + 72 * n
    b_rhs = 20 * nnz + 4 * (n + 1) + 44 * n
    b_ion = {"tt2006": 352, "crn": 376}.get(model, 80) * n
    return b_rhs * steps + b_it * iters, b_ion * steps


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.p = None

    def __enter__(self):
        import threading
        self.lines, self.out = [], ""
        self.first = threading.Event()
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
            return self

        def reader():
            for line in self.p.stdout:
                self.lines.append(line)
                self.first.set()
            self.first.set()

        self.t = threading.Thread(target=reader, daemon=True)
        self.t.start()
        self.first.wait(timeout=10.0)   # nvidia-smi is up (its start-up can exceed a short timed region)
        self.n0 = len(self.lines)       # samples from before the timed region are dropped
        return self

    def __exit__(self, *a):
        if self.p is not None:
            n_end = len(self.lines)
            t0 = time.time()
            while len(self.lines) <= n_end and time.time() - t0 < 1.0:   # one sample after the region
                time.sleep(0.02)
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.t.join(timeout=2)
            kept = self.lines[self.n0:] or self.lines[-1:]
            self.out = "".join(kept)

    def summary(self):
        rows = [r.split(",") for r in self.out.strip().splitlines() if r.count(",") >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({nm for r in rows for nm, v in zip(names, r[5:9]) if "Active" in v and "Not" not in v})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def oracle_sample(w, steps=20, warmup=3, preroll=None):
    """The CPU oracle (as it stands) on a bounded sample of the workload -- same dx,
    dt, model, stimulus style and tolerances on the smaller slab `sample_dims` --
    at all host cores (OpenMP on its independent per-row / per-node loops): the
    oracle prerolls the sample into the workload's timing window itself, runs
    `warmup` steps, then times `steps` steps.  No library code on this path."""
    import oracle as O
    sample = {"biv": w.get("sample_h"), "sphere": w.get("sample_level")}.get(w["stim"], w.get("sample_dims"))
    xyz, tets, stims, region, fibre = make_inputs(w, sample)
    E = tets.shape[0]
    cfg = O.Config(dt=w["dt"], model=w["model"], chi=CHI, cm=CM, abs_tol=1e-5, rel_tol=1e-5, max_iters=100)
    sim = O.Monodomain(xyz, tets, np.zeros(E, np.int32) if region is None else region,
                       G.uniform_fibres(E) if fibre is None else fibre, {0: SIGMA, 1: SIGMA}, cfg,
                       [O.Stimulus(*s) for s in stims])
    n = xyz.shape[0]
    allc = host_threads()
    O.set_threads(allc)
    pre = w["preroll"] if preroll is None else preroll
    sim.run(pre + warmup)
    sim.reports.clear()
    t0 = time.perf_counter()
    sim.run(steps)
    el = time.perf_counter() - t0
    iters = float(np.mean([r.iters for r in sim.reports]))
    return dict(value=n * steps / el, unit="node-steps/s", cores=allc, kind="oracle",
                cpu_model=cpu_model(), nproc=os.cpu_count(), ms_per_step=1e3 * el / steps,
                sample=(f"BiV recipe at h={sample} mm" if w["stim"] == "biv" else
                        f"icosphere level {sample} (same edge length)" if w["stim"] == "sphere" else
                        f"{sample[0]}x{sample[1]}x{sample[2]} grid") +
                       f" ({n} nodes, same dx/dt/model/stimulus style), prerolled by the oracle {pre} + {warmup} "
                       f"steps, {steps} steps timed ({el:.1f} s at {allc} threads), mean PCG iters {iters:.1f}")


def host_threads():
    """Host cores this process may run on (the oracle's "all cores" leg): the CPU
    affinity set, not OMP_NUM_THREADS, which torchrun sets to 1 per rank."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def ncu_traffic(workload, iters_per_step, rhs=True):
    """DRAM bytes per step of the PCG path (rhs_kernel + pcg_kernel) from the committed
    ncu --set full capture, the pcg part rescaled to the timed mean iteration count."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            e = json.load(f).get(workload)
        if e is None:
            return None
        return (e["rhs_bytes"] if rhs else 0.0) + e["pcg_bytes"] * iters_per_step / e["iters"]
    except Exception:
        return None


def ionic_roofline(workload, model, n, ionic_ms_per_step):
    """FP64 roofline of the ionic kernel (FP64-ALU bound for TT2006 /
    CRN): ncu-counted FP64 work per node (profiles/ncu_fp64.json) x nodes over the
    live kernel time, against the measured DFMA rate."""
    if model not in ("tt2006", "crn") or not ionic_ms_per_step:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_fp64.json")) as f:
            d = json.load(f)
        e = d.get(workload) or d["slab10M_tt" if model == "tt2006" else "slab10M_crn"]
    except Exception:
        return None
    ach = e["flop_per_node"] * n / (ionic_ms_per_step / 1e3) / 1e12
    return {"kernel": e["kernel"], "bound": "fp64", "achieved": ach, "peak": d["peak_tflops"],
            "unit": "TFLOP/s", "frac": ach / d["peak_tflops"], "flop_per_node": e["flop_per_node"],
            "fp64_pipe_active_ncu": e["fp64_pipe_active_ncu"],
            "peak_source": "measured DFMA rate (profiles/r01_probe_fp64.txt)",
            "work_source": "ncu FP64 instruction counts per node (profiles/ncu_fp64.json)",
            "ns_per_node_step": ionic_ms_per_step * 1e6 / n,
            "note": "frac counts flops, and the flops per node are the current kernel's (r02 cut them from "
                    "2418 to ~1745 for TT2006 with table exp/log and fewer Newton steps), so a leaner kernel "
                    "lowers it at equal speed; fp64_pipe_active_ncu is the hardware utilisation"}


def run_reference(args, w):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cb = oracle_sample(w, steps=args.steps, warmup=args.warmup)
    line = {
        "impl": "reference", "metric": "node-steps/s", "value": cb["value"], "unit": "node-steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": cb["ms_per_step"], "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "model": w["model"], "dt_ms": w["dt"],
                   "note": "reference arm = the CPU oracle (no reference code exists; BASELINE.md)"},
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "node-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-rcm", action="store_true")
    ap.add_argument("--partitions", type=int, default=1, help="row-block partitions on this GPU")
    ap.add_argument("--pcg-variant", type=int, default=-1,
                    help="-1 automatic (default), 0 direct loads, 1 TMA-staged, 2 direct + 16-bit indices, "
                         "3 L2-resident matrix, 4 all slots of a row in flight, 6 single-reduction (Chronopoulos-Gear) PCG")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--preroll", type=int, default=None)
    ap.add_argument("--dist", action="store_true", help="use the NCCL path even at world size 1")
    ap.add_argument("--windows", type=int, default=3, help="timed windows of K steps (median reported)")
    ap.add_argument("--weak", action="store_true",
                    help="multi-GPU (torchrun / --dist): weak scaling, a (100 N) x 250 x 100 slab = 2.5 M nodes per GPU "
                         "(SURVEY 8d C5); default strong scaling of the workload")
    ap.add_argument("--no-north-star", action="store_true",
                    help="skip the slab10M_tt sub-record of the default run")
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, w)
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    rank, world, local = dist_env()
    if w.get("cohort"):
        return run_cohort(args, w)
    if world > 1 or args.dist:
        import bench_dist
        return bench_dist.main(args, w)

    import torch

    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream()
    line = measure_grid(args, args.workload, w, local, stream, preroll=args.preroll, e2e_steps=args.e2e_steps,
                        cpu=not args.no_cpu_baseline)
    # the north-star workload (BASELINE north_star: ~10 M-node TT2006 slab, CG path
    # >= 60 % of the HBM roofline) rides along as a sub-record of the default run
    if args.workload == DEFAULT_WORKLOAD and not args.no_north_star:
        try:
            ns = measure_grid(args, "slab10M_tt", WORKLOADS["slab10M_tt"], local, stream, preroll=None,
                              e2e_steps=0, cpu=not args.no_cpu_baseline)
            line["north_star"] = {k: ns[k] for k in ("value", "unit", "ms_per_step", "windows_ms_per_step",
                                                     "sim_ms_per_wall_s", "pcg_iters_per_step", "config",
                                                     "roofline", "ionic_roofline", "cpu_baseline", "clocks",
                                                     "gpu_launches", "setup_s")}
            line["north_star"]["what"] = ("BASELINE north_star target workload, measured in the same run with "
                                          "the same protocol (K steps per window, median of the windows)")
        except Exception as ex:  # report, never lose the primary line
            line["north_star"] = {"error": repr(ex)}
    print(json.dumps(line), flush=True)


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline_injected(w, V_dims, device, stream, steps=20):
    """The CPU oracle (as it stands) timed on this host beside the GPU run, on a
    bounded sample of the workload (same dx, dt, model, stimulus style and
    tolerances on the slab `V_dims`) STARTED IN THE TIMING WINDOW: the sample is
    prerolled by the library (the workload's preroll steps; a timing baseline,
    not a parity input), its state injected into the oracle, then `steps` oracle
    steps are timed at 1 thread and at all host cores (OpenMP on the oracle's
    independent per-row / per-node loops; bitwise the same results)."""
    import oracle as O
    import paper_2510_12011_b200 as T
    xyz, tets, stims, region, fibre = make_inputs(w, V_dims)
    E = tets.shape[0]
    n = xyz.shape[0]
    cfg = T.tc_config_default(dt=w["dt"], model=w["model"], chi=CHI, cm=CM, abs_tol=1e-5, rel_tol=1e-5,
                              max_iters=100)
    g = T.Monodomain(xyz, tets, region, fibre, {0: SIGMA, 1: SIGMA}, cfg, stims, device=device, stream=stream)
    g.step(w["preroll"])
    s = g.get_state()
    g.close()
    ns = {"tt2006": 18, "crn": 20, "ms": 1}[w["model"]]
    Vk, Vkm1, U = s[:n], s[n:2 * n], s[2 * n:(2 + ns) * n].reshape(ns, n)
    k0 = int(round(s[-2]))
    ocfg = O.Config(dt=w["dt"], model=w["model"], chi=CHI, cm=CM, abs_tol=1e-5, rel_tol=1e-5, max_iters=100)
    sim = O.Monodomain(xyz, tets, np.zeros(E, np.int32) if region is None else region,
                       G.uniform_fibres(E) if fibre is None else fibre, {0: SIGMA, 1: SIGMA}, ocfg,
                       [O.Stimulus(*st) for st in stims])
    allc = host_threads()
    res = {}
    try:
        for th in (1, allc):
            O.set_threads(th)
            sim.set_state(Vk, Vkm1, U, k0)
            sim.reports.clear()
            t0 = time.perf_counter()
            for _ in range(steps):
                sim.step()
            el = time.perf_counter() - t0
            res[th] = dict(value=n * steps / el, seconds=el, threads=th,
                           pcg_iters_per_step=float(np.mean([r.iters for r in sim.reports])))
    finally:
        O.set_threads(allc)
    return dict(value=res[allc]["value"], unit="node-steps/s", cores=allc, kind="oracle",
                threads_1=res[1], threads_all=res[allc], cpu_model=cpu_model(), nproc=os.cpu_count(),
                sample=(f"BiV recipe at h={V_dims} mm" if w["stim"] == "biv" else
                        f"icosphere level {V_dims}" if w["stim"] == "sphere" else
                        f"{V_dims[0]}x{V_dims[1]}x{V_dims[2]} slab") + f" ({n} nodes) of the same workload "
                       f"(dx/dt/model/stimulus/tolerances), state after the workload's {w['preroll']} preroll "
                       f"steps injected, {steps} timed steps at 1 thread and at {allc} threads; "
                       f"value = all threads")


def measure_grid(args, name, w, local, stream, preroll=None, e2e_steps=20, cpu=True):
    """One single-GPU workload: setup, preroll into the timing window, W warm-up
    steps, then `args.windows` windows of exactly K steps each (CUDA events on the
    library's stream, synchronised on both sides); value = the median window."""
    import torch
    import paper_2510_12011_b200 as T
    xyz, tets, stims, region, fibre = make_inputs(w)
    E = tets.shape[0]
    elem_key = "triangles" if tets.shape[1] == 3 else "tets"
    n = xyz.shape[0]
    cfg = T.tc_config_default(dt=w["dt"], model=w["model"], chi=CHI, cm=CM, abs_tol=1e-5, rel_tol=1e-5,
                              max_iters=100, use_rcm=0 if args.no_rcm else 1,
                              pcg_variant=args.pcg_variant, partitions=args.partitions)
    t0 = time.perf_counter()
    sim = T.Monodomain(xyz, tets, region, fibre, {0: SIGMA, 1: SIGMA}, cfg, stims,
                       device=local, stream=stream.cuda_stream)
    t_setup = time.perf_counter() - t0
    del tets
    info = T.tc_matrix_info(sim.ctx)
    eng = T.tc_engine_info(sim.ctx)
    preroll = w["preroll"] if preroll is None else preroll
    if preroll:
        sim.step(preroll)                   # move into the timing window (propagating front)
    sim.step(args.warmup)
    T.tc_profile(sim.ctx, True)
    T.tc_profile_read(sim.ctx, reset=True)
    torch.cuda.synchronize()
    wins = []
    with ClockSampler(local) as clk:
        for _ in range(max(1, args.windows)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            stats = sim.step(args.steps)
            e1.record(stream)
            torch.cuda.synchronize()
            prof = T.tc_profile_read(sim.ctx, reset=True)
            wins.append((e0.elapsed_time(e1), int(stats["iters"].sum()), prof))
    T.tc_profile(sim.ctx, False)
    order = sorted(range(len(wins)), key=lambda i: wins[i][0])
    ms, iters, prof = wins[order[len(order) // 2]]
    value = n * args.steps / (ms / 1e3)

    # roofline of the dominant kernel: the cooperative PCG kernel (RHS + Alg. 1);
    # with the ionic || RHS pipeline the profile's PCG time is the PCG kernel alone
    pipe = T.tc_pipeline_info(sim.ctx) if eng["engine"] == "grid" else {"chunks": 0, "rows_per_chunk": 0}
    peaks, which = measured_peaks()
    nnz = info["nnz"]
    b_cg, b_ion = bytes_per_step(n, nnz, iters, w["model"], args.steps)
    if pipe["chunks"]:
        b_cg -= (20 * nnz + 4 * (n + 1) + 44 * n) * args.steps      # RHS bytes overlap the ionic kernel
    cg_s = prof["pcg_ms"] / 1e3
    achieved = b_cg / cg_s / 1e9 if cg_s > 0 else None
    traffic = ncu_traffic(name, iters / args.steps, rhs=not pipe["chunks"])
    kname = ("PCG path per step: rhs_kernel + cooperative pcg_kernel (Eq. 3 RHS + Alg. 1)" if eng["engine"] == "grid"
             else "cohort_kernel (cluster engine: the whole step, ionic + RHS + Alg. 1, one launch per call)")
    if pipe["chunks"]:
        kname = (f"cooperative pcg_kernel (Alg. 1; the RHS runs in {pipe['chunks']} chunks overlapped with the ionic "
                 "kernel and is not counted)")
    roof = {"kernel": kname,
            "bound": "hbm",
            "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"] if achieved else None,
            "traffic": traffic, "peak_source": which,
            "frac_of_nominal_8TBs": achieved / 8000.0 if achieved else None,
            "bytes_model": ("per step: iters*(12nnz+4(n+1)+72n) (SURVEY 8d; RHS overlapped with the ionic kernel)"
                            if pipe["chunks"] else
                            "per step: 20nnz+4(n+1)+44n + iters*(12nnz+4(n+1)+72n) (SURVEY 8d)"),
            "ionic_rhs_pipeline": pipe,
            "algorithmic_bytes_per_step": b_cg / args.steps,
            "traffic_unit": "DRAM bytes per step of the same kernels (ncu, profiles/ncu_traffic.json)",
            "share_of_step": prof["pcg_ms"] / ms,
            "ionic_ms_per_step": prof["ionic_ms"] / args.steps,
            "pcg_ms_per_step": prof["pcg_ms"] / args.steps,
            "pcg_ms_per_iter": prof["pcg_ms"] / max(iters, 1)}

    # end to end through the C ABI with host buffers: every step loads a full
    # state (V^k, V^{k-1}, u^k) from pinned host memory and returns V^{k+1} to
    # pinned host memory; tc_step_io overlaps the copies with the compute
    e2e = None
    if e2e_steps > 0:
        st = sim.get_state()
        ke = e2e_steps
        hin = torch.empty(st.shape[0], dtype=torch.float64, pin_memory=True).numpy()
        hin[:] = st
        hout = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
        T.tc_step_io_repeat(sim.ctx, hin, hout, 1)   # warm: staging buffers and copy streams
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        T.tc_step_io_repeat(sim.ctx, hin, hout, ke)
        e2e_s = time.perf_counter() - t0
        e2e = {"value": n * ke / e2e_s, "unit": "node-steps/s", "h2d_bytes_per_step": int(hin.nbytes),
               "d2h_bytes_per_step": int(hout.nbytes), "steps": ke,
               "what": "tc_step_io (stride 0): per step the full state (V^k, V^{k-1}, u^k) H2D from one pinned "
                       "host buffer, one step, V^{k+1} D2H to one pinned host buffer; copies of neighbouring steps "
                       "overlap the compute (two copy streams), wall clock over all steps incl. pipeline fill "
                       "and drain"}
        del hin, hout
    sim.close()

    cpu_res = None
    if cpu:
        try:
            cpu_res = cpu_baseline_injected(w, w["cpu_dims"], local, stream.cuda_stream)
        except Exception as ex:  # report, never fail the bench on the baseline leg
            cpu_res = {"error": repr(ex)}
    return {
        "metric": "node-steps/s", "value": value, "unit": "node-steps/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "windows_ms_per_step": [wv[0] / args.steps for wv in wins],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": name, "baseline_config": w["cfg"], "nodes": n, "nnz": nnz,
                   elem_key: int(E), "model": w["model"], "dt_ms": w["dt"], "dx_mm": w["dx"],
                   "grid": mesh_desc(w), "tol": "abs=rel=1e-5, max 100 (P:316)",
                   "rcm": not args.no_rcm, "preroll_steps": preroll, "pcg_variant": info["pcg_variant"],
                   "engine": eng,
                   "wide_slices": info.get("wide_slices"),
                   "timing": f"{len(wins)} windows of {args.steps} steps, median reported",
                   "l2": f"inputs larger than L2 (A+K+col {(20 * info['nnz_pad']) / 1e9:.2f} GB >> 126 MB)"
                         if n > 1_000_000 else "small problem: L2-resident",
                   "parallelism": "1 GPU"},
        "sim_ms_per_wall_s": args.steps * w["dt"] / (ms / 1e3),
        "pcg_iters_per_step": iters / args.steps,
        "setup_s": t_setup,
        "roofline": roof,
        "ionic_roofline": ionic_roofline(name, w["model"], n, prof["ionic_ms"] / args.steps),
        "cpu_baseline": cpu_res,
        "e2e": e2e,
        "gpu_launches": int(round(prof["launches"])),
        "clocks": clk.summary(),
    }


def run_cohort(args, w):
    """f1: every member advanced by one tc_cohort_step launch per timed call."""
    import torch
    import paper_2510_12011_b200 as T
    rank, world, local = dist_env()
    if world > 1:   # replicas only: every rank runs its own cohort
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream()
    if w["stim"] == "sphere":
        members = G.sphere_cohort_members(w["cohort"], seed=G.SEED + rank, level=w["level"], radius=w["radius"])
    else:
        members = G.cohort_members(w["cohort"], seed=G.SEED + rank, base=w.get("member_base", (41, 15, 7)),
                                   dx=w["dx"])
    sims = []
    t0 = time.perf_counter()
    for m in members:
        cfg = T.tc_config_default(dt=w["dt"], model=w["model"], chi=CHI, cm=CM, abs_tol=1e-5, rel_tol=1e-5,
                                  max_iters=100)
        sims.append(T.Monodomain(m["xyz"], m["tets"], None, m["fibre"],
                                 {0: (SIGMA[0] * m["sigma_scale"], SIGMA[1] * m["sigma_scale"])}, cfg,
                                 [(m["stim_nodes"], 0.0, 2.0, 50.0)], device=local,
                                 stream=stream.cuda_stream))
        for name, f in m["param_factors"].items():
            T.tc_set_ionic_param(sims[-1].ctx, name, T.tc_get_ionic_param(sims[-1].ctx, name) * f)
    co = T.Cohort(sims)
    t_setup = time.perf_counter() - t0
    info = co.info()
    n_nodes = [T.tc_num_nodes(s.ctx) for s in sims]
    nnz = [T.tc_matrix_info(s.ctx)["nnz"] for s in sims]
    N = int(sum(n_nodes))
    co.step(w["preroll"], want_stats=False)
    co.step(args.warmup, want_stats=False)
    torch.cuda.synchronize()
    engines = sorted({T.tc_engine_info(s_.ctx)["engine"] for s_ in sims})
    big = engines == ["grid"]   # large members: grid-engine kernels per member, sharing the GPU
    launches0 = sum(T.tc_profile_read(s_.ctx)["launches"] for s_ in sims)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        stats = co.step(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = int(round(sum(T.tc_profile_read(s_.ctx)["launches"] for s_ in sims) - launches0))
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = N * world * args.steps / (ms / 1e3)
    b_cg = b_ion = 0.0
    for mi in range(len(sims)):
        bc, bi = bytes_per_step(n_nodes[mi], nnz[mi], int(stats["iters"][mi].sum()), w["model"], args.steps)
        b_cg += bc
        b_ion += bi
    peaks, which = measured_peaks()
    achieved = (b_cg + b_ion) / (ms / 1e3) / 1e9
    roof = {"kernel": ("per-member grid-engine kernels (ionic, RHS + cooperative PCG shaped for a share of the GPU) "
                       "on per-member streams running side by side" if big else
                       "cohort_kernel (cluster engine, one cluster per member, whole step per launch)"),
            "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": None, "peak_source": which,
            "bytes_model": "per member and step: B_ion + 20nnz+4(n+1)+44n + iters*(12nnz+4(n+1)+72n) (SURVEY 8d)",
            "note": ("members' matrices and vectors stream from HBM (together far larger than L2)" if big else
                     "members are shared-memory / L2 resident: latency-bound (cluster barriers, DSMEM), "
                     "the HBM fraction is the algorithmic-byte rate, not a bandwidth claim")}
    # end to end through the C ABI with host buffers: every member's state H2D, one cohort step, V D2H
    hin = []
    for s_ in sims:
        st_ = s_.get_state()
        h = torch.empty(st_.shape[0], dtype=torch.float64, pin_memory=True).numpy()
        h[:] = st_
        hin.append(h)
    hout = [torch.empty(n_, dtype=torch.float64, pin_memory=True).numpy() for n_ in n_nodes]
    ke = max(1, args.e2e_steps)
    co.set_states(hin)   # untimed: the first call allocates each member's staging (tc_step_io buffers)
    torch.cuda.synchronize()
    split = [0.0, 0.0, 0.0]
    t0 = time.perf_counter()
    for _ in range(ke):
        ta = time.perf_counter()
        co.set_states(hin)
        tb = time.perf_counter()
        co.step(1, want_stats=False)
        tc_ = time.perf_counter()
        co.get_v(hout)
        td = time.perf_counter()
        split[0] += tb - ta; split[1] += tc_ - tb; split[2] += td - tc_
    e2e_s = time.perf_counter() - t0
    e2e = {"value": N * world * ke / e2e_s, "unit": "node-steps/s",
           "h2d_bytes_per_step": int(sum(h.nbytes for h in hin)), "d2h_bytes_per_step": int(sum(h.nbytes for h in hout)),
           "what": "per step: tc_cohort_set_states (every member's state, pinned host) + tc_cohort_step(1) + tc_cohort_get_v (every member's V)",
           "split_ms_per_step": {"set_state": 1e3 * split[0] / ke, "cohort_step": 1e3 * split[1] / ke,
                                 "get_v": 1e3 * split[2] / ke}}
    iters = float(stats["iters"].mean())
    co.close()
    for s_ in sims:
        s_.close()
    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline:
        try:
            import oracle as O
            m = members[0]
            E = m["tets"].shape[0]
            if w["model"] == "ms":
                names = ["tau_in", "tau_out", "tau_open", "tau_close", "v_gate", "V_min", "V_max"]
                prm = O.ms_default_params().copy()
            else:
                names = O.tt_param_names()
                prm = O.tt_default_params().copy()
            for k_, f_ in m["param_factors"].items():
                prm[names.index(k_)] *= f_
            cfg = O.Config(dt=w["dt"], model=w["model"], chi=CHI, cm=CM, abs_tol=1e-5, rel_tol=1e-5,
                           max_iters=100, params=prm)
            osim = O.Monodomain(m["xyz"], m["tets"], np.zeros(E, np.int32), m["fibre"],
                                {0: (SIGMA[0] * m["sigma_scale"], SIGMA[1] * m["sigma_scale"])}, cfg,
                                [O.Stimulus(m["stim_nodes"], 0.0, 2.0, 50.0)])
            O.set_threads(1)
            k_, t1 = 0, time.perf_counter()
            while time.perf_counter() - t1 < 15.0 and k_ < 800:
                osim.step()
                k_ += 1
            el = time.perf_counter() - t1
            O.set_threads(O.max_threads())
            cpu = dict(value=n_nodes[0] * k_ / el, unit="node-steps/s", cores=1, kind="oracle",
                       sample=f"member 0 ({n_nodes[0]} nodes), first {k_} steps from rest, {el:.1f} s single-thread")
        except Exception as ex:
            cpu = {"error": str(ex)}
    line = {
        "metric": "node-steps/s", "value": value, "unit": "node-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "baseline_config": w["cfg"], "members": len(sims),
                   "nodes_total": N, "nodes_min": int(min(n_nodes)), "nodes_max": int(max(n_nodes)),
                   "model": w["model"], "dt_ms": w["dt"], "dx_mm": w["dx"], "tol": "abs=rel=1e-5, max 100 (P:316)",
                   "preroll_steps": w["preroll"], "cohort": info,
                   "engines": engines,
                   "l2": ("inputs larger than L2 (every member's matrix streamed each step)" if big else
                          "small problems: L2 / shared-memory resident by design (cluster engine)"),
                   "parallelism": "replicas only" if world > 1 else "1 GPU"},
        "sim_ms_per_wall_s": args.steps * w["dt"] / (ms / 1e3),
        "pcg_iters_per_step": iters, "setup_s": t_setup, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
