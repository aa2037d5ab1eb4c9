"""bench_dist.py -- the N>1 leg of bench.py (one process per GPU under torchrun).

Every rank passes the same global mesh to the library, which cuts the RCM-ordered
system into WORLD_SIZE row blocks (rank r owns block r) and runs the persistent
peer-memory PCG (halos and reductions over NVLink by the kernel itself), or the
split-phase PCG with NCCL when peer mappings are unavailable.
Timing: barrier + cudaSynchronize on both sides, CUDA events on the library's
stream, max over ranks; rank 0 prints the JSON line.  scaling = "strong"
(the global workload is fixed as N grows)."""
from __future__ import annotations

import json
import os
import time

import numpy as np


def main(args, w):
    # every rank runs the host setup (pattern, RCM, partition plan) with OpenMP:
    # share the host cores between the ranks of this node instead of oversubscribing
    # (torchrun sets OMP_NUM_THREADS=1 for nproc > 1; an explicit larger value is kept)
    nloc = int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1")))
    nthr = max(1, (os.cpu_count() or 1) // max(1, nloc))
    if os.environ.get("OMP_NUM_THREADS", "1") == "1":
        os.environ["OMP_NUM_THREADS"] = str(nthr)
    else:
        nthr = int(os.environ["OMP_NUM_THREADS"])
    import torch
    torch.set_num_threads(nthr)   # the process-wide OpenMP runtime is shared with libtcb200
    import torch.distributed as dist

    import bench
    import paper_2510_12011_b200 as T

    rank, world, local = bench.dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")        # bootstrap only (NCCL id, timing max)
    uid = [T.tc_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    stream = torch.cuda.current_stream()
    weak = getattr(args, "weak", False) and w.get("dims") and w["stim"] == "face"
    dims = (100 * world, 250, 100) if weak else None     # SURVEY 8(d) C5 weak unit: 2.5 M nodes per GPU
    xyz, tets, stims, region, fibre = bench.make_inputs(w, dims)
    E = tets.shape[0]
    n = xyz.shape[0]
    cfg = T.tc_config_default(dt=w["dt"], model=w["model"], chi=bench.CHI, cm=bench.CM, abs_tol=1e-5,
                              rel_tol=1e-5, max_iters=100, use_rcm=0 if args.no_rcm else 1)
    t0 = time.perf_counter()
    sim = T.Monodomain(xyz, tets, region, fibre, {0: bench.SIGMA, 1: bench.SIGMA}, cfg, stims,
                       device=local, stream=stream.cuda_stream, comm=(rank, world, uid[0]))
    t_setup = time.perf_counter() - t0
    del tets
    info = T.tc_matrix_info(sim.ctx)
    preroll = w["preroll"] if args.preroll is None else args.preroll
    if preroll:
        sim.step(preroll)
    sim.step(args.warmup)
    T.tc_profile(sim.ctx, True)
    T.tc_profile_read(sim.ctx, reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    with bench.ClockSampler(local) as clk:
        e0.record(stream)
        stats = sim.step(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    ms_local = e0.elapsed_time(e1)
    prof = T.tc_profile_read(sim.ctx, reset=True)
    t = torch.tensor([ms_local], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    iters = int(stats["iters"].sum())
    value = n * args.steps / (ms / 1e3)
    # roofline of this rank's PCG path (its rows): same algorithmic byte model
    peaks, which = bench.measured_peaks()
    n_loc = int(info["nslices"]) * 32
    nnz_loc = int(info["nnz_pad"])
    b_cg, _ = bench.bytes_per_step(n_loc, nnz_loc, iters, w["model"], args.steps)
    cg_s = prof["pcg_ms"] / 1e3
    achieved = b_cg / cg_s / 1e9 if cg_s > 0 else None
    # end to end: global state H2D (each rank uploads its block), step, V gathered to host
    st = sim.get_state()
    hin = torch.empty(st.shape[0], dtype=torch.float64, pin_memory=True).numpy()
    hin[:] = st
    hout = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    ke = max(1, args.e2e_steps)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(ke):
        T.tc_set_state(sim.ctx, hin)
        T.tc_step(sim.ctx, 1, want_stats=False)
        T.tc_get_v(sim.ctx, hout)
    e2e_local = time.perf_counter() - t0
    t = torch.tensor([e2e_local], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    sim.close()
    if rank == 0:
        line = {
            "metric": "node-steps/s", "value": value, "unit": "node-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "baseline_config": w["cfg"], "nodes": n,
                       "nnz": int(info["nnz"]), "model": w["model"], "dt_ms": w["dt"],
                       "dx_mm": w["dx"], "grid": list(dims) if weak else bench.mesh_desc(w),
                       "rcm": not args.no_rcm,
                       "preroll_steps": preroll, "parallelism": f"row blocks x{world} ({info['path']} PCG: "
                                      + ("NVLink peer memory" if info["path"] == "peer" else "NCCL") + ")",
                       "ghosts_rank0": int(info["ghosts"]),
                       "l2": "inputs larger than L2" if n > 1_000_000 else "small problem"},
            "sim_ms_per_wall_s": args.steps * w["dt"] / (ms / 1e3),
            "pcg_iters_per_step": iters / args.steps,
            "setup_s": t_setup,
            "roofline": {"kernel": f"{info['path']} PCG path (rank 0 rows)", "bound": "hbm",
                         "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"] if achieved else None,
                         "traffic": None, "peak_source": which,
                         "pcg_ms_per_step": prof["pcg_ms"] / args.steps,
                         "ionic_ms_per_step": prof["ionic_ms"] / args.steps},
            "cpu_baseline": None,
            "e2e": {"value": n * ke / e2e_s, "unit": "node-steps/s",
                    "h2d_bytes_per_step": int(hin.nbytes), "d2h_bytes_per_step": int(hout.nbytes)},
            "gpu_launches": int(round(prof["launches"])),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
