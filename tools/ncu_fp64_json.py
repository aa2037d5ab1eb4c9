#!/usr/bin/env python
"""Rewrite the slab10M_tt / slab10M_crn entries of profiles/ncu_fp64.json (and the
TT2006 entries that reuse the 10 M per-node work) from the ncu FP64 instruction
counts that tools/ncu_fp64.sh captured:

  python tools/ncu_fp64_json.py <round tag, e.g. r01g>   (reads profiles/<tag>_fp64ops_*.csv)

flop = 2 dfma + dadd + dmul (thread-level, predicated on); per node = / 10 M."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NODES = 250 * 200 * 200


def read(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    m = {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in rows}
    name = rows[0]["Kernel Name"].split("(")[0]
    return name, m


def main():
    tag = sys.argv[1]
    p = os.path.join(ROOT, "profiles", "ncu_fp64.json")
    data = json.load(open(p))
    for wl in ("slab10M_tt", "slab10M_crn"):
        src = os.path.join("profiles", f"{tag}_fp64ops_{wl}.csv")
        name, m = read(os.path.join(ROOT, src))
        fma = m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
        add = m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
        mul = m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
        ent = data.get(wl, {})
        ent.update(kernel=name, flop_per_node=round((2 * fma + add + mul) / NODES, 4),
                   fp64_inst_per_node=round((fma + add + mul) / NODES, 4),
                   fp64_pipe_active_ncu=round(m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"] / 100, 4),
                   ncu_ms=m["gpu__time_duration.sum"] / 1e6, capture=src)
        data[wl] = ent
    tt = data["slab10M_tt"]
    for k, v in data.items():
        if isinstance(v, dict) and k not in ("slab10M_tt", "slab10M_crn") and v.get("kernel") == "ionic_tt_kernel":
            v.update({f: tt[f] for f in ("flop_per_node", "fp64_inst_per_node", "fp64_pipe_active_ncu", "ncu_ms")})
    data["_what"] = data["_what"].split("profiles/r01")[0] + f"profiles/{tag}_fp64ops_*.csv (tools/ncu_fp64.sh)); " \
        "flop = 2 dfma + dadd + dmul; peak = measured DFMA rate (profiles/r01_probe_fp64.txt, 34.2 TFLOP/s)"
    json.dump(data, open(p, "w"), indent=1)
    print(json.dumps({k: data[k] for k in ("slab10M_tt", "slab10M_crn")}, indent=1))


if __name__ == "__main__":
    main()
