#!/usr/bin/env python
"""DRAM bytes of the PCG path of one captured time step (rhs_kernel +
pcg_kernel) from an ncu --set full report -> profiles/ncu_traffic.json, which
bench.py reads for roofline.traffic (rescaled to the timed mean iteration count).

  python tools/ncu_traffic.py <workload> <report.ncu-rep> <iters_of_captured_step> <capture_summary>
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    wl, rep, iters, summ = sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    rhs = pcg = 0.0
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "")
        b = float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])
        unit = rows[1][h.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        if "rhs_kernel" in name:
            rhs = b * scale
        elif "pcg_kernel" in name:
            pcg = b * scale
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    data = json.load(open(p)) if os.path.exists(p) else {}
    data[wl] = {"rhs_bytes": rhs, "pcg_bytes": pcg, "iters": iters, "capture": summ}
    if rhs == 0.0:   # variant 4 with the RHS fused into the PCG kernel: pcg_bytes holds both
        data[wl]["rhs_fused"] = True
    json.dump(data, open(p, "w"), indent=1)
    print(wl, data[wl])


if __name__ == "__main__":
    main()
