#!/usr/bin/env python
"""N-version benchmark at Table 3's settings (dt 0.005 ms, dx 0.5 /
0.2 / 0.1 mm, 100 ms): LAT along the P1 -> P8 diagonal (21 samples) for each
dx, on the GPU.  Writes the table as JSON (argv[1], default stdout).
Same runner as tests/test_gpu_nversion.py."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2510_12011_b200 as T  # noqa: E402
from test_gpu_nversion import DT, T_END, TOL, run_gpu  # noqa: E402

t3 = json.load(open(os.path.join(ROOT, "tests", "golden", "table3_nversion.json")))
out = {"what": "LAT (ms) along the P1 (0,0,0) -> P8 (20,7,3) diagonal, 21 samples s = 0, 0.05, ..., 1 "
               "(nearest node, ties lowest index), PAPER.md Table 3 N-version settings",
       "dt_ms": DT, "t_end_ms": T_END, "pcg_abs_tol": TOL, "s": list(np.linspace(0, 1, 21)), "runs": {}}
for dx in t3["dx_mm"]:
    t0 = time.time()
    lat, lrt, iters, diag, xyz = run_gpu(T, t3, dx)
    out["runs"][str(dx)] = {"nodes": int(xyz.shape[0]), "lat_diag_ms": [float(v) for v in lat[diag]],
                            "lat_P8_ms": float(lat[diag[-1]]), "all_activated": bool((lat >= 0).all()),
                            "mean_pcg_iters": float(np.mean(iters)), "wall_s": time.time() - t0}
r = out["runs"]
out["refinement_gap_P8_ms"] = {"0.5-0.2": r["0.5"]["lat_P8_ms"] - r["0.2"]["lat_P8_ms"],
                               "0.2-0.1": r["0.2"]["lat_P8_ms"] - r["0.1"]["lat_P8_ms"]}
s = json.dumps(out, indent=1)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(s)
print(s)
