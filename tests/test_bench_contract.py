"""CPU checks of what bench.py reports (no GPU): the workloads are the configs
BASELINE.json / SURVEY 8 name, the closed-form pattern size of a Kuhn slab
equals the oracle's assembled pattern on small grids and the survey's counts at
full size, and the algorithmic bytes are SURVEY 8(d)'s formulas."""
import importlib.util
import json
import os
import sys

import numpy as np
import pytest

import meshgen as G
import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    argv = sys.argv
    sys.argv = ["bench.py"]
    try:
        spec.loader.exec_module(b)
    finally:
        sys.argv = argv
    return b


@pytest.mark.parametrize("dims", [(2, 2, 2), (3, 4, 5), (7, 3, 2), (6, 6, 6)])
def test_kuhn_nnz_equals_the_assembled_pattern(bench, dims):
    """n + 2 x (axis + face-diagonal + body-diagonal edges) of the Kuhn split
    (reading M1) = the entries of the oracle's pattern of the generated mesh."""
    xyz, tets = G.kuhn_box(*dims, 0.5)
    rp, col = O.pattern(xyz.shape[0], tets)
    assert bench.kuhn_nnz(*dims) == rp[-1]
    assert rp[-1] == col.shape[0]


def test_full_size_counts_match_the_survey(bench):
    """C* 10,000,000 nodes / 148,882,598 entries, C5 20,000,000 /
    298,163,398, C3 442,401 / 6,455,601, C1 4,305 / 56,769."""
    for dims, n, nnz in (((250, 200, 200), 10_000_000, 148_882_598), ((400, 250, 200), 20_000_000, 298_163_398),
                         ((201, 71, 31), 442_401, 6_455_601), ((41, 15, 7), 4_305, 56_769)):
        assert int(np.prod(dims)) == n
        assert bench.kuhn_nnz(*dims) == nnz, dims


def test_workloads_are_the_named_configs(bench):
    W = bench.WORKLOADS
    assert bench.DEFAULT_WORKLOAD == "slab20M_ms"
    d = W["slab20M_ms"]                       # configs[4]: ~20M-node MS slab
    assert d["cfg"] == 4 and d["model"] == "ms" and np.prod(d["dims"]) == 20_000_000
    d = W["slab10M_tt"]                       # north star: ~10M-node TT2006 slab
    assert d["cfg"] == "north_star" and d["model"] == "tt2006" and np.prod(d["dims"]) == 10_000_000
    d = W["nversion_dx0.1_tt"]                # configs[2]: dx 0.1, TT2006, dt 0.01
    assert d["cfg"] == 2 and d["dx"] == 0.1 and d["dt"] == 0.01 and d["model"] == "tt2006"
    d = W["nversion_dx0.5_tt"]                # configs[0]: dx 0.5, TT2006, dt 0.05
    assert d["cfg"] == 0 and d["dx"] == 0.5 and d["dt"] == 0.05
    assert W["biv3M_tt"]["cfg"] == 3 and W["biv3M_tt"]["model"] == "tt2006"
    cfgs = json.load(open(os.path.join(ROOT, "BASELINE.json")))["configs"]
    assert "20M" in cfgs[4] and "Mitchell" in cfgs[4] and "dx=0.1" in cfgs[2] and "dx=0.5" in cfgs[0]
    for name, w in W.items():
        assert w["model"] in ("ms", "tt2006", "crn"), name
        assert w["dt"] > 0 and w["preroll"] >= 0, name


def test_algorithmic_bytes_are_survey_8d(bench):
    n, nnz, it, steps = 1000, 15000, 70, 10
    cg, ion = bench.bytes_per_step(n, nnz, it, "tt2006", steps)
    b_it = 12 * nnz + 4 * (n + 1) + 72 * n
    b_rhs = 20 * nnz + 4 * (n + 1) + 44 * n
    assert cg == steps * b_rhs + it * b_it
    assert ion == steps * 352 * n
    assert bench.bytes_per_step(n, nnz, it, "ms", steps)[1] == steps * 80 * n
