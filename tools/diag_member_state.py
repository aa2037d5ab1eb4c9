#!/usr/bin/env python
"""Save the GPU state of cohort100 member 8 (grid engine) just before and after
the step that produced a NaN (diagnosis of the fast-exp / reciprocal range)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import meshgen as G  # noqa: E402
from diag_member_nan import build  # noqa: E402


def main():
    import paper_2510_12011_b200 as T
    i = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    m = G.cohort_members(100, seed=G.SEED)[i]
    s = build(T, m, "grid")
    L = T.tc_state_len(s.ctx)
    prev = None
    for k in range(1000):
        buf = np.empty(L)
        T._L.tc_get_state(s.ctx, T._ptr(buf), L)
        try:
            s.step(1)
        except T.TcError as ex:
            after = np.empty(L)
            T._L.tc_get_state(s.ctx, T._ptr(after), L)
            np.savez(os.path.join(ROOT, "gpurun_out", f"r01g_state_m{i}.npz"), before=buf, after=after, k=k,
                     err=str(ex))
            print("saved", k, ex)
            return
    print("no NaN")


if __name__ == "__main__":
    main()
