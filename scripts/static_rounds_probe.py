"""Per-round anatomy of a static solve (diagnostics, host-stepped through
SolverParams.instrument): sink excess, excess holders and where they sit.

    python scripts/static_rounds_probe.py --side 4900
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_01235_b200 as mfx  # noqa: E402
from paper_2511_01235_b200 import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--side", type=int, default=4900)
a = ap.parse_args()
w = a.side
us, vs, caps, s, t = gen.road_graph(w, w, 0, 0.21)
n = w * w
g = mfx.build_bicsr(mfx.EdgeListGraph(n, us, vs, caps))
t0 = time.time()


def cb(st, gg, rnd, label):
    if label != "bfs":
        return
    ex = st.excess
    h = st.height
    hold = np.flatnonzero(ex > 0)
    hold = hold[(hold != s) & (hold != t)]
    act = hold[h[hold] < n]
    r, c = act // w, act % w
    dist = (w - 1 - r) + (w - 1 - c)
    print(f"round {rnd}: t excess {ex[t]}  holders {len(hold)} (excess {ex[hold].sum()})  active {len(act)}"
          f" (excess {ex[act].sum()})  labels {h[act].min() if len(act) else '-'}..{h[act].max() if len(act) else '-'}"
          f"  manhattan-to-t {dist.min() if len(act) else '-'}..{dist.max() if len(act) else '-'}"
          f"  [{time.time() - t0:.1f} s]", flush=True)


r = mfx.solve_static(g, s, t, mfx.SolverParams(instrument=cb))
print("flow", r.flow_value, "rounds", r.rounds)
