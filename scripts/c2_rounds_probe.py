"""Per-round anatomy of one C2 dynamic batch (diagnostics, host-stepped via
SolverParams.instrument): active vertices after each relabel, their labels,
excess, and how many of them are still active at the next relabel.

    python scripts/c2_rounds_probe.py [--side 2048]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_01235_b200 as mfx  # noqa: E402
from paper_2511_01235_b200 import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--side", type=int, default=2048)
a = ap.parse_args()
us, vs, caps, s, t = gen.grid_graph(a.side, a.side, 0)
n = a.side * a.side + 2
g = mfx.build_bicsr(mfx.EdgeListGraph(n, us, vs, caps))
st = mfx.solve_static(g, s, t).state
el = g.to_edge_list()
bu, bv, bc, _ = gen.sparse_batch(n, el.us, el.vs, el.caps, s, t, 10000, "mixed", 0)
prev = {}


def cb(st, gg, rnd, label):
    ex, h = st.excess, st.height
    act = np.flatnonzero((ex > 0) & (h < n))
    act = act[(act != s) & (act != t)]
    if label == "bfs":
        kept = len(np.intersect1d(act, prev.get("act", np.empty(0, np.int64))))
        deficit = -ex[(ex < 0) & (np.arange(n) != s)].sum()
        hl = h[act]
        print(f"round {rnd} relabel: active {act.size} (excess {ex[act].sum()}), "
              f"labels {np.percentile(hl, [0, 50, 90, 100]).astype(int).tolist() if act.size else '-'}, "
              f"still active from the last relabel {kept}, deficit left {deficit}, "
              f"reached {(h < n).sum()}", flush=True)
        prev["act"] = act
    else:
        print(f"round {rnd} after push+repair: active {act.size} (excess {ex[act].sum()})", flush=True)


r = mfx.solve_dynamic(st, g, mfx.UpdateBatch(bu, bv, bc), mfx.SolverParams(instrument=cb))
print("flow", r.flow_value, "rounds", r.rounds)
