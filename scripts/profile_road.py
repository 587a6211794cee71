"""Road-shaped static solve for ncu (diagnostics): build, a warm-up static
solve, then one static solve.  Launch order of solve_kernel: [warm, static].

    ncu --set full -k regex:solve_kernel --launch-skip 1 --launch-count 1 \
        python scripts/profile_road.py --side 2048
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_01235_b200 as mfx  # noqa: E402
from paper_2511_01235_b200 import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--side", type=int, default=2048)
a = ap.parse_args()
us, vs, caps, s, t = gen.road_graph(a.side, a.side, 0, 0.21)
g = mfx.build_bicsr(mfx.EdgeListGraph(a.side * a.side, us, vs, caps))
for _ in range(2):
    r = mfx.solve_static(g, s, t)
    print("static", r.flow_value, r.rounds, round(r.device["ms_total"], 2), "ms", flush=True)
