"""Static-solve A/B of engine knobs on one graph (diagnostics): every knob
setting solves the same graph `--reps` times; prints mean / min ms, rounds.

    python scripts/static_ab.py --graph road --side 4900 --knobs '' MFX_L2_WINDOW=0
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
ap.add_argument("--graph", default="road")
ap.add_argument("--side", type=int, default=4900)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--knobs", nargs="*", default=[""])
a = ap.parse_args()
if a.graph == "road":
    us, vs, caps, s, t = gen.road_graph(a.side, a.side, 0, 0.21)
    n = a.side * a.side
elif a.graph == "rmat":
    us, vs, caps, s, t = gen.rmat_graph(a.side, 16, 0)
    n = 1 << a.side
else:
    us, vs, caps, s, t = gen.grid_graph(a.side, a.side, 0)
    n = a.side * a.side + 2
g = mfx.build_bicsr(mfx.EdgeListGraph(n, us, vs, caps))
st = mfx.init_residuals(g, s, t)
mfx.resolve_static(g, st)
for spec in a.knobs * 2:  # two passes: interleaved A/B
    kv_all = dict(kv.split("=") for kv in spec.split(",") if kv)
    env = {k: v for k, v in kv_all.items() if k.isupper()}  # MFX_* environment knobs
    params = mfx.SolverParams(**{k: int(v) for k, v in kv_all.items() if not k.isupper()})
    os.environ.update(env)
    ms, rounds = [], []
    for _ in range(a.reps):
        r = mfx.resolve_static(g, st, params)
        ms.append(r.device["ms_total"])
        rounds.append(r.rounds)
    d = r.device
    print(f"{spec or 'default':32s} mean {np.mean(ms):8.2f} ms  min {np.min(ms):8.2f}  rounds {rounds}"
          f"  levels {d['bfs_levels']} epochs {d['bfs_epochs']} waves {d['waves']}"
          f"  bfs {d['ns_bfs'] / 1e6:.1f} push {d['ns_push'] / 1e6:.1f} ms", flush=True)
    for k in env:
        os.environ.pop(k)
