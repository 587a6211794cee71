"""Host overhead of one solve_dynamic_device call (diagnostics): wall time
per call vs the device's own ms_total, on the C4 chain.

    python scripts/host_overhead.py [--side 4900] [--batches 40]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_01235_b200 as mfx  # noqa: E402
from paper_2511_01235_b200 import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--side", type=int, default=4900)
ap.add_argument("--batches", type=int, default=40)
a = ap.parse_args()
us, vs, caps, s, t = gen.road_graph(a.side, a.side, 0, 0.21)
n = a.side * a.side
g = mfx.build_bicsr(mfx.EdgeListGraph(n, us, vs, caps))
st = mfx.solve_static(g, s, t).state
el = g.to_edge_list()
c = el.caps.copy()
dev = []
for i in range(a.batches):
    bu, bv, bc, pick = gen.sparse_batch(n, el.us, el.vs, c, s, t, 10000, "mixed", i)
    c[pick] = bc
    dev.append(tuple(torch.from_numpy(x).cuda() for x in (bu, bv, bc)))
torch.cuda.synchronize()
p = mfx.SolverParams()
wall, devms = [], []
for i, (bu, bv, bc) in enumerate(dev):
    t0 = time.perf_counter()
    r = mfx.solve_dynamic_device(st, g, 10000, bu.data_ptr(), bv.data_ptr(), bc.data_ptr(), p)
    wall.append((time.perf_counter() - t0) * 1e3)
    devms.append(r.device["ms_total"])
    st = r.state
wall, devms = np.array(wall[3:]), np.array(devms[3:])
print(f"wall per call {wall.mean():.3f} ms, device ms_total {devms.mean():.3f} ms, "
      f"host overhead {np.mean(wall - devms) * 1e3:.1f} us (median {np.median(wall - devms) * 1e3:.1f})")
