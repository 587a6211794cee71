"""Global relabel heights vs the oracle's FIFO BFS for several bfs_local
values (diagnostics for the CTA-local ring)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2511_01235_b200 as mf  # noqa: E402
from paper_2511_01235_b200 import gen  # noqa: E402
from test_gpu_parity import instance  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "grid64"
n, us, vs, caps, s, t = instance(name)
g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
ref = None
for bl in ["-1", "1", "2", "4", "8", "16", "32", "64", "128", "4096"]:
    os.environ["MFX_BFS_LOCAL"] = bl
    st = mf.init_residuals(g, s, t)
    mf.saturate_source(st, g)
    reached = mf.backward_bfs(st, g)
    h = np.asarray(st.height).copy()
    if ref is None:
        ref = h
    bad = np.flatnonzero(h != ref)
    print(f"bfs_local {bl:>5}: reached {reached} mismatches {bad.size}"
          + (f" e.g. v={bad[:5].tolist()} got {h[bad[:5]].tolist()} want {ref[bad[:5]].tolist()}" if bad.size else ""))
