"""Static C2 solve: rounds / pushes / relabels / repairs (diagnostics)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_01235_b200 as mfx  # noqa: E402
from paper_2511_01235_b200 import gen  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
us, vs, caps, s, t = gen.grid_graph(side, side, 0)
g = mfx.build_bicsr(mfx.EdgeListGraph(side * side + 2, us, vs, caps))
for _ in range(2):
    r = mfx.solve_static(g.copy(), s, t)
    print(f"flow {r.flow_value} rounds {r.rounds} pushes {r.pushes} relabels {r.relabels} "
          f"repairs {r.repairs} ms {r.device['ms_solve']:.2f} waves {r.device['waves']}")
