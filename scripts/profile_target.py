"""Small, deterministic workload for ncu: build C2 (or a smaller grid), one
warm-up static solve, one static solve, then `--batches` dynamic batches.
Launch order of mfx::solve_kernel: [warm static, static, dyn 1, dyn 2, ...,
relabel 1, ...].

    ncu --set full -k regex:solve_kernel --launch-skip 2 --launch-count 1 \
        python scripts/profile_target.py      # profiles dynamic batch 1
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_01235_b200 as mfx  # noqa: E402
from paper_2511_01235_b200 import gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=2048)
    ap.add_argument("--batch", type=int, default=10000)
    ap.add_argument("--batches", type=int, default=2)
    ap.add_argument("--relabels", type=int, default=0,
                    help="then this many dynamic global relabels (WHAT_BFS launches)")
    args = ap.parse_args()
    us, vs, caps, s, t = gen.grid_graph(args.side, args.side, 0)
    n = args.side * args.side + 2
    g = mfx.build_bicsr(mfx.EdgeListGraph(n, us, vs, caps))
    mfx.solve_static(g, s, t)
    r = mfx.solve_static(g, s, t)
    el = g.to_edge_list()
    c = el.caps.copy()
    st = r.state
    out = [("static", r.flow_value, r.device["ms_solve"])]
    for i in range(args.batches):
        bu, bv, bc, pick = gen.fast_batch(n, el.us, el.vs, c, s, t, args.batch, "mixed", i)
        c[pick] = bc
        rr = mfx.solve_dynamic(st, g, mfx.UpdateBatch(bu, bv, bc))
        out.append((f"dyn{i}", rr.flow_value, rr.device["ms_solve"]))
        st = rr.state
    for i in range(args.relabels):  # BFS alone on the last state (dynamic bases)
        out.append((f"relabel{i}", mfx.backward_bfs_dynamic(st, g), 0.0))
    for row in out:
        print(*row)


if __name__ == "__main__":
    main()
