"""Per-batch anatomy of the C4 headline chain (diagnostics): the bench's
chained sparse_batch batches, each solve's device counters and phase split,
plus the per-barrier trace of the slowest batch when MFX_TRACE_CAP is set.

    python scripts/c4_probe.py [--side 4900] [--batches 13] [--knobs MFX_X=1,...]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import paper_2511_01235_b200 as mfx  # noqa: E402
from paper_2511_01235_b200 import gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=4900)
    ap.add_argument("--graph", default="road")
    ap.add_argument("--batches", type=int, default=13)
    ap.add_argument("--batch", type=int, default=10000)
    ap.add_argument("--knobs", nargs="*", default=[""])
    args = ap.parse_args()
    if args.graph == "road":
        us, vs, caps, s, t = gen.road_graph(args.side, args.side, 0, 0.21)
        n = args.side * args.side
    else:
        us, vs, caps, s, t = gen.grid_graph(args.side, args.side, 0)
        n = args.side * args.side + 2
    g0 = mfx.build_bicsr(mfx.EdgeListGraph(n, us, vs, caps))
    el = g0.to_edge_list()
    c = el.caps.copy()
    chain = []
    for i in range(args.batches):
        bu, bv, bc, pick = gen.sparse_batch(n, el.us, el.vs, c, s, t, args.batch, "mixed", i)
        c[pick] = bc
        chain.append((bu, bv, bc))
    for spec in args.knobs:
        env = dict(kv.split("=") for kv in spec.split(",") if kv)
        for k, v in env.items():
            os.environ[k] = v
        g = g0.copy()
        r = mfx.solve_static(g, s, t)
        d = r.device
        print(json.dumps({"knobs": spec or "default", "static_ms": round(d["ms_total"], 2),
                          "rounds": r.rounds, "levels": d["bfs_levels"], "epochs": d["bfs_epochs"],
                          "waves": d["waves"], "bfs_ms": round(d["ns_bfs"] / 1e6, 2),
                          "push_ms": round(d["ns_push"] / 1e6, 2)}), flush=True)
        st = r.state
        rows = []
        for i, (bu, bv, bc) in enumerate(chain):
            rr = mfx.solve_dynamic(st, g, mfx.UpdateBatch(bu, bv, bc))
            d = rr.device
            rows.append(d["ms_total"])
            print(json.dumps({"batch": i, "ms": round(d["ms_total"], 3), "flow": rr.flow_value,
                              "rounds": rr.rounds, "levels": d["bfs_levels"],
                              "epochs": d["bfs_epochs"], "waves": d["waves"],
                              "bfs_ms": round(d["ns_bfs"] / 1e6, 3),
                              "push_ms": round(d["ns_push"] / 1e6, 3),
                              "repair_ms": round(d["ns_repair"] / 1e6, 3),
                              "pushes": rr.pushes, "relabels": rr.relabels}), flush=True)
            if os.environ.get("MFX_TRACE_CAP"):
                import trace as T
                T.report(f"batch {i}", rr.state, g, rr)
            st = rr.state
        print(f"# {spec or 'default'}: mean {np.mean(rows[3:]):.2f} ms over batches 3..", flush=True)
        for k in env:
            os.environ.pop(k, None)


if __name__ == "__main__":
    main()
