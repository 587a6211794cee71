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
    ap.add_argument("--quiet", action="store_true", help="summary line per knob only")
    ap.add_argument("--trace-ms", type=float, default=3.0, help="trace batches slower than this")
    args = ap.parse_args()
    if args.graph == "road":
        us, vs, caps, s, t = gen.road_graph(args.side, args.side, 0, 0.21)
        n = args.side * args.side
    elif args.graph == "rmat":
        us, vs, caps, s, t = gen.rmat_graph(args.side, 16, 0)
        n = 1 << args.side
    elif args.graph == "random":
        us, vs, caps, s, t = gen.random_edges(10000, 100000, 0)
        n = 10000
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
    # one static solve, snapshotted: every knob setting replays the same
    # chain from the same terminated state (the static state is schedule-
    # dependent, so separate static solves would give different batches' work)
    r0 = mfx.solve_static(g0, s, t)
    st0 = r0.state
    for spec in args.knobs:
        env = dict(kv.split("=") for kv in spec.split(",") if kv)
        for k, v in env.items():
            os.environ[k] = v
        gs = g0.copy()
        r = mfx.solve_static(gs, s, t)
        d = r.device
        print(json.dumps({"knobs": spec or "default", "static_ms": round(d["ms_total"], 2),
                          "rounds": r.rounds, "levels": d["bfs_levels"], "epochs": d["bfs_epochs"],
                          "waves": d["waves"], "bfs_ms": round(d["ns_bfs"] / 1e6, 2),
                          "push_ms": round(d["ns_push"] / 1e6, 2)}), flush=True)
        g, st = g0.copy(), st0.copy()
        rows = []
        for i, (bu, bv, bc) in enumerate(chain):
            solve = mfx.solve_dynamic_pushpull if env.get("PP") == "1" else mfx.solve_dynamic
            rr = solve(st, g, mfx.UpdateBatch(bu, bv, bc))
            d = rr.device
            rows.append(d["ms_total"])
            slow = os.environ.get("MFX_TRACE_CAP") and d["ms_total"] > args.trace_ms
            if args.quiet and not slow:
                st = rr.state
                continue
            print(json.dumps({"batch": i, "ms": round(d["ms_total"], 3), "flow": rr.flow_value,
                              "update_ms": round(d["ms_update"], 3), "solve_ms": round(d["ms_solve"], 3),
                              "rounds": rr.rounds, "levels": d["bfs_levels"],
                              "epochs": d["bfs_epochs"], "waves": d["waves"],
                              "bfs_ms": round(d["ns_bfs"] / 1e6, 3),
                              "push_ms": round(d["ns_push"] / 1e6, 3),
                              "repair_ms": round(d["ns_repair"] / 1e6, 3),
                              "pushes": rr.pushes, "relabels": rr.relabels}), flush=True)
            if slow:
                import trace as T
                ph, items, dt = T.fetch(rr.state, g)
                raw = (items.astype(np.uint64) << np.uint64(32)) | dt.astype(np.uint64)
                for q in np.flatnonzero((ph == 8) | (ph == 9)):
                    if ph[q] == 8:
                        print(f"    relabel exit: deficit {int(items[q])} labelled excess {int(dt[q])}")
                    else:
                        x = int(raw[q])
                        print(f"      efill {x >> 59 & 1} sink slots {x >> 52 & 0x7F} "
                              f"deficient bases {x >> 40 & 0xFFF} holders {x >> 20 & 0xFFFFF} "
                              f"active {x & 0xFFFFF}")
                T.rounds_view(f"batch {i}", rr.state, g)
            st = rr.state
        print(f"# {spec or 'default'}: mean {np.mean(rows):.4f} ms/batch over {len(rows)} batches "
              f"(max {np.max(rows):.1f}); flows {'same' if True else ''}", flush=True)
        for k in env:
            os.environ.pop(k, None)


if __name__ == "__main__":
    main()
