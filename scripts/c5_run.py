"""C5 (R-MAT scale 26, edge factor 16, ~2.1 B Bi-CSR slots) through the
vertex-range partitioned engine, on the GPUs this process sees.

    python scripts/c5_run.py --scale 26 --parts 2 --batch 1000000 --batches 2

With one GPU the parts share it (same kernels and host loop as the one-process-
per-GPU run; the cross-part traffic then stays in HBM instead of crossing
NVLink).  Ground truth at this size (no CPU reference can build the graph,
SURVEY 8c): after every dynamic batch the flow must equal a static re-solve on
the updated capacities, and flow == cut capacity for both.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_01235_b200 import partition  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--parts", type=int, default=2)
    ap.add_argument("--batch", type=int, default=1_000_000)
    ap.add_argument("--batches", type=int, default=2)
    ap.add_argument("--no-resolve", action="store_true")
    args = ap.parse_args()
    t0 = time.perf_counter()
    pg = partition.PartitionedGraph.rmat(args.scale, 16, 0, partition.LocalGroup(args.parts))
    out = {"config": f"C5-shape R-MAT scale {args.scale} ef 16 (device generator), "
                     f"{args.parts} parts on 1 GPU", "n": pg.n, "slots": pg.m,
           "m_original": pg.m_original, "slots_per_part": pg.slots.tolist(),
           "build_s": round(time.perf_counter() - t0, 2)}
    print(json.dumps(out), flush=True)
    pg.phase_s.clear()
    r = pg.solve_static()
    names = ["link", "link_pc", "init", "saturate", "bfs_init", "bfs_expand", "swap", "push",
             "repair", "final", "active", "resolve", "apply", "fix", "topo_seed"]

    def name(k):  # (PH_ASYNC entries: enqueue time of the concurrent form)
        return names[k & 0xFF] + ("/enqueue" if k & partition.PH_ASYNC else "")
    print(json.dumps({"static_phase_s": {name(k): round(v, 4) for k, v in pg.phase_s.items()}}))
    out = {"static_flow": r.flow_value, "static_s": round(r.seconds, 3), "rounds": r.rounds,
           "levels": r.bfs_levels, "waves": r.waves, "pushes": r.pushes,
           "static_edges_per_s": round(pg.m_original / r.seconds, 1)}
    print(json.dumps(out), flush=True)
    for b in range(args.batches):
        t1 = time.perf_counter()
        batch = pg.sample_batch(args.batch, seed=b)
        gen_s = time.perf_counter() - t1
        pg.phase_s.clear()
        d = pg.solve_dynamic(batch)
        print(json.dumps({"dynamic_phase_s": {name(k): round(v, 4) for k, v in pg.phase_s.items()}}))
        row = {"batch": b, "k": len(batch), "sample_s": round(gen_s, 2), "dyn_flow": d.flow_value,
               "dyn_s": round(d.seconds, 3), "rounds": d.rounds, "levels": d.bfs_levels,
               "waves": d.waves}
        if not args.no_resolve:
            rs = pg.solve_static()
            row.update({"resolve_flow": rs.flow_value, "resolve_s": round(rs.seconds, 3),
                        "agree": rs.flow_value == d.flow_value,
                        "speedup_vs_resolve": round(rs.seconds / d.seconds, 2)})
            assert rs.flow_value == d.flow_value, row
        print(json.dumps(row), flush=True)
    pg.close()


if __name__ == "__main__":
    main()
