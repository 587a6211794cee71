"""Parameter sweep on the GPU: static solve + chained dynamic batches for
several solver knobs; prints per-setting timing and phase split, and checks
every setting agrees on every flow.

    python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 3 \
        --knobs 'max_waves=0' 'max_waves=8' 'wave_mult=4,wave_add=32' 'MFX_TAIL_LOCAL=0'

Knobs are SolverParams fields, or MFX_* environment knobs (read per solve;
MFX_VARIANT is fixed per graph at its first solve, so it needs its own run).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_01235_b200 as mfx  # noqa: E402
from paper_2511_01235_b200 import gen  # noqa: E402


def instance(kind, side, scale):
    if kind == "grid":
        us, vs, caps, s, t = gen.grid_graph(side, side, 0)
        return side * side + 2, us, vs, caps, s, t
    if kind == "rmat":
        us, vs, caps, s, t = gen.rmat_graph(scale, 16, 0)
        return 1 << scale, us, vs, caps, s, t
    if kind == "road":
        us, vs, caps, s, t = gen.road_graph(side, side, 0, 0.21)
        return side * side, us, vs, caps, s, t
    if kind == "random":
        us, vs, caps, s, t = gen.random_edges(10000, 100000, 0)
        return 10000, us, vs, caps, s, t
    raise ValueError(kind)


ENV_SET = set()


def parse_knobs(spec):
    out = {}
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        out[k] = int(v) if v.lstrip("-").isdigit() else v
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--graph", default="grid")
    ap.add_argument("--side", type=int, default=2048)
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--batch", type=int, default=10000)
    ap.add_argument("--batches", type=int, default=3)
    ap.add_argument("--knobs", nargs="+", default=[""])
    ap.add_argument("--barrier", action="store_true")
    args = ap.parse_args()
    n, us, vs, caps, s, t = instance(args.graph, args.side, args.scale)
    t0 = time.perf_counter()
    g = mfx.build_bicsr(mfx.EdgeListGraph(n, us, vs, caps))
    print(f"# {args.graph} n={n} S={g.m} m_orig={g.m_original} build {time.perf_counter()-t0:.2f}s "
          f"cap_bytes={g.cap_bytes}", flush=True)
    if args.barrier:
        import ctypes
        from paper_2511_01235_b200 import _lib
        st = mfx.init_residuals(g, s, t)
        for bps in (1, 2, 3, 4):
            ns = ctypes.c_double()
            _lib.check(_lib.load().mfx_bench_barrier(g.handle, st.handle, 20000, bps,
                                                     ctypes.byref(ns)))
            print(f"# grid barrier: {bps} CTA/SM -> {ns.value:.0f} ns", flush=True)
    el = g.to_edge_list()
    chain = []
    c = el.caps.copy()
    for i in range(args.batches):
        bu, bv, bc, pick = gen.fast_batch(n, el.us, el.vs, c, s, t, args.batch, "mixed", i)
        c[pick] = bc
        chain.append((bu, bv, bc))
    ref_flows = None
    base = g.copy()
    for spec in args.knobs:
        kn = parse_knobs(spec)
        pp = bool(kn.pop("pp", 0))  # O2 push-pull dynamic solves
        for k in ENV_SET:
            os.environ.pop(k, None)
        ENV_SET.clear()
        for k in [k for k in kn if k.startswith("MFX_")]:  # engine env knobs
            os.environ[k] = str(kn.pop(k))
            ENV_SET.add(k)
        p = mfx.SolverParams(**kn)
        gg = base.copy()
        mfx.solve_static(gg, s, t, p)  # warm
        r = mfx.solve_static(gg, s, t, p)
        d = r.device
        row = {"knobs": spec or "default", "static_ms": round(d["ms_total"], 2),
               "st_rounds": r.rounds, "st_levels": d["bfs_levels"], "st_epochs": d["bfs_epochs"], "st_waves": d["waves"],
               "st_bfs_ms": round(d["ns_bfs"] / 1e6, 2), "st_push_ms": round(d["ns_push"] / 1e6, 2),
               "st_repair_ms": round(d["ns_repair"] / 1e6, 2), "st_pushes": r.pushes,
               "st_relabels": r.relabels, "st_GBs": round(d["bytes_alg"] / d["ms_solve"] / 1e6, 1)}
        flows = [r.flow_value]
        st = r.state
        dyn = []
        for bu, bv, bc in chain:
            solve = mfx.solve_dynamic_pushpull if pp else mfx.solve_dynamic
            rr = solve(st, gg, mfx.UpdateBatch(bu, bv, bc), p)
            flows.append(rr.flow_value)
            dd = rr.device
            dyn.append((dd["ms_total"], rr.rounds, dd["bfs_levels"], dd["waves"], dd["ns_bfs"] / 1e6,
                        dd["ns_push"] / 1e6, dd["ns_repair"] / 1e6, dd["ms_update"], dd["bfs_epochs"]))
            st = rr.state
        a = np.array(dyn)
        row.update({"dyn_ms": round(a[:, 0].mean(), 2), "dyn_rounds": round(a[:, 1].mean(), 1),
                    "dyn_levels": round(a[:, 2].mean(), 1), "dyn_waves": round(a[:, 3].mean(), 1),
                    "dyn_bfs_ms": round(a[:, 4].mean(), 2), "dyn_push_ms": round(a[:, 5].mean(), 2),
                    "dyn_repair_ms": round(a[:, 6].mean(), 2), "dyn_update_ms": round(a[:, 7].mean(), 3),
                    "dyn_epochs": round(a[:, 8].mean(), 1)})
        rep = mfx.verify_gpu(st, gg, flows[-1])
        row["verified"] = rep.ok
        if ref_flows is None:
            ref_flows = flows
        row["flows_agree"] = flows == ref_flows
        print(json.dumps(row), flush=True)
    print("# flows", ref_flows)


if __name__ == "__main__":
    main()
