"""Regenerate the golden fixtures from the LIVE reference (run in the build
container, where /root/reference exists; the GPU box only reads the output).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.json (flows, sizes, sha256 of reference arrays,
reference error messages) and tests/golden/golden.npz (full arrays for the
small cases).  Every value below is produced by the reference package
``dynmaxflow`` itself (build_bicsr, solve_static(deterministic=True),
solve_dynamic, bfs_heights, apply_updates/recompute_excess/saturate_source,
generate_batch, random_graph); only the C2-C4 *shapes* come from this repo's
generator (the reference ships no grid/R-MAT/road generator).
"""

import hashlib
import json
import os
import sys

import numpy as np

REF = os.environ.get("DYNMAXFLOW_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import dynmaxflow as mf  # noqa: E402  (the reference)
from dynmaxflow import kernels as K  # noqa: E402

from paper_2511_01235_b200 import gen  # noqa: E402  (shapes only)


def sha(a) -> str:
    a = np.asarray(a)
    if a.dtype == np.bool_:
        a = a.astype(np.uint8)
    else:
        a = a.astype(np.int64)
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


ARR = {}


def put(name, a):
    a = np.asarray(a)
    ARR[name] = a.astype(np.uint8) if a.dtype == np.bool_ else a.astype(np.int64)


def det():
    return mf.SolverParams(deterministic=True)


def graph_record(csr):
    return {
        "n": csr.n, "S": csr.m, "m_original": csr.m_original,
        "diag": [csr.diagnostics.self_loops_dropped, csr.diagnostics.parallel_edges_merged,
                 csr.diagnostics.reverse_stubs_added],
        "sha": {k: sha(getattr(csr, k)) for k in
                ("offsets", "adj", "src", "rev", "cap0", "is_original")},
    }


def bfs(st, csr, bases, forbidden):
    h = st.height.copy()
    q = np.empty(csr.n, np.int64)
    K.bfs_heights(csr.offsets, csr.adj, csr.rev, st.cf, h, np.asarray(bases, np.int64),
                  csr.n, False, forbidden, np.empty(0, np.int8), -1, q)
    return h


def prephase(st, csr, batch):
    """apply_updates + recompute_excess + saturate_source (dynamic.py:157-159)."""
    st2, g2 = st.copy(), csr.copy()
    mf.apply_updates(st2, g2, batch)
    mf.recompute_excess(st2, g2)
    mf.saturate_source(st2, g2)
    return st2, g2


def dyn_bases(st):
    mask = mf.deficient_mask(st)
    mask[st.sink] = True
    return np.flatnonzero(mask)


def case_instance(name, n, us, vs, caps, s, t, batches, full_arrays, record, source=None):
    """Build, deterministic static solve, BFS checkpoints, then chained
    dynamic batches (each batch drawn by the reference generate_batch from the
    current normalized edge list)."""
    g = mf.EdgeListGraph(n, np.asarray(us, np.int64), np.asarray(vs, np.int64),
                         np.asarray(caps, np.int64))
    csr = mf.build_bicsr(g)
    rec = {"s": int(s), "t": int(t), "n": int(n), "graph": graph_record(csr),
           "source": source, "input_sha": [sha(g.us), sha(g.vs), sha(g.caps)]}
    if full_arrays:
        put(f"{name}/in_us", g.us)
        put(f"{name}/in_vs", g.vs)
        put(f"{name}/in_caps", g.caps)
        for k in ("offsets", "adj", "src", "rev", "cap0", "is_original"):
            put(f"{name}/{k}", getattr(csr, k))
    res = mf.solve_static(csr, s, t, det())
    rec["static_flow"] = res.flow_value
    rec["static_rounds_det"] = res.rounds
    st = res.state
    rec["static_state_sha"] = {k: sha(getattr(st, k)) for k in ("cf", "excess", "height")}
    # BFS checkpoint on the post-saturation state (state.py:42-59 then the
    # first global relabel of solver.py:216)
    st0 = mf.init_residuals(csr, s, t)
    mf.saturate_source(st0, csr)
    h0 = bfs(st0, csr, [t], -1)
    rec["bfs_sat_sha"] = sha(h0)
    rec["sat_sha"] = {k: sha(getattr(st0, k)) for k in ("cf", "excess")}
    if full_arrays:
        put(f"{name}/sat_cf", st0.cf)
        put(f"{name}/sat_excess", st0.excess)
        put(f"{name}/bfs_sat_h", h0)
    chain = []
    cur_st, cur_g = st, csr
    for bi, (kind, pct_or_k, seed) in enumerate(batches):
        el = cur_g.to_edge_list()
        pct = pct_or_k if isinstance(pct_or_k, float) else gen.pct_for_count(pct_or_k, el.m)
        batch = mf.generate_batch(el, s, t, mf.BatchSpec(pct=pct, kind=kind, seed=seed))
        pre_st, pre_g = prephase(cur_st, cur_g, batch)
        hb = bfs(pre_st, pre_g, dyn_bases(pre_st), s)
        entry = {
            "kind": kind, "pct": pct, "seed": seed, "k": len(batch),
            "batch_sha": [sha(batch.us), sha(batch.vs), sha(batch.new_caps)],
            "prior_state_sha": {k: sha(getattr(cur_st, k)) for k in ("cf", "excess", "height")},
            "pre_sha": {"cf": sha(pre_st.cf), "excess": sha(pre_st.excess),
                        "cap0": sha(pre_g.cap0)},
            "bfs_dyn_sha": sha(hb),
        }
        if full_arrays:
            for k in ("cf", "excess", "height"):
                put(f"{name}/b{bi}/prior_{k}", getattr(cur_st, k))
            put(f"{name}/b{bi}/prior_cap0", cur_g.cap0)
            put(f"{name}/b{bi}/us", batch.us)
            put(f"{name}/b{bi}/vs", batch.vs)
            put(f"{name}/b{bi}/caps", batch.new_caps)
            put(f"{name}/b{bi}/pre_cf", pre_st.cf)
            put(f"{name}/b{bi}/pre_excess", pre_st.excess)
            put(f"{name}/b{bi}/pre_cap0", pre_g.cap0)
            put(f"{name}/b{bi}/bfs_dyn_h", hb)
        r = mf.solve_dynamic(cur_st.copy(), cur_g.copy(), batch, det())
        entry["flow"] = r.flow_value
        entry["rounds_det"] = r.rounds
        entry["state_sha"] = {k: sha(getattr(r.state, k)) for k in ("cf", "excess", "height")}
        # independent check: static solve on the updated graph
        upd = mf.build_bicsr(mf.updated_edge_list(cur_g, batch))
        entry["resolve_flow"] = mf.solve_static(upd, s, t, det()).flow_value
        assert entry["resolve_flow"] == entry["flow"], (name, bi)
        chain.append(entry)
        cur_st, cur_g = r.state, r.graph
    rec["chain"] = chain
    record[name] = rec
    print(f"{name}: n={n} S={csr.m} static={rec['static_flow']} "
          f"chain={[c['flow'] for c in chain]}", flush=True)


def error_messages():
    out = {}
    cases = {
        "n0": (0, [], [], []),
        "src_range": (3, [0, 5], [1, 2], [1, 1]),
        "dst_range": (3, [0, 1], [1, -1], [1, 1]),
        "neg_cap": (3, [0, 1], [1, 2], [1, -4]),
    }
    for key, (n, us, vs, caps) in cases.items():
        try:
            mf.build_bicsr(mf.EdgeListGraph(n, np.asarray(us, np.int64),
                                            np.asarray(vs, np.int64), np.asarray(caps, np.int64)))
        except mf.GraphError as exc:
            out["graph/" + key] = str(exc)
    g = mf.EdgeListGraph.from_edges(4, [(0, 1, 3), (0, 2, 2), (1, 3, 2), (2, 3, 3), (1, 2, 1)])
    csr = mf.build_bicsr(g)
    res = mf.solve_static(csr, 0, 3, det())
    bcases = {
        "neg": [(0, 1, 2), (1, 3, -1)],
        "unknown": [(0, 1, 2), (0, 3, 5)],
        "stub": [(1, 0, 5)],
        "dup": [(1, 3, 1), (0, 1, 2), (1, 3, 4), (0, 1, 3)],
    }
    for key, ups in bcases.items():
        try:
            mf.apply_updates(res.state.copy(), csr.copy(), mf.UpdateBatch.from_updates(ups))
        except mf.BatchError as exc:
            out["batch/" + key] = str(exc)
    for key, (s, t) in {"s_range": (7, 1), "t_range": (0, -1), "same": (2, 2)}.items():
        try:
            mf.solve_static(csr, s, t)
        except ValueError as exc:
            out["endpoints/" + key] = str(exc)
    return out


def main():
    record = {}
    # SPEC examples
    spec_graphs = {
        "spec_single": (2, [(0, 1, 7)], 0, 1),
        "spec_parallel": (2, [(0, 1, 3), (0, 1, 4)], 0, 1),
        "spec_mutual": (3, [(0, 1, 5), (1, 0, 2), (1, 2, 1)], 0, 2),
        "diamond": (4, [(0, 1, 3), (0, 2, 2), (1, 3, 2), (2, 3, 3), (1, 2, 1)], 0, 3),
        "chain4": (4, [(0, 1, 5), (1, 2, 5), (2, 3, 5)], 0, 3),
        "star": (6, [(0, 1, 2), (0, 2, 2), (1, 5, 1), (2, 5, 1), (3, 5, 4), (4, 5, 4)], 0, 5),
        "split": (4, [(0, 1, 3), (2, 3, 3)], 0, 3),
        "k33": (8, [(0, a, 1) for a in (1, 2, 3)] + [(b, 7, 1) for b in (4, 5, 6)]
                + [(a, b, 1) for a in (1, 2, 3) for b in (4, 5, 6)], 0, 7),
        "sat_mutual": (3, [(0, 1, 4), (1, 0, 1), (1, 2, 9)], 0, 2),
    }
    for name, (n, edges, s, t) in spec_graphs.items():
        us = [e[0] for e in edges]
        vs = [e[1] for e in edges]
        caps = [e[2] for e in edges]
        case_instance(name, n, us, vs, caps, s, t, [], True, record)
    # dynamic SPEC examples on the diamond
    g = mf.EdgeListGraph.from_edges(4, [(0, 1, 3), (0, 2, 2), (1, 3, 2), (2, 3, 3), (1, 2, 1)])
    csr = mf.build_bicsr(g)
    base = mf.solve_static(csr, 0, 3, det())
    record["diamond_dyn"] = {}
    for key, ups in {"dec01": [(0, 1, 1)], "inc13": [(1, 3, 4)], "empty": []}.items():
        r = mf.solve_dynamic(base.state.copy(), csr.copy(), mf.UpdateBatch.from_updates(ups), det())
        record["diamond_dyn"][key] = {"updates": ups, "flow": r.flow_value, "rounds": r.rounds}

    # SPEC acceptance-1/2 style random instances (small; full arrays kept)
    rng = np.random.default_rng(1234)
    for i in range(24):
        n = int(rng.integers(2, 201))
        m = int(rng.integers(1, 2001))
        g, s, t = mf.random_graph(n, m, seed=i)
        kinds = [("inc", 5.0, i), ("dec", 10.0, i + 1), ("mixed", 25.0, i + 2), ("mixed", 1.0, i + 3)]
        case_instance(f"rand{i}", n, g.us, g.vs, g.caps, s, t, kinds, True, record,
                      {"gen": "random_graph", "args": [n, m, i]})

    # C1 = reference random_graph(10000, 100000, seed=0) + a 1,000-update mixed batch
    g, s, t = mf.random_graph(10000, 100000, seed=0)
    case_instance("C1", 10000, g.us, g.vs, g.caps, s, t,
                  [("mixed", 1000, 0), ("mixed", 1000, 1)], False, record,
                  {"gen": "random_graph", "args": [10000, 100000, 0]})

    # scaled-down C2/C3/C4 shapes (CPU-reference anchors for the full configs)
    us, vs, caps, s, t = gen.grid_graph(64, 64, seed=0)
    case_instance("grid64", 64 * 64 + 2, us, vs, caps, s, t,
                  [("mixed", 200, 0), ("inc", 100, 1), ("dec", 100, 2)], False, record,
                  {"gen": "grid_graph", "args": [64, 64, 0]})
    us, vs, caps, s, t = gen.rmat_graph(12, 16, seed=0)
    case_instance("rmat12", 1 << 12, us, vs, caps, s, t,
                  [("mixed", 500, 0), ("mixed", 2000, 1)], False, record,
                  {"gen": "rmat_graph", "args": [12, 16, 0]})
    us, vs, caps, s, t = gen.road_graph(48, 48, seed=0, p_vert=0.2)
    case_instance("road48", 48 * 48, us, vs, caps, s, t,
                  [("mixed", 100, 0), ("mixed", 100, 1)], False, record,
                  {"gen": "road_graph", "args": [48, 48, 0, 0.2]})
    us, vs, caps, s, t = gen.grid_graph(256, 256, seed=0)
    case_instance("grid256", 256 * 256 + 2, us, vs, caps, s, t, [("mixed", 1000, 0)], False, record,
                  {"gen": "grid_graph", "args": [256, 256, 0]})

    record["errors"] = error_messages()
    record["reference"] = {"backend": mf.backend_name(), "numpy": np.__version__,
                           "version": mf.__version__}
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(record, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **ARR)
    print("wrote", len(ARR), "arrays")


if __name__ == "__main__":
    main()
