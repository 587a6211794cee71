"""O2 push-pull dynamic solve (reference dynamic.py:292-377) on the GPU: the
flow after every chained batch equals the reference's (golden fixtures, made
with solve_dynamic; the reference states push-pull gives the identical
value), plain and push-pull batches interleave on one state, and a state
without a cut certificate is rejected like the reference."""
import json
import os

import numpy as np
import pytest

from golden_data import load
from paper_2511_01235_b200 import gen

pytestmark = pytest.mark.gpu
G = load()


@pytest.fixture(scope="module")
def mf():
    import paper_2511_01235_b200 as m
    return m


def instance(name):
    rec = G.rec[name]
    if f"{name}/in_us" in G.arr:
        return (rec["n"], G.arr[f"{name}/in_us"], G.arr[f"{name}/in_vs"],
                G.arr[f"{name}/in_caps"], rec["s"], rec["t"])
    src = rec["source"]
    us, vs, caps, s, t = gen.source_edges(src["gen"], src["args"])
    return rec["n"], us, vs, caps, s, t


@pytest.mark.parametrize("name", ["rand0", "rand1", "rand5", "rand7", "rand13", "rand16", "rand20",
                                  "C1", "grid64", "grid256", "rmat12", "road48"])
@pytest.mark.parametrize("interleave", [False, True])
def test_pushpull_chain_matches_reference(mf, name, interleave):
    rec = G.rec[name]
    n, us, vs, caps, s, t = instance(name)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    st = mf.solve_static(g, s, t).state
    keep = g.is_original.astype(bool)
    for j, entry in enumerate(rec["chain"]):
        spec = gen.BatchSpec(entry["pct"], entry["kind"], entry["seed"])
        bu, bv, bc, _ = gen.batch_arrays(n, g.src[keep], g.adj[keep], g.cap0[keep], s, t, spec)
        fn = mf.solve_dynamic if (interleave and j % 2) else mf.solve_dynamic_pushpull
        r = fn(st, g, mf.UpdateBatch(bu, bv, bc))
        assert r.flow_value == entry["flow"] == r.certificate.cut_capacity, (name, j)
        rep = mf.verify_gpu(r.state, g, r.flow_value)
        assert rep.ok, rep.problems
        st = r.state


def test_pushpull_full_size_c2_matches_reference(mf):
    with open(os.path.join(os.path.dirname(__file__), "golden", "large.json")) as fh:
        rec = json.load(fh)["C2"]
    us, vs, caps, s, t = gen.grid_graph(*rec["args"])
    n = rec["n"]
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    st = mf.solve_static(g, s, t).state
    el = g.to_edge_list()
    ecaps = el.caps.copy()
    for entry in rec["chain"]:
        bu, bv, bc, pick = gen.fast_batch(n, el.us, el.vs, ecaps, s, t, entry["k"], "mixed",
                                          entry["seed"])
        ecaps[pick] = bc
        r = mf.solve_dynamic_pushpull(st, g, mf.UpdateBatch(bu, bv, bc))
        assert r.flow_value == entry["flow"]
        st = r.state


def test_pushpull_requires_cut_certificate(mf):
    edges = [(0, 1, 3), (0, 2, 2), (1, 3, 2), (2, 3, 3), (1, 2, 1)]
    g = mf.build_bicsr(mf.EdgeListGraph.from_edges(4, edges))
    st = mf.init_residuals(g, 0, 3)  # heights all 0: t is not on the B side of any cut
    with pytest.raises(mf.SolverError):
        mf.solve_dynamic_pushpull(st, g, mf.UpdateBatch.from_updates([(0, 1, 1)]))
    st = mf.solve_static(g, 0, 3).state
    r = mf.solve_dynamic_pushpull(st, g, mf.UpdateBatch.from_updates([(0, 1, 1)]))
    assert r.flow_value == 3
    with pytest.raises(mf.BatchError):
        mf.solve_dynamic_pushpull(r.state, g, mf.UpdateBatch.from_updates([(1, 0, 1)]))
