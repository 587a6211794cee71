"""Reference-signature helpers that run without a GPU: the generators
(reference bench.py:66-147) and the independent max-flow checks
(reference oracle.py:20-101), against the reference-generated goldens and,
when the unmodified reference is installed (baseline/_ref), against it."""
import os
import sys

import numpy as np
import pytest

import paper_2511_01235_b200 as mf
from golden_data import load, sha

G = load()
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref():
    p = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(p, "dynmaxflow")):
        pytest.skip("reference not installed in baseline/_ref")
    if p not in sys.path:
        sys.path.insert(0, p)
    import dynmaxflow
    return dynmaxflow


def test_random_graph_reference_signature():
    g, s, t = mf.random_graph(500, 4000, seed=3)
    assert isinstance(g, mf.EdgeListGraph) and (s, t) == (0, 499)
    us, vs, caps, s2, t2 = mf.random_edges(500, 4000, seed=3)
    assert np.array_equal(g.us, us) and np.array_equal(g.caps, caps) and (s2, t2) == (s, t)
    rec = G.rec["C1"]
    g1, s1, t1 = mf.random_graph(10000, 100000, seed=0)
    assert (s1, t1) == (rec["s"], rec["t"])


def test_generate_batch_reference_signature_and_errors():
    """UpdateBatch out, draw for draw the golden chain's first batch; a
    non-normalized list raises the reference's GraphError."""
    g, s, t = mf.random_graph(300, 3000, seed=5)
    csr_like = _normalize(g)
    b = mf.generate_batch(csr_like, s, t, mf.BatchSpec(10.0, "mixed", 2))
    assert isinstance(b, mf.UpdateBatch) and len(b) == int(np.ceil(10.0 * csr_like.m / 100))
    bu, bv, bc, _ = mf.batch_arrays(csr_like.n, csr_like.us, csr_like.vs, csr_like.caps, s, t,
                                    mf.BatchSpec(10.0, "mixed", 2))
    assert np.array_equal(b.us, bu) and np.array_equal(b.new_caps, bc)
    dup = mf.EdgeListGraph(3, np.array([0, 0]), np.array([1, 1]), np.array([2, 3]))
    with pytest.raises(mf.GraphError, match="normalized edge list"):
        mf.generate_batch(dup, 0, 2, mf.BatchSpec(50.0, "inc", 0))


def _normalize(g):
    """Unique (u, v) pairs, caps summed, self-loops dropped (graph.py:138-147)."""
    keep = g.us != g.vs
    key = g.us[keep] * g.n + g.vs[keep]
    uk, inv = np.unique(key, return_inverse=True)
    caps = np.zeros(uk.size, np.int64)
    np.add.at(caps, inv, g.caps[keep])
    return mf.EdgeListGraph(g.n, uk // g.n, uk % g.n, caps)


def test_generate_batch_matches_reference():
    ref = _ref()
    rg, s, t = ref.random_graph(400, 4000, seed=8)
    el = ref.build_bicsr(rg).to_edge_list()
    for kind, seed in (("mixed", 0), ("inc", 1), ("dec", 2)):
        rb = ref.generate_batch(el, s, t, ref.BatchSpec(pct=7.5, kind=kind, seed=seed))
        ob = mf.generate_batch(mf.EdgeListGraph(el.n, el.us, el.vs, el.caps), s, t,
                               mf.BatchSpec(7.5, kind, seed))
        assert [sha(ob.us), sha(ob.vs), sha(ob.new_caps)] == \
            [sha(rb.us), sha(rb.vs), sha(rb.new_caps)]


@pytest.mark.parametrize("name", [k for k in G.cases()][:12])
def test_dinic_maxflow_equals_golden_static_flow(name):
    rec = G.rec[name]
    if f"{name}/in_us" in G.arr:
        us, vs, caps = (G.arr[f"{name}/in_{k}"] for k in ("us", "vs", "caps"))
        n, s, t = rec["n"], rec["s"], rec["t"]
    else:
        from paper_2511_01235_b200 import gen
        us, vs, caps, s, t = gen.source_edges(rec["source"]["gen"], rec["source"]["args"])
        n = rec["n"]
    if s == t:
        pytest.skip("degenerate case")
    assert mf.dinic_maxflow(mf.EdgeListGraph(n, us, vs, caps), s, t) == rec["static_flow"]


def test_exhaustive_min_cut_small():
    rng = np.random.default_rng(3)
    for _ in range(20):
        n = int(rng.integers(3, 9))
        m = int(rng.integers(1, 20))
        us, vs = rng.integers(0, n, m), rng.integers(0, n, m)
        caps = rng.integers(0, 30, m)
        g = mf.EdgeListGraph(n, us, vs, caps)
        assert mf.exhaustive_min_cut(g, 0, n - 1) == mf.dinic_maxflow(g, 0, n - 1)
    with pytest.raises(ValueError, match="limited to 20"):
        mf.exhaustive_min_cut(mf.EdgeListGraph(30, np.array([0]), np.array([1]),
                                               np.array([1])), 0, 29)
