"""Full-size configurations (BASELINE.json C2-C4) on the GPU.

C2 / C3 and the scaled grid / R-MAT / road anchors: the static flow and every
chained batch flow equal the LIVE reference's (tests/golden/large.json,
written by tests/golden/make_golden_large.py), and the device verifier passes
after every batch.  C4 at full scale (24 M vertices) has no CPU ground truth
(hours on the reference); there the dynamic flow after each batch must equal
a GPU static re-solve on the updated capacities, with the device certificate
(flow == cut, saturated A->B, idle B->A) as the duality proof.
"""
import json
import os

import numpy as np
import pytest

from paper_2511_01235_b200 import gen

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "large.json")) as _fh:
    LARGE = json.load(_fh)
NAMES = sorted(k for k in LARGE if not k.startswith("_"))


@pytest.fixture(scope="module")
def mf():
    import paper_2511_01235_b200 as m
    return m


def instance(rec):
    us, vs, caps, s, t = gen.source_edges(rec["gen"], rec["args"])
    assert (s, t) == (rec["s"], rec["t"])
    return rec["n"], us, vs, caps, s, t


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("wide", [False, True])
def test_reference_flows_full_size(mf, name, wide):
    """``wide``: the same chains on int64 residual storage (both solve-kernel
    builds: v256 on the grids / roads, v512 on R-MAT)."""
    rec = LARGE[name]
    n, us, vs, caps, s, t = instance(rec)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps), wide=wide)
    assert g.cap_bytes == (8 if wide else 4)
    assert (g.m, g.m_original) == (rec["S"], rec["m_original"])
    res = mf.solve_static(g, s, t)
    assert res.flow_value == rec["static_flow"] == res.certificate.cut_capacity
    el = g.to_edge_list()
    ecaps = el.caps.copy()
    st = res.state
    for entry in rec["chain"]:
        bu, bv, bc, pick = gen.fast_batch(n, el.us, el.vs, ecaps, s, t, entry["k"], "mixed",
                                          entry["seed"])
        ecaps[pick] = bc
        r = mf.solve_dynamic(st, g, mf.UpdateBatch(bu, bv, bc))
        assert r.flow_value == entry["flow"] == r.certificate.cut_capacity, (entry, r.flow_value)
        rep = mf.verify_gpu(r.state, g, r.flow_value)
        assert rep.ok, rep.problems
        st = r.state


@pytest.mark.parametrize("side,batches,wide", [(4900, 3, False), (4900, 2, True)])
def test_c4_road_dynamic_equals_static_resolve(mf, side, batches, wide):
    """C4 (road, 24 M vertices, BFS depth ~10^4): no CPU ground truth, so
    dynamic == GPU static re-solve after every batch, both certified."""
    us, vs, caps, s, t = gen.road_graph(side, side, 0, 0.21)
    n = side * side
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps), wide=wide)
    res = mf.solve_static(g, s, t)
    assert res.flow_value == res.certificate.cut_capacity
    el = g.to_edge_list()
    ecaps = el.caps.copy()
    st = res.state
    scratch = mf.init_residuals(g, s, t)
    for b in range(batches):
        bu, bv, bc, pick = gen.fast_batch(n, el.us, el.vs, ecaps, s, t, 10_000, "mixed", b)
        ecaps[pick] = bc
        r = mf.solve_dynamic(st, g, mf.UpdateBatch(bu, bv, bc))
        rs = mf.resolve_static(g, scratch)
        assert r.flow_value == rs.flow_value == r.certificate.cut_capacity
        assert mf.verify_gpu(r.state, g, r.flow_value).ok
        st = r.state


def test_c2_terminal_hub_rows(mf):
    """The C2 source and sink rows hold ~2.1 M slots each (grid-wide
    expansion path); saturation moves exactly the source row's capacity."""
    rec = LARGE["C2"]
    n, us, vs, caps, s, t = instance(rec)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    off = g.offsets
    assert off[s + 1] - off[s] > 2_000_000 and off[t + 1] - off[t] > 2_000_000
    st = mf.init_residuals(g, s, t)
    mf.saturate_source(st, g)
    row = slice(off[s], off[s + 1])
    assert int(st.excess[s]) == -int(g.cap0[row].sum())
    assert np.all(st.cf[row] == 0)
