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


def _single_device_rmat(mf, scale):
    import ctypes

    import torch

    from paper_2511_01235_b200 import _lib
    n = 1 << scale
    m = n * 16
    e = [torch.empty(m, dtype=torch.int64, device="cuda:0") for _ in range(3)]
    s, t = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.load().mfx_rmat_device(scale, 16, 0, 0.57, 0.19, 0.19, 0, e[0].data_ptr(),
                                           e[1].data_ptr(), e[2].data_ptr(), ctypes.byref(s),
                                           ctypes.byref(t)))
    g = mf.build_bicsr_device(n, e[0].data_ptr(), e[1].data_ptr(), e[2].data_ptr(), m)
    del e
    torch.cuda.empty_cache()
    return g, s.value, t.value


def _c5_single_chain(mf, scale, batches, k, static_flow=None):
    """The C5 generator on the single-device engine (the 2.1 B slots of
    scale 26 fit its int32 layout): the static flow equals the partitioned
    engine's on the same device-drawn graph, and every chained batch of
    device-sampled mixed updates equals a static re-solve, flow == cut."""
    from paper_2511_01235_b200 import gen, partition
    g, s, t = _single_device_rmat(mf, scale)
    res = mf.solve_static(g, s, t)
    assert res.flow_value == res.certificate.cut_capacity > 0
    if static_flow is None:  # (both engines at once do not fit one GPU at scale 26)
        pg = partition.PartitionedGraph.rmat(scale, 16, 0, partition.LocalGroup(2))
        assert pg.solve_static().flow_value == res.flow_value
        pg.close()
    else:
        assert res.flow_value == static_flow
    st = res.state
    for b in range(batches):
        bu, bv, bc = gen.device_sample_batch(g, s, t, k, "mixed", seed=b)
        assert bu.size == k
        r = mf.solve_dynamic(st, g, mf.UpdateBatch(bu, bv, bc))
        assert r.flow_value == r.certificate.cut_capacity
        rs = mf.resolve_static(g, mf.init_residuals(g, s, t))
        assert rs.flow_value == r.flow_value, (scale, b)
        st = r.state


def test_c5_generator_single_device_scale22(mf):
    _c5_single_chain(mf, 22, 2, 1_000_000)


@pytest.mark.slow
@pytest.mark.skipif(not os.environ.get("MFX_SLOW"), reason="opt-in (minutes): MFX_SLOW=1")
def test_c5_full_single_device(mf):
    """Full C5 (R-MAT 26, 2,103,824,774 slots) on one B200; 13,488,105 is the
    partitioned engine's static flow on the same device-drawn graph
    (profiles/round2/bench_lines.jsonl, C5 with 4 parts)."""
    _c5_single_chain(mf, 26, 2, 1_000_000, static_flow=13488105)
