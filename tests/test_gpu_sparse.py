"""Sparse relabels: a relabel whose predecessor reached few
vertices keeps the list of what it reaches, and the next relabel resets and
seeds from that list instead of all n vertices.  The invariant that makes
this exact is {v : h[v] < n} == the list; it is checked after every solve of
chained batches, and every flow equals the full-pass engine's
(MFX_SPARSE=0 MFX_TRACK=0) and passes the device verifier.
"""
import ctypes

import numpy as np
import pytest

from paper_2511_01235_b200 import _lib, gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mf():
    import paper_2511_01235_b200 as m
    return m


def reached_list(st, n):
    buf = (ctypes.c_int32 * max(1, n))()
    cnt = ctypes.c_int64()
    _lib.check(_lib.load().mfx_reached_list(st.handle, buf, n, ctypes.byref(cnt)))
    if cnt.value < 0:
        return None
    return np.frombuffer(buf, dtype=np.int32, count=cnt.value).copy()


def instance(kind, side):
    if kind == "road":
        us, vs, caps, s, t = gen.road_graph(side, side, 0, 0.21)
        return side * side, us, vs, caps, s, t
    if kind == "grid":
        us, vs, caps, s, t = gen.grid_graph(side, side, 0)
        return side * side + 2, us, vs, caps, s, t
    us, vs, caps, s, t = gen.rmat_graph(side, 16, 0)
    return 1 << side, us, vs, caps, s, t


def chain(n, us, vs, caps, s, t, k, count, seed0):
    caps = np.array(caps, np.int64, copy=True)
    out = []
    for j in range(count):
        bu, bv, bc, pick = gen.fast_batch(n, us, vs, caps, s, t, k, "mixed", seed0 + j)
        caps[pick] = bc
        out.append((bu, bv, bc))
    return out


def run_chain(mf, n, us, vs, caps, s, t, batches, check_list):
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    res = mf.solve_static(g, s, t)
    flows, listed = [res.flow_value], 0
    st = res.state
    for bu, bv, bc in batches:
        r = mf.solve_dynamic(st, g, mf.UpdateBatch(bu, bv, bc))
        assert r.flow_value == r.certificate.cut_capacity
        rep = mf.verify_gpu(r.state, g, r.flow_value)
        assert rep.ok, rep.problems
        flows.append(r.flow_value)
        st = r.state
        if check_list:
            lst = reached_list(st, n)
            if lst is not None:
                listed += 1
                assert len(np.unique(lst)) == len(lst), "duplicate entries"
                assert np.array_equal(np.sort(lst), np.flatnonzero(st.height < n))
    return flows, listed


@pytest.mark.parametrize("kind,side,k", [("road", 64, 200), ("road", 256, 2000), ("road", 512, 4000),
                                         ("grid", 64, 300), ("rmat", 12, 2000)])
def test_sparse_relabels_exact(mf, kind, side, k, monkeypatch):
    n, us, vs, caps, s, t = instance(kind, side)
    el = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps)).to_edge_list()  # (normalised: R-MAT)
    us, vs, caps = el.us, el.vs, el.caps.copy()
    if kind == "road":  # thin sink edges: the cut sits at the sink corner, as in C4
        caps[vs == t] = 1
    batches = chain(n, us, vs, caps, s, t, k, 8, 31)
    flows, listed = run_chain(mf, n, us, vs, caps, s, t, batches, check_list=True)
    monkeypatch.setenv("MFX_SPARSE", "0")
    monkeypatch.setenv("MFX_TRACK", "0")
    full, _ = run_chain(mf, n, us, vs, caps, s, t, batches, check_list=False)
    assert flows == full
    if kind == "road":  # its sink side is a corner: the lists are in use
        assert listed > 0


def test_state_copy_keeps_the_list(mf):
    n, us, vs, caps, s, t = instance("road", 128)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    res = mf.solve_static(g, s, t)
    (bu, bv, bc), = chain(n, us, vs, caps, s, t, 500, 1, 5)
    r = mf.solve_dynamic(res.state, g, mf.UpdateBatch(bu, bv, bc))
    lst = reached_list(r.state, n)
    snap = r.state.copy()
    lst2 = reached_list(snap, n)
    if lst is None:
        assert lst2 is None
    else:
        assert np.array_equal(lst, lst2)
        assert np.array_equal(np.sort(lst2), np.flatnonzero(snap.height < n))
    # an upload invalidates it
    snap.upload(snap.cf, snap.excess, snap.height)
    assert reached_list(snap, n) is None
