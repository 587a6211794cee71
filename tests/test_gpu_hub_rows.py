"""Hub rows on the device path: the cooperative push's CTA rows take 4
consecutive slots per thread and one ordered scan per chunk (solve.cu
push_coop, pass 2), the warp-row BFS expansion and the repair scan keep 4
slots in flight per lane.  Star-shaped graphs put the whole flow through
rows of 1K-40K slots, where every chunk boundary, the first-minimum slot
offset and the excess running out mid-chunk occur; the flow is known in
closed form (s -> hub -> leaf_i -> t: sum of min(a_i, b_i) when s's edge is
wide), checked static and after chained capacity batches, plus the C oracle's
Dinic (oracle.py:199) on a two-hub variant.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mf():
    import paper_2511_01235_b200 as m
    return m


def star(k, seed):
    """s = 0, hub = 1, leaves 2..k+1, t = k+2."""
    rng = np.random.default_rng(seed)
    a = rng.integers(1, 100, k)
    b = rng.integers(1, 100, k)
    leaves = np.arange(2, k + 2, dtype=np.int64)
    t = k + 2
    us = np.concatenate([[0], np.ones(k, np.int64), leaves])
    vs = np.concatenate([[1], leaves, np.full(k, t, np.int64)])
    caps = np.concatenate([[10 ** 8], a, b]).astype(np.int64)
    return k + 3, us, vs, caps, 0, t, a, b


@pytest.mark.parametrize("k", [1000, 1500, 4099, 40000])
def test_star_hub_flow_static_and_dynamic(mf, k):
    n, us, vs, caps, s, t, a, b = star(k, k)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    r = mf.solve_static(g, s, t)
    assert r.flow_value == int(np.minimum(a, b).sum()) == r.certificate.cut_capacity
    rng = np.random.default_rng(7)
    st = r.state
    for j in range(4):
        # re-weight a random set of hub -> leaf and leaf -> t edges
        pick = rng.choice(k, size=k // 5, replace=False)
        na = rng.integers(0, 100, pick.size)
        nb = rng.integers(0, 100, pick.size)
        leaves = pick + 2
        bu = np.concatenate([np.ones(pick.size, np.int64), leaves]).astype(np.int64)
        bv = np.concatenate([leaves, np.full(pick.size, t, np.int64)]).astype(np.int64)
        bc = np.concatenate([na, nb]).astype(np.int64)
        a[pick], b[pick] = na, nb
        rr = mf.solve_dynamic(st, g, mf.UpdateBatch(bu, bv, bc))
        assert rr.flow_value == int(np.minimum(a, b).sum()) == rr.certificate.cut_capacity, j
        rep = mf.verify_gpu(rr.state, g, rr.flow_value)
        assert rep.ok, rep.problems
        st = rr.state


def test_two_hubs_against_oracle_dinic(mf):
    """Two hubs sharing their leaves, a bottleneck source edge: the flow is
    not the closed form; the C oracle's Dinic decides."""
    rng = np.random.default_rng(3)
    k = 6000
    leaves = np.arange(3, k + 3, dtype=np.int64)
    t = k + 3
    us = np.concatenate([[0, 0], np.ones(k, np.int64), np.full(k, 2, np.int64), leaves])
    vs = np.concatenate([[1, 2], leaves, leaves, np.full(k, t, np.int64)])
    caps = np.concatenate([[150000, 90000], rng.integers(1, 60, 2 * k),
                           rng.integers(1, 100, k)]).astype(np.int64)
    n = k + 4
    og = O.build_bicsr(n, us, vs, caps)
    want, _ = O.dinic(og, 0, t)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    r = mf.solve_static(g, 0, t)
    assert r.flow_value == want == r.certificate.cut_capacity
