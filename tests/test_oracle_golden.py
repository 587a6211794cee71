"""Pins the CPU oracle (oracle/mfx_oracle.c) and the input generators to the
fixtures produced by the live reference (tests/golden/make_golden.py).

The oracle runs the reference's deterministic schedule, so besides flow values
its terminal states, saturation, BFS heights and dynamic pre-phase arrays must
match the reference byte-for-byte (sha256 of the int64 arrays).
"""
import numpy as np
import pytest

import oracle as O
from golden_data import load, sha
from paper_2511_01235_b200 import gen

G = load()


def instance(name):
    rec = G.rec[name]
    if f"{name}/in_us" in G.arr:
        return (rec["n"], G.arr[f"{name}/in_us"], G.arr[f"{name}/in_vs"],
                G.arr[f"{name}/in_caps"], rec["s"], rec["t"])
    src = rec["source"]
    us, vs, caps, s, t = gen.source_edges(src["gen"], src["args"])
    return rec["n"], us, vs, caps, s, t


def batch_for(name, cur_g, entry, s, t):
    el_us, el_vs = cur_g.src[cur_g.is_original], cur_g.adj[cur_g.is_original]
    el_caps = cur_g.cap0[cur_g.is_original]
    spec = gen.BatchSpec(entry["pct"], entry["kind"], entry["seed"])
    bu, bv, bc, _ = gen.batch_arrays(cur_g.n, el_us, el_vs, el_caps, s, t, spec)
    return bu, bv, bc


CASES = G.cases()
FAST = [c for c in CASES if c not in ("grid256",)]


@pytest.mark.parametrize("name", CASES)
def test_generators_reproduce_reference_inputs(name):
    n, us, vs, caps, s, t = instance(name)
    assert [sha(us), sha(vs), sha(caps)] == G.rec[name]["input_sha"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_build_bit_exact(name):
    n, us, vs, caps, s, t = instance(name)
    g = O.build_bicsr(n, us, vs, caps)
    ref = G.rec[name]["graph"]
    assert g.m == ref["S"] and g.m_original == ref["m_original"]
    assert list(g.diag) == ref["diag"]
    for k in ("offsets", "adj", "src", "rev", "cap0", "is_original"):
        assert sha(getattr(g, k)) == ref["sha"][k], k


@pytest.mark.parametrize("name", FAST)
def test_oracle_static_and_chain(name):
    """Saturation, first BFS, deterministic static state, and every chained
    batch's pre-phase / BFS / flow, all against the reference."""
    rec = G.rec[name]
    n, us, vs, caps, s, t = instance(name)
    g = O.build_bicsr(n, us, vs, caps)
    # saturate_source + first global relabel (state.py:42-59, kernels.py:168)
    cf = g.cap0.copy()
    ex = np.zeros(n, np.int64)
    O.saturate_source(g, s, cf, ex)
    assert sha(cf) == rec["sat_sha"]["cf"] and sha(ex) == rec["sat_sha"]["excess"]
    h, _ = O.bfs_heights(g, cf, [t], -1)
    assert sha(h) == rec["bfs_sat_sha"]
    r, st = O.solve_static(g, s, t)
    assert r.status == 0
    assert r.flow == rec["static_flow"] == r.cut
    assert r.rounds == rec["static_rounds_det"]
    assert {k: sha(getattr(st, k)) for k in ("cf", "excess", "height")} == rec["static_state_sha"]
    for entry in rec["chain"]:
        bu, bv, bc = batch_for(name, g, entry, s, t)
        assert [sha(bu), sha(bv), sha(bc)] == entry["batch_sha"]
        # pre-phase, bit-exact (dynamic.py:157-159)
        g2, st2 = g.copy(), st.copy()
        rc, bad = O.apply_updates(g2, st2.cf, bu, bv, bc)
        assert rc == 0
        O.recompute_excess(g2, st2.cf, st2.excess)
        O.saturate_source(g2, s, st2.cf, st2.excess)
        assert sha(st2.cf) == entry["pre_sha"]["cf"]
        assert sha(st2.excess) == entry["pre_sha"]["excess"]
        assert sha(g2.cap0) == entry["pre_sha"]["cap0"]
        bases = [v for v in range(n) if v == t or (v != s and st2.excess[v] < 0)]
        hb, _ = O.bfs_heights(g2, st2.cf, bases, s)
        assert sha(hb) == entry["bfs_dyn_sha"]
        r = O.solve_dynamic(g, st, bu, bv, bc)
        assert r.status == 0
        assert r.flow == entry["flow"] == r.cut
        assert {k: sha(getattr(st, k)) for k in ("cf", "excess", "height")} == entry["state_sha"]


def test_oracle_diamond_dynamic_examples():
    """SPEC.md:300-302 via the reference's recorded answers."""
    rec = G.rec["diamond_dyn"]
    for key, ent in rec.items():
        g = O.build_bicsr(4, [0, 0, 1, 2, 1], [1, 2, 3, 3, 2], [3, 2, 2, 3, 1])
        _, st = O.solve_static(g, 0, 3)
        ups = ent["updates"]
        r = O.solve_dynamic(g, st, [u[0] for u in ups], [u[1] for u in ups], [u[2] for u in ups])
        assert r.flow == ent["flow"]
        assert r.rounds == ent["rounds"]


def test_oracle_batch_errors():
    """_resolve_batch error order (dynamic.py:63-88)."""
    g = O.build_bicsr(4, [0, 0, 1, 2, 1], [1, 2, 3, 3, 2], [3, 2, 2, 3, 1])
    _, st = O.solve_static(g, 0, 3)
    cf = st.cf.copy()
    assert O.apply_updates(g.copy(), cf, [0, 1], [1, 3], [2, -1]) == (1, 1)
    assert O.apply_updates(g.copy(), cf, [0, 0], [1, 3], [2, 5]) == (2, 1)
    assert O.apply_updates(g.copy(), cf, [1], [0], [5]) == (2, 0)
    assert O.apply_updates(g.copy(), cf, [1, 0, 1, 0], [3, 1, 3, 1], [1, 2, 4, 3]) == (3, 3)
    assert np.array_equal(cf, st.cf)
