"""GPU parity: the CUDA path (through the C-ABI) against the reference-generated
golden fixtures and the CPU oracle.

Bit-exact: Bi-CSR build arrays, saturation, global-relabel heights, the
dynamic pre-phase (cf / excess / cap0).  Value-exact: flow and cut after the
static solve and after every chained batch, plus the device verifier.
"""
import numpy as np
import pytest

import oracle as O
from golden_data import load, sha
from paper_2511_01235_b200 import gen

pytestmark = pytest.mark.gpu

G = load()
CASES = G.cases()
SMALL = G.cases(with_arrays=True)


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


def chain_batch(g_src, g_adj, g_orig, cap0, n, s, t, entry):
    keep = g_orig.astype(bool)
    spec = gen.BatchSpec(entry["pct"], entry["kind"], entry["seed"])
    bu, bv, bc, _ = gen.batch_arrays(n, g_src[keep], g_adj[keep], cap0[keep], s, t, spec)
    return bu, bv, bc


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("wide", [False, True])
def test_build_bit_exact(mf, name, wide):
    n, us, vs, caps, s, t = instance(name)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps), wide=wide)
    ref = G.rec[name]["graph"]
    assert g.m == ref["S"] and g.m_original == ref["m_original"]
    d = g.diagnostics
    assert [d.self_loops_dropped, d.parallel_edges_merged, d.reverse_stubs_added] == ref["diag"]
    for k in ("offsets", "adj", "src", "rev", "cap0", "is_original"):
        assert sha(getattr(g, k)) == ref["sha"][k], k
    assert g.cap_bytes == (8 if wide else 4)


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("wide", [False, True])
def test_saturate_and_global_relabel_bit_exact(mf, name, wide):
    n, us, vs, caps, s, t = instance(name)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps), wide=wide)
    st = mf.init_residuals(g, s, t)
    mf.saturate_source(st, g)
    assert np.array_equal(st.cf, G.arr[f"{name}/sat_cf"])
    assert np.array_equal(st.excess, G.arr[f"{name}/sat_excess"])
    mf.backward_bfs(st, g)
    assert np.array_equal(st.height, G.arr[f"{name}/bfs_sat_h"])


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("wide", [False, True])
def test_dynamic_prephase_and_bfs_bit_exact(mf, name, wide):
    """Given the reference's terminated state, the fused device pre-phase
    equals apply_updates + recompute_excess + saturate_source byte for byte,
    and the dynamic global relabel equals backward_bfs_dynamic."""
    rec = G.rec[name]
    n, s, t = rec["n"], rec["s"], rec["t"]
    for bi, entry in enumerate(rec["chain"]):
        a = lambda k: G.arr[f"{name}/b{bi}/{k}"]  # noqa: E731
        g = mf.upload_bicsr(n, G.arr[f"{name}/offsets"], G.arr[f"{name}/adj"],
                            G.arr[f"{name}/rev"], a("prior_cap0"), G.arr[f"{name}/is_original"],
                            wide=wide)
        assert g.cap_bytes == (8 if wide else 4)
        st = mf.init_residuals(g, s, t)
        st.upload(a("prior_cf"), a("prior_excess"), a("prior_height"))
        mf.dynamic_prephase(st, g, mf.UpdateBatch(a("us"), a("vs"), a("caps")))
        assert np.array_equal(st.cf, a("pre_cf"))
        assert np.array_equal(st.excess, a("pre_excess"))
        assert np.array_equal(g.cap0, a("pre_cap0"))
        mf.backward_bfs_dynamic(st, g)
        assert np.array_equal(st.height, a("bfs_dyn_h"))


@pytest.mark.parametrize("name", ["C1", "grid64", "rmat12", "road48"])
def test_prephase_bit_exact_from_oracle_state(mf, name):
    """Larger cases: the oracle reproduces the reference's deterministic
    terminal state (pinned in test_oracle_golden); upload it and compare the
    device pre-phase against the reference's hashes."""
    rec = G.rec[name]
    n, us, vs, caps, s, t = instance(name)
    og = O.build_bicsr(n, us, vs, caps)
    _, ost = O.solve_static(og, s, t)
    for entry in rec["chain"]:
        bu, bv, bc = chain_batch(og.src, og.adj, og.is_original, og.cap0, n, s, t, entry)
        g = mf.upload_bicsr(n, og.offsets, og.adj, og.rev, og.cap0, og.is_original)
        st = mf.init_residuals(g, s, t)
        st.upload(ost.cf, ost.excess, ost.height)
        mf.dynamic_prephase(st, g, mf.UpdateBatch(bu, bv, bc))
        assert sha(st.cf) == entry["pre_sha"]["cf"]
        assert sha(st.excess) == entry["pre_sha"]["excess"]
        assert sha(g.cap0) == entry["pre_sha"]["cap0"]
        mf.backward_bfs_dynamic(st, g)
        assert sha(st.height) == entry["bfs_dyn_sha"]
        O.solve_dynamic(og, ost, bu, bv, bc)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("wide", [False, True])
def test_static_and_chained_dynamic_flows(mf, name, wide):
    """Flow and cut after the static solve and after every chained batch
    equal the reference's; the device verifier passes each time.  ``wide``
    runs the int64-residual builds of the solve kernel and pre-phase."""
    rec = G.rec[name]
    n, us, vs, caps, s, t = instance(name)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps), wide=wide)
    assert g.cap_bytes == (8 if wide else 4)
    res = mf.solve_static(g, s, t)
    assert res.flow_value == rec["static_flow"]
    assert res.certificate.cut_capacity == res.flow_value
    rep = mf.verify_gpu(res.state, g, res.flow_value)
    assert rep.ok, rep.problems
    st = res.state
    for entry in rec["chain"]:
        bu, bv, bc = chain_batch(g.src, g.adj, g.is_original, g.cap0, n, s, t, entry)
        assert [sha(bu), sha(bv), sha(bc)] == entry["batch_sha"]
        r = mf.solve_dynamic(st, g, mf.UpdateBatch(bu, bv, bc))
        assert r.flow_value == entry["flow"], (name, entry["seed"])
        assert r.certificate.cut_capacity == r.flow_value
        rep = mf.verify_gpu(r.state, g, r.flow_value)
        assert rep.ok, rep.problems
        # GPU static re-solve on the updated capacities agrees
        g2 = mf.build_bicsr(g.to_edge_list(), wide=wide)
        assert mf.solve_static(g2, s, t).flow_value == entry["flow"]
        st = r.state


def test_reference_semantics_certificate_with_reference_layout(mf):
    """The device state is consumable by reference-style verifiers: the A
    mask is {h == n}, cut recomputed on the host from downloaded arrays."""
    name = "rand3"
    rec = G.rec[name]
    n, us, vs, caps, s, t = instance(name)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    res = mf.solve_static(g, s, t)
    a = res.certificate.a_mask
    assert np.array_equal(a, res.state.height == n)
    crossing = g.is_original & a[g.src] & ~a[g.adj]
    assert int(g.cap0[crossing].sum()) == res.flow_value == rec["static_flow"]
    assert (res.state.cf[crossing] == 0).all()
    f = np.maximum(g.cap0 - res.state.cf, 0)
    assert (res.state.cf + res.state.cf[g.rev] == g.cap0 + g.cap0[g.rev]).all()
    back = g.is_original & ~a[g.src] & a[g.adj]
    assert (f[back] == 0).all()


def test_diamond_dynamic_spec_examples(mf):
    rec = G.rec["diamond_dyn"]
    for key, ent in rec.items():
        g = mf.build_bicsr(mf.EdgeListGraph.from_edges(
            4, [(0, 1, 3), (0, 2, 2), (1, 3, 2), (2, 3, 3), (1, 2, 1)]))
        base = mf.solve_static(g, 0, 3)
        assert base.flow_value == 5
        r = mf.solve_dynamic(base.state, g, mf.UpdateBatch.from_updates(ent["updates"]))
        assert r.flow_value == ent["flow"]


def test_error_messages_match_reference(mf):
    errs = G.rec["errors"]
    cases = {
        "n0": (0, [], [], []),
        "src_range": (3, [0, 5], [1, 2], [1, 1]),
        "dst_range": (3, [0, 1], [1, -1], [1, 1]),
        "neg_cap": (3, [0, 1], [1, 2], [1, -4]),
    }
    for key, (n, us, vs, caps) in cases.items():
        with pytest.raises(mf.GraphError) as ei:
            mf.build_bicsr(mf.EdgeListGraph(n, np.array(us, np.int64), np.array(vs, np.int64),
                                            np.array(caps, np.int64)))
        assert str(ei.value) == errs["graph/" + key]
    g = mf.build_bicsr(mf.EdgeListGraph.from_edges(
        4, [(0, 1, 3), (0, 2, 2), (1, 3, 2), (2, 3, 3), (1, 2, 1)]))
    res = mf.solve_static(g, 0, 3)
    before = (res.state.cf.copy(), res.state.excess.copy(), g.cap0.copy())
    bcases = {
        "neg": [(0, 1, 2), (1, 3, -1)],
        "unknown": [(0, 1, 2), (0, 3, 5)],
        "stub": [(1, 0, 5)],
        "dup": [(1, 3, 1), (0, 1, 2), (1, 3, 4), (0, 1, 3)],
    }
    for key, ups in bcases.items():
        with pytest.raises(mf.BatchError) as ei:
            mf.solve_dynamic(res.state, g, mf.UpdateBatch.from_updates(ups))
        assert str(ei.value) == errs["batch/" + key]
        # all-or-nothing: nothing was mutated
        assert np.array_equal(res.state.cf, before[0])
        assert np.array_equal(res.state.excess, before[1])
        assert np.array_equal(g.cap0, before[2])
    for key, (s, t) in {"s_range": (7, 1), "t_range": (0, -1), "same": (2, 2)}.items():
        with pytest.raises(ValueError) as ei:
            mf.solve_static(g, s, t)
        assert str(ei.value) == errs["endpoints/" + key]
    # the state is still usable after rejected batches
    r = mf.solve_dynamic(res.state, g, mf.UpdateBatch.from_updates([(0, 1, 1)]))
    assert r.flow_value == 3


def test_edge_cases(mf):
    # single vertex pair, no path, isolated vertices, empty batch, empty edge list
    g = mf.build_bicsr(mf.EdgeListGraph.from_edges(2, [(0, 1, 7)]))
    assert mf.solve_static(g, 0, 1).flow_value == 7
    g = mf.build_bicsr(mf.EdgeListGraph.from_edges(4, [(0, 1, 3), (2, 3, 3)]))
    r = mf.solve_static(g, 0, 3)
    assert r.flow_value == 0 and r.certificate.cut_capacity == 0
    r2 = mf.solve_dynamic(r.state, g, mf.UpdateBatch.from_updates([]))
    assert r2.flow_value == 0 and r2.rounds == 0
    g = mf.build_bicsr(mf.EdgeListGraph(5, np.empty(0, np.int64), np.empty(0, np.int64),
                                        np.empty(0, np.int64)))
    assert g.m == 0
    assert mf.solve_static(g, 0, 4).flow_value == 0
    # self-loops only
    g = mf.build_bicsr(mf.EdgeListGraph.from_edges(3, [(1, 1, 5), (2, 2, 4)]))
    assert g.m == 0 and g.diagnostics.self_loops_dropped == 2


def test_wide_capacities(mf):
    """Pair sums beyond int32 select int64 residual storage automatically."""
    big = 3_000_000_000
    g = mf.build_bicsr(mf.EdgeListGraph.from_edges(
        4, [(0, 1, big), (0, 2, big), (1, 3, big // 2), (2, 3, big), (1, 2, 7)]))
    assert g.cap_bytes == 8
    r = mf.solve_static(g, 0, 3)
    og = O.build_bicsr(4, [0, 0, 1, 2, 1], [1, 2, 3, 3, 2], [big, big, big // 2, big, 7])
    assert r.flow_value == O.solve_static(og, 0, 3)[0].flow
    # an int32 graph rejects a batch that would overflow its storage
    g32 = mf.build_bicsr(mf.EdgeListGraph.from_edges(3, [(0, 1, 5), (1, 2, 5)]))
    r = mf.solve_static(g32, 0, 2)
    with pytest.raises(ValueError):
        mf.solve_dynamic(r.state, g32, mf.UpdateBatch.from_updates([(0, 1, big)]))
    gw = mf.build_bicsr(mf.EdgeListGraph.from_edges(3, [(0, 1, 5), (1, 2, 5)]), wide=True)
    r = mf.solve_static(gw, 0, 2)
    r2 = mf.solve_dynamic(r.state, gw, mf.UpdateBatch.from_updates([(0, 1, big), (1, 2, big)]))
    assert r2.flow_value == big


@pytest.mark.parametrize("seed", range(40))
def test_random_vs_oracle(mf, seed):
    """SPEC acceptance 1/2 style: random graphs, static + inc/dec/mixed
    chains, several kernel knobs; every flow equals the oracle's."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 400))
    m = int(rng.integers(1, 4000))
    us, vs, caps, s, t = gen.random_edges(n, m, seed)
    knobs = [dict(), dict(kernel_cycles=1), dict(kernel_cycles=64), dict(mode="topology"),
             dict(max_waves=1), dict(max_waves=3, kernel_cycles=2),
             dict(schedule="async"), dict(schedule="async", async_budget=1),
             dict(schedule="async", async_budget=2, kernel_cycles=3),
             dict(blocks_per_sm=1)][seed % 10]
    params = mf.SolverParams(**knobs)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    og = O.build_bicsr(n, us, vs, caps)
    res = mf.solve_static(g, s, t, params)
    ores, ost = O.solve_static(og, s, t)
    assert res.flow_value == ores.flow
    st = res.state
    for j, (kind, pct) in enumerate([("inc", 5.0), ("dec", 10.0), ("mixed", 25.0), ("mixed", 1.0)]):
        el_us, el_vs, el_caps = og.src[og.is_original], og.adj[og.is_original], og.cap0[og.is_original]
        bu, bv, bc, _ = gen.batch_arrays(n, el_us, el_vs, el_caps, s, t,
                                           gen.BatchSpec(pct, kind, seed * 10 + j))
        r = mf.solve_dynamic(st, g, mf.UpdateBatch(bu, bv, bc), params)
        orr = O.solve_dynamic(og, ost, bu, bv, bc)
        assert r.flow_value == orr.flow, (seed, kind)
        rep = mf.verify_gpu(r.state, g, r.flow_value)
        assert rep.ok, rep.problems
        st = r.state


def test_instrument_invariants(mf):
    """SPEC acceptance 4 on the device path: at every round boundary cf >= 0,
    residual-sum conservation, sum(excess) == 0."""
    us, vs, caps, s, t = gen.random_edges(80, 600, 5)
    g = mf.build_bicsr(mf.EdgeListGraph(80, us, vs, caps))
    seen = []

    def hook(st, gg, rnd, label):
        cf, ex = st.cf, st.excess
        assert (cf >= 0).all()
        assert (cf + cf[gg.rev] == gg.cap0 + gg.cap0[gg.rev]).all()
        assert ex.sum() == 0
        seen.append((rnd, label))

    res = mf.solve_static(g, s, t, mf.SolverParams(instrument=hook))
    og = O.build_bicsr(80, us, vs, caps)
    assert res.flow_value == O.solve_static(og, s, t)[0].flow
    assert seen and seen[0] == (0, "bfs")
    el = g.to_edge_list()
    bu, bv, bc, _ = gen.batch_arrays(80, el.us, el.vs, el.caps, s, t, gen.BatchSpec(20.0, "mixed", 1))
    r = mf.solve_dynamic(res.state, g, mf.UpdateBatch(bu, bv, bc), mf.SolverParams(instrument=hook))
    g2 = mf.build_bicsr(g.to_edge_list())
    assert r.flow_value == mf.solve_static(g2, s, t).flow_value


def test_state_copy_and_graph_copy_semantics(mf):
    us, vs, caps, s, t = gen.random_edges(300, 3000, 9)
    g = mf.build_bicsr(mf.EdgeListGraph(300, us, vs, caps))
    res = mf.solve_static(g, s, t)
    snap_st, snap_g = res.state.copy(), g.copy()
    cap_before = g.cap0.copy()
    el = g.to_edge_list()
    bu, bv, bc, _ = gen.batch_arrays(300, el.us, el.vs, el.caps, s, t, gen.BatchSpec(10.0, "dec", 2))
    r1 = mf.solve_dynamic(res.state, g, mf.UpdateBatch(bu, bv, bc))
    # the snapshot is untouched and can replay the same batch
    assert np.array_equal(snap_g.cap0, cap_before)
    assert not np.array_equal(g.cap0, cap_before)
    r2 = mf.solve_dynamic(snap_st, snap_g, mf.UpdateBatch(bu, bv, bc))
    assert r1.flow_value == r2.flow_value
    assert np.array_equal(g.cap0, snap_g.cap0)
    # device restore
    st3 = res.state.copy()
    st3.assign(snap_st)
    assert np.array_equal(st3.cf, snap_st.cf)


def test_edge_indices_and_reverse(mf):
    us, vs, caps, s, t = gen.random_edges(50, 300, 4)
    g = mf.build_bicsr(mf.EdgeListGraph(50, us, vs, caps))
    idx = g.edge_indices(g.src, g.adj)
    assert np.array_equal(idx, np.arange(g.m))
    assert g.edge_index(0, 0) == -1
    for i in range(0, g.m, 7):
        assert mf.reverse_edge(g, mf.reverse_edge(g, i)) == i
    with pytest.raises(mf.GraphError):
        mf.reverse_edge(g, g.m)


@pytest.mark.parametrize("name", ["rand3", "grid64", "rmat12", "C1"])
def test_global_relabel_strict_retry_path(mf, name, monkeypatch):
    """The safety net of the label-correcting global relabel (a frontier
    overflow redoes it in strict mode; device_flags bit 3 forces that path):
    heights stay bit-exact and flows stay the reference's."""
    rec = G.rec[name]
    n, us, vs, caps, s, t = instance(name)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    p = mf.SolverParams(device_flags=8)
    res = mf.solve_static(g, s, t, p)
    assert res.flow_value == rec["static_flow"] == res.certificate.cut_capacity
    monkeypatch.setenv("MFX_FLAGS", "8")
    st = mf.init_residuals(g, s, t)
    mf.saturate_source(st, g)
    mf.backward_bfs(st, g)
    assert sha(st.height) == rec["bfs_sat_sha"]


SCHEDULES = [
    {"MFX_BFS_LOCAL": "16"},                                   # short CTA-local BFS runs
    {"MFX_BFS_LOCAL": "4096", "MFX_LQ_CAP": "64"},              # long runs, tiny ring (spills)
    {"MFX_WAVE_TIME": "0"},                                    # no push-phase time budget
    {"MFX_WAVE_TIME": "2", "MFX_TAIL_LOCAL": "0"},              # tight budget, no CTA-0 tails
    {"MFX_TAIL_LOCAL": "4096", "MFX_BFS_LOCAL_MAX": "1"},       # large tails, grid-wide BFS
]


@pytest.mark.parametrize("env", SCHEDULES, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
@pytest.mark.parametrize("name", ["grid64", "rmat12", "rand3"])
def test_schedule_knobs_keep_reference_results(mf, name, env, monkeypatch):
    """The schedule knobs change only the order of work:
    global-relabel heights stay bit-exact and every chained flow stays the
    reference's."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rec = G.rec[name]
    n, us, vs, caps, s, t = instance(name)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    st = mf.init_residuals(g, s, t)
    mf.saturate_source(st, g)
    mf.backward_bfs(st, g)
    assert sha(st.height) == rec["bfs_sat_sha"]
    res = mf.solve_static(g, s, t)
    assert res.flow_value == rec["static_flow"] == res.certificate.cut_capacity
    st = res.state
    for entry in rec["chain"]:  # (the batches update g's capacities)
        bu, bv, bc = chain_batch(g.src, g.adj, g.is_original, g.cap0, n, s, t, entry)
        r = mf.solve_dynamic(st, g, mf.UpdateBatch(bu, bv, bc))
        assert r.flow_value == entry["flow"] == r.certificate.cut_capacity, (name, entry["seed"])
        st = r.state


@pytest.mark.parametrize("name", [c for c in CASES if c not in ("grid256",)])
def test_deterministic_mode_states_bit_exact(mf, name):
    """SolverParams(deterministic=True): the device runs each round's push
    and repair serially in worklist order, so the whole final state -- cf,
    excess, height -- after the static solve and after every chained batch
    is byte-identical to the reference's deterministic runs (state_sha from
    the live reference), rounds included."""
    rec = G.rec[name]
    n, us, vs, caps, s, t = instance(name)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    det = mf.SolverParams(deterministic=True)
    res = mf.solve_static(g, s, t, det)
    assert res.flow_value == rec["static_flow"]
    assert res.rounds == rec["static_rounds_det"]
    st = res.state
    assert {k: sha(getattr(st, k)) for k in ("cf", "excess", "height")} == rec["static_state_sha"]
    for entry in rec["chain"]:
        bu, bv, bc = chain_batch(g.src, g.adj, g.is_original, g.cap0, n, s, t, entry)
        r = mf.solve_dynamic(st, g, mf.UpdateBatch(bu, bv, bc), det)
        assert r.flow_value == entry["flow"]
        assert r.rounds == entry["rounds_det"]
        st = r.state
        assert {k: sha(getattr(st, k)) for k in ("cf", "excess", "height")} == entry["state_sha"]
