"""Vertex-range partitioned engine on one GPU: P = 1..4 parts
hosted by one process (same-device peer pointers: the same kernels and the
same host loop as the multi-GPU run), and P = 2 processes sharing the GPU
through CUDA IPC with a gloo group (the one-process-per-GPU plumbing).

Checks: each part's rows are exactly its slice of the reference Bi-CSR
(rev mapped back to global slots equals the reference rev); the global
relabel heights equal the reference's; the static flow and every chained
batch flow equal the reference's (golden fixtures); batch errors raise the
reference's exceptions and leave the state untouched.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from golden_data import load, sha
from paper_2511_01235_b200 import gen

pytestmark = pytest.mark.gpu

G = load()
NAMES = ["rand0", "rand3", "rand7", "rand16", "rand20", "C1", "grid64", "rmat12", "road48"]


@pytest.fixture(scope="module")
def mf():
    import paper_2511_01235_b200 as m
    return m


@pytest.fixture(scope="module")
def part():
    from paper_2511_01235_b200 import partition
    return partition


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


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("name", ["rand3", "grid64", "rmat12"])
def test_parts_are_slices_of_the_reference_layout(mf, part, name, P):
    n, us, vs, caps, s, t = instance(name)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    pg = part.PartitionedGraph(n, us, vs, caps, s, t, part.LocalGroup(P))
    assert pg.m == g.m and pg.m_original == g.m_original
    off, adj, rev, cap0, orig = [], [], [], [], []
    for r in range(P):
        d = pg.download(r)
        lo = int(pg.bounds[r])
        off.append(d["off"][:-1] + pg.slot_base[r])
        adj.append(d["adj"])
        owner = np.searchsorted(pg.bounds, d["adj"], side="right") - 1
        rev.append(pg.slot_base[owner] + d["rev"])
        cap0.append(d["cap0"])
        orig.append(d["orig"])
        assert int(d["off"][-1]) == pg.slots[r]
        assert np.array_equal(g.offsets[lo:int(pg.bounds[r + 1]) + 1] - g.offsets[lo], d["off"])
    assert np.array_equal(np.concatenate(off + [[g.m]]), g.offsets)
    for got, want in ((adj, g.adj), (rev, g.rev), (cap0, g.cap0), (orig, g.is_original)):
        assert np.array_equal(np.concatenate(got), np.asarray(want, np.int64))
    pg.close()


@pytest.mark.parametrize("bottom_up", ["0", "16", "1000000000"], ids=["topdown", "auto", "bottomup"])
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("name", ["rand3", "rand7", "grid64", "rmat12"])
def test_global_relabel_heights_bit_exact(mf, part, name, P, bottom_up, monkeypatch):
    """Saturated state -> backward BFS (bases {t}): heights equal the
    reference's bfs_heights (golden sha over the whole height array), with
    top-down levels only, the automatic direction switch, and bottom-up
    levels throughout."""
    monkeypatch.setenv("MFX_PART_BOTTOM_UP", bottom_up)
    n, us, vs, caps, s, t = instance(name)
    pg = part.PartitionedGraph(n, us, vs, caps, s, t, part.LocalGroup(P))
    pg.init_residuals()
    pg.saturate_source()
    pg.global_relabel(dynamic=False)
    h = np.concatenate([pg.download(r)["height"] for r in range(P)])
    assert sha(h) == G.rec[name]["bfs_sat_sha"]
    pg.close()


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("name", NAMES)
def test_static_and_chained_dynamic_flows(mf, part, name, P):
    rec = G.rec[name]
    n, us, vs, caps, s, t = instance(name)
    if P > n:
        pytest.skip("more parts than vertices")
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))  # batch sampling only
    pg = part.PartitionedGraph(n, us, vs, caps, s, t, part.LocalGroup(P))
    res = pg.solve_static()
    assert res.flow_value == rec["static_flow"] == res.cut_capacity
    cap0 = np.asarray(g.cap0, np.int64).copy()
    for entry in rec["chain"]:
        bu, bv, bc = chain_batch(g.src, g.adj, g.is_original, cap0, n, s, t, entry)
        r = pg.solve_dynamic(mf.UpdateBatch(bu, bv, bc))
        assert r.flow_value == entry["flow"] == r.cut_capacity, (name, P, entry["seed"])
        assert pg.active_count() == 0
        cap0[g.edge_indices(bu, bv)] = bc
    pg.close()


@pytest.mark.parametrize("outbox", ["0", "2", "64"])
@pytest.mark.parametrize("name", ["grid64", "rmat12"])
def test_cut_slot_outboxes(mf, part, name, outbox, monkeypatch):
    """Cut-slot pushes buffered per destination part and applied by the owner
    after the push phase (part.cu part_inbox_kernel): off (direct remote
    updates), tiny outboxes that overflow into the direct path mid-phase, and
    a small one; the golden static and chained flows hold in every mode."""
    monkeypatch.setenv("MFX_PART_OUTBOX", outbox)
    rec = G.rec[name]
    n, us, vs, caps, s, t = instance(name)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    pg = part.PartitionedGraph(n, us, vs, caps, s, t, part.LocalGroup(3))
    res = pg.solve_static()
    assert res.flow_value == rec["static_flow"] == res.cut_capacity
    cap0 = np.asarray(g.cap0, np.int64).copy()
    for entry in rec["chain"][:3]:
        bu, bv, bc = chain_batch(g.src, g.adj, g.is_original, cap0, n, s, t, entry)
        r = pg.solve_dynamic(mf.UpdateBatch(bu, bv, bc))
        assert r.flow_value == entry["flow"] == r.cut_capacity
        assert pg.active_count() == 0
        cap0[g.edge_indices(bu, bv)] = bc
    pg.close()


def test_batch_errors_match_reference_and_leave_state(mf, part):
    """The reference's error cases (tests/golden/make_golden.py) on the
    diamond, split over 2 parts: same exception text, state untouched."""
    errs = G.rec["errors"]
    edges = [(0, 1, 3), (0, 2, 2), (1, 3, 2), (2, 3, 3), (1, 2, 1)]
    us, vs, caps = (np.array([e[c] for e in edges], np.int64) for c in range(3))
    pg = part.PartitionedGraph(4, us, vs, caps, 0, 3, part.LocalGroup(2))
    assert pg.solve_static().flow_value == 5
    cases = {
        "neg": [(0, 1, 2), (1, 3, -1)],
        "unknown": [(0, 1, 2), (0, 3, 5)],
        "stub": [(1, 0, 5)],
        "dup": [(1, 3, 1), (0, 1, 2), (1, 3, 4), (0, 1, 3)],
    }
    for key, ups in cases.items():
        with pytest.raises(mf.BatchError) as ei:
            pg.solve_dynamic(mf.UpdateBatch.from_updates(ups))
        assert str(ei.value) == errs["batch/" + key], key
    # state untouched: the SPEC example (0->1): 3 -> 1 gives 3
    assert pg.solve_dynamic(mf.UpdateBatch.from_updates([(0, 1, 1)])).flow_value == 3
    pg.close()


def test_full_size_c3_two_parts_matches_reference(mf, part):
    """C3 (R-MAT 20, 31.4 M slots) split over 2 parts: static + chained
    batches equal the live reference (tests/golden/large.json)."""
    import json
    with open(os.path.join(os.path.dirname(__file__), "golden", "large.json")) as fh:
        rec = json.load(fh)["C3"]
    us, vs, caps, s, t = gen.rmat_graph(*rec["args"])
    n = rec["n"]
    pg = part.PartitionedGraph(n, us, vs, caps, s, t, part.LocalGroup(2))
    assert pg.m == rec["S"]
    assert pg.solve_static().flow_value == rec["static_flow"]
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    el = g.to_edge_list()
    ecaps = el.caps.copy()
    for entry in rec["chain"][:2]:
        bu, bv, bc, pick = gen.fast_batch(n, el.us, el.vs, ecaps, s, t, entry["k"], "mixed",
                                          entry["seed"])
        ecaps[pick] = bc
        assert pg.solve_dynamic(mf.UpdateBatch(bu, bv, bc)).flow_value == entry["flow"]
    pg.close()


def test_two_processes_ipc_gloo(tmp_path):
    """One process per part (the multi-GPU launch shape): two ranks share
    cuda:0 through CUDA IPC, torch.distributed (gloo) carries the handles
    and the per-phase barrier / all-reduce."""
    script = os.path.join(os.path.dirname(__file__), "part_worker.py")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", WORLD_SIZE="2")
    procs = [subprocess.Popen([sys.executable, script, str(r), str(tmp_path / f"out{r}.txt")],
                              env=dict(env, RANK=str(r)), stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = [p.communicate(timeout=300)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    got = [open(tmp_path / f"out{r}.txt").read().split() for r in range(2)]
    assert got[0] == got[1]
    rec = G.rec["grid64"]
    assert [int(x) for x in got[0]] == [rec["static_flow"]] + [e["flow"] for e in rec["chain"]]


def test_device_rmat_sampler_and_dynamic_equals_resolve(part):
    """Device-generated R-MAT (C5 generator at scale 14) over 3 parts:
    sampled batches are valid mixed updates, and after each the dynamic
    flow equals a static re-solve on the updated capacities."""
    pg = part.PartitionedGraph.rmat(14, 16, 3, part.LocalGroup(3))
    f0 = pg.solve_static().flow_value
    assert f0 > 0
    for b in range(3):
        batch = pg.sample_batch(2000, seed=b)
        assert len(batch) == 2000
        keys = batch.us * pg.n + batch.vs
        assert np.unique(keys).size == len(batch) and np.all(batch.new_caps >= 0)
        d = pg.solve_dynamic(batch)
        s = pg.solve_static()
        assert d.flow_value == s.flow_value == d.cut_capacity
    pg.close()


def _rmat_chain(part, scale, P, k, batches):
    pg = part.PartitionedGraph.rmat(scale, 16, 0, part.LocalGroup(P))
    st = pg.solve_static()
    assert st.flow_value == st.cut_capacity > 0
    for b in range(batches):
        batch = pg.sample_batch(k, seed=b)
        assert len(batch) == k
        d = pg.solve_dynamic(batch)
        assert d.flow_value == d.cut_capacity
        s = pg.solve_static()  # static re-solve on the updated capacities
        assert s.flow_value == d.flow_value == s.cut_capacity, (scale, P, b)
    pg.close()


@pytest.mark.parametrize("P", [2, 4])
def test_rmat22_partition_million_update_batches(part, P):
    """C5's generator at scale 22 (131 M slots) over P parts with C5-sized
    batches of 10^6 mixed updates: dynamic == static re-solve, flow == cut."""
    _rmat_chain(part, 22, P, 1_000_000, 2)


@pytest.mark.slow
@pytest.mark.skipif(not os.environ.get("MFX_SLOW"), reason="opt-in (minutes): MFX_SLOW=1")
@pytest.mark.parametrize("scale,P", [(24, 2), (24, 4), (26, 4)])
def test_rmat_large_partition_million_update_batches(part, scale, P):
    """R-MAT 24 (521 M slots) and full C5 (R-MAT 26, 2.1 B slots) on one
    GPU, 10^6-update batches, dynamic == static re-solve."""
    _rmat_chain(part, scale, P, 1_000_000, 2)


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("name", ["rand3", "grid64", "rmat12", "road48"])
def test_topology_mode_and_instrument(mf, part, name, P):
    """mode="topology" (solver.py:167-175: every non-terminal works each
    round) gives the reference's flows on the partition too, and the
    instrument hook sees every round's relabel and repair
    (solver.py:219-241; the partitioned state is the PartitionedGraph)."""
    rec = G.rec[name]
    n, us, vs, caps, s, t = instance(name)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    pg = part.PartitionedGraph(n, us, vs, caps, s, t, part.LocalGroup(P))
    seen = []

    def hook(st, gg, rnd, label):
        assert st is pg and gg is pg
        seen.append((rnd, label))

    p = mf.SolverParams(mode="topology", instrument=hook)
    res = pg.solve_static(p)
    assert res.flow_value == rec["static_flow"] == res.cut_capacity
    assert seen[0] == (0, "bfs") and seen[-1] == (res.rounds, "bfs")
    assert [x for x in seen if x[1] == "repair"] == [(r, "repair") for r in range(res.rounds)]
    cap0 = np.asarray(g.cap0, np.int64).copy()
    for entry in rec["chain"]:
        bu, bv, bc = chain_batch(g.src, g.adj, g.is_original, cap0, n, s, t, entry)
        r = pg.solve_dynamic(mf.UpdateBatch(bu, bv, bc), mf.SolverParams(mode="topology"))
        assert r.flow_value == entry["flow"] == r.cut_capacity, (name, P, entry["seed"])
        cap0[g.edge_indices(bu, bv)] = bc
    pg.close()
