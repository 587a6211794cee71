"""GPU stress and safety-net tests.

* The CTA-local BFS ring is a polled structure (warps spin on slot and
  counter words in shared memory; `compute-sanitizer racecheck` flags it by
  design), so its correctness is argued, not tool-checked.  These tests
  repeat the bit-exact global relabel (static and dynamic bases,
  kernels.py:168-215 via solver.py:155-164 / dynamic.py:125-133) 50 times per
  graph under randomised ring schedules: back-off, ring capacity, labels per
  epoch.  Any lost or duplicated ring item shows up as a wrong height.
* The operation ceiling (solver.py:37-44, 196-200) and the device watchdog
  have never fired in an ordinary run; here both are forced, the error
  classes and texts are checked, and the handles stay usable afterwards.
"""
import random

import numpy as np
import pytest

import oracle as O
from golden_data import load, sha
from paper_2511_01235_b200 import gen

pytestmark = pytest.mark.gpu

G = load()


@pytest.fixture(scope="module")
def mf():
    import paper_2511_01235_b200 as m
    return m


def instance(name):
    rec = G.rec[name]
    src = rec["source"]
    us, vs, caps, s, t = gen.source_edges(src["gen"], src["args"])
    return rec["n"], us, vs, caps, s, t


_TERMINAL = {}


def terminal(name):
    """The oracle's terminated static state (= the reference's, pinned in
    test_oracle_golden) and the first chained batch of the golden record."""
    if name not in _TERMINAL:
        rec = G.rec[name]
        n, us, vs, caps, s, t = instance(name)
        og = O.build_bicsr(n, us, vs, caps)
        _, ost = O.solve_static(og, s, t)
        entry = rec["chain"][0]
        keep = og.is_original.astype(bool)
        spec = gen.BatchSpec(entry["pct"], entry["kind"], entry["seed"])
        bu, bv, bc, _ = gen.batch_arrays(n, og.src[keep], og.adj[keep], og.cap0[keep], s, t, spec)
        _TERMINAL[name] = (og, ost, (bu, bv, bc), entry)
    return _TERMINAL[name]


RING_SLEEP = ["0", "20", "64", "300", "1000"]
LQ_CAP = ["8", "64", "256", "2048"]
BFS_LOCAL = ["2", "16", "128", "1024"]


@pytest.mark.parametrize("name", ["grid64", "rmat12", "road48"])
def test_bfs_ring_stress_bit_exact(mf, name, monkeypatch):
    rec = G.rec[name]
    n, us, vs, caps, s, t = instance(name)
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    og, ost, (bu, bv, bc), entry = terminal(name)
    rng = random.Random(hash(name) & 0xFFFF)
    for it in range(50):
        env = {"MFX_RING_SLEEP": rng.choice(RING_SLEEP), "MFX_LQ_CAP": rng.choice(LQ_CAP),
               "MFX_BFS_LOCAL": rng.choice(BFS_LOCAL)}
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        st = mf.init_residuals(g, s, t)
        mf.saturate_source(st, g)
        mf.backward_bfs(st, g)
        assert sha(st.height) == rec["bfs_sat_sha"], (it, env)
        gd = mf.upload_bicsr(n, og.offsets, og.adj, og.rev, og.cap0, og.is_original)
        sd = mf.init_residuals(gd, s, t)
        sd.upload(ost.cf, ost.excess, ost.height)
        mf.dynamic_prephase(sd, gd, mf.UpdateBatch(bu, bv, bc))
        mf.backward_bfs_dynamic(sd, gd)
        assert sha(sd.height) == entry["bfs_dyn_sha"], (it, env)


def test_operation_ceiling_raises_and_recovers(mf, monkeypatch):
    """A ceiling below the work a solve needs aborts it on the device with the
    reference's SolverError text (solver.py:196-200); the graph solves
    normally afterwards."""
    rec = G.rec["grid64"]
    n, us, vs, caps, s, t = instance("grid64")
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    monkeypatch.setenv("MFX_CEILING", "10")
    with pytest.raises(mf.SolverError, match="exceeded the termination ceiling 10"):
        mf.solve_static(g, s, t)
    monkeypatch.delenv("MFX_CEILING")
    res = mf.solve_static(g, s, t)
    assert res.flow_value == rec["static_flow"] == res.certificate.cut_capacity


def test_dynamic_ceiling_raises(mf, monkeypatch):
    rec = G.rec["rmat12"]
    n, us, vs, caps, s, t = instance("rmat12")
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    res = mf.solve_static(g, s, t)
    assert res.flow_value == rec["static_flow"]
    _, _, (bu, bv, bc), entry = terminal("rmat12")
    monkeypatch.setenv("MFX_CEILING", "1")
    with pytest.raises(mf.SolverError, match="termination ceiling 1"):
        mf.solve_dynamic(res.state, g, mf.UpdateBatch(bu, bv, bc))


def test_watchdog_aborts_instead_of_hanging(mf, monkeypatch):
    """The device watchdog (timeout_s / $MFX_TIMEOUT_S) ends a solve past its
    deadline with DeviceTimeout rather than spinning; the next solve on the
    same graph is unaffected."""
    rec = G.rec["road48"]
    n, us, vs, caps, s, t = instance("road48")
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    with pytest.raises(mf.DeviceTimeout, match="watchdog"):
        mf.solve_static(g, s, t, mf.SolverParams(timeout_s=1e-9))
    monkeypatch.setenv("MFX_TIMEOUT_S", "1e-9")
    with pytest.raises(mf.DeviceTimeout):
        mf.solve_static(g, s, t)
    monkeypatch.delenv("MFX_TIMEOUT_S")
    res = mf.solve_static(g, s, t)
    assert res.flow_value == rec["static_flow"] == res.certificate.cut_capacity
    rep = mf.verify_gpu(res.state, g, res.flow_value)
    assert rep.ok, rep.problems
