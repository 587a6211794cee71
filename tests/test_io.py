"""File formats (reference io.py) through the native readers: every sample in
tests/golden/io/ parses to the reference's arrays or raises the reference's
exception with the same text (tests/golden/make_golden_io.py ran the live
reference).  Graph and edge-list parsing are host-only; update files are
validated against a device graph (GPU tests)."""
import json
import os

import numpy as np
import pytest

from paper_2511_01235_b200 import io as mio

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")
with open(os.path.join(HERE, "io.json")) as _fh:
    GOLD = json.load(_fh)


def check(rec, fn):
    if "error" in rec:
        with pytest.raises(Exception) as ei:
            fn()
        assert type(ei.value).__name__ == rec["error"]
        assert str(ei.value).replace(HERE + "/", "") == rec["message"]
        return None
    return fn()


@pytest.mark.parametrize("name", sorted(k for k in GOLD if k.endswith(".max")))
def test_parse_graph_matches_reference(name):
    rec = GOLD[name]
    out = check(rec, lambda: mio.parse_graph(os.path.join(HERE, name)))
    if out is not None:
        g, s, t = out
        want = rec["ok"]
        assert (g.n, s, t) == (want["n"], want["s"], want["t"])
        for k in ("us", "vs", "caps"):
            assert getattr(g, k).tolist() == want[k]


@pytest.mark.parametrize("key", sorted(k for k in GOLD if "|" in k))
def test_parse_edge_list_matches_reference(key):
    name, one = key.split("|")
    rec = GOLD[key]
    out = check(rec, lambda: mio.parse_edge_list(os.path.join(HERE, name), one_indexed=one == "1"))
    if out is not None:
        want = rec["ok"]
        assert out.n == want["n"]
        for k in ("us", "vs", "caps"):
            assert getattr(out, k).tolist() == want[k]


def test_parse_error_attributes_and_missing_file(tmp_path):
    with pytest.raises(mio.ParseError) as ei:
        mio.parse_graph(os.path.join(HERE, "bad_arc_neg.max"))
    assert ei.value.lineno == 4 and ei.value.path.endswith("bad_arc_neg.max")
    with pytest.raises(FileNotFoundError):
        mio.parse_graph(tmp_path / "absent.max")


def test_write_then_parse_round_trip(tmp_path):
    from paper_2511_01235_b200 import EdgeListGraph, UpdateBatch, gen
    us, vs, caps, s, t = gen.random_edges(300, 3000, seed=5)
    p = tmp_path / "g.max"
    mio.write_graph(p, EdgeListGraph(300, us, vs, caps), s, t)
    g, s2, t2 = mio.parse_graph(p)
    assert (g.n, s2, t2) == (300, s, t)
    assert np.array_equal(g.us, us) and np.array_equal(g.vs, vs) and np.array_equal(g.caps, caps)
    text = p.read_text().splitlines()
    assert text[:3] == ["p max 300 3000", f"n {s + 1} s", f"n {t + 1} t"]
    assert text[3] == f"a {us[0] + 1} {vs[0] + 1} {caps[0]}"
    q = tmp_path / "u.txt"
    b = UpdateBatch(us[:5], vs[:5], caps[:5] + 1)
    mio.write_updates(q, b)
    assert q.read_text().splitlines()[0] == f"u {us[0] + 1} {vs[0] + 1} {caps[0] + 1}"


def test_results_csv_round_trip(tmp_path):
    r = [mio.ResultRecord("g", "dynamic", "mixed", 1.5, 42, 3, 1.0, 2.0, 0.5, 3.5, True),
         mio.ResultRecord("g", "static", "inc", 10.0, 7, 1, 0.25, 0.125, 0.0, 0.375, False)]
    p = tmp_path / "r.csv"
    mio.write_results(p, r, {"backend": "cuda-sm_100a", "reps": 3})
    lines = p.read_text().splitlines()
    assert lines[0] == "# backend=cuda-sm_100a" and lines[2] == ",".join(mio.RESULT_FIELDS)
    assert lines[3] == "g,dynamic,mixed,1.5,42,3,1.000,2.000,0.500,3.500,true"
    assert mio.read_results(p) == r


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(k for k in GOLD if k.endswith(".txt") and "|" not in k))
def test_parse_updates_matches_reference(name):
    import paper_2511_01235_b200 as mf
    g, s, t = mio.parse_graph(os.path.join(HERE, "ok_diamond.max"))
    csr = mf.build_bicsr(g)
    out = check(GOLD[name], lambda: mio.parse_updates(os.path.join(HERE, name), csr))
    if out is not None:
        want = GOLD[name]["ok"]
        assert out.us.tolist() == want["us"] and out.vs.tolist() == want["vs"]
        assert out.new_caps.tolist() == want["caps"]


@pytest.mark.gpu
def test_run_benchmark_schema_and_plot_data(tmp_path):
    """Reference bench.py run_benchmark schema on the GPU engine: three modes
    per spec, identical verified flows, gnuplot tables per kind."""
    import paper_2511_01235_b200 as mf
    g, s, t = mf.random_graph(400, 4000, seed=3)  # reference signature
    specs = [mf.BatchSpec(5.0, "mixed", 0), mf.BatchSpec(10.0, "inc", 1), mf.BatchSpec(5.0, "dec", 2)]
    recs = mf.run_benchmark(g, s, t, specs, reps=2, instance="r400")
    assert [r.mode for r in recs] == list(mf.BENCH_MODES) * 3
    for i in range(0, 9, 3):
        assert len({r.flow_value for r in recs[i:i + 3]}) == 1
        assert all(r.verified and r.total_ms > 0 for r in recs[i:i + 3])
    paths = mf.write_plot_data(recs, tmp_path)
    assert sorted(os.path.basename(p) for p in paths) == ["dec.dat", "inc.dat", "mixed.dat"]
    lines = open(paths[0]).read().splitlines()
    assert lines[0] == "# pct dynamic pushpull static" and len(lines) == 2
    mio.write_results(tmp_path / "r.csv", recs)
    back = mio.read_results(tmp_path / "r.csv")  # (times round-trip at 3 decimals)
    assert [(r.mode, r.flow_value, r.verified) for r in back] == \
        [(r.mode, r.flow_value, r.verified) for r in recs]
    assert all(abs(a.total_ms - b.total_ms) < 1e-3 for a, b in zip(back, recs))
