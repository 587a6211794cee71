"""The reference-side binding actually runs: a temporary
copy of the UNMODIFIED reference package (baseline/_ref/dynmaxflow) gets
``integration/dynmaxflow/_mfx.py`` plus the two call-site guards
(``integration/apply_patch.py``), and with ``DYNMAXFLOW_MFX_LIB`` pointing at
libmfx.so the reference's own ``solve_static`` / ``solve_dynamic`` --
driven by the reference's own ``build_bicsr``, ``generate_batch``,
``verify_cut`` and ``run_benchmark`` -- reproduce the golden flows after
every chained batch.  Runs in a subprocess so the patched package never
meets the test process's imports."""
import json
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = os.path.join(ROOT, "baseline", "_ref", "dynmaxflow")
LIB = os.path.join(ROOT, "paper_2511_01235_b200", "_lib", "libmfx.so")

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[2])
import dynmaxflow as R
from golden_data import load
assert R.__file__.startswith(sys.argv[1]), R.__file__
G = load()
out = {}
for name in json.loads(sys.argv[3]):
    rec = G.rec[name]
    n, s, t = rec["n"], rec["s"], rec["t"]
    if f"{name}/in_us" in G.arr:
        us, vs, caps = (G.arr[f"{name}/in_{k}"] for k in ("us", "vs", "caps"))
    else:
        src = rec["source"]
        if src["gen"] == "random_graph":
            e, s2, t2 = R.random_graph(*src["args"])
            us, vs, caps = e.us, e.vs, e.caps
        else:
            sys.path.insert(0, sys.argv[4])
            from paper_2511_01235_b200 import gen
            us, vs, caps, _, _ = gen.source_edges(src["gen"], src["args"])
    g = R.build_bicsr(R.EdgeListGraph(n, us, vs, caps))
    res = R.solve_static(g, s, t)
    assert type(res) is R.FlowResult and type(res.certificate) is R.CutCertificate
    assert R.verify_cut(res.certificate, g, res.state, res.flow_value).ok
    flows = [res.flow_value]
    st = res.state
    for e in rec["chain"]:
        b = R.generate_batch(g.to_edge_list(), s, t, R.BatchSpec(pct=e["pct"], kind=e["kind"],
                                                                seed=e["seed"]))
        r = R.solve_dynamic(st, g, b)
        rep = R.verify_cut(r.certificate, g, r.state, r.flow_value)
        assert rep.ok, rep.problems
        pre = R.verify_preflow(R.construct_flow(r.state, g), g, s, t, r.state.excess)
        assert pre.ok, pre.problems
        flows.append(r.flow_value)
        st, g = r.state, r.graph
    out[name] = flows
# reference error classes and texts through the backend
g = R.build_bicsr(R.EdgeListGraph(4, np.array([0, 1, 2]), np.array([1, 2, 3]), np.array([5, 4, 3])))
r = R.solve_static(g, 0, 3)
try:
    R.solve_dynamic(r.state, g, R.UpdateBatch.from_updates([(0, 1, 2), (2, 1, 1)]))
    raise SystemExit("no BatchError")
except R.BatchError as e:
    out["_batch_error"] = str(e)
try:
    R.solve_static(g, 2, 2)
except ValueError as e:
    out["_value_error"] = str(e)
# the reference's own benchmark harness on top of the backend
recs = R.run_benchmark(R.EdgeListGraph(4, np.array([0, 1, 2]), np.array([1, 2, 3]),
                                       np.array([5, 4, 3])), 0, 3,
                       [R.BatchSpec(pct=50.0, kind="mixed", seed=1)], reps=1, instance="tiny")
out["_bench_modes"] = sorted({x.mode for x in recs})
print(json.dumps(out))
"""


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not installed in baseline/_ref")
def test_reference_package_with_mfx_backend(tmp_path, golden):
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import apply_patch
    pkg = tmp_path / "dynmaxflow"
    shutil.copytree(REF, pkg)
    apply_patch.patch(str(pkg))
    names = ["diamond", "rand0", "rand5", "rand13", "C1", "grid64", "rmat12", "road48"]
    names = [n for n in names if n in golden.rec]
    env = dict(os.environ, DYNMAXFLOW_MFX_LIB=LIB, PYTHONPATH=str(tmp_path))
    p = subprocess.run([sys.executable, "-c", SCRIPT, str(tmp_path), HERE, json.dumps(names), ROOT],
                       capture_output=True, text=True, env=env, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    out = json.loads(p.stdout.strip().splitlines()[-1])
    for name in names:
        rec = golden.rec[name]
        assert out[name] == [rec["static_flow"]] + [e["flow"] for e in rec["chain"]], name
    assert out["_batch_error"] == "update 1 targets edge 2->1 which is not an edge of the original graph"
    assert out["_value_error"] == "source and sink must differ"
    assert len(out["_bench_modes"]) >= 2
