"""Golden cases for the file formats, from the LIVE reference io.py (run in the
build container; the GPU box and the CPU tests only read the output).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_io.py

Writes the sample files under tests/golden/io/ and io.json: for every file the
reference's parse result (arrays) or its exception class and message.
"""
import json
import os
import sys

import numpy as np

REF = os.environ.get("DYNMAXFLOW_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import dynmaxflow as mf  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")

GRAPHS = {
    "ok_diamond.max": "c diamond\np max 4 5\nn 1 s\nn 4 t\na 1 2 3\na 1 3 2\na 2 4 2\na 3 4 3\na 2 3 1\n",
    "ok_comments.max": "# hash comment\n\n   c indented comment\np   max\t3 2\nn 1 s\nn 3 t\n  a 1 2 +7  \na 2 3 1_0\ncomment line\n",
    "ok_selfloop.max": "p max 3 4\nn 1 s\nn 3 t\na 1 1 5\na 1 2 4\na 1 2 6\na 2 3 9\n",
    "ok_zero_arcs.max": "p max 2 0\nn 1 s\nn 2 t\n",
    "bad_dup_p.max": "p max 2 1\np max 2 1\n",
    "bad_p_format.max": "p min 2 1\n",
    "bad_p_int.max": "p max two 1\n",
    "bad_sizes.max": "p max 0 1\n",
    "bad_node_first.max": "n 1 s\np max 2 1\n",
    "bad_node_kind.max": "p max 2 1\nn 1 x\n",
    "bad_node_id.max": "p max 2 1\nn 1.5 s\n",
    "bad_node_range.max": "p max 2 1\nn 3 s\n",
    "bad_dup_source.max": "p max 2 1\nn 1 s\nn 2 s\n",
    "bad_dup_sink.max": "p max 2 1\nn 1 t\nn 2 t\n",
    "bad_arc_first.max": "a 1 2 3\n",
    "bad_too_many.max": "p max 2 1\nn 1 s\nn 2 t\na 1 2 1\na 2 1 1\n",
    "bad_arc_fields.max": "p max 2 1\nn 1 s\nn 2 t\na 1 2\n",
    "bad_arc_int.max": "p max 2 1\nn 1 s\nn 2 t\na 1 2 x'y\n",
    "bad_arc_range.max": "p max 2 1\nn 1 s\nn 2 t\na 1 3 4\n",
    "bad_arc_neg.max": "p max 2 1\nn 1 s\nn 2 t\na 1 2 -4\n",
    "bad_kind.max": "p max 2 1\nx 1 2\n",
    "bad_missing_p.max": "c nothing\n",
    "bad_missing_s.max": "p max 2 1\nn 2 t\na 1 2 1\n",
    "bad_missing_t.max": "p max 2 1\nn 1 s\na 1 2 1\n",
    "bad_arc_count.max": "p max 2 2\nn 1 s\nn 2 t\na 1 2 1\n",
    "bad_underscore.max": "p max 2 1\nn 1 s\nn 2 t\na 1 2 1__0\n",
}
EDGE_LISTS = {
    "ok_edges.txt": "# u v cap\n0 1 5\n1 2 3\n0 2 1\n",
    "ok_edges1.txt": "1 2 5\n2 3 3\n",
    "bad_edges_fields.txt": "0 1\n",
    "bad_edges_int.txt": "0 1 z\n",
    "bad_edges_neg.txt": "0 -1 2\n",
    "bad_edges_cap.txt": "0 1 -2\n",
    "bad_edges_empty.txt": "c none\n",
}
UPDATES = {  # against ok_diamond.max
    "ok_upd.txt": "c batch\nu 1 2 1\nu 3 4 5\n",
    "bad_upd_kind.txt": "x 1 2 1\n",
    "bad_upd_fields.txt": "u 1 2\n",
    "bad_upd_int.txt": "u 1 2 q\n",
    "bad_upd_range.txt": "u 1 9 1\n",
    "bad_upd_neg.txt": "u 1 2 -1\n",
    "bad_upd_unknown.txt": "u 1 4 1\n",
    "bad_upd_stub.txt": "u 2 1 1\n",
    "bad_upd_dup.txt": "u 1 2 1\nu 1 2 2\n",
}


def run(fn):
    try:
        r = fn()
    except Exception as exc:  # noqa: BLE001
        return {"error": type(exc).__name__, "message": str(exc).replace(HERE + "/", "")}
    return {"ok": r}


def main():
    os.makedirs(HERE, exist_ok=True)
    out = {}
    for d in (GRAPHS, EDGE_LISTS, UPDATES):
        for name, text in d.items():
            with open(os.path.join(HERE, name), "w") as fh:
                fh.write(text)
    for name in GRAPHS:
        def f(name=name):
            g, s, t = mf.parse_graph(os.path.join(HERE, name))
            return {"n": g.n, "us": g.us.tolist(), "vs": g.vs.tolist(), "caps": g.caps.tolist(),
                    "s": s, "t": t}
        out[name] = run(f)
    for name in EDGE_LISTS:
        for one in (False, True):
            def f(name=name, one=one):
                g = mf.parse_edge_list(os.path.join(HERE, name), one_indexed=one)
                return {"n": g.n, "us": g.us.tolist(), "vs": g.vs.tolist(), "caps": g.caps.tolist()}
            out[f"{name}|{int(one)}"] = run(f)
    g, _, _ = mf.parse_graph(os.path.join(HERE, "ok_diamond.max"))
    csr = mf.build_bicsr(g)
    for name in UPDATES:
        def f(name=name):
            b = mf.parse_updates(os.path.join(HERE, name), csr)
            return {"us": b.us.tolist(), "vs": b.vs.tolist(), "caps": b.new_caps.tolist()}
        out[name] = run(f)
    with open(os.path.join(HERE, "io.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print(len(out), "cases")


if __name__ == "__main__":
    main()
