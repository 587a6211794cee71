"""Full-scale golden flows for the BASELINE.json configs, from the LIVE
reference (run in the build container, where /root/reference exists; the GPU
box only reads tests/golden/large.json).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_large.py [C2 C3 road512 ...]

For each config: reference ``build_bicsr`` + ``solve_static`` (numba backend,
threads = nproc), then a chain of ``solve_dynamic`` batches drawn with this
repo's ``gen.fast_batch`` (reference generate_batch semantics, O(m)) from the
capacities the previous batch left.  Records the static flow, every chained
flow, the batch seeds/sizes and the reference wall times (this container's
host, for context only).  The C4 road config at full scale (24 M vertices)
and C5 (R-MAT 26) do not finish on the reference CPU path; road512/road1024
are the scaled-down anchors of the same generator.
"""

import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("DYNMAXFLOW_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import dynmaxflow as ref  # noqa: E402  (the reference)

from paper_2511_01235_b200 import gen  # noqa: E402  (shapes + batch sampler only)

OUT = os.path.join(HERE, "large.json")

# name -> (generator, args, [(batch size, seed), ...])
CONFIGS = {
    "C2": ("grid_graph", [2048, 2048, 0], [(10_000, s) for s in range(4)]),
    "C3": ("rmat_graph", [20, 16, 0], [(1_000, 0), (10_000, 1), (100_000, 2), (10_000, 3)]),
    "rmat18": ("rmat_graph", [18, 16, 0], [(1_000, 0), (10_000, 1), (100_000, 2)]),
    "grid512": ("grid_graph", [512, 512, 0], [(10_000, s) for s in range(4)]),
    "road256": ("road_graph", [256, 256, 0, 0.21], [(1_000, 0), (10_000, 1), (1_000, 2)]),
    "road512": ("road_graph", [512, 512, 0, 0.21], [(1_000, 0), (10_000, 1)]),
}


def n_of(name, args):
    g = CONFIGS[name][0]
    if g == "grid_graph":
        return args[0] * args[1] + 2
    if g == "rmat_graph":
        return 1 << args[0]
    return args[0] * args[1]


def run(name):
    gname, args, chain = CONFIGS[name]
    us, vs, caps, s, t = getattr(gen, gname)(*args)
    n = n_of(name, args)
    params = ref.SolverParams(threads=os.cpu_count())
    t0 = time.perf_counter()
    csr = ref.build_bicsr(ref.EdgeListGraph(n, us, vs, caps))
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    res = ref.solve_static(csr, s, t, params)
    t_static = time.perf_counter() - t0
    rec = {"gen": gname, "args": args, "n": n, "s": int(s), "t": int(t), "S": int(csr.m),
           "m_original": int(csr.m_original), "static_flow": int(res.flow_value),
           "static_rounds": int(res.rounds), "ref_build_s": round(t_build, 2),
           "ref_static_s": round(t_static, 2), "threads": os.cpu_count(), "chain": []}
    print(name, "static", res.flow_value, f"{t_static:.1f}s", flush=True)
    el = csr.to_edge_list()
    ecaps = el.caps.copy()
    st, g = res.state, res.graph
    for k, seed in chain:
        bu, bv, bc, pick = gen.fast_batch(n, el.us, el.vs, ecaps, s, t, k, "mixed", seed)
        ecaps[pick] = bc
        t0 = time.perf_counter()
        r = ref.solve_dynamic(st, g, ref.UpdateBatch(bu, bv, bc), params)
        dt = time.perf_counter() - t0
        st, g = r.state, r.graph
        rec["chain"].append({"k": k, "seed": seed, "flow": int(r.flow_value),
                             "rounds": int(r.rounds), "ref_s": round(dt, 2)})
        print(name, "batch", k, seed, r.flow_value, f"{dt:.1f}s", flush=True)
    return rec


def main():
    names = sys.argv[1:] or list(CONFIGS)
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            data = json.load(fh)
    data["_meta"] = {"generator": "tests/golden/make_golden_large.py", "reference": REF,
                     "backend": ref.backend_name() if hasattr(ref, "backend_name") else "numba",
                     "batches": "gen.fast_batch(n, el.us, el.vs, caps_after_prev, s, t, k, "
                                "'mixed', seed) over csr.to_edge_list()"}
    for name in names:
        data[name] = run(name)
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
