"""Benchmark harness with the reference's record schema (bench.py:150-230):
per batch spec, the dynamic solve, the O2 push-pull solve and a from-scratch
static solve on the updated graph, each timed over ``reps`` fresh device
copies; per-phase medians go into :class:`~paper_2511_01235_b200.io.ResultRecord`
rows, and :func:`write_plot_data` writes one gnuplot table per batch kind.

The repetitions restart from device snapshots (``BiCsrGraph.copy`` /
``SolverState.copy``: D2D copies), the static leg's graph build is outside
its timer as in the reference, and "verified" means the device verifier
(``verify_gpu``: the checks of oracle.verify_cut) passed on every
repetition and all three modes agreed on the flow value.
"""

import os
import statistics
import time

from .dynamic import UpdateBatch, solve_dynamic, solve_dynamic_pushpull, updated_edge_list
from .gen import BatchSpec, batch_arrays
from .graph import EdgeListGraph, build_bicsr
from .io import ResultRecord
from .solver import SolverParams, solve_static
from .verify import verify_gpu

BENCH_MODES = ("dynamic", "pushpull", "static")
_PHASES = ("bfs", "push", "repair")


def _time_mode(mode, csr, prior, batch, s, t, params, reps):
    """(median ms per phase + total, rounds, flow, all certificates ok)."""
    samples = {k: [] for k in (*_PHASES, "total")}
    ok, res = True, None
    for _ in range(max(1, reps)):
        if mode == "static":
            graph = build_bicsr(updated_edge_list(csr, batch))  # untimed, as the reference
            t0 = time.perf_counter()
            res = solve_static(graph, s, t, params)
        else:
            graph, state = csr.copy(), prior.state.copy()
            fn = solve_dynamic if mode == "dynamic" else solve_dynamic_pushpull
            t0 = time.perf_counter()
            res = fn(state, graph, batch, params)
        samples["total"].append(time.perf_counter() - t0)
        for k in _PHASES:
            samples[k].append(res.phase_times[k])
        ok = ok and verify_gpu(res.state, graph, res.flow_value).ok
    med = {k: 1e3 * statistics.median(v) for k, v in samples.items()}
    return med, res.rounds, res.flow_value, ok


def run_benchmark(g: EdgeListGraph, s: int, t: int, specs: list[BatchSpec],
                  params: SolverParams | None = None, reps: int = 3,
                  instance: str = "graph") -> list[ResultRecord]:
    """reference bench.py:153-207 on the GPU engine."""
    params = params or SolverParams()
    csr = build_bicsr(g)
    el = csr.to_edge_list()
    prior = solve_static(csr, s, t, params)
    out = []
    for spec in specs:
        batch = UpdateBatch(*batch_arrays(el.n, el.us, el.vs, el.caps, s, t, spec)[:3])
        runs = {m: _time_mode(m, csr, prior, batch, s, t, params, reps) for m in BENCH_MODES}
        agree = len({r[2] for r in runs.values()}) == 1
        for m in BENCH_MODES:
            med, rounds, flow, ok = runs[m]
            out.append(ResultRecord(instance, m, spec.canonical_kind(), spec.pct, flow, rounds,
                                    med["bfs"], med["push"], med["repair"], med["total"],
                                    bool(ok and agree)))
    return out


def write_plot_data(records: list[ResultRecord], directory) -> list[str]:
    """One ``<kind>.dat`` per batch kind: batch % then the median total ms
    of each mode (reference bench.py:210-230)."""
    by_kind: dict[str, dict[float, dict[str, float]]] = {}
    for r in records:
        by_kind.setdefault(r.batch_kind, {}).setdefault(r.batch_pct, {})[r.mode] = r.total_ms
    paths = []
    for kind in sorted(by_kind):
        path = os.path.join(directory, f"{kind}.dat")
        lines = ["# pct " + " ".join(BENCH_MODES)]
        for pct, row in sorted(by_kind[kind].items()):
            lines.append(f"{pct:g} " + " ".join(f"{row.get(m, float('nan')):.3f}"
                                                 for m in BENCH_MODES))
        with open(path, "w") as fh:
            fh.write("\n".join(lines) + "\n")
        paths.append(path)
    return paths
