"""File formats (mirror of reference io.py): DIMACS max-flow graphs, update
batches and the benchmark result CSV.

The graph / update / edge-list readers and writers are native
(csrc/io.cpp, one buffered pass, same accept / reject rules and error text as
the reference, io.py:33-182) so multi-million-edge inputs go straight to the
GPU builder.  The result CSV (io.py:185-238) is a few rows and stays Python.
"""

import csv
import ctypes
import os
from dataclasses import dataclass, fields

import numpy as np

from . import _lib as L
from .dynamic import BatchError, UpdateBatch
from .graph import BiCsrGraph, EdgeListGraph


class ParseError(ValueError):
    """Malformed input file; message carries the file path and line number
    (io.py:20-26)."""

    def __init__(self, path, lineno, message):
        super().__init__(f"{path}:{lineno}: {message}")
        self.path = str(path)
        self.lineno = lineno


def _read(fn, path, *args):
    path = os.fspath(path)
    with open(path):  # the reference's open(): FileNotFoundError / IsADirectoryError
        pass
    lib = L.load()
    h = ctypes.c_void_p()
    rc = fn(path.encode(), *args, ctypes.byref(h))
    if rc == L.MFX_PARSE_ERROR:
        raise ParseError(path, int(lib.mfx_io_error_line()), L.last_error())
    L.check(rc)
    try:
        info = np.zeros(4, np.int64)
        L.check(lib.mfx_edges_info(h, L.ptr64(info)))
        m = int(info[1])
        us, vs, caps = (np.empty(m, np.int64) for _ in range(3))
        L.check(lib.mfx_edges_get(h, L.ptr64(us), L.ptr64(vs), L.ptr64(caps)))
    finally:
        lib.mfx_edges_free(h)
    return int(info[0]), us, vs, caps, int(info[2]), int(info[3])


def parse_graph(path) -> tuple[EdgeListGraph, int, int]:
    """Read a DIMACS-max file; returns the edge list plus source and sink
    (io.py:33-109)."""
    n, us, vs, caps, s, t = _read(L.load().mfx_io_parse_graph, path)
    return EdgeListGraph(n, us, vs, caps), s, t


def write_graph(path, g: EdgeListGraph, source: int, sink: int) -> None:
    """io.py:112-118."""
    us, vs, caps = (L.as_i64(a) for a in (g.us, g.vs, g.caps))
    rc = L.load().mfx_io_write_graph(os.fspath(path).encode(), g.n, g.m, source, sink,
                                      L.ptr64(us), L.ptr64(vs), L.ptr64(caps))
    if rc == L.MFX_PARSE_ERROR:
        raise OSError(L.last_error())
    L.check(rc)


def resolve_batch(g: BiCsrGraph, batch: UpdateBatch) -> np.ndarray:
    """Edge slots a batch targets, with the reference's checks and messages
    (dynamic.py:63-88): negative capacity, unknown or stub edge, duplicate.
    The lookup runs on the device (BiCsrGraph.edge_indices)."""
    if len(batch) == 0:
        return np.empty(0, dtype=np.int64)
    neg = np.flatnonzero(batch.new_caps < 0)
    if neg.size:
        k = int(neg[0])
        raise BatchError(f"update {k} ({int(batch.us[k])}->{int(batch.vs[k])}): "
                         f"negative capacity {int(batch.new_caps[k])}")
    idx = g.edge_indices(batch.us, batch.vs)
    known = (idx >= 0) & g.is_original[np.maximum(idx, 0)]
    bad = np.flatnonzero(~known)
    if bad.size:
        k = int(bad[0])
        raise BatchError(f"update {k} targets edge {int(batch.us[k])}->{int(batch.vs[k])} "
                         f"which is not an edge of the original graph")
    order = np.argsort(idx, kind="stable")
    dup = np.flatnonzero(idx[order][1:] == idx[order][:-1])
    if dup.size:
        k = int(order[dup[0] + 1])
        raise BatchError(f"duplicate update for edge {int(batch.us[k])}->{int(batch.vs[k])}")
    return idx


def parse_updates(path, g: BiCsrGraph) -> UpdateBatch:
    """Read an update file and validate every edge against the graph
    (io.py:121-144)."""
    _, us, vs, caps, _, _ = _read(L.load().mfx_io_parse_updates, path, g.n)
    batch = UpdateBatch(us, vs, caps)
    resolve_batch(g, batch)  # existence + duplicate validation
    return batch


def write_updates(path, batch: UpdateBatch) -> None:
    """io.py:147-150."""
    us, vs, caps = batch.arrays()
    rc = L.load().mfx_io_write_updates(os.fspath(path).encode(), us.size, L.ptr64(us),
                                       L.ptr64(vs), L.ptr64(caps))
    if rc == L.MFX_PARSE_ERROR:
        raise OSError(L.last_error())
    L.check(rc)


def parse_edge_list(path, one_indexed: bool = False) -> EdgeListGraph:
    """Whitespace ``u v cap`` edge list; n = largest id + 1 (io.py:153-182)."""
    n, us, vs, caps, _, _ = _read(L.load().mfx_io_parse_edge_list, path, 1 if one_indexed else 0)
    return EdgeListGraph(n, us, vs, caps)


# ---------------------------------------------------------------------------
# benchmark result CSV (io.py:185-238)
# ---------------------------------------------------------------------------
@dataclass
class ResultRecord:
    """One benchmark measurement, serialized as a CSV row."""

    instance: str
    mode: str
    batch_kind: str
    batch_pct: float
    flow_value: int
    rounds: int
    bfs_ms: float
    push_ms: float
    repair_ms: float
    total_ms: float
    verified: bool


RESULT_FIELDS = [f.name for f in fields(ResultRecord)]


def _cells(r: ResultRecord) -> list:
    return [r.instance, r.mode, r.batch_kind, f"{r.batch_pct:g}", r.flow_value, r.rounds,
            *(f"{x:.3f}" for x in (r.bfs_ms, r.push_ms, r.repair_ms, r.total_ms)),
            "true" if r.verified else "false"]


def write_results(path_or_file, records: list[ResultRecord], metadata: dict | None = None) -> None:
    """Header row + one row per record; metadata as '# key=value' lines
    (io.py:205-222)."""
    if isinstance(path_or_file, (str, bytes)) or hasattr(path_or_file, "__fspath__"):
        with open(path_or_file, "w", newline="") as fh:
            write_results(fh, records, metadata)
        return
    path_or_file.writelines(f"# {k}={v}\n" for k, v in (metadata or {}).items())
    out = csv.writer(path_or_file)
    out.writerow(RESULT_FIELDS)
    out.writerows(_cells(r) for r in records)


_CAST = (str, str, str, float, int, int, float, float, float, float, lambda x: x == "true")


def read_results(path) -> list[ResultRecord]:
    """Inverse of write_results (io.py:225-238)."""
    with open(path, newline="") as fh:
        table = list(csv.reader(ln for ln in fh if not ln.startswith("#")))
    if not table or table[0] != RESULT_FIELDS:
        raise ParseError(path, 1, f"unexpected CSV header {table[0] if table else []}")
    return [ResultRecord(*(cast(x) for cast, x in zip(_CAST, row))) for row in table[1:]]
