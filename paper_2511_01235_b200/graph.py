"""Bi-CSR graph on the device (mirror of reference graph.py).

``build_bicsr`` runs the GPU builder (csrc/build.cu) and returns a
:class:`BiCsrGraph` whose arrays live in HBM; the numpy attributes
(``offsets``, ``adj``, ``src``, ``rev``, ``cap0``, ``is_original``) are
downloaded lazily in the reference's int64 layout, so reference-style code
(and the reference's own verifiers) can read them unchanged.
"""

import ctypes
from dataclasses import dataclass
from typing import Iterable, Iterator

import numpy as np

from . import _lib as L


class GraphError(ValueError):
    """Malformed graph input (bad vertex id, negative capacity, ...)."""


L.register_error(L.MFX_GRAPH_ERROR, GraphError)


@dataclass(frozen=True)
class EdgeListGraph:
    """Directed capacitated edge list (reference graph.py:19-61); may hold
    self-loops and parallel edges, which build_bicsr normalises away."""

    n: int
    us: np.ndarray
    vs: np.ndarray
    caps: np.ndarray

    @classmethod
    def from_edges(cls, n: int, edges: Iterable[tuple[int, int, int]]) -> "EdgeListGraph":
        rows = list(edges)
        cols = [np.fromiter((r[c] for r in rows), dtype=np.int64, count=len(rows))
                for c in range(3)]
        return cls(n, *cols)

    @property
    def m(self) -> int:
        return int(self.us.shape[0])

    def edges(self) -> Iterator[tuple[int, int, int]]:
        for u, v, c in zip(self.us.tolist(), self.vs.tolist(), self.caps.tolist()):
            yield u, v, c

    def validate(self) -> None:
        """Same checks and messages as the reference (graph.py:48-61); the
        GPU builder repeats them on the device."""
        if self.n <= 0:
            raise GraphError(f"vertex count must be positive, got {self.n}")
        for label, arr in (("source", self.us), ("target", self.vs)):
            bad = np.flatnonzero((arr < 0) | (arr >= self.n))
            if bad.size:
                i = int(bad[0])
                raise GraphError(f"edge {i}: {label} vertex {int(arr[i])} out of range [0, {self.n})")
        neg = np.flatnonzero(self.caps < 0)
        if neg.size:
            i = int(neg[0])
            raise GraphError(f"edge {i}: negative capacity {int(self.caps[i])}")


@dataclass
class BuildDiagnostics:
    self_loops_dropped: int = 0
    parallel_edges_merged: int = 0
    reverse_stubs_added: int = 0


class _Handle:
    """Owns one mfx_graph*."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr:
            try:
                L.load().mfx_graph_free(self.ptr)
            except Exception:
                pass
            self.ptr = None


class BiCsrGraph:
    """Device-resident Bi-CSR (reference graph.py:71-123).

    The topology is immutable and shared by :meth:`copy`; ``cap0`` is private
    per copy and is what :func:`solve_dynamic` mutates on the device.
    """

    def __init__(self, handle: _Handle):
        self._h = handle
        info = L.GraphInfo()
        L.check(L.load().mfx_graph_info_get(handle.ptr, ctypes.byref(info)))
        self.n = int(info.n)
        self.m = int(info.S)
        self._m_original = int(info.m_original)
        self.cap_bytes = int(info.cap_bytes)
        self.device = int(info.device)
        self.diagnostics = BuildDiagnostics(int(info.self_loops_dropped),
                                            int(info.parallel_edges_merged),
                                            int(info.reverse_stubs_added))
        self._topo_cache = None   # shared across copies (immutable)
        self._cap0_cache = None
        self._keys = None

    # -- device handle -------------------------------------------------------
    @property
    def handle(self):
        return self._h.ptr

    def _invalidate(self):
        self._cap0_cache = None

    # -- lazily downloaded arrays (reference int64 layout) -------------------
    def _topology(self):
        if self._topo_cache is None:
            off = np.empty(self.n + 1, np.int64)
            adj = np.empty(self.m, np.int64)
            src = np.empty(self.m, np.int64)
            rev = np.empty(self.m, np.int64)
            orig = np.empty(self.m, np.uint8)
            L.check(L.load().mfx_graph_download(self.handle, L.ptr64(off), L.ptr64(adj),
                                                L.ptr64(src), L.ptr64(rev), None, L.ptr8(orig)))
            self._topo_cache = {"offsets": off, "adj": adj, "src": src, "rev": rev,
                                "is_original": orig.astype(bool)}
            for arr in self._topo_cache.values():
                arr.setflags(write=False)
        return self._topo_cache

    @property
    def offsets(self):
        return self._topology()["offsets"]

    @property
    def adj(self):
        return self._topology()["adj"]

    @property
    def src(self):
        return self._topology()["src"]

    @property
    def rev(self):
        return self._topology()["rev"]

    @property
    def is_original(self):
        return self._topology()["is_original"]

    @property
    def cap0(self):
        """Current capacities: a read-only downloaded snapshot (the device
        copy is the truth; write through :meth:`set_cap0`)."""
        if self._cap0_cache is None:
            c = np.empty(self.m, np.int64)
            L.check(L.load().mfx_graph_download(self.handle, None, None, None, None,
                                                L.ptr64(c), None))
            c.setflags(write=False)  # a snapshot: in-place writes would be lost, so they raise
            self._cap0_cache = c
        return self._cap0_cache

    def set_cap0(self, cap0) -> None:
        c = L.as_i64(cap0)
        if c.shape != (self.m,):
            raise ValueError(f"cap0 must have shape ({self.m},)")
        L.check(L.load().mfx_graph_set_cap0(self.handle, L.ptr64(c)))
        self._invalidate()

    @property
    def m_original(self) -> int:
        return self._m_original

    def sorted_keys(self) -> np.ndarray:
        """Ascending ``u * n + v`` slot keys (graph.py:95-99)."""
        if self._keys is None:
            self._keys = self.src * np.int64(self.n) + self.adj
        return self._keys

    def edge_indices(self, us, vs) -> np.ndarray:
        """Slot indices for directed pairs; -1 where absent (graph.py:101-108),
        looked up on the device."""
        us, vs = L.as_i64(us), L.as_i64(vs)
        shape = np.broadcast(us, vs).shape
        us, vs = (np.ascontiguousarray(np.broadcast_to(a, shape).ravel()) for a in (us, vs))
        out = np.empty(us.size, np.int64)
        if us.size:
            L.check(L.load().mfx_edge_indices(self.handle, us.size, L.ptr64(us), L.ptr64(vs),
                                              L.ptr64(out)))
        return out.reshape(shape)

    def edge_index(self, u: int, v: int) -> int:
        return int(self.edge_indices(np.array([u]), np.array([v]))[0])

    def to_edge_list(self) -> EdgeListGraph:
        """Normalized edge list: original slots only (graph.py:113-117)."""
        keep = self.is_original
        return EdgeListGraph(self.n, self.src[keep].copy(), self.adj[keep].copy(),
                             self.cap0[keep].copy())

    def copy(self) -> "BiCsrGraph":
        """Shares the device topology, private capacities (graph.py:119-123)."""
        out = L.vp()
        L.check(L.load().mfx_graph_copy(self.handle, ctypes.byref(out)))
        g = BiCsrGraph(_Handle(out))
        g._topo_cache = self._topo_cache
        g._keys = self._keys
        return g

    def __repr__(self):
        return (f"BiCsrGraph(n={self.n}, m={self.m}, m_original={self.m_original}, "
                f"cap_bytes={self.cap_bytes}, device={self.device})")


def build_bicsr(g: EdgeListGraph, device: int = 0, wide: bool = False) -> BiCsrGraph:
    """Normalise an edge list and build the Bi-CSR on the GPU
    (reference graph.py:126-174; arrays bit-identical to the reference's).

    ``wide`` forces int64 residual storage (otherwise int32 whenever every
    pair capacity sum fits)."""
    us, vs, caps = L.as_i64(g.us), L.as_i64(g.vs), L.as_i64(g.caps)
    out = L.vp()
    L.check(L.load().mfx_graph_build(int(g.n), us.size, L.ptr64(us), L.ptr64(vs), L.ptr64(caps),
                                     device, int(bool(wide)), ctypes.byref(out)))
    return BiCsrGraph(_Handle(out))


def build_bicsr_device(n: int, d_us: int, d_vs: int, d_caps: int, m: int, device: int = 0,
                       wide: bool = False) -> BiCsrGraph:
    """Build from edge arrays already resident in device memory (raw
    pointers, e.g. ``torch.Tensor.data_ptr()``)."""
    out = L.vp()
    L.check(L.load().mfx_graph_build_device(int(n), int(m), d_us, d_vs, d_caps, device,
                                            int(bool(wide)), ctypes.byref(out)))
    return BiCsrGraph(_Handle(out))


def upload_bicsr(n, offsets, adj, rev, cap0, is_original, device: int = 0,
                 wide: bool = False) -> BiCsrGraph:
    """Upload a reference-layout Bi-CSR as-is (parity tests)."""
    off, a, r, c = (L.as_i64(x) for x in (offsets, adj, rev, cap0))
    o = np.ascontiguousarray(np.asarray(is_original).astype(np.uint8))
    out = L.vp()
    L.check(L.load().mfx_graph_from_bicsr(int(n), a.size, L.ptr64(off), L.ptr64(a), L.ptr64(r),
                                          L.ptr64(c), L.ptr8(o), device, int(bool(wide)),
                                          ctypes.byref(out)))
    return BiCsrGraph(_Handle(out))


def reverse_edge(g: BiCsrGraph, i: int) -> int:
    """Paired reverse slot; an involution (graph.py:177-181)."""
    if not 0 <= i < g.m:
        raise GraphError(f"edge index {i} out of range [0, {g.m})")
    return int(g.rev[i])
