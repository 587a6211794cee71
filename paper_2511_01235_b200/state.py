"""Device-resident solver state (mirror of reference state.py).

``cf`` / ``excess`` / ``height`` live in HBM (cf in the graph's residual
width, excess int64, height int32); the numpy attributes are downloaded
lazily in the reference's int64 layout.
"""

import ctypes

import numpy as np

from . import _lib as L
from .graph import BiCsrGraph


class _Handle:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr:
            try:
                L.load().mfx_state_free(self.ptr)
            except Exception:
                pass
            self.ptr = None


class SolverState:
    """cf / excess / height of one (source, sink) pair (state.py:16-27)."""

    def __init__(self, handle: _Handle, graph: BiCsrGraph, source: int, sink: int):
        self._h = handle
        self._graph = graph
        self.source = int(source)
        self.sink = int(sink)
        self.n_vertices = graph.n
        self._cache = None

    @property
    def handle(self):
        return self._h.ptr

    def _invalidate(self):
        self._cache = None

    def _arrays(self):
        if self._cache is None:
            g = self._graph
            cf = np.empty(g.m, np.int64)
            ex = np.empty(g.n, np.int64)
            h = np.empty(g.n, np.int64)
            L.check(L.load().mfx_state_download(self.handle, L.ptr64(cf), L.ptr64(ex), L.ptr64(h)))
            for arr in (cf, ex, h):  # snapshots of device memory: write through upload()
                arr.setflags(write=False)
            self._cache = (cf, ex, h)
        return self._cache

    @property
    def cf(self) -> np.ndarray:
        return self._arrays()[0]

    @property
    def excess(self) -> np.ndarray:
        return self._arrays()[1]

    @property
    def height(self) -> np.ndarray:
        return self._arrays()[2]

    def upload(self, cf=None, excess=None, height=None) -> None:
        """Overwrite any of the arrays (int64, reference layout)."""
        args = []
        for a, size in ((cf, self._graph.m), (excess, self.n_vertices), (height, self.n_vertices)):
            if a is None:
                args.append(None)
                continue
            a = L.as_i64(a)
            if a.shape != (size,):
                raise ValueError(f"array of shape {a.shape}, expected ({size},)")
            args.append(a)
        ptrs = [None if a is None else L.ptr64(a) for a in args]
        L.check(L.load().mfx_state_upload(self.handle, *ptrs))
        self._invalidate()

    def copy(self) -> "SolverState":
        """Device snapshot (state.py:25-27)."""
        out = L.vp()
        L.check(L.load().mfx_state_copy(self.handle, ctypes.byref(out)))
        return SolverState(_Handle(out), self._graph, self.source, self.sink)

    def assign(self, other: "SolverState") -> None:
        """Restore from a snapshot taken with :meth:`copy` (device copy)."""
        L.check(L.load().mfx_state_assign(self.handle, other.handle))
        self.source, self.sink = other.source, other.sink
        self._invalidate()

    def __repr__(self):
        return f"SolverState(n={self.n_vertices}, source={self.source}, sink={self.sink})"


def init_residuals(g: BiCsrGraph, source: int, sink: int) -> SolverState:
    """cf = cap0, excess = 0, height = 0 (state.py:30-39), on the device."""
    out = L.vp()
    L.check(L.load().mfx_state_create(g.handle, int(source), int(sink), ctypes.byref(out)))
    return SolverState(_Handle(out), g, source, sink)


def saturate_source(st: SolverState, g: BiCsrGraph) -> None:
    """Push the full residual of every source-outgoing slot (state.py:42-59)."""
    L.check(L.load().mfx_saturate_source(st.handle, g.handle))
    st._invalidate()


def _mask(st: SolverState, which: int) -> np.ndarray:
    out = np.empty(st.n_vertices, np.uint8)
    L.check(L.load().mfx_mask(st.handle, which, L.ptr8(out)))
    return out.astype(bool)


def active_mask(st: SolverState) -> np.ndarray:
    """Positive excess, height below n, not s/t (state.py:62-67)."""
    return _mask(st, 0)


def deficient_mask(st: SolverState) -> np.ndarray:
    """Negative excess, not s/t (state.py:70-75)."""
    return _mask(st, 1)
