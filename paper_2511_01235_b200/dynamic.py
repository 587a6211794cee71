"""Incremental max-flow after a batch of capacity updates (mirror of
reference dynamic.py).

``solve_dynamic`` is one C-ABI call: the O(k + deg s) batch pre-phase
(validate, apply, reverse over-capacity flow, move endpoint excess,
re-saturate the source; csrc/state.cu) and the persistent solve kernel with
the sink and every deficient vertex as height-0 bases (dynamic.py:146-175).
``st`` and ``g``'s capacities are mutated on the device, so batches chain by
passing ``res.state`` / ``res.graph`` back in.
"""

import ctypes
from dataclasses import dataclass
from typing import Iterable

import numpy as np

from . import _lib as L
from .graph import BiCsrGraph, EdgeListGraph
from .solver import (FlowResult, SolverError, SolverParams, _instrumented_rounds, _result)
from .state import SolverState


class BatchError(ValueError):
    """Update batch references a missing edge or contains duplicates."""


L.register_error(L.MFX_BATCH_ERROR, BatchError)


@dataclass(frozen=True)
class UpdateBatch:
    """Edge re-weightings (u, v, new_cap) applied atomically as one batch
    (dynamic.py:39-60)."""

    us: np.ndarray
    vs: np.ndarray
    new_caps: np.ndarray

    @classmethod
    def from_updates(cls, updates: Iterable[tuple[int, int, int]]) -> "UpdateBatch":
        rows = list(updates)
        cols = [np.fromiter((r[c] for r in rows), dtype=np.int64, count=len(rows))
                for c in range(3)]
        return cls(*cols)

    def __len__(self) -> int:
        return int(self.us.shape[0])

    def updates(self):
        for u, v, c in zip(self.us.tolist(), self.vs.tolist(), self.new_caps.tolist()):
            yield u, v, c

    def arrays(self):
        return L.as_i64(self.us), L.as_i64(self.vs), L.as_i64(self.new_caps)


def apply_updates(st: SolverState, g: BiCsrGraph, batch: UpdateBatch) -> None:
    """Fold new capacities into the residuals on the device
    (dynamic.py:91-111); validation happens before any write."""
    us, vs, cs = batch.arrays()
    L.check(L.load().mfx_apply_updates(g.handle, st.handle, us.size, L.ptr64(us), L.ptr64(vs),
                                       L.ptr64(cs)))
    st._invalidate()
    g._invalidate()


def recompute_excess(st: SolverState, g: BiCsrGraph) -> None:
    """excess from the constructed flow, O(n + S) on the device
    (dynamic.py:114-116)."""
    L.check(L.load().mfx_recompute_excess(st.handle, g.handle))
    st._invalidate()


def dynamic_prephase(st: SolverState, g: BiCsrGraph, batch: UpdateBatch) -> None:
    """apply_updates + recompute_excess + saturate_source as the fused O(k)
    device pre-phase of solve_dynamic (bit-identical result)."""
    us, vs, cs = batch.arrays()
    L.check(L.load().mfx_dynamic_prephase(g.handle, st.handle, us.size, L.ptr64(us),
                                          L.ptr64(vs), L.ptr64(cs)))
    st._invalidate()
    g._invalidate()


def backward_bfs_dynamic(st: SolverState, g: BiCsrGraph) -> int:
    """Global relabel with the sink and every deficient vertex as bases and
    the source pinned at n (dynamic.py:125-133); returns #reached."""
    reached = ctypes.c_int64()
    L.check(L.load().mfx_global_relabel(st.handle, g.handle, 1, ctypes.byref(reached)))
    st._invalidate()
    return int(reached.value)


def solve_dynamic(st: SolverState, g: BiCsrGraph, batch: UpdateBatch,
                  params: SolverParams | None = None) -> FlowResult:
    """Recompute the max flow after a capacity-update batch
    (dynamic.py:146-175).  Mutates ``st`` and ``g``'s capacities in place."""
    params = params or SolverParams()
    params.validate()
    p = params.to_c()
    if params.instrument is not None:
        dynamic_prephase(st, g, batch)
        return _instrumented_rounds(st, g, p, params.instrument, dynamic=True)
    us, vs, cs = batch.arrays()
    r = L.Result()
    L.check(L.load().mfx_solve_dynamic(g.handle, st.handle, us.size, L.ptr64(us), L.ptr64(vs),
                                       L.ptr64(cs), ctypes.byref(p), ctypes.byref(r)))
    return _result(r, st, g)


def solve_dynamic_pushpull(st: SolverState, g: BiCsrGraph, batch: UpdateBatch,
                           params: SolverParams | None = None) -> FlowResult:
    """Dynamic recompute with the push and pull pipelines of O2
    (dynamic.py:292-377): the prior terminal heights give the cut (A =
    {h == n}); after the batch every A->B residual is pushed across, the B
    side pushes overflow to the sink and its deficits while the A side pulls
    its deficits from the source and its overflow (region-restricted, one
    device round loop for both), then ordinary rounds connect what is left.
    Same flow value as :func:`solve_dynamic`."""
    params = params or SolverParams()
    params.validate()
    p = params.to_c()
    us, vs, cs = batch.arrays()
    r = L.Result()
    if params.instrument is not None:
        # the reference hands instrument to the final ordinary pass only
        # (dynamic.py:366-369): device pipelines, then host-stepped rounds
        L.check(L.load().mfx_pushpull_regions(g.handle, st.handle, us.size, L.ptr64(us),
                                              L.ptr64(vs), L.ptr64(cs), ctypes.byref(p),
                                              ctypes.byref(r)))
        st._invalidate()
        g._invalidate()
        return _instrumented_rounds(st, g, p, params.instrument, dynamic=True,
                                    round_base=int(r.rounds), reset=False)
    L.check(L.load().mfx_solve_dynamic_pushpull(g.handle, st.handle, us.size, L.ptr64(us),
                                                L.ptr64(vs), L.ptr64(cs), ctypes.byref(p),
                                                ctypes.byref(r)))
    return _result(r, st, g)


def solve_dynamic_device(st: SolverState, g: BiCsrGraph, k: int, d_us: int, d_vs: int,
                         d_caps: int, params: SolverParams | None = None) -> FlowResult:
    """solve_dynamic with the batch already resident in device memory (raw
    int64 device pointers)."""
    params = params or SolverParams()
    p = params.to_c()
    r = L.Result()
    L.check(L.load().mfx_solve_dynamic_device(g.handle, st.handle, int(k), d_us, d_vs, d_caps,
                                              ctypes.byref(p), ctypes.byref(r)))
    return _result(r, st, g)


def updated_edge_list(g: BiCsrGraph, batch: UpdateBatch) -> EdgeListGraph:
    """The updated graph as a fresh normalized edge list (dynamic.py:380-387);
    ``g`` is left untouched.  The batch is validated like apply_updates."""
    gg = g.copy()
    us, vs, cs = batch.arrays()
    L.check(L.load().mfx_apply_updates(gg.handle, None, us.size, L.ptr64(us), L.ptr64(vs),
                                       L.ptr64(cs)))
    gg._invalidate()
    keep = g.is_original
    return EdgeListGraph(g.n, g.src[keep].copy(), g.adj[keep].copy(), gg.cap0[keep].copy())


__all__ = ["BatchError", "UpdateBatch", "apply_updates", "recompute_excess", "dynamic_prephase",
           "backward_bfs_dynamic", "solve_dynamic", "solve_dynamic_device", "solve_dynamic_pushpull", "updated_edge_list",
           "SolverError"]
