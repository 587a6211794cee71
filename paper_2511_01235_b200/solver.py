"""Static max-flow on the device (mirror of reference solver.py).

``solve_static`` is one C-ABI call: init + source saturation + the persistent
solve kernel (global relabel -> push waves -> repair, until the device finds
no active vertex) + flow and cut.  The host never sees a round boundary
unless ``SolverParams.instrument`` is set, in which case the same kernel is
stepped one phase at a time so the callback can observe every round
(solver.py:219-241).
"""

import ctypes
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib as L
from .graph import BiCsrGraph
from .state import SolverState, active_mask, init_residuals, saturate_source


class SolverError(RuntimeError):
    """Operation ceiling exceeded or a terminal consistency check failed."""


L.register_error(L.MFX_SOLVER_ERROR, SolverError)

MODES = ("data", "topology")
SCHEDULES = ("waves", "async")  # device push-phase schedule (not a reference knob)


def operation_ceiling(n: int, m_original: int) -> int:
    """Bound on pushes + relabels for one solve (solver.py:37-44); the device
    saturates it to 64 bits."""
    return n * n + n * m_original + 4 * n * n * (n + m_original)


@dataclass
class SolverParams:
    """Solver knobs (solver.py:47-84).

    kernel_cycles / mode / instrument / deterministic have the reference
    meaning: ``deterministic=True`` runs each round's push and repair phases
    serially in worklist order on the device (the global relabel stays
    parallel; its heights are unique), so the final cf / excess / height are
    byte-identical to the reference's deterministic runs -- a parity and
    tracing mode, not a fast one.  ``threads`` sizes the reference's host
    thread pool and has no device meaning (accepted, unused).  Device knobs: ``max_waves`` (push waves per
    round before the next global relabel, 0 = until the active list drains),
    ``timeout_s`` (device watchdog; 0 = $MFX_TIMEOUT_S or 600 s), ``blocks_per_sm`` (persistent grid),
    ``bfs_local`` (BFS levels a CTA may run ahead on its own between two grid
    barriers of the global relabel; 0 = auto: 128 on short-row graphs, strict
    on long-row graphs; < 0 = strict level-synchronous BFS).
    """

    kernel_cycles: int = 0
    mode: str = "data"
    deterministic: bool = False
    threads: int = 0
    instrument: Optional[Callable] = None
    max_waves: int = 0
    timeout_s: float = 0.0
    blocks_per_sm: int = 0
    wave_mult: int = 0
    wave_add: int = 0
    schedule: str = "waves"
    async_budget: int = 0
    bfs_local: int = 0
    bfs_local_max: int = 0
    device_flags: int = 0

    def resolve_threads(self) -> int:
        return 1

    def resolve_kernel_cycles(self, g: BiCsrGraph) -> int:
        if self.kernel_cycles > 0:
            return self.kernel_cycles
        if self.kernel_cycles < 0:
            raise ValueError("kernel_cycles must be >= 1 (or 0 for the default)")
        return max(1, -(-g.m_original // g.n))

    def validate(self) -> None:
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")

    def to_c(self) -> L.Params:
        self.validate()
        if self.kernel_cycles < 0:
            raise ValueError("kernel_cycles must be >= 1 (or 0 for the default)")
        if self.schedule not in SCHEDULES:
            raise ValueError(f"schedule must be one of {SCHEDULES}, got {self.schedule!r}")
        return L.Params(int(self.kernel_cycles), MODES.index(self.mode), int(self.max_waves),
                        float(self.timeout_s), int(self.blocks_per_sm), int(self.device_flags),
                        int(self.wave_mult), int(self.wave_add),
                        SCHEDULES.index(self.schedule), int(self.async_budget),
                        int(self.bfs_local), int(self.bfs_local_max), int(bool(self.deterministic)),
                        0)


@dataclass
class CutCertificate:
    """A = {height == n} (source side), cut = sum of original A->B
    capacities (solver.py:87-105)."""

    a_mask: np.ndarray
    cut_capacity: int

    @property
    def partition_a(self) -> np.ndarray:
        return np.flatnonzero(self.a_mask)

    @property
    def partition_b(self) -> np.ndarray:
        return np.flatnonzero(~self.a_mask)


class _LazyCertificate(CutCertificate):
    """Certificate whose A mask is downloaded on first access."""

    def __init__(self, st: SolverState, cut: int):
        self._st = st
        self._mask = None
        self.cut_capacity = int(cut)

    @property
    def a_mask(self):
        if self._mask is None:
            out = np.empty(self._st.n_vertices, np.uint8)
            L.check(L.load().mfx_mask(self._st.handle, 2, L.ptr8(out)))
            self._mask = out.astype(bool)
        return self._mask

    @a_mask.setter
    def a_mask(self, v):
        self._mask = v


@dataclass
class FlowResult:
    """Reference FlowResult (solver.py:108-118) plus device statistics."""

    flow_value: int
    rounds: int
    phase_times: dict
    certificate: CutCertificate
    pushes: int = 0
    relabels: int = 0
    repairs: int = 0
    state: SolverState = None
    graph: BiCsrGraph = None
    device: dict = field(default_factory=dict)


def _result(r: L.Result, st: SolverState, g: BiCsrGraph) -> FlowResult:
    st._invalidate()
    g._invalidate()
    times = {"bfs": r.ns_bfs * 1e-9, "push": r.ns_push * 1e-9, "repair": r.ns_repair * 1e-9}
    return FlowResult(int(r.flow), int(r.rounds), times, _LazyCertificate(st, r.cut),
                      int(r.pushes), int(r.relabels), int(r.repairs), st, g, r.as_dict())


def backward_bfs(st: SolverState, g: BiCsrGraph) -> int:
    """Global relabel from the sink (solver.py:155-164); returns #reached."""
    reached = ctypes.c_int64()
    L.check(L.load().mfx_global_relabel(st.handle, g.handle, 0, ctypes.byref(reached)))
    st._invalidate()
    return int(reached.value)


def active_worklist(st: SolverState, mode: str = "data") -> np.ndarray:
    """Active vertices, or all but s/t in topology mode (solver.py:167-175)."""
    if mode == "topology":
        mask = np.ones(st.n_vertices, dtype=bool)
        mask[st.source] = False
        mask[st.sink] = False
        return np.flatnonzero(mask)
    return np.flatnonzero(active_mask(st))


def extract_certificate(st: SolverState, g: BiCsrGraph) -> CutCertificate:
    """Cut certificate of a terminated state (solver.py:178-184)."""
    if bool(active_mask(st).any()):
        raise SolverError("certificate requested before termination")
    cut = ctypes.c_int64()
    L.check(L.load().mfx_certificate(st.handle, g.handle, ctypes.byref(cut), None))
    return _LazyCertificate(st, cut.value)


def _validate_endpoints(g: BiCsrGraph, source: int, sink: int) -> None:
    if not 0 <= source < g.n:
        raise ValueError(f"source {source} out of range [0, {g.n})")
    if not 0 <= sink < g.n:
        raise ValueError(f"sink {sink} out of range [0, {g.n})")
    if source == sink:
        raise ValueError("source and sink must differ")


def _instrumented_rounds(st: SolverState, g: BiCsrGraph, p: L.Params, instrument,
                         dynamic: bool, round_base: int = 0, reset: bool = True) -> FlowResult:
    """Host-stepped variant of the device round loop (solver.py:204-241):
    static rounds relabel from {t} with nothing forbidden, dynamic ones from
    {t} U deficient with s forbidden.  ``round_base``/``reset``: continue the
    counters of an earlier device phase (push-pull's final pass)."""
    lib = L.load()
    active = ctypes.c_int64()
    r = L.Result()
    rnd = round_base
    first = 0x10 if reset else 0
    dyn = 1 if dynamic else 0
    while True:
        L.check(lib.mfx_step(g.handle, st.handle, ctypes.byref(p), 0 | first, dyn,
                             ctypes.byref(active), ctypes.byref(r)))
        first = 0
        st._invalidate()
        instrument(st, g, rnd, "bfs")
        if active.value == 0:
            break
        L.check(lib.mfx_step(g.handle, st.handle, ctypes.byref(p), 1, dyn, None,
                             ctypes.byref(r)))
        st._invalidate()
        instrument(st, g, rnd, "repair")
        rnd += 1
    L.check(lib.mfx_step(g.handle, st.handle, ctypes.byref(p), 2, dyn, None, ctypes.byref(r)))
    res = _result(r, st, g)
    if res.flow_value != res.certificate.cut_capacity:
        raise SolverError(f"flow {res.flow_value} does not match cut capacity "
                          f"{res.certificate.cut_capacity}")
    return res


def solve_static(g: BiCsrGraph, source: int, sink: int,
                 params: SolverParams | None = None) -> FlowResult:
    """Maximum flow on a static graph (solver.py:253-283), solved on the GPU.

    Returns the flow value with the cut certificate whose capacity equals it;
    the terminal device state is attached for chaining into
    :func:`~paper_2511_01235_b200.dynamic.solve_dynamic`.
    """
    params = params or SolverParams()
    params.validate()
    _validate_endpoints(g, source, sink)
    p = params.to_c()
    st = init_residuals(g, source, sink)
    if params.instrument is not None:
        saturate_source(st, g)
        return _instrumented_rounds(st, g, p, params.instrument, dynamic=False)
    r = L.Result()
    L.check(L.load().mfx_solve_static(g.handle, st.handle, ctypes.byref(p), ctypes.byref(r)))
    return _result(r, st, g)


def resolve_static(g: BiCsrGraph, st: SolverState, params: SolverParams | None = None) -> FlowResult:
    """Static solve into an existing state object (no allocation): the GPU
    static re-solve used as the dynamic solver's comparison point."""
    params = params or SolverParams()
    p = params.to_c()
    if st.source == st.sink:
        raise ValueError("source and sink must differ")
    r = L.Result()
    L.check(L.load().mfx_solve_static(g.handle, st.handle, ctypes.byref(p), ctypes.byref(r)))
    return _result(r, st, g)
