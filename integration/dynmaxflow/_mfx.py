"""Optional B200 backend for the reference package ``dynmaxflow``.

This is the file a dynmaxflow maintainer adds as ``dynmaxflow/_mfx.py``
(INTEGRATION.md).  With ``DYNMAXFLOW_MFX_LIB=/path/to/libmfx.so`` set, the
two guarded call sites route to it:

* ``solver.solve_static``   (solver.py:253)  -> ``mfx_solve_static``
* ``dynamic.solve_dynamic`` (dynamic.py:146) -> ``mfx_solve_dynamic``

It speaks only the C-ABI of include/mfx.h through ctypes (plain pointers,
int64 arrays) and returns the reference's own ``FlowResult`` /
``CutCertificate`` objects.  Reference semantics are kept: the solvers
mutate ``SolverState`` arrays and ``g.cap0`` in place (the device results
are written back into the caller's numpy arrays), errors raise the
reference's exception classes with the reference's messages, and the
returned state chains into the next ``solve_dynamic``.  The device handles
ride on the objects as ``g._mfx`` / ``st._mfx``; an object without one
(e.g. a ``copy()``) is uploaded from its host arrays on first use.
"""
import ctypes
import os

import numpy as np

from .graph import GraphError
from .solver import CutCertificate, FlowResult, SolverError, SolverParams, _validate_endpoints
from .state import init_residuals

_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_vp = ctypes.c_void_p


class _Params(ctypes.Structure):  # mfx_params
    _fields_ = [("kernel_cycles", ctypes.c_int64), ("mode", ctypes.c_int32),
                ("max_waves", ctypes.c_int32), ("timeout_s", ctypes.c_double),
                ("blocks_per_sm", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("wave_mult", ctypes.c_int32), ("wave_add", ctypes.c_int32),
                ("schedule", ctypes.c_int32), ("async_budget", ctypes.c_int32),
                ("bfs_local", ctypes.c_int32), ("bfs_local_max", ctypes.c_int32),
                ("deterministic", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class _Result(ctypes.Structure):  # mfx_result
    _fields_ = [(k, ctypes.c_int64) for k in (
        "flow", "cut", "rounds", "pushes", "relabels", "repairs", "bfs_levels", "waves",
        "bytes_alg", "updates")] + \
        [(k, ctypes.c_double) for k in (
            "ns_bfs", "ns_push", "ns_repair", "ms_update", "ms_solve", "ms_total")] + \
        [("status", ctypes.c_int32), ("launches", ctypes.c_int32),
         ("async_items", ctypes.c_int64), ("bfs_epochs", ctypes.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(os.environ["DYNMAXFLOW_MFX_LIB"])
        L.mfx_last_error.restype = ctypes.c_char_p
        L.mfx_graph_from_bicsr.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, _i64p, _i64p,
                                           _i64p, _u8p, ctypes.c_int, ctypes.c_int,
                                           ctypes.POINTER(_vp)]
        L.mfx_graph_download.argtypes = [_vp, _i64p, _i64p, _i64p, _i64p, _i64p, _u8p]
        L.mfx_graph_free.argtypes = [_vp]
        L.mfx_graph_free.restype = None
        L.mfx_state_create.argtypes = [_vp, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(_vp)]
        L.mfx_state_upload.argtypes = [_vp, _i64p, _i64p, _i64p]
        L.mfx_state_download.argtypes = [_vp, _i64p, _i64p, _i64p]
        L.mfx_state_free.argtypes = [_vp]
        L.mfx_state_free.restype = None
        L.mfx_solve_static.argtypes = [_vp, _vp, ctypes.POINTER(_Params),
                                       ctypes.POINTER(_Result)]
        L.mfx_solve_dynamic.argtypes = [_vp, _vp, ctypes.c_int64, _i64p, _i64p, _i64p,
                                        ctypes.POINTER(_Params), ctypes.POINTER(_Result)]
        _lib = L
    return _lib


def _errors():
    from .dynamic import BatchError  # dynamic imports solver: resolve lazily
    return {1: GraphError, 2: BatchError, 3: SolverError, 4: ValueError}


def _check(rc):
    if rc:
        raise _errors().get(rc, RuntimeError)(lib().mfx_last_error().decode())


def _p(a, t=_i64p):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(t)


class _Handle:
    def __init__(self, ptr, free):
        self.ptr, self._free = ptr, free

    def __del__(self):
        try:
            self._free(self.ptr)
        except Exception:
            pass


def _graph(g):
    """Device copy of a reference BiCsrGraph (cached on the object)."""
    h = getattr(g, "_mfx", None)
    if h is None:
        out = _vp()
        arrs = [np.ascontiguousarray(x, dtype=np.int64) for x in (g.offsets, g.adj, g.rev, g.cap0)]
        orig = np.ascontiguousarray(g.is_original, dtype=np.uint8)
        _check(lib().mfx_graph_from_bicsr(g.n, g.m, *(_p(a) for a in arrs), _p(orig, _u8p),
                                          0, 0, ctypes.byref(out)))
        h = g._mfx = _Handle(out, lib().mfx_graph_free)
    return h.ptr


def _state(st, g):
    """Device copy of a reference SolverState (cached on the object)."""
    h = getattr(st, "_mfx", None)
    gp = _graph(g)
    if h is None or h.graph != gp:  # new object, or used with another graph object
        out = _vp()
        _check(lib().mfx_state_create(gp, st.source, st.sink, ctypes.byref(out)))
        h = st._mfx = _Handle(out, lib().mfx_state_free)
        h.graph = gp
        _check(lib().mfx_state_upload(out, _p(st.cf), _p(st.excess), _p(st.height)))
    return h.ptr


def _params(params: SolverParams) -> _Params:
    p = _Params()
    p.kernel_cycles = params.kernel_cycles  # 0 = the reference default rule on the device
    p.mode = 0 if params.mode == "data" else 1
    p.deterministic = int(bool(params.deterministic))
    return p


def _write_back(st, g, dev_state):
    """Reference semantics: the caller's arrays hold the solved state."""
    _check(lib().mfx_state_download(dev_state, _p(st.cf), _p(st.excess), _p(st.height)))
    _check(lib().mfx_graph_download(_graph(g), None, None, None, None, _p(g.cap0), None))


def _result(r: _Result, st, g) -> FlowResult:
    cert = CutCertificate(st.height == st.n_vertices, int(r.cut))
    times = {"bfs": r.ns_bfs * 1e-9, "push": r.ns_push * 1e-9, "repair": r.ns_repair * 1e-9}
    return FlowResult(int(r.flow), int(r.rounds), times, cert, int(r.pushes), int(r.relabels),
                      int(r.repairs), st, g)


def solve_static(g, source, sink, params=None) -> FlowResult:
    params = params or SolverParams()
    params.validate()
    _validate_endpoints(g, source, sink)
    params.resolve_kernel_cycles(g)  # same ValueError as the reference for kernel_cycles < 0
    st = init_residuals(g, source, sink)
    dev = _state(st, g)
    r = _Result()
    _check(lib().mfx_solve_static(_graph(g), dev, ctypes.byref(_params(params)), ctypes.byref(r)))
    _write_back(st, g, dev)
    return _result(r, st, g)


def solve_dynamic(st, g, batch, params=None) -> FlowResult:
    params = params or SolverParams()
    params.validate()
    params.resolve_kernel_cycles(g)
    dev = _state(st, g)
    us, vs, caps = (np.ascontiguousarray(a, dtype=np.int64)
                    for a in (batch.us, batch.vs, batch.new_caps))
    r = _Result()
    _check(lib().mfx_solve_dynamic(_graph(g), dev, len(us), _p(us), _p(vs), _p(caps),
                                   ctypes.byref(_params(params)), ctypes.byref(r)))
    _write_back(st, g, dev)
    return _result(r, st, g)
