"""ctypes binding of libmfx.so (include/mfx.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2511_01235_b200/csrc``).  There is no fallback: if the shared object is
missing or no CUDA device is visible, every solver entry point raises.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# $MFX_LIB_PATH: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("MFX_LIB_PATH") or os.path.join(_HERE, "_lib", "libmfx.so")

MFX_OK = 0
MFX_GRAPH_ERROR = 1
MFX_BATCH_ERROR = 2
MFX_SOLVER_ERROR = 3
MFX_VALUE_ERROR = 4
MFX_CUDA_ERROR = 5
MFX_TIMEOUT = 6
MFX_PARSE_ERROR = 7

i64 = ctypes.c_int64
i32 = ctypes.c_int32
p_i64 = ctypes.POINTER(ctypes.c_int64)
p_u8 = ctypes.POINTER(ctypes.c_uint8)
vp = ctypes.c_void_p


class GraphInfo(ctypes.Structure):
    _fields_ = [("n", i64), ("S", i64), ("m_original", i64), ("self_loops_dropped", i64),
                ("parallel_edges_merged", i64), ("reverse_stubs_added", i64),
                ("cap_bytes", i32), ("device", i32)]


class Params(ctypes.Structure):
    _fields_ = [("kernel_cycles", i64), ("mode", i32), ("max_waves", i32),
                ("timeout_s", ctypes.c_double), ("blocks_per_sm", i32), ("flags", i32),
                ("wave_mult", i32), ("wave_add", i32), ("schedule", i32),
                ("async_budget", i32), ("bfs_local", i32), ("bfs_local_max", i32),
                ("deterministic", i32), ("reserved", i32)]


class Result(ctypes.Structure):
    _fields_ = [("flow", i64), ("cut", i64), ("rounds", i64), ("pushes", i64),
                ("relabels", i64), ("repairs", i64), ("bfs_levels", i64), ("waves", i64),
                ("bytes_alg", i64), ("updates", i64), ("ns_bfs", ctypes.c_double),
                ("ns_push", ctypes.c_double), ("ns_repair", ctypes.c_double),
                ("ms_update", ctypes.c_double), ("ms_solve", ctypes.c_double),
                ("ms_total", ctypes.c_double), ("status", i32), ("launches", i32),
                ("async_items", i64), ("bfs_epochs", i64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class VerifyReport(ctypes.Structure):
    _fields_ = [(k, i64) for k in (
        "negative_cf", "pair_violations", "excess_mismatch", "excess_sum", "active_vertices",
        "unsaturated_ab", "loaded_ba", "cut_capacity", "flow_at_bases", "source_in_b",
        "sink_in_a", "first_bad_slot")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# exported symbol -> (restype, argtypes); tests check every declaration in
# include/mfx.h is exported.
SIGNATURES = {
    "mfx_version": (ctypes.c_int, []),
    "mfx_last_error": (ctypes.c_char_p, []),
    "mfx_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "mfx_launch_count": (i64, []),
    "mfx_graph_build": (ctypes.c_int, [i64, i64, p_i64, p_i64, p_i64, ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(vp)]),
    "mfx_graph_build_device": (ctypes.c_int, [i64, i64, vp, vp, vp, ctypes.c_int, ctypes.c_int,
                                              ctypes.POINTER(vp)]),
    "mfx_graph_from_bicsr": (ctypes.c_int, [i64, i64, p_i64, p_i64, p_i64, p_i64, p_u8,
                                            ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]),
    "mfx_graph_info_get": (ctypes.c_int, [vp, ctypes.POINTER(GraphInfo)]),
    "mfx_graph_download": (ctypes.c_int, [vp, p_i64, p_i64, p_i64, p_i64, p_i64, p_u8]),
    "mfx_graph_copy": (ctypes.c_int, [vp, ctypes.POINTER(vp)]),
    "mfx_graph_set_cap0": (ctypes.c_int, [vp, p_i64]),
    "mfx_edge_indices": (ctypes.c_int, [vp, i64, p_i64, p_i64, p_i64]),
    "mfx_graph_free": (None, [vp]),
    "mfx_state_create": (ctypes.c_int, [vp, i64, i64, ctypes.POINTER(vp)]),
    "mfx_state_copy": (ctypes.c_int, [vp, ctypes.POINTER(vp)]),
    "mfx_state_assign": (ctypes.c_int, [vp, vp]),
    "mfx_state_upload": (ctypes.c_int, [vp, p_i64, p_i64, p_i64]),
    "mfx_state_download": (ctypes.c_int, [vp, p_i64, p_i64, p_i64]),
    "mfx_state_free": (None, [vp]),
    "mfx_saturate_source": (ctypes.c_int, [vp, vp]),
    "mfx_mask": (ctypes.c_int, [vp, ctypes.c_int, p_u8]),
    "mfx_global_relabel": (ctypes.c_int, [vp, vp, ctypes.c_int, p_i64]),
    "mfx_solve_static": (ctypes.c_int, [vp, vp, ctypes.POINTER(Params), ctypes.POINTER(Result)]),
    "mfx_solve_dynamic": (ctypes.c_int, [vp, vp, i64, p_i64, p_i64, p_i64,
                                         ctypes.POINTER(Params), ctypes.POINTER(Result)]),
    "mfx_solve_dynamic_device": (ctypes.c_int, [vp, vp, i64, vp, vp, vp,
                                                ctypes.POINTER(Params), ctypes.POINTER(Result)]),
    "mfx_solve_dynamic_pushpull": (ctypes.c_int, [vp, vp, i64, p_i64, p_i64, p_i64,
                                                  ctypes.POINTER(Params), ctypes.POINTER(Result)]),
    "mfx_pushpull_regions": (ctypes.c_int, [vp, vp, i64, p_i64, p_i64, p_i64,
                                            ctypes.POINTER(Params), ctypes.POINTER(Result)]),
    "mfx_apply_updates": (ctypes.c_int, [vp, vp, i64, p_i64, p_i64, p_i64]),
    "mfx_dynamic_prephase": (ctypes.c_int, [vp, vp, i64, p_i64, p_i64, p_i64]),
    "mfx_recompute_excess": (ctypes.c_int, [vp, vp]),
    "mfx_step": (ctypes.c_int, [vp, vp, ctypes.POINTER(Params), ctypes.c_int, ctypes.c_int,
                                p_i64, ctypes.POINTER(Result)]),
    "mfx_certificate": (ctypes.c_int, [vp, vp, p_i64, p_u8]),
    "mfx_verify": (ctypes.c_int, [vp, vp, ctypes.POINTER(VerifyReport)]),
    "mfx_bench_barrier": (ctypes.c_int, [vp, vp, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_double)]),
    "mfx_trace_fetch": (ctypes.c_int, [vp, vp, ctypes.POINTER(ctypes.c_uint64), i64, p_i64]),
    "mfx_reached_list": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_int32), i64, p_i64]),
    "mfx_bench_chase": (ctypes.c_int, [vp, i64, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
    "mfx_sample_batch": (ctypes.c_int, [vp, i64, i64, i64, i64, ctypes.c_uint64, ctypes.c_double,
                                        p_i64, p_i64, p_i64, p_i64]),
    "mfx_transfer_bytes": (ctypes.c_int, [i64, p_i64, p_i64]),
    "mfx_host_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(vp)]),
    "mfx_host_free": (ctypes.c_int, [vp]),
    "mfx_graph_stream": (vp, [vp]),
    # vertex-range partition
    "mfx_part_create": (ctypes.c_int, [i64, ctypes.c_int, ctypes.c_int, p_i64, i64, vp, vp, vp,
                                       i64, i64, ctypes.c_int, ctypes.POINTER(vp)]),
    "mfx_part_create_host": (ctypes.c_int, [i64, ctypes.c_int, ctypes.c_int, p_i64, i64, p_i64,
                                            p_i64, p_i64, i64, i64, ctypes.c_int,
                                            ctypes.POINTER(vp)]),
    "mfx_part_free": (None, [vp]),
    "mfx_part_info": (ctypes.c_int, [vp, p_i64]),
    "mfx_part_export": (ctypes.c_int, [vp, vp, i64, p_i64]),
    "mfx_part_attach": (ctypes.c_int, [vp, ctypes.c_int, vp, i64]),
    "mfx_part_attach_local": (ctypes.c_int, [vp, vp]),
    "mfx_part_phase": (ctypes.c_int, [vp, ctypes.c_int, p_i64, p_i64]),
    "mfx_part_sync": (ctypes.c_int, [vp]),
    "mfx_part_stage_batch": (ctypes.c_int, [vp, i64, p_i64, p_i64, p_i64, p_i64, i64]),
    "mfx_part_download": (ctypes.c_int, [vp, p_i64, p_i64, p_i64, p_i64, p_i64, p_u8, p_i64,
                                         p_i64]),
    "mfx_part_sample_batch": (ctypes.c_int, [vp, i64, i64, ctypes.c_uint64, ctypes.c_double,
                                             p_i64, p_i64, p_i64, p_i64]),
    "mfx_io_parse_graph": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(vp)]),
    "mfx_io_parse_updates": (ctypes.c_int, [ctypes.c_char_p, i64, ctypes.POINTER(vp)]),
    "mfx_io_parse_edge_list": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(vp)]),
    "mfx_edges_info": (ctypes.c_int, [vp, p_i64]),
    "mfx_edges_get": (ctypes.c_int, [vp, p_i64, p_i64, p_i64]),
    "mfx_edges_free": (None, [vp]),
    "mfx_io_error_line": (i64, []),
    "mfx_io_write_graph": (ctypes.c_int, [ctypes.c_char_p, i64, i64, i64, i64, p_i64, p_i64,
                                          p_i64]),
    "mfx_io_write_updates": (ctypes.c_int, [ctypes.c_char_p, i64, p_i64, p_i64, p_i64]),
    "mfx_rmat_device": (ctypes.c_int, [ctypes.c_int, i64, ctypes.c_uint64, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_int, vp, vp,
                                       vp, p_i64, p_i64]),
    "mfx_part_bounds_device": (ctypes.c_int, [i64, i64, vp, vp, ctypes.c_int, ctypes.c_int,
                                              p_i64]),
}

_lib = None


class LibraryMissing(RuntimeError):
    """libmfx.so is not built: there is no CPU fallback for the solver."""


def load():
    """Load libmfx.so (no CUDA call is made at load time)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                f"or `make -C {os.path.join(_HERE, 'csrc')}` (no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    return load().mfx_last_error().decode("utf-8", "replace")


def ptr64(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags["C_CONTIGUOUS"], (a.dtype, a.flags)
    return a.ctypes.data_as(p_i64)


def ptr8(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(p_u8)


def as_i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


_RAISERS = {}


def register_error(code, cls):
    _RAISERS[code] = cls


class CudaError(RuntimeError):
    """A CUDA runtime error inside libmfx."""


class DeviceTimeout(RuntimeError):
    """The device watchdog of a solve expired."""


def check(rc: int):
    if rc == MFX_OK:
        return
    msg = last_error()
    cls = _RAISERS.get(rc)
    if cls is None:
        cls = {MFX_VALUE_ERROR: ValueError, MFX_CUDA_ERROR: CudaError,
               MFX_TIMEOUT: DeviceTimeout}.get(rc, RuntimeError)
    raise cls(msg)


def launch_count() -> int:
    return int(load().mfx_launch_count())


class HostBuffer:
    """Pinned (page-locked) int64 host array for end-to-end timing."""

    def __init__(self, count: int):
        self._p = vp()
        check(load().mfx_host_alloc(max(1, count) * 8, ctypes.byref(self._p)))
        buf = (ctypes.c_int64 * max(1, count)).from_address(self._p.value)
        self.array = np.frombuffer(buf, dtype=np.int64, count=count)

    def free(self):
        if self._p:
            self.array = None
            load().mfx_host_free(self._p)
            self._p = vp()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
