"""Vertex-range partitioned max-flow across GPUs (config C5).

The reference has no multi-device path (multi-GPU is "future work",
PAPER.md:732-733).  C5 (R-MAT 26, ~2.1 B Bi-CSR slots) exceeds the int32 slot
layout of one device, so it is the one configuration that shards.  Part r of
P owns the vertices ``[bounds[r], bounds[r+1])`` and their rows of the global
Bi-CSR (csrc/part.cu).  Peers reach each other's arrays through device
pointers: same-GPU pointers or NVLink P2P for parts hosted by one process
(:class:`LocalGroup`), CUDA IPC mappings when each GPU has its own process
(:class:`TorchGroup`, ``torch.distributed`` for the plumbing).

The host drives the reference round loop (solver.py:204-241) one phase at a
time (level-synchronous global relabel, push waves, repair, finalize) with a
barrier and a small all-reduce between phases; the math of every phase runs in
sm_100a kernels (csrc/part.cu).  Flow values match the single-GPU engine and
the reference (tests/test_gpu_partition.py).
"""

import ctypes
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .dynamic import BatchError, UpdateBatch
from .solver import SolverError, SolverParams, operation_ceiling

PH_LINK, PH_LINK_PC, PH_INIT, PH_SATURATE, PH_BFS_INIT, PH_BFS_EXPAND, PH_SWAP, PH_PUSH, \
    PH_REPAIR, PH_FINAL, PH_ACTIVE, PH_BATCH_RESOLVE, PH_BATCH_APPLY, PH_BATCH_FIX, \
    PH_TOPO_SEED = range(15)
BLOB_BYTES = 16 * 64  # B_NBUF CUDA IPC handles (csrc/part.cu)
PH_ASYNC = 0x100  # MFX_PH_ASYNC (include/mfx.h): enqueue only
# phases the host reads nothing back from (their out[] is unused by the round loop)
ASYNC_PHASES = (PH_BFS_INIT, PH_BFS_EXPAND, PH_PUSH, PH_REPAIR)
NONE = np.iinfo(np.int64).max


def balanced_bounds(n: int, us, vs, nparts: int) -> np.ndarray:
    """Contiguous vertex ranges with about equal Bi-CSR slot counts (a row
    holds the out-edges and the reverse stubs of the in-edges)."""
    if not 1 <= nparts <= 8:
        raise ValueError(f"nparts must be in [1, 8], got {nparts}")
    if nparts > n:
        raise ValueError(f"cannot split {n} vertices into {nparts} parts")
    us, vs = np.asarray(us, np.int64), np.asarray(vs, np.int64)
    deg = np.bincount(us, minlength=n)[:n] + np.bincount(vs, minlength=n)[:n] + 1
    cum = np.cumsum(deg)
    out = [0]
    for p in range(1, nparts):
        b = int(np.searchsorted(cum, cum[-1] * p / nparts, side="left")) + 1
        b = max(b, out[-1] + 1)
        b = min(b, n - (nparts - p))
        out.append(b)
    out.append(n)
    return np.asarray(out, np.int64)


def route(bounds: np.ndarray, us: np.ndarray) -> np.ndarray:
    """Owner part of each update's tail vertex (-1 when out of range)."""
    n = int(bounds[-1])
    own = np.searchsorted(bounds, us, side="right") - 1
    own[(us < 0) | (us >= n)] = -1
    return own


def combine_errors(blocks) -> np.ndarray:
    """Merge per-part batch error blocks (csrc/part.cu PartErr): first
    offending update per kind; the duplicate reported is the one on the
    globally smallest duplicated slot (same rule as the single-GPU path)."""
    out = np.full(8, NONE, np.int64)
    for b in blocks:
        b = np.asarray(b, np.int64)
        out[0] = min(out[0], b[0])
        out[1] = min(out[1], b[1])
        out[4] = min(out[4], b[4])
        if b[2] < out[2]:
            out[2], out[3] = b[2], b[3]
    return out


def batch_exception(err, us, vs, caps):
    """The reference's exception for a rejected batch (dynamic.py:63-88),
    worded like the single-GPU path (csrc/api.cu batch_error)."""
    if err[0] != NONE:
        j = int(err[0])
        return BatchError(f"update {j} ({us[j]}->{vs[j]}): negative capacity {caps[j]}")
    if err[1] != NONE:
        j = int(err[1])
        return BatchError(f"update {j} targets edge {us[j]}->{vs[j]} which is not an edge of "
                          f"the original graph")
    if err[3] != NONE:
        j = int(err[3])
        return BatchError(f"duplicate update for edge {us[j]}->{vs[j]}")
    if err[4] != NONE:
        j = int(err[4])
        return ValueError(f"update {j} ({us[j]}->{vs[j]}): capacity {caps[j]} overflows the "
                          f"int32 residual storage of the partitioned engine")
    return None


# ---------------------------------------------------------------------------
# groups: who hosts which parts, and the host-side collectives
# ---------------------------------------------------------------------------
class LocalGroup:
    """All P parts in this process: on one GPU (same-device pointers) or on
    several (NVLink P2P).  Phases run part after part, which is one valid
    interleaving of the concurrent schedule (every cross-part update is an
    atomic)."""

    def __init__(self, nparts: int, devices=None):
        self.nparts = int(nparts)
        self.local_ranks = list(range(self.nparts))
        self.devices = list(devices) if devices is not None else [0] * self.nparts
        if len(self.devices) != self.nparts:
            raise ValueError("one device per part")

    def allreduce(self, arr: np.ndarray, op: str = "sum") -> np.ndarray:
        return np.asarray(arr, np.int64)  # the caller already combined all local parts

    def allgather(self, obj):
        return [obj]

    def barrier(self):
        pass


class TorchGroup:
    """One part per process (``torch.distributed``; gloo or NCCL)."""

    def __init__(self, device: int | None = None):
        import torch
        import torch.distributed as dist
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised")
        self.dist = dist
        self.torch = torch
        self.rank = dist.get_rank()
        self.nparts = dist.get_world_size()
        self.local_ranks = [self.rank]
        self.devices = [device if device is not None else 0]
        self.nccl = dist.get_backend() == "nccl"

    def _tensor(self, arr):
        t = self.torch.as_tensor(np.asarray(arr, np.int64))
        return t.cuda() if self.nccl else t

    def allreduce(self, arr: np.ndarray, op: str = "sum") -> np.ndarray:
        t = self._tensor(arr)
        ro = {"sum": self.dist.ReduceOp.SUM, "max": self.dist.ReduceOp.MAX,
              "min": self.dist.ReduceOp.MIN}[op]
        self.dist.all_reduce(t, op=ro)
        return t.cpu().numpy()

    def allgather(self, obj):
        out = [None] * self.nparts
        self.dist.all_gather_object(out, obj)
        return out

    def barrier(self):
        if self.nccl:
            self.dist.barrier(device_ids=[self.torch.cuda.current_device()])
        else:
            self.dist.barrier()


# ---------------------------------------------------------------------------
@dataclass
class PartFlowResult:
    """Flow of a partitioned solve (fields as FlowResult, solver.py:108-118)."""

    flow_value: int
    cut_capacity: int
    rounds: int
    pushes: int = 0
    relabels: int = 0
    repairs: int = 0
    bfs_levels: int = 0
    waves: int = 0
    seconds: float = 0.0
    device: dict = field(default_factory=dict)


class PartitionedGraph:
    """A graph split by vertex range over the parts of ``group``, with the
    solver state of one (source, sink) pair.

    ``us/vs/caps`` are the whole edge list (every part selects the edges
    touching its range on the device); pass ``device_edges=(d_us, d_vs,
    d_caps, m)`` (device pointers) instead to build from device memory.
    """

    def __init__(self, n, us, vs, caps, source, sink, group=None, bounds=None,
                 device_edges=None):
        self.lib = L.load()
        self.calls = 0
        self.phase_s = {}  # host-observed seconds per phase kind (synchronous calls)
        self.group = group or LocalGroup(1)
        self.n = int(n)
        self.source, self.sink = int(source), int(sink)
        P = self.group.nparts
        if bounds is None:
            if us is None:
                raise ValueError("bounds are required when building from device edges")
            bounds = balanced_bounds(self.n, us, vs, P)
        self.bounds = L.as_i64(bounds)
        if self.bounds.shape[0] != P + 1:
            raise ValueError("bounds must have nparts + 1 entries")
        self.handles = {}
        for r, dev in zip(self.group.local_ranks, self.group.devices):
            h = ctypes.c_void_p()
            if device_edges is not None:
                d_us, d_vs, d_caps, m = device_edges
                L.check(self.lib.mfx_part_create(self.n, P, r, L.ptr64(self.bounds), int(m), d_us,
                                                 d_vs, d_caps, self.source, self.sink, int(dev),
                                                 ctypes.byref(h)))
            else:
                a, b, c = L.as_i64(us), L.as_i64(vs), L.as_i64(caps)
                L.check(self.lib.mfx_part_create_host(self.n, P, r, L.ptr64(self.bounds), a.size,
                                                      L.ptr64(a), L.ptr64(b), L.ptr64(c),
                                                      self.source, self.sink, int(dev),
                                                      ctypes.byref(h)))
            self.handles[r] = h
        self._connect()
        self._phase_all(PH_LINK)
        self.group.barrier()
        self._phase_all(PH_LINK_PC)
        self.group.barrier()
        infos = {}
        for r, h in self.handles.items():
            info = np.zeros(8, np.int64)
            L.check(self.lib.mfx_part_info(h, L.ptr64(info)))
            infos[r] = info
        every = {}
        for d in self.group.allgather({r: v.tolist() for r, v in infos.items()}):
            every.update(d)
        self.info = {int(r): np.asarray(v, np.int64) for r, v in every.items()}
        self.slots = np.array([self.info[r][2] for r in range(P)], np.int64)
        self.slot_base = np.concatenate([[0], np.cumsum(self.slots)[:-1]]).astype(np.int64)
        self.m = int(self.slots.sum())
        self.m_original = int(sum(self.info[r][3] for r in range(P)))
        self.stamp = 0
        self.terminated = False
        # global relabel: levels whose frontier exceeds 1/div of the unreached
        # vertices run bottom-up (0 = always top-down)
        self.bottom_up_div = int(os.environ.get("MFX_PART_BOTTOM_UP", "16"))
        self.async_phases = os.environ.get("MFX_PART_ASYNC", "1") != "0"

    # -- plumbing ------------------------------------------------------------
    def _connect(self):
        if isinstance(self.group, LocalGroup):
            for r, h in self.handles.items():
                for q, g in self.handles.items():
                    if q != r:
                        L.check(self.lib.mfx_part_attach_local(h, g))
            return
        (r, h), = self.handles.items()
        blob = ctypes.create_string_buffer(BLOB_BYTES)
        ln = ctypes.c_int64()
        L.check(self.lib.mfx_part_export(h, blob, BLOB_BYTES, ctypes.byref(ln)))
        blobs = self.group.allgather(bytes(blob.raw[:ln.value]))
        for q, b in enumerate(blobs):
            if q != r:
                buf = ctypes.create_string_buffer(b, len(b))
                L.check(self.lib.mfx_part_attach(h, q, buf, len(b)))
        self.group.barrier()

    def _phase(self, r, phase, args=()):
        a = np.zeros(8, np.int64)
        a[:len(args)] = args
        out = np.zeros(8, np.int64)
        self.calls += 1  # one phase = a few launches + up to 64 B of counters read back
        t0 = time.perf_counter()
        L.check(self.lib.mfx_part_phase(self.handles[r], phase, L.ptr64(a), L.ptr64(out)))
        self.phase_s[phase] = self.phase_s.get(phase, 0.0) + time.perf_counter() - t0
        return out

    def _phase_all(self, phase, args=None):
        """Run one phase on every local part; args: dict rank -> tuple.

        Phases whose results the host does not read run concurrently when one
        process hosts several parts: every part's phase is enqueued on its own
        stream, then all are awaited (the multi-GPU schedule on one process;
        every cross-part update is an atomic, so any interleaving is valid).
        $MFX_PART_ASYNC=0 runs them part after part."""
        if (phase in ASYNC_PHASES and len(self.handles) > 1 and self.async_phases):
            outs = {}
            for r in self.handles:
                outs[r] = self._phase(r, phase | PH_ASYNC, (args or {}).get(r, ()))
            t0 = time.perf_counter()
            for r in self.handles:
                L.check(self.lib.mfx_part_sync(self.handles[r]))
            self.phase_s[phase | PH_ASYNC] = (self.phase_s.get(phase | PH_ASYNC, 0.0)
                                              + time.perf_counter() - t0)
            return outs
        return {r: self._phase(r, phase, (args or {}).get(r, ())) for r in self.handles}

    def _sum(self, outs, idx) -> np.ndarray:
        local = np.zeros(len(idx), np.int64)
        for o in outs.values():
            local += o[list(idx)]
        return self.group.allreduce(local, "sum")

    # -- the round loop (solver.py:204-241) ------------------------------------
    def _global_relabel(self, dyn: int):
        self._phase_all(PH_BFS_INIT, {r: (dyn,) for r in self.handles})
        self.group.barrier()
        outs = self._phase_all(PH_SWAP)
        tot = int(self._sum(outs, (0, 1)).sum())
        reached = int(self._sum(outs, (5,))[0])
        cur, L_ = 0, 0
        while tot > 0:
            # direction-optimising: a level whose frontier holds more than
            # 1/bottom_up_div of the unreached vertices runs bottom-up
            up = int(self.bottom_up_div > 0 and tot * self.bottom_up_div > self.n - reached)
            self._phase_all(PH_BFS_EXPAND, {r: (L_, cur, o[0], o[1], dyn, up) for r, o in outs.items()})
            self.group.barrier()
            outs = self._phase_all(PH_SWAP)
            tot = int(self._sum(outs, (0, 1)).sum())
            reached = int(self._sum(outs, (5,))[0])
            cur ^= 1
            L_ += 1
        return outs, L_

    def _rounds(self, params: SolverParams, dyn: int, t0: float):
        kc = params.kernel_cycles or max(1, -(-self.m_original // self.n))
        ceiling = operation_ceiling(self.n, self.m_original)
        timeout = params.timeout_s if params.timeout_s > 0 else 600.0
        st = dict(rounds=0, pushes=0, relabels=0, repairs=0, levels=0, waves=0)
        base = self._sum({r: self._stats(r) for r in self.handles}, (0, 1, 2))
        rnd = 0
        while True:
            outs, depth = self._global_relabel(dyn)
            st["levels"] += depth
            if params.instrument is not None:  # (solver.py:219-241: the state is this object)
                params.instrument(self, self, rnd, "bfs")
            active = int(self._sum(outs, (4,))[0])
            if active == 0:
                break
            if params.mode == "topology":  # every non-terminal works this round
                self._phase_all(PH_TOPO_SEED)
                self.group.barrier()
                outs = self._phase_all(PH_SWAP)
            budget = params.max_waves if params.max_waves > 0 else 2 * depth // 4 + 4
            begin = {r: (0, 0) for r in outs}
            end = {r: (int(o[2]), int(o[3])) for r, o in outs.items()}
            waves = 0
            while True:
                self.stamp += 1
                self._phase_all(PH_PUSH, {r: (begin[r][0], end[r][0], begin[r][1], end[r][1], kc,
                                              self.stamp) for r in outs})
                self.group.barrier()
                outs = self._phase_all(PH_SWAP)
                waves += 1
                new = {r: (int(o[2]), int(o[3])) for r, o in outs.items()}
                grown, ovf = (int(x) for x in self._sum(
                    {r: np.array([new[r][0] - end[r][0] + new[r][1] - end[r][1], o[6]], np.int64)
                     for r, o in outs.items()}, (0, 1)))
                begin, end = end, new
                if grown == 0 or waves >= budget or ovf:
                    break
            rcap = {r: int(self.info[r][4]) for r in outs}
            self._phase_all(PH_REPAIR, {r: (min(end[r][0], rcap[r]), min(end[r][1], rcap[r]))
                                        for r in outs})
            self.group.barrier()
            st["rounds"] += 1
            st["waves"] += waves
            if params.instrument is not None:
                params.instrument(self, self, rnd, "repair")
            rnd += 1
            if time.perf_counter() - t0 > timeout:
                raise L.DeviceTimeout(f"partitioned solve exceeded {timeout:.0f} s after "
                                      f"{st['rounds']} rounds")
        counts = self._sum({r: self._stats(r) for r in self.handles}, (0, 1, 2)) - base
        st["pushes"], st["relabels"], st["repairs"] = (int(x) for x in counts)
        if st["pushes"] + st["relabels"] > ceiling:
            raise SolverError("push/relabel count exceeded the termination ceiling")
        fin = self._phase_all(PH_FINAL, {r: (int(o[7]),) for r, o in outs.items()})
        flow, cut = (int(x) for x in self._sum(fin, (0, 1)))
        return flow, cut, st

    def _stats(self, r):
        """Cumulative pushes, relabels, repairs, bytes of part r (device
        counters; an empty repair phase only reads them)."""
        return self._phase(r, PH_REPAIR, (0, 0))

    def _finish(self, flow, cut, st, t0) -> PartFlowResult:
        secs = float(self.group.allreduce(np.array([int((time.perf_counter() - t0) * 1e9)]),
                                          "max")[0]) * 1e-9
        if flow != cut:
            raise SolverError(f"flow {flow} does not match cut capacity {cut}")
        self.terminated = True
        return PartFlowResult(flow, cut, st["rounds"], st["pushes"], st["relabels"],
                              st["repairs"], st["levels"], st["waves"], secs,
                              {"parts": self.group.nparts, "slots": self.m})

    # -- public API --------------------------------------------------------------
    def solve_static(self, params: SolverParams | None = None) -> PartFlowResult:
        """solve_static (solver.py:253-283) over the partition set."""
        params = params or SolverParams()
        params.validate()
        self.group.barrier()
        t0 = time.perf_counter()
        self._phase_all(PH_INIT)
        self.group.barrier()
        self._phase_all(PH_SATURATE, {r: (0,) for r in self.handles})
        self.group.barrier()
        flow, cut, st = self._rounds(params, 1, t0)
        return self._finish(flow, cut, st, t0)

    def global_relabel(self, dynamic: bool = False) -> int:
        """backward_bfs / backward_bfs_dynamic (solver.py:155-164,
        dynamic.py:125-133) on the current state; returns #reached."""
        outs, _ = self._global_relabel(1 if dynamic else 0)
        self.terminated = False
        return int(self._sum(outs, (5,))[0])

    def saturate_source(self):
        self._phase_all(PH_SATURATE, {r: (0,) for r in self.handles})
        self.group.barrier()
        self.terminated = False

    def init_residuals(self):
        self._phase_all(PH_INIT)
        self.group.barrier()
        self.terminated = False

    def active_count(self) -> int:
        return int(self._sum(self._phase_all(PH_ACTIVE), (0,))[0])

    def solve_dynamic(self, batch: UpdateBatch, params: SolverParams | None = None
                      ) -> PartFlowResult:
        """solve_dynamic (dynamic.py:146-175): route each update to the part
        owning its tail, validate everywhere before any write, apply, repair
        over-capacity flow, re-saturate, then rounds with the sink and every
        deficient vertex as bases."""
        params = params or SolverParams()
        params.validate()
        if self.active_count() != 0:
            raise SolverError("solve_dynamic requires a terminated solver state")
        us, vs, caps = batch.arrays()
        k = us.size
        self.group.barrier()
        t0 = time.perf_counter()
        own = route(self.bounds, us)
        gidx = np.arange(k, dtype=np.int64)
        host_err = np.full(8, NONE, np.int64)
        if (caps < 0).any():
            host_err[0] = int(np.flatnonzero(caps < 0)[0])
        if (own < 0).any():
            host_err[1] = int(np.flatnonzero(own < 0)[0])
        for r, h in self.handles.items():
            sel = own == r
            a, b, c, j = (np.ascontiguousarray(x[sel]) for x in (us, vs, caps, gidx))
            L.check(self.lib.mfx_part_stage_batch(h, a.size, L.ptr64(a), L.ptr64(b), L.ptr64(c),
                                                  L.ptr64(j), int(self.slot_base[r])))
        blocks = list(self._phase_all(PH_BATCH_RESOLVE).values()) + [host_err]
        local = combine_errors(blocks)
        # all-reduce: min over kinds; the duplicate pair follows its slot
        red = self.group.allreduce(local[[0, 1, 2, 4]], "min")
        dupk = self.group.allreduce(np.array([local[3] if local[2] == red[2] else NONE]), "min")
        err = np.array([red[0], red[1], red[2], dupk[0], red[3], NONE, NONE, NONE], np.int64)
        exc = batch_exception(err, us, vs, caps)
        self._phase_all(PH_BATCH_APPLY, {r: (0 if exc else 1,) for r in self.handles})
        self.group.barrier()
        if exc is not None:
            raise exc
        self._phase_all(PH_BATCH_FIX)
        self.group.barrier()
        self._phase_all(PH_SATURATE, {r: (0,) for r in self.handles})
        self.group.barrier()
        flow, cut, st = self._rounds(params, 1, t0)
        return self._finish(flow, cut, st, t0)

    def sample_batch(self, k: int, seed: int, bias: float = 10.0) -> UpdateBatch:
        """A mixed batch of k updates drawn on the device from the current
        capacities (gen.py fast_batch semantics: half decrements on positive
        edges, half increments, bias on s-out / t-in edges), split over the
        parts in proportion to their original edges; (u, v)-sorted."""
        P = self.group.nparts
        share = np.array([self.info[r][3] for r in range(P)], np.float64)
        share = share / max(share.sum(), 1.0)

        def split(x):
            c = np.floor(share * x).astype(np.int64)
            c[: x - int(c.sum())] += 1
            return c
        kd, ki = split(k // 2), split(k - k // 2)
        got = {}
        for r, h in self.handles.items():
            want = int(kd[r] + ki[r])
            a, b, c = (np.zeros(max(want, 1), np.int64) for _ in range(3))
            n_out = ctypes.c_int64()
            L.check(self.lib.mfx_part_sample_batch(h, int(kd[r]), int(ki[r]),
                                                   int(seed) * 131 + r, float(bias), L.ptr64(a),
                                                   L.ptr64(b), L.ptr64(c), ctypes.byref(n_out)))
            got[r] = (a[:n_out.value], b[:n_out.value], c[:n_out.value])
        every = {}
        for d in self.group.allgather({r: tuple(x.tolist() for x in v) for r, v in got.items()}):
            every.update(d)
        us = np.concatenate([np.asarray(every[r][0], np.int64) for r in range(P)])
        vs = np.concatenate([np.asarray(every[r][1], np.int64) for r in range(P)])
        cs = np.concatenate([np.asarray(every[r][2], np.int64) for r in range(P)])
        order = np.lexsort((vs, us))
        return UpdateBatch(us[order], vs[order], cs[order])

    @classmethod
    def rmat(cls, scale: int, edge_factor: int = 16, seed: int = 0, group=None, device: int = 0,
             a: float = 0.57, b: float = 0.19, c: float = 0.19):
        """C5-shaped graph generated on the device (csrc/gen.cu: the gen.py
        R-MAT recursion with a counter-based stream) and split by slot-
        balanced vertex ranges; every rank draws the same edge list on its
        own GPU and keeps the edges touching its range."""
        import torch
        group = group or LocalGroup(1)
        lib = L.load()
        n = 1 << scale
        m = n * edge_factor
        dev = f"cuda:{group.devices[0]}"
        e = [torch.empty(m, dtype=torch.int64, device=dev) for _ in range(3)]
        s, t = ctypes.c_int64(), ctypes.c_int64()
        L.check(lib.mfx_rmat_device(scale, edge_factor, seed, a, b, c, group.devices[0],
                                    e[0].data_ptr(), e[1].data_ptr(), e[2].data_ptr(),
                                    ctypes.byref(s), ctypes.byref(t)))
        bounds = np.zeros(group.nparts + 1, np.int64)
        L.check(lib.mfx_part_bounds_device(n, m, e[0].data_ptr(), e[1].data_ptr(), group.nparts,
                                           group.devices[0], L.ptr64(bounds)))
        if len(set(group.devices)) > 1:
            raise ValueError("device generation expects the local parts on one GPU")
        pg = cls(n, None, None, None, s.value, t.value, group, bounds=bounds,
                 device_edges=(e[0].data_ptr(), e[1].data_ptr(), e[2].data_ptr(), m))
        del e
        torch.cuda.empty_cache()
        return pg

    def download(self, r: int) -> dict:
        """Local arrays of part r (int64): off, adj, rev, cap0, cf, orig,
        excess, height."""
        h = self.handles[r]
        lo, hi, S = (int(x) for x in self.info[r][:3])
        nl = hi - lo
        out = {k: np.zeros(nl + 1 if k == "off" else S, np.int64)
               for k in ("off", "adj", "rev", "cap0", "cf")}
        out["orig"] = np.zeros(S, np.uint8)
        out["excess"] = np.zeros(nl, np.int64)
        out["height"] = np.zeros(nl, np.int64)
        L.check(self.lib.mfx_part_download(h, L.ptr64(out["off"]), L.ptr64(out["adj"]),
                                           L.ptr64(out["rev"]), L.ptr64(out["cap0"]),
                                           L.ptr64(out["cf"]), L.ptr8(out["orig"]),
                                           L.ptr64(out["excess"]), L.ptr64(out["height"])))
        return out

    def close(self):
        for h in self.handles.values():
            self.lib.mfx_part_free(h)
        self.handles = {}

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
