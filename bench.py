"""Benchmark for BASELINE.json's metric: dynamic max-flow ms per update batch
(against a GPU static re-solve) and static max-flow edges/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config auto|C1|C2|C3|C4|C5]

Headline (N = 1, ``--config auto``): C4, the largest single-GPU config of
BASELINE.json -- a road-shaped lattice of 24,010,000 vertices / 58,104,530
directed edges, corner to corner, chained batches of 10,000 mixed updates.
C1-C3 are the same measurement on the other single-GPU configs.

A step = one chained batch through solve_dynamic:

* ``value``: K steps with the batches resident in HBM, CUDA events on the
  engine's stream, max over ranks.
* ``e2e``: the SAME K batches replayed from a device snapshot of the state
  and capacities taken before the timed region, through the public API
  ``solve_dynamic(st, g, UpdateBatch(...))`` from pinned host arrays (H2D of
  the batch and D2H of the result inside the timed region).  Its flows must
  equal the ``value`` leg's.
* ``roofline``: the persistent solve kernel (one launch per batch):
  algorithmic bytes counted on the device / its event-timed duration,
  against MEASURED_PEAKS.json; ``traffic`` = ncu DRAM bytes of the same
  kernel on the same config and batch index, read from
  profiles/ncu_<config>_solve_kernel.json only when that capture was taken
  from the current kernel sources (hash), else null.
* ``cpu_baseline``: the C oracle port (1 thread) on one batch of the same
  workload continuing from the GPU's terminated state, wall-clock capped
  (a capped sample is a lower bound and says so).

N > 1 (torchrun, or ``--gpus N`` which re-launches itself under torchrun):
the one multi-GPU path of the north star, C5 -- R-MAT vertex-range
partitioned, one part per rank (``--scale``, default 26).  ``--config C5`` at
N = 1 runs the same partition code with ``--parts`` parts on one GPU.

``--impl reference`` runs the unmodified reference package
(baseline/_ref, numba, all host threads) on the same config: for C4 its
static solve is infeasible (thousands of O(n) rounds), so its start state is
a maximum flow from the oracle's Dinic restatement (not timed) and each
batch is capped through the reference's own ``instrument`` hook; a capped
batch reports its elapsed time as a lower bound.  A scaled road anchor
(512^2, ``threads=nproc`` and ``threads=1``) runs to completion beside it.
"""

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "dynamic maxflow ms per update batch vs static recompute; static maxflow edges/s"

# config -> (generator, args, batch size, description)
CONFIGS = {
    "C1": ("random", (10000, 100000), 1000,
           "C1: random graph 10K vertices / 100K edges (reference random_graph, seed 0)"),
    "C2": ("grid", (2048,), 10000,
           "C2: 2048x2048 4-neighbour grid + terminal edge per pixel (caps U[1,100], seed 0)"),
    "C3": ("rmat", (20,), 10000,
           "C3: R-MAT scale 20 ef 16 (0.57,0.19,0.19), caps U[1,100], seed 0"),
    "C4": ("road", (4900,), 10000,
           "C4: road-shaped lattice 4900x4900 (every row link, vertical links p=0.21, "
           "column 0 kept), both directions, caps U[1,100], corner to corner"),
    # one GPU: the whole graph on the single-device engine (2.10 B slots fit
    # the int32 layout); N > 1 GPUs: the vertex-range partition (bench_c5)
    "C5": ("rmat_device", (26,), 1_000_000,
           "C5: R-MAT scale 26 ef 16 (0.57,0.19,0.19; device generator, seed 0), caps U[1,100]"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="auto", choices=["auto", "C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--batch", type=int, default=0, help="updates per batch (0: the config's)")
    ap.add_argument("--side", type=int, default=0, help="grid/road side override (scaled runs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-cap-s", type=float, default=30.0, help="cap of the cpu_baseline sample")
    ap.add_argument("--ref-cap-s", type=float, default=120.0,
                    help="reference arm: wall-clock cap per batch")
    ap.add_argument("--ref-budget-s", type=float, default=240.0,
                    help="reference arm: wall-clock budget for the chained batches")
    ap.add_argument("--profile", action="store_true",
                    help="ncu mode: static solve, W warm-up batches, then K batches inside the "
                         "NVTX range 'timed' (no e2e / re-solve / cpu legs)")
    ap.add_argument("--scale", type=int, default=26, help="C5 R-MAT scale")
    ap.add_argument("--parts", type=int, default=4, help="C5 parts when run as one process")
    ap.add_argument("--engine", default="single", choices=["single", "part"],
                    help="C5 on one GPU: the single-device engine, or the partition (--parts)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch plumbing only (ranks, collectives, max-over-ranks, JSON line); "
                         "no engine calls -- runs without a GPU")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# launch / ranks
# ---------------------------------------------------------------------------
def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_relaunch(args):
    """``--gpus N`` outside torchrun: re-run this script as N ranks."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def dist_setup():
    """One process per GPU.  NCCL when every rank has its own GPU; gloo
    when ranks share devices (one-GPU boxes) or there is no GPU."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg, device, backend = None, 0, None
    import torch
    ngpu = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if ngpu:
        device = local % ngpu
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if ngpu >= world else "gloo"
        if ngpu:
            torch.cuda.set_device(device)
        dist.init_process_group(backend=backend)
        pg = dist
    return rank, world, device, pg, backend


def barrier(pg, backend, device):
    if pg is None:
        return
    if backend == "nccl":
        pg.barrier(device_ids=[device])
    else:
        pg.barrier()


def max_over_ranks(pg, backend, x: float, device: int) -> float:
    if pg is None:
        return x
    import torch
    dev = f"cuda:{device}" if backend == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """NVML SM clock and throttle-reason sampling during the timed region
    (the profiling recipe's clocks line)."""

    NAMES = {"applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
             "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
             "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100}

    def __init__(self, device: int):
        self.device = device
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.reasons.update(k for k, b in self.NAMES.items() if r & b)
                    except Exception:
                        pass
                    self._stop.wait(0.02)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        busy = [s for s in self.samples if s > 0]
        return {"sm_mhz": float(statistics.median(busy)) if busy else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# evidence helpers
# ---------------------------------------------------------------------------
def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def kernel_source_hash() -> str:
    """Hash of everything that determines the solve kernel's code."""
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2511_01235_b200", "csrc")
    for name in sorted(os.listdir(csrc)):
        if name.endswith((".cu", ".cuh", ".h", ".cpp")) or name == "Makefile":
            with open(os.path.join(csrc, name), "rb") as fh:
                h.update(name.encode() + b"\0" + fh.read())
    with open(os.path.join(ROOT, "include", "mfx.h"), "rb") as fh:
        h.update(fh.read())
    return h.hexdigest()[:16]


def load_traffic(config: str):
    """ncu DRAM bytes per solve-kernel launch for this config, valid only
    if captured from the current kernel sources."""
    path = os.path.join(ROOT, "profiles", f"ncu_{config}_solve_kernel.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
    except Exception:
        return None, "no ncu capture for this config"
    if d.get("src_hash") != kernel_source_hash():
        return None, f"stale ncu capture ({os.path.basename(path)} src_hash {d.get('src_hash')})"
    return d, os.path.relpath(path, ROOT)


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def make_instance(cfg: str, side: int = 0):
    from paper_2511_01235_b200 import gen
    kind, a, _, _ = CONFIGS[cfg]
    if kind == "random":
        us, vs, caps, s, t = gen.random_edges(*a, seed=0)
        return a[0], us, vs, caps, s, t
    if kind == "grid":
        w = side or a[0]
        us, vs, caps, s, t = gen.grid_graph(w, w, seed=0)
        return w * w + 2, us, vs, caps, s, t
    if kind == "rmat":
        us, vs, caps, s, t = gen.rmat_graph(a[0], 16, seed=0)
        return 1 << a[0], us, vs, caps, s, t
    w = side or a[0]
    us, vs, caps, s, t = gen.road_graph(w, w, seed=0, p_vert=0.21)
    return w * w, us, vs, caps, s, t


def make_chain(n, el_us, el_vs, el_caps, s, t, count, k, seed0):
    """``count`` chained mixed batches, each drawn from the capacities the
    previous one left (gen.sparse_batch: reference generate_batch law)."""
    from paper_2511_01235_b200 import gen
    caps = np.array(el_caps, np.int64, copy=True)
    out = []
    for i in range(count):
        bu, bv, bc, pick = gen.sparse_batch(n, el_us, el_vs, caps, s, t, k, "mixed", seed0 + i)
        caps[pick] = bc
        out.append((bu, bv, bc))
    return out


def workload_block(args, cfg, k, world):
    desc = CONFIGS[cfg][3]
    if args.side:
        desc += f" [scaled: side {args.side}]"
    return {"workload": f"{desc}; chained batches of {k} mixed updates (bias 10, "
                        f"gen.sparse_batch = reference generate_batch law)",
            "config": cfg, "batch_updates": k,
            "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
            "l2": "inputs larger than L2 (Bi-CSR + state > 126 MB)" if cfg != "C1"
            else "graph fits in L2 (C1: ~3 MB); no flush"}


# ---------------------------------------------------------------------------
# our arm, single GPU configs
# ---------------------------------------------------------------------------
def bench_ours(args, cfg, rank, world, dev, pg, backend):
    import ctypes

    import torch

    import paper_2511_01235_b200 as mfx
    from paper_2511_01235_b200 import _lib

    L = _lib.load()
    k = args.batch or CONFIGS[cfg][2]
    device_graph = CONFIGS[cfg][0] == "rmat_device"
    if device_graph:  # C5: drawn and built on the device (1.07 B edges)
        n = 1 << args.scale
        m = n * 16
        e = [torch.empty(m, dtype=torch.int64, device=f"cuda:{dev}") for _ in range(3)]
        s_, t_ = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(L.mfx_rmat_device(args.scale, 16, 0, 0.57, 0.19, 0.19, dev, e[0].data_ptr(),
                                     e[1].data_ptr(), e[2].data_ptr(), ctypes.byref(s_),
                                     ctypes.byref(t_)))
        s, t = s_.value, t_.value
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g = mfx.build_bicsr_device(n, e[0].data_ptr(), e[1].data_ptr(), e[2].data_ptr(), m,
                                   device=dev)
        build_s = time.perf_counter() - t0
        del e
        torch.cuda.empty_cache()
    else:
        n, us, vs, caps, s, t = make_instance(cfg, args.side)
        t0 = time.perf_counter()
        g = mfx.build_bicsr(mfx.EdgeListGraph(n, us, vs, caps), device=dev)
        build_s = time.perf_counter() - t0
        del us, vs, caps
    params = mfx.SolverParams()
    res = mfx.solve_static(g, s, t, params)  # warm
    static_ms = [res.device["ms_total"]]
    if not args.profile:
        for _ in range(2):
            res = mfx.solve_static(g, s, t, params)
            static_ms.append(res.device["ms_total"])
    st = res.state
    W, K = args.warmup, args.steps
    if device_graph:  # chained device draws, each from the capacities the last one left
        from paper_2511_01235_b200 import gen
        gs, chain = g.copy(), []
        for i in range(W + K):
            b = gen.device_sample_batch(gs, s, t, k, "mixed", seed=1000 * rank + i)
            _lib.check(L.mfx_apply_updates(gs.handle, None, b[0].size, _lib.ptr64(b[0]),
                                           _lib.ptr64(b[1]), _lib.ptr64(b[2])))  # (capacities only)
            chain.append(b)
        del gs
    else:
        el = g.to_edge_list()
        chain = make_chain(n, el.us, el.vs, el.caps, s, t, W + K, k, 1000 * rank)
    dbat = [tuple(torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{dev}") for a in b)
            for b in chain]
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(L.mfx_graph_stream(g.handle), device=dev)
    for i in range(W):
        bu, bv, bc = dbat[i]
        mfx.solve_dynamic_device(st, g, k, bu.data_ptr(), bv.data_ptr(), bc.data_ptr(), params)
    # snapshots for the e2e replay and the O2 push-pull replay of the same batches
    g_snap, st_snap = (None, None) if args.profile else (g.copy(), st.copy())
    g_pp, st_pp = (None, None) if args.profile else (g.copy(), st.copy())
    torch.cuda.synchronize()

    rows = []
    launches0 = mfx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        barrier(pg, backend, dev)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("timed")
        ev0.record(stream)
        for i in range(W, W + K):
            bu, bv, bc = dbat[i]
            r = mfx.solve_dynamic_device(st, g, k, bu.data_ptr(), bv.data_ptr(), bc.data_ptr(),
                                         params)
            d = r.device
            rows.append((r.flow_value, r.rounds, d["ms_solve"], d["bytes_alg"], d["bfs_epochs"],
                         d["waves"], d["bfs_levels"], d["ms_total"]))
        ev1.record(stream)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        barrier(pg, backend, dev)
    launches = mfx.launch_count() - launches0
    elapsed = max_over_ranks(pg, backend, ev0.elapsed_time(ev1), dev)
    a = np.array(rows, dtype=np.float64)
    out = {"cfg": cfg, "k": k, "n": n, "S": g.m, "m_orig": g.m_original, "build_s": build_s,
           "static_ms": min(static_ms), "static_flow": res.flow_value,
           "static_rounds": res.rounds, "elapsed_ms": elapsed, "flows": [int(x) for x in a[:, 0]],
           "rounds": a[:, 1], "solve_ms": a[:, 2], "bytes_alg": a[:, 3], "epochs": a[:, 4],
           "waves": a[:, 5], "levels": a[:, 6], "launches": launches, "clocks": clk.summary(),
           "cap_bytes": g.cap_bytes}
    if args.profile:
        return out

    # ---- e2e: same batches, public API, pinned host memory, from the snapshot
    pinned = []
    for bu, bv, bc in chain[W:]:
        hb = [mfx.HostBuffer(bu.size) for _ in range(3)]
        for h, x in zip(hb, (bu, bv, bc)):
            h.array[:] = x
        pinned.append(hb)
    barrier(pg, backend, dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_flows = []
    for hb in pinned:
        r = mfx.solve_dynamic(st_snap, g_snap, mfx.UpdateBatch(hb[0].array, hb[1].array,
                                                               hb[2].array), params)
        e2e_flows.append(r.flow_value)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(pg, backend, (time.perf_counter() - t0) * 1e3, dev)
    assert e2e_flows == out["flows"], (e2e_flows, out["flows"])
    h2d, d2h = ctypes.c_int64(), ctypes.c_int64()
    L.mfx_transfer_bytes(k, ctypes.byref(h2d), ctypes.byref(d2h))
    out.update(e2e_ms_per_step=e2e_ms / K, e2e_h2d=int(h2d.value), e2e_d2h=int(d2h.value))
    del g_snap, st_snap

    # ---- the reference bench's second dynamic mode (bench.py:150-198):
    # solve_dynamic_pushpull (O2) on the same batches from the same state
    pp_ms, pp_flows = [], []
    for i in range(W, W + K):
        r = mfx.solve_dynamic_pushpull(st_pp, g_pp, mfx.UpdateBatch(*chain[i]), params)
        pp_ms.append(r.device["ms_total"])
        pp_flows.append(r.flow_value)
        st_pp = r.state
    assert pp_flows == out["flows"], (pp_flows, out["flows"])
    out["pushpull_ms"] = pp_ms
    del g_pp, st_pp

    # ---- GPU static re-solve on the updated capacities (the comparison point)
    st2 = mfx.init_residuals(g, s, t)
    rs = []
    for _ in range(2):
        rr = mfx.resolve_static(g, st2, params)
        rs.append(rr.device["ms_total"])
    assert rr.flow_value == out["flows"][-1], (rr.flow_value, out["flows"][-1])
    out.update(resolve_ms=min(rs), resolve_flow=rr.flow_value)
    rep = mfx.verify_gpu(st, g, out["flows"][-1])
    assert rep.ok, rep.problems
    del st2

    # ---- grid-barrier cost, for the latency floor of the solve kernel
    ns = ctypes.c_double()
    _lib.check(L.mfx_bench_barrier(g.handle, st.handle, 2000, 0, ctypes.byref(ns)))
    out["barrier_ns"] = ns.value
    cns = ctypes.c_double()  # dependent-load latency: the latency roofline's unit
    _lib.check(L.mfx_bench_chase(g.handle, 1 << 30, 20000, ctypes.byref(cns)))
    out["chase_ns"] = cns.value

    if rank == 0 and world == 1 and not args.no_cpu_baseline and not device_graph:
        out["cpu_baseline"] = cpu_sample(g, st, s, t, n, k, args)
    elif device_graph:
        out["cpu_baseline"] = {"value": None, "unit": "ms/batch", "cores": 1, "kind": "port",
                               "sample": "not run: the C oracle cannot hold the 2.1 B-slot graph "
                                         "in host memory within the bench's time budget"}
    return out


def cpu_sample(g, st, s, t, n, k, args):
    """The C oracle (test infrastructure, 1 thread) on one batch of the same
    workload, from the GPU's terminated state, capped at --cpu-cap-s."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    og = O.OracleGraph(n, g.m, g.offsets.copy(), g.adj.copy(), g.src.copy(), g.rev.copy(),
                       g.cap0.copy(), g.is_original.copy(), (0, 0, 0))
    ost = O.OracleState(st.cf.astype(np.int64), st.excess.astype(np.int64),
                        st.height.astype(np.int64), s, t)
    keep = og.is_original
    (bu, bv, bc), = make_chain(n, og.src[keep], og.adj[keep], og.cap0[keep], s, t, 1, k, 99991)
    O.set_time_cap(args.cpu_cap_s)
    t0 = time.perf_counter()
    r = O.solve_dynamic(og, ost, bu, bv, bc)
    dt = time.perf_counter() - t0
    O.set_time_cap(0)
    capped = r.status == 5
    return {"value": round(dt * 1e3, 1), "unit": "ms/batch", "cores": 1, "kind": "port",
            "lower_bound": capped,
            "sample": (f"1 batch of {k} mixed updates (C oracle: deterministic single-thread "
                       f"restatement of the reference rounds) from the GPU's terminated state; "
                       + (f"capped at {args.cpu_cap_s:.0f} s after {r.rounds} rounds "
                          f"(value is a lower bound)" if capped else
                          f"flow {r.flow}, {r.rounds} rounds"))}


def emit_ours(args, out, world):
    K = args.steps
    peak, peak_src = load_peaks()
    solve_ms = out["solve_ms"]
    kernel_ms = float(np.mean(solve_ms))
    bytes_launch = float(np.mean(out["bytes_alg"]))
    achieved = bytes_launch / 1e9 / (kernel_ms / 1e3) if kernel_ms > 0 else 0.0
    traffic, tsrc = load_traffic(out["cfg"])
    barriers = float(np.mean(out["epochs"] + out["waves"]))
    bar_us = out.get("barrier_ns", 0.0) / 1e3
    # latency roofline: the critical path of a launch is a chain of dependent
    # global accesses -- ~4 per BFS label (row offsets/height -> row -> head
    # heights -> relaxing atomic) and ~5 per push wave (+ the CTA-0 list
    # hand-off) -- at the measured cache-missing load latency, plus the grid
    # barriers at their measured cost
    chain = float(np.mean(4 * out["levels"] + 5 * out["waves"]))
    load_us = out.get("chase_ns", 0.0) / 1e3
    lat_floor_ms = (chain * load_us + barriers * bar_us) / 1e3
    value = out["elapsed_ms"] / K
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "ms/batch", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(value, 4),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "int32" if out["cap_bytes"] == 4 else "int64", "data": "synthetic",
        "config": workload_block(args, out["cfg"], out["k"], world),
        "graph": {"n": out["n"], "slots": out["S"], "m_original": out["m_orig"],
                  "build_s": round(out["build_s"], 2)},
        "static_maxflow_edges_per_s": round(out["m_orig"] / (out["static_ms"] / 1e3), 1),
        "static_ms": round(out["static_ms"], 3), "static_rounds": out["static_rounds"],
        "gpu_static_resolve_ms": round(out["resolve_ms"], 3) if "resolve_ms" in out else None,
        "dynamic_speedup_vs_gpu_static_resolve": (round(out["resolve_ms"] / value, 2)
                                                  if "resolve_ms" in out else None),
        "flow_static": out["static_flow"], "flows": out["flows"],
        "pushpull_ms_per_batch": (round(float(np.mean(out["pushpull_ms"])), 4)
                                  if "pushpull_ms" in out else None),
        "pushpull_speedup_vs_gpu_static_resolve": (
            round(out["resolve_ms"] / float(np.mean(out["pushpull_ms"])), 2)
            if "pushpull_ms" in out and "resolve_ms" in out else None),
        "per_batch_ms": [round(x, 3) for x in out["solve_ms"]],
        "rounds_per_batch": round(float(np.mean(out["rounds"])), 2),
        "gpu_launches": out["launches"],
        "roofline": {
            "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 5), "peak_source": peak_src,
            "traffic": (traffic or {}).get("dram_bytes_per_launch"),
            "traffic_source": tsrc,
            "kernel": "solve_kernel (persistent cooperative, one launch per batch)",
            "bytes_alg_per_launch": int(bytes_launch),
            "kernel_ms_per_launch": round(kernel_ms, 4),
            "latency": {"grid_barriers_per_launch": round(barriers, 1),
                        "barrier_us": round(bar_us, 2),
                        "barrier_floor_ms": round(barriers * bar_us / 1e3, 4),
                        "bfs_levels_per_launch": round(float(np.mean(out["levels"])), 1),
                        "push_waves_per_launch": round(float(np.mean(out["waves"])), 1),
                        "dependent_loads_per_launch": round(chain, 1),
                        "load_latency_us": round(load_us, 3),
                        "floor_ms": round(lat_floor_ms, 4),
                        "frac": round(lat_floor_ms / kernel_ms, 4) if kernel_ms else None,
                        "model": "critical path = (4 x BFS labels + 5 x push waves) dependent "
                                 "loads at the measured pointer-chase latency + grid barriers "
                                 "at their measured cost; frac = that floor / kernel time"},
        },
        "clocks": out["clocks"],
        "kernel_src_hash": kernel_source_hash(),
    }
    if "e2e_ms_per_step" in out:
        line["e2e"] = {"value": round(out["e2e_ms_per_step"], 4), "unit": "ms/batch",
                       "h2d_bytes_per_step": out["e2e_h2d"], "d2h_bytes_per_step": out["e2e_d2h"],
                       "same_batches_as_value": True}
    if "cpu_baseline" in out:
        line["cpu_baseline"] = out["cpu_baseline"]
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# C5: vertex-range partition (the multi-GPU path)
# ---------------------------------------------------------------------------
def bench_c5(args, rank, world, dev, pg, backend):
    import torch

    from paper_2511_01235_b200 import partition
    group = partition.TorchGroup(device=dev) if world > 1 else \
        partition.LocalGroup(args.parts, [dev] * args.parts)
    t0 = time.perf_counter()
    g = partition.PartitionedGraph.rmat(args.scale, 16, 0, group, device=dev)
    build_s = time.perf_counter() - t0
    st = g.solve_static()
    W, K = args.warmup, args.steps
    k = args.batch or 1_000_000
    for i in range(W):
        g.solve_dynamic(g.sample_batch(k, seed=i))
    timed, flows, phases = [], [], []
    calls0 = g.calls
    with ClockSampler(dev) as clk:
        for i in range(W, W + K):
            b = g.sample_batch(k, seed=i)  # device sampler, outside the timed solve
            barrier(pg, backend, dev)
            torch.cuda.synchronize()
            r = g.solve_dynamic(b)  # host batch in, counters out (end to end)
            torch.cuda.synchronize()
            timed.append(r.seconds)  # max over ranks inside solve_dynamic
            flows.append(r.flow_value)
            phases.append({"rounds": r.rounds, "bfs_levels": r.bfs_levels, "waves": r.waves})
    calls = (g.calls - calls0) / K
    rs = g.solve_static()
    assert rs.flow_value == flows[-1], (rs.flow_value, flows[-1])
    ms = 1e3 * sum(timed) / K
    if rank != 0:
        return
    parts = group.nparts
    line = {
        "metric": METRIC, "value": round(ms, 3), "unit": "ms/batch", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(ms, 3), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"C5: R-MAT scale {args.scale} ef 16 (device generator, seed 0), "
                               f"{g.m} Bi-CSR slots, chained batches of {k} mixed "
                               f"updates (device sampler, bias 10)",
                   "config": "C5", "parts": parts,
                   "parallelism": f"vertex-range partition, {parts} parts on {world} rank(s), "
                                  f"collectives {backend or 'none (one process)'}",
                   "l2": "inputs larger than L2"},
        "static_maxflow_edges_per_s": round(g.m_original / st.seconds, 1),
        "static_ms": round(1e3 * st.seconds, 3), "build_s": round(build_s, 2),
        "gpu_static_resolve_ms": round(1e3 * rs.seconds, 3),
        "dynamic_speedup_vs_gpu_static_resolve": round(rs.seconds * 1e3 / ms, 2),
        "flow_static": st.flow_value, "flows": flows, "resolve_agrees": True,
        "per_batch": {k2: round(float(np.mean([p[k2] for p in phases])), 2)
                      for k2 in ("rounds", "bfs_levels", "waves")},
        "e2e": {"value": round(ms, 3), "unit": "ms/batch", "h2d_bytes_per_step": 32 * k,
                "d2h_bytes_per_step": int(64 * calls)},
        "host_calls_per_batch": round(calls, 1),
        "roofline": None, "clocks": clk.summary(),
        "note": "host-driven per phase; the roofline line is the single-GPU bench",
    }
    print(json.dumps(line), flush=True)
    g.close()


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
class _Capped(Exception):
    pass


def _ref_dynamic(ref, st, g, batch, params, cap_s):
    """One reference solve_dynamic, stopped through its instrument hook
    (called after every global relabel, solver.py:219-241) once past cap."""
    t0 = time.perf_counter()
    rounds = [0]

    def hook(_st, _g, rnd, label):
        rounds[0] = rnd
        if time.perf_counter() - t0 > cap_s:
            raise _Capped()

    params.instrument = hook
    try:
        r = ref.solve_dynamic(st, g, batch, params)
        return time.perf_counter() - t0, r, False
    except _Capped:
        return time.perf_counter() - t0, rounds[0], True
    finally:
        params.instrument = None


def bench_reference(args, cfg, world):
    """The unmodified reference package on the host cores, same config."""
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    cores = os.cpu_count() or 1
    try:
        import dynmaxflow as ref
    except Exception as e:  # pragma: no cover - install missing
        print(json.dumps({"impl": "reference", "unavailable": f"baseline/_ref import failed: {e}"}))
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    k = args.batch or CONFIGS[cfg][2]
    params = ref.SolverParams(threads=cores)
    tg, ts, tt = ref.random_graph(50, 300, seed=0)  # warm the numba JIT (bench.py protocol)
    g0 = ref.build_bicsr(tg)
    ref.solve_dynamic(ref.solve_static(g0, ts, tt, params).state, g0,
                      ref.UpdateBatch.from_updates([]), params)
    n, us, vs, caps, s, t = make_instance(cfg, args.side)
    t0 = time.perf_counter()
    csr = ref.build_bicsr(ref.EdgeListGraph(n, us, vs, caps))
    build_s = time.perf_counter() - t0
    del us, vs, caps
    notes = {}
    static_s = None
    if cfg == "C4" and not args.side:
        # start state: a maximum flow from the oracle's Dinic restatement
        import oracle as O
        og = O.OracleGraph(n, csr.m, csr.offsets, csr.adj, csr.src, csr.rev, csr.cap0,
                           csr.is_original, (0, 0, 0))
        t0 = time.perf_counter()
        flow0, ost = O.terminated_state(og, s, t)
        notes["start_state"] = (f"max flow {flow0} from oracle Dinic (oracle.py:20-84 restated), "
                                f"{time.perf_counter() - t0:.1f} s, not timed; reference static "
                                f"solve infeasible (~10^4 rounds of O(n) BFS)")
        st = ref.SolverState(ost.cf, ost.excess, ost.height, s, t, n)
        g = csr
    else:
        t0 = time.perf_counter()
        prior = ref.solve_static(csr, s, t, params)
        static_s = time.perf_counter() - t0
        st, g = prior.state, csr
    el = csr.to_edge_list()
    chain = make_chain(n, el.us, el.vs, el.caps, s, t, max(1, args.steps), k, 0)
    times, capped_any, done = [], False, 0
    tb = time.perf_counter()
    for bu, bv, bc in chain:
        dt, r, capped = _ref_dynamic(ref, st, g, ref.UpdateBatch(bu, bv, bc), params,
                                     args.ref_cap_s)
        times.append(dt)
        if capped:
            capped_any = True
            notes["capped_batch"] = (f"batch {len(times) - 1} unfinished after {dt:.1f} s "
                                     f"(round {r}); value is a lower bound")
            break
        done += 1
        st, g = r.state, r.graph
        if time.perf_counter() - tb > args.ref_budget_s:
            break
    ms = 1e3 * sum(times) / len(times)
    anchor = ref_anchor(ref, args, cores) if cfg == "C4" and not args.side else None
    sample = (f"{done} chained batch(es) of {k} mixed updates completed"
              + (", then one capped" if capped_any else "") +
              f" (per-batch cap {args.ref_cap_s:.0f} s, budget {args.ref_budget_s:.0f} s); "
              f"build_bicsr {build_s:.1f} s not timed")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(ms, 3), "unit": "ms/batch",
        "n_gpus": world, "steps": len(times), "warmup": 0, "ms_per_step": round(ms, 3),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "lower_bound": capped_any,
        "config": dict(workload_block(args, cfg, k, 1),
                       parallelism=f"{cores} host threads (numba, SolverParams(threads={cores}))"),
        "static_ms": round(1e3 * static_s, 1) if static_s else None,
        "static_maxflow_edges_per_s": round(csr.m_original / static_s, 1) if static_s else None,
        "per_batch_ms": [round(1e3 * x, 1) for x in times],
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms/batch", "cores": cores,
                         "kind": "reference", "sample": sample, "lower_bound": capped_any},
        "e2e": {"value": round(ms, 3), "unit": "ms/batch", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "notes": notes,
    }
    if anchor:
        line["scaled_anchor"] = anchor
    print(json.dumps(line), flush=True)


def ref_anchor(ref, args, cores):
    """C4's generator at 512^2 run to completion by the reference:
    static solve and chained batches, threads=nproc and threads=1."""
    from paper_2511_01235_b200 import gen
    side = 512
    us, vs, caps, s, t = gen.road_graph(side, side, seed=0, p_vert=0.21)
    n = side * side
    out = {"graph": f"road {side}x{side} (C4 generator), n={n}, m={us.size}"}
    csr0 = ref.build_bicsr(ref.EdgeListGraph(n, us, vs, caps))
    k = max(1, round(10000 * csr0.m_original / 58104530))
    el = csr0.to_edge_list()
    chain = make_chain(n, el.us, el.vs, el.caps, s, t, 2, k, 0)
    out["batch_updates"] = k
    for thr in (cores, 1):
        p = ref.SolverParams(threads=thr)
        csr = csr0.copy()
        t0 = time.perf_counter()
        prior = ref.solve_static(csr, s, t, p)
        st_s = time.perf_counter() - t0
        st, g, dts, flows = prior.state, csr, [], []
        for bu, bv, bc in chain:
            t0 = time.perf_counter()
            r = ref.solve_dynamic(st, g, ref.UpdateBatch(bu, bv, bc), p)
            dts.append(time.perf_counter() - t0)
            st, g = r.state, r.graph
            flows.append(r.flow_value)
        out[f"threads_{thr}"] = {"static_ms": round(1e3 * st_s, 1), "static_rounds": prior.rounds,
                                 "static_flow": prior.flow_value,
                                 "dynamic_ms_per_batch": round(1e3 * float(np.mean(dts)), 1),
                                 "flows": flows}
    return out


# ---------------------------------------------------------------------------
def main():
    args = parse()
    maybe_relaunch(args)
    rank, world, dev, pg, backend = dist_setup()
    cfg = args.config
    if cfg == "auto":
        cfg = "C5" if world > 1 else "C4"
    if args.dry_run:
        barrier(pg, backend, dev)
        t = max_over_ranks(pg, backend, float(rank + 1), dev)
        if rank == 0:
            print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "config": cfg,
                              "backend": backend, "max_over_ranks_check": t}), flush=True)
        return
    if args.impl == "reference":
        if rank == 0:
            if cfg == "C5":
                print(json.dumps({"impl": "reference", "unavailable":
                                  "the reference's numpy build_bicsr cannot hold the 2.1 B-slot "
                                  "C5 graph (SURVEY 6.2); C5 parity = dynamic vs GPU static "
                                  "re-solve"}))
            else:
                bench_reference(args, cfg, world)
        return
    if cfg == "C5" and (world > 1 or args.engine == "part"):
        bench_c5(args, rank, world, dev, pg, backend)
        return
    out = bench_ours(args, cfg, rank, world, dev, pg, backend)
    if rank == 0:
        emit_ours(args, out, world)


if __name__ == "__main__":
    main()
