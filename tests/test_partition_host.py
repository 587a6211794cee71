"""Host-side logic of the partitioned engine (no GPU): slot-balanced vertex
ranges, batch routing, per-part error merging with the reference's precedence,
and the torch.distributed group (gloo, world_size 2) that carries the IPC
blobs and the per-phase all-reduces of the multi-GPU run."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as tmp

from paper_2511_01235_b200 import gen
from paper_2511_01235_b200.partition import (NONE, LocalGroup, balanced_bounds, batch_exception,
                                             combine_errors, route)


def test_balanced_bounds_cover_and_balance():
    us, vs, caps, s, t = gen.rmat_graph(12, 16, 0)
    n = 1 << 12
    for P in (1, 2, 3, 4, 8):
        b = balanced_bounds(n, us, vs, P)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) > 0)
        w = np.bincount(us, minlength=n) + np.bincount(vs, minlength=n) + 1
        per = np.add.reduceat(w, b[:-1])
        assert per.max() <= per.sum() / P + w.max()  # within one row of the ideal split


def test_balanced_bounds_rejects_bad_counts():
    with pytest.raises(ValueError):
        balanced_bounds(4, [0], [1], 9)
    with pytest.raises(ValueError):
        balanced_bounds(2, [0], [1], 3)


def test_route_by_tail_vertex():
    b = np.array([0, 3, 7, 10], np.int64)
    us = np.array([0, 2, 3, 6, 7, 9, -1, 10], np.int64)
    assert route(b, us).tolist() == [0, 0, 1, 1, 2, 2, -1, -1]


def test_combine_errors_precedence():
    a = np.array([5, NONE, 40, 7, NONE, NONE, NONE, NONE], np.int64)
    b = np.array([NONE, 3, 12, 9, 2, NONE, NONE, NONE], np.int64)
    e = combine_errors([a, b])
    assert e[0] == 5 and e[1] == 3 and e[4] == 2
    assert (e[2], e[3]) == (12, 9)  # duplicate on the globally smallest slot


def test_batch_exception_texts():
    from paper_2511_01235_b200 import BatchError
    us, vs, caps = [0, 1], [1, 3], [2, -1]
    none = np.full(8, NONE, np.int64)
    e = none.copy()
    e[0] = 1
    x = batch_exception(e, us, vs, caps)
    assert isinstance(x, BatchError) and str(x) == "update 1 (1->3): negative capacity -1"
    e = none.copy()
    e[1] = 0
    assert str(batch_exception(e, us, vs, caps)) == (
        "update 0 targets edge 0->1 which is not an edge of the original graph")
    e = none.copy()
    e[3] = 1
    assert str(batch_exception(e, us, vs, caps)) == "duplicate update for edge 1->3"
    assert batch_exception(none, us, vs, caps) is None


def test_local_group_is_identity():
    g = LocalGroup(3)
    assert g.local_ranks == [0, 1, 2] and g.devices == [0, 0, 0]
    assert g.allreduce(np.array([1, 2])).tolist() == [1, 2]
    assert g.allgather({"x": 1}) == [{"x": 1}]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, q):
    import torch.distributed as dist

    from paper_2511_01235_b200.partition import TorchGroup
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    g = TorchGroup()
    out = {
        "ranks": (g.rank, g.nparts, g.local_ranks),
        "sum": g.allreduce(np.array([rank + 1, 10 * rank], np.int64), "sum").tolist(),
        "max": g.allreduce(np.array([rank, -rank], np.int64), "max").tolist(),
        "min": g.allreduce(np.array([rank, NONE if rank else 5], np.int64), "min").tolist(),
        "gather": g.allgather({rank: [rank, rank * 2]}),
    }
    # error merge across ranks exactly as PartitionedGraph.solve_dynamic does
    local = np.array([NONE, 4 + rank, 30 - rank, 100 + rank, NONE, NONE, NONE, NONE], np.int64)
    red = g.allreduce(local[[0, 1, 2, 4]], "min")
    dupk = g.allreduce(np.array([local[3] if local[2] == red[2] else NONE]), "min")
    out["err"] = [int(red[0]), int(red[1]), int(red[2]), int(dupk[0]), int(red[3])]
    g.barrier()
    dist.destroy_process_group()
    q.put((rank, out))


def test_torch_group_gloo_world2():
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        o = res[r]
        assert o["ranks"] == (r, 2, [r])
        assert o["sum"] == [3, 10]
        assert o["max"] == [1, 0]
        assert o["min"] == [0, 5]
        assert o["gather"] == [{0: [0, 0]}, {1: [1, 2]}]
        assert o["err"] == [NONE, 4, 29, 101, NONE]
