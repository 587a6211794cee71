"""The reference's structural verifiers and independent max-flow checks,
re-exported under the reference names (reference __init__.py:12-14,
oracle.py:20-258) so code written against ``dynmaxflow`` finds them.

They are correctness tools, not the solve path: they run on host arrays
(the device state is downloaded lazily), with the reference's report types
and message texts.  The constraint checks of a terminated solve also run on
the device as :func:`~paper_2511_01235_b200.verify.verify_gpu`.
"""

from dataclasses import dataclass

import numpy as np

from .graph import BiCsrGraph, EdgeListGraph
from .solver import CutCertificate
from .state import SolverState


@dataclass
class ConstructedFlow:
    """Per-slot flow recovered from residuals (oracle.py:104-108)."""

    f: np.ndarray


@dataclass
class PreflowReport:
    ok: bool
    problems: list
    imbalance: np.ndarray


@dataclass
class CutReport:
    ok: bool
    problems: list


@dataclass
class DistanceLabels:
    d: np.ndarray


def _i64(a):
    return np.asarray(a, dtype=np.int64)


def construct_flow(st: SolverState, g: BiCsrGraph) -> ConstructedFlow:
    """f = max(0, cap0 - cf) per slot; rejects a state whose pair sums are
    not conserved (oracle.py:111-123)."""
    cf, cap0, rev = _i64(st.cf), _i64(g.cap0), _i64(g.rev)
    bad = np.flatnonzero(cf + cf[rev] != cap0 + cap0[rev])
    if bad.size:
        i = int(bad[0])
        src, adj = g.src, g.adj
        raise ValueError(f"residual-sum conservation violated on edge slot {i} "
                         f"({int(src[i])}->{int(adj[i])}); state corrupt")
    return ConstructedFlow(np.maximum(cap0 - cf, 0))


def verify_preflow(flow: ConstructedFlow, g: BiCsrGraph, s: int, t: int,
                   expected_excess=None) -> PreflowReport:
    """Capacity bounds and per-vertex imbalance (oracle.py:133-172)."""
    problems = []
    f, cap0 = _i64(flow.f), _i64(g.cap0)
    over = np.flatnonzero(f > cap0)
    if over.size:
        i = int(over[0])
        problems.append(f"{over.size} edge(s) exceed capacity, first at slot {i}: "
                        f"f={int(f[i])} > cap={int(cap0[i])}")
    neg = np.flatnonzero(f < 0)
    if neg.size:
        problems.append(f"{neg.size} negative flow entries, first at slot {int(neg[0])}")
    n = g.n
    imbalance = _exact_imbalance(g, f)
    if expected_excess is not None:
        exp = _i64(expected_excess)
        bad = np.flatnonzero(imbalance != exp)
        if bad.size:
            v = int(bad[0])
            problems.append(f"{bad.size} vertices where imbalance differs from tracked "
                            f"excess, first v={v}: {int(imbalance[v])} != {int(exp[v])}")
    else:
        interior = np.ones(n, dtype=bool)
        interior[s] = interior[t] = False
        bad = np.flatnonzero(interior & (imbalance != 0))
        if bad.size:
            problems.append(f"conservation violated at {bad.size} interior vertices, "
                            f"first v={int(bad[0])}")
    return PreflowReport(not problems, problems, imbalance)


def _exact_imbalance(g, f):
    out = np.zeros(g.n, dtype=np.int64)
    np.add.at(out, _i64(g.adj), f)
    np.subtract.at(out, _i64(g.src), f)
    return out


def verify_cut(cert: CutCertificate, g: BiCsrGraph, st: SolverState,
               claimed_flow: int) -> CutReport:
    """Cut certificate against the claimed flow (oracle.py:182-225)."""
    problems = []
    a = np.asarray(cert.a_mask, dtype=bool)
    if not a[st.source]:
        problems.append("source is not on cut side A")
    if a[st.sink]:
        problems.append("sink is not on cut side B")
    src, adj, orig = _i64(g.src), _i64(g.adj), np.asarray(g.is_original, bool)
    cap0, cf = _i64(g.cap0), _i64(st.cf)
    crossing = orig & a[src] & ~a[adj]
    recomputed = int(cap0[crossing].sum())
    if recomputed != cert.cut_capacity:
        problems.append(f"stored cut capacity {cert.cut_capacity} != recomputed {recomputed}")
    if cert.cut_capacity != claimed_flow:
        problems.append(f"cut capacity {cert.cut_capacity} != claimed flow {claimed_flow}")
    unsat = np.flatnonzero(crossing & (cf != 0))
    if unsat.size:
        i = int(unsat[0])
        problems.append(f"{unsat.size} A->B edge(s) not saturated, first "
                        f"{int(src[i])}->{int(adj[i])} cf={int(cf[i])}")
    try:
        f = construct_flow(st, g).f
    except ValueError as exc:
        problems.append(str(exc))
    else:
        loaded = np.flatnonzero(orig & ~a[src] & a[adj] & (f != 0))
        if loaded.size:
            i = int(loaded[0])
            problems.append(f"{loaded.size} B->A edge(s) carry flow, first "
                            f"{int(src[i])}->{int(adj[i])} f={int(f[i])}")
    return CutReport(not problems, problems)


def residual_distances(st: SolverState, g: BiCsrGraph, bases) -> DistanceLabels:
    """Multi-source BFS distance to ``bases`` over residual edges in their
    flow direction (oracle.py:233-258), level-synchronous over numpy
    frontiers (independent of the device BFS)."""
    n = g.n
    off, adj, rev, cf = _i64(g.offsets), _i64(g.adj), _i64(g.rev), _i64(st.cf)
    d = np.full(n, n, dtype=np.int64)
    front = np.unique(_i64(bases))
    d[front] = 0
    level = 0
    while front.size:
        lo, hi = off[front], off[front + 1]
        cnt = hi - lo
        slots = np.repeat(lo - np.cumsum(np.r_[0, cnt[:-1]]), cnt) + np.arange(cnt.sum())
        v = adj[slots]
        ok = (d[v] == n) & (cf[rev[slots]] > 0)
        nxt = np.unique(v[ok])
        level += 1
        d[nxt] = level
        front = nxt
    return DistanceLabels(d)


def dinic_maxflow(g: EdgeListGraph, s: int, t: int) -> int:
    """Exact max-flow value by an independent blocking-flow solver (the role
    of oracle.py:20-55): scipy's Dinic on the edge list with parallel edges
    merged and self-loops dropped."""
    if s == t:
        raise ValueError("source and sink must differ")
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import maximum_flow
    us, vs, caps = _i64(g.us), _i64(g.vs), _i64(g.caps)
    keep = us != vs
    us, vs, caps = us[keep], vs[keep], caps[keep]
    if caps.size and int(caps.max()) >= 2 ** 31:
        raise ValueError("dinic_maxflow check supports capacities below 2^31")
    m = csr_matrix((caps.astype(np.int32), (us, vs)), shape=(g.n, g.n))
    m.sum_duplicates()
    if m.nnz == 0:
        return 0
    return int(maximum_flow(m, s, t, method="dinic").flow_value)


def exhaustive_min_cut(g: EdgeListGraph, s: int, t: int) -> int:
    """Minimum s-t cut by enumerating every bipartition of the free
    vertices (oracle.py:87-101); at most 20 free vertices."""
    free = np.array([v for v in range(g.n) if v != s and v != t], dtype=np.int64)
    if free.size > 20:
        raise ValueError("exhaustive cut enumeration limited to 20 free vertices")
    us, vs, caps = _i64(g.us), _i64(g.vs), _i64(g.caps)
    masks = np.arange(1 << free.size, dtype=np.int64)
    bit = np.full(g.n, -1, dtype=np.int64)
    bit[free] = np.arange(free.size)

    def side_a(x):  # per edge endpoint, per bipartition: in A?
        if x == s:
            return np.ones(masks.size, bool)
        if x == t:
            return np.zeros(masks.size, bool)
        return (masks >> bit[x]) & 1 == 1

    best = np.zeros(masks.size, dtype=np.int64)
    for u, v, c in zip(us.tolist(), vs.tolist(), caps.tolist()):
        best += np.where(side_a(u) & ~side_a(v), c, 0)
    return int(best.min())
