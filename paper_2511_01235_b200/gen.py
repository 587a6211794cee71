"""Synthetic instances and update batches for the five benchmark shapes.

Host-side input synthesis (numpy), not part of the solve path.

* :func:`random_graph` draws the same numbers, in the same order, as the
  reference's ``random_graph`` (reference bench.py:124-147), so config C1 is
  the reference's own instance.
* :func:`grid_graph`, :func:`rmat_graph`, :func:`road_graph` are the C2-C5
  shapes of SURVEY.md Appendix B.
* :func:`generate_batch` reproduces the reference's biased batch sampler
  (reference bench.py:66-121) draw for draw; :func:`fast_batch` has the same
  inc/dec/mixed/bias semantics with an O(m) weighted sampler
  (exponential-race keys) for graphs where ``rng.choice(p=...)`` is too slow.
"""

import math
import warnings
from dataclasses import dataclass

import numpy as np

KINDS = {"inc": "inc", "incremental": "inc", "dec": "dec", "decremental": "dec",
         "mixed": "mixed"}


@dataclass(frozen=True)
class BatchSpec:
    """Batch recipe: ``pct`` of the edges re-weighted, ``kind`` in
    inc/dec/mixed, ``bias`` = sampling weight of s-out / t-in edges
    (reference bench.py:30-56)."""

    pct: float
    kind: str
    seed: int
    bias: float = 10.0

    def canonical_kind(self) -> str:
        try:
            return KINDS[self.kind]
        except KeyError:
            raise ValueError(
                f"kind must be one of {sorted(set(KINDS))}, got {self.kind!r}") from None

    def validate(self) -> None:
        if not (0 < self.pct <= 100):
            raise ValueError(f"pct must be in (0, 100], got {self.pct}")
        if self.bias < 1:
            raise ValueError(f"bias must be >= 1, got {self.bias}")
        self.canonical_kind()


def pct_for_count(k: int, m: int) -> float:
    """Percentage that yields exactly ``k`` updates (ceil semantics of
    reference bench.py:84); naive ``100*k/m`` can round up to k+1."""
    return 100.0 * (k - 0.5) / m


# ----------------------------------------------------------------------------
# graphs
# ----------------------------------------------------------------------------

def random_edges(n: int, m: int, seed: int, cap_lo: int = 1, cap_hi: int = 100):
    """C1 generator; identical draws to reference bench.py:124-147.
    Returns ``(us, vs, caps, s, t)`` as int64 arrays (the array form of
    :func:`random_graph`)."""
    if n < 2:
        raise ValueError("need at least two vertices")
    rng = np.random.default_rng(seed)
    s, t = 0, n - 1
    forced = min(n - 1, max(1, m // 8), m // 2)
    out_heads = rng.integers(1, n, forced, dtype=np.int64)       # s -> *
    in_tails = rng.integers(0, n - 1, forced, dtype=np.int64)    # * -> t
    n_rand = m - 2 * forced
    rand_u = rng.integers(0, n, n_rand, dtype=np.int64)
    rand_v = rng.integers(0, n, n_rand, dtype=np.int64)
    us = np.concatenate([np.full(forced, s, np.int64), in_tails, rand_u])
    vs = np.concatenate([out_heads, np.full(forced, t, np.int64), rand_v])
    caps = rng.integers(cap_lo, cap_hi + 1, us.shape[0], dtype=np.int64)
    return us, vs, caps, s, t


def grid_graph(w: int, h: int, seed: int = 0):
    """C2: 4-neighbour grid, both directions, plus one terminal edge per
    pixel (s->p with prob 1/2 else p->t); caps U[1,100].  s = w*h,
    t = w*h+1."""
    rng = np.random.default_rng(seed)
    pix = np.arange(w * h, dtype=np.int64).reshape(h, w)
    s, t = w * h, w * h + 1
    blocks_u = [pix[:, :-1], pix[:, 1:], pix[:-1, :], pix[1:, :]]
    blocks_v = [pix[:, 1:], pix[:, :-1], pix[1:, :], pix[:-1, :]]
    us = [b.ravel() for b in blocks_u]
    vs = [b.ravel() for b in blocks_v]
    flat = pix.ravel()
    fg = rng.random(w * h) < 0.5
    us += [np.full(int(fg.sum()), s, np.int64), flat[~fg]]
    vs += [flat[fg], np.full(int((~fg).sum()), t, np.int64)]
    us = np.concatenate(us)
    vs = np.concatenate(vs)
    caps = rng.integers(1, 101, us.shape[0], dtype=np.int64)
    return us, vs, caps, s, t


def rmat_graph(scale: int, edge_factor: int = 16, seed: int = 0,
               a: float = 0.57, b: float = 0.19, c: float = 0.19):
    """C3/C5: R-MAT without label permutation; duplicates and self-loops left
    for the Bi-CSR build.  s = argmax out-degree, t = argmax in-degree != s."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    m = n * edge_factor
    us = np.zeros(m, np.int64)
    vs = np.zeros(m, np.int64)
    ab, abc = a + b, a + b + c
    for bit in range(scale):
        r = rng.random(m)
        us |= (r >= ab).astype(np.int64) << bit
        vs |= (((r >= a) & (r < ab)) | (r >= abc)).astype(np.int64) << bit
    caps = rng.integers(1, 101, m, dtype=np.int64)
    s = int(np.argmax(np.bincount(us, minlength=n)))
    indeg = np.bincount(vs, minlength=n).astype(np.int64)
    indeg[s] = -1
    t = int(np.argmax(indeg))
    return us, vs, caps, s, t


def road_graph(w: int, h: int, seed: int = 0, p_vert: float = 0.2):
    """C4: sparse lattice with every horizontal link and vertical links kept
    with probability ``p_vert`` (column 0 always kept), both directions;
    s = corner (0,0), t = opposite corner.  Long BFS depth (~w+h)."""
    rng = np.random.default_rng(seed)
    pix = np.arange(w * h, dtype=np.int64).reshape(h, w)
    keep = rng.random((h - 1, w)) < p_vert
    keep[:, 0] = True
    fu = np.concatenate([pix[:, :-1].ravel(), pix[:-1, :][keep]])
    fv = np.concatenate([pix[:, 1:].ravel(), pix[1:, :][keep]])
    us = np.concatenate([fu, fv])
    vs = np.concatenate([fv, fu])
    caps = rng.integers(1, 101, us.shape[0], dtype=np.int64)
    return us, vs, caps, 0, w * h - 1


def config_graph(name: str):
    """(n, us, vs, caps, s, t) for the named benchmark configuration."""
    if name == "C1":
        us, vs, caps, s, t = random_edges(10000, 100000, seed=0)
        return 10000, us, vs, caps, s, t
    if name == "C2":
        us, vs, caps, s, t = grid_graph(2048, 2048, seed=0)
        return 2048 * 2048 + 2, us, vs, caps, s, t
    if name == "C3":
        us, vs, caps, s, t = rmat_graph(20, 16, seed=0)
        return 1 << 20, us, vs, caps, s, t
    if name == "C4":
        us, vs, caps, s, t = road_graph(4900, 4900, seed=0, p_vert=0.21)
        return 4900 * 4900, us, vs, caps, s, t
    raise ValueError(f"unknown config {name!r}")


# ----------------------------------------------------------------------------
# batches
# ----------------------------------------------------------------------------

def _check_normalized(n, us, vs):
    keys = us * np.int64(n) + vs
    if np.unique(keys).size != us.size:
        raise ValueError("batch generation expects a normalized edge list "
                         "(unique directed pairs)")


def _inc(rng, old):
    return rng.integers(old + 1, 2 * old + 11, dtype=np.int64)


def _dec(rng, old):
    return rng.integers(np.zeros_like(old), old, dtype=np.int64)


def _choice(rng, pool, weights, k):
    if k == 0:
        return np.empty(0, np.int64)
    w = weights[pool]
    return rng.choice(pool, size=k, replace=False, p=w / w.sum()).astype(np.int64)


def batch_arrays(n, us, vs, caps, s, t, spec: BatchSpec):
    """Draw-for-draw reproduction of the reference sampler
    (reference bench.py:66-121) on edge arrays.  Returns (us, vs, new_caps,
    pick) sorted by (u, v); ``pick`` indexes the input edge list.  Raises
    ValueError on a non-normalized list (:func:`generate_batch` raises the
    reference's GraphError)."""
    spec.validate()
    kind = spec.canonical_kind()
    us, vs, caps = (np.asarray(a, np.int64) for a in (us, vs, caps))
    m = us.size
    if m == 0:
        e = np.empty(0, np.int64)
        return e, e, e, e
    _check_normalized(n, us, vs)
    k = math.ceil(spec.pct * m / 100)
    if k > m:
        warnings.warn(f"batch of {k} updates clamped to the {m} existing edges")
        k = m
    weights = np.ones(m)
    weights[(us == s) | (vs == t)] *= spec.bias
    rng = np.random.default_rng(spec.seed)
    every = np.arange(m, dtype=np.int64)
    positive = np.flatnonzero(caps > 0)
    if kind == "inc":
        pick = _choice(rng, every, weights, k)
        new = _inc(rng, caps[pick])
    elif kind == "dec":
        if positive.size < k:
            warnings.warn(f"decremental batch clamped to the {positive.size} "
                          f"positive-capacity edges")
            k = positive.size
        pick = _choice(rng, positive, weights, k)
        new = _dec(rng, caps[pick])
    else:
        n_dec = min(k // 2, positive.size)
        dec_pick = _choice(rng, positive, weights, n_dec)
        remaining = np.setdiff1d(every, dec_pick)
        n_inc = min(k - n_dec, remaining.size)
        inc_pick = _choice(rng, remaining, weights, n_inc)
        pick = np.concatenate([dec_pick, inc_pick])
        new = np.concatenate([_dec(rng, caps[dec_pick]), _inc(rng, caps[inc_pick])])
    order = np.lexsort((vs[pick], us[pick]))
    pick = pick[order]
    return us[pick], vs[pick], new[order], pick


def fast_batch(n, us, vs, caps, s, t, k: int, kind: str = "mixed", seed: int = 0,
               bias: float = 10.0):
    """Same semantics as :func:`generate_batch` for exactly ``k`` updates,
    sampling without replacement by exponential-race keys (E_i / w_i,
    smallest first), which is distributed like sequential weighted draws.
    O(m); meant for the multi-million-edge configs."""
    kind = KINDS[kind]
    us, vs, caps = (np.asarray(a, np.int64) for a in (us, vs, caps))
    m = us.size
    k = min(k, m)
    rng = np.random.default_rng(seed)
    w = np.ones(m)
    w[(us == s) | (vs == t)] = bias
    race = rng.exponential(size=m) / w
    positive = caps > 0

    def smallest(mask, cnt):
        idx = np.flatnonzero(mask)
        cnt = min(cnt, idx.size)
        if cnt == 0:
            return np.empty(0, np.int64)
        part = np.argpartition(race[idx], cnt - 1)[:cnt]
        return idx[part]

    if kind == "inc":
        pick = smallest(np.ones(m, bool), k)
        new = _inc(rng, caps[pick])
    elif kind == "dec":
        pick = smallest(positive, k)
        new = _dec(rng, caps[pick])
    else:
        dec_pick = smallest(positive, k // 2)
        rest = np.ones(m, bool)
        rest[dec_pick] = False
        inc_pick = smallest(rest, k - dec_pick.size)
        pick = np.concatenate([dec_pick, inc_pick])
        new = np.concatenate([_dec(rng, caps[dec_pick]), _inc(rng, caps[inc_pick])])
    order = np.lexsort((vs[pick], us[pick]))
    pick = pick[order]
    return us[pick], vs[pick], new[order], pick



def _race_smallest(rng, m, excluded, heavy, bias, cnt):
    """The ``cnt`` smallest exponential-race keys E_i / w_i over the edges
    [0, m) minus ``excluded`` (sorted; weight 1) plus ``heavy`` (weight
    ``bias``), without a key per light edge: the positions of the j smallest
    of M iid Exp(1) keys form a uniform random subset, and their values are
    the order statistics sum_{i<=j} E_i / (M - i + 1)."""
    M = m - excluded.size
    c = min(cnt, M)
    if c:
        ranks = rng.choice(M, size=c, replace=False).astype(np.int64)
        # rank among the non-excluded edges -> edge index
        shift = excluded - np.arange(excluded.size, dtype=np.int64)
        light = ranks + np.searchsorted(shift, ranks, side="right")
        vals = np.cumsum(rng.exponential(size=c) / (M - np.arange(c, dtype=np.float64)))
    else:
        light, vals = np.empty(0, np.int64), np.empty(0)
    idx = np.concatenate([light, heavy])
    key = np.concatenate([vals, rng.exponential(size=heavy.size) / bias])
    take = min(cnt, idx.size)
    return idx[np.argsort(key, kind="stable")[:take]]


def sparse_batch(n, us, vs, caps, s, t, k: int, kind: str = "mixed", seed: int = 0,
                 bias: float = 10.0):
    """:func:`fast_batch`'s law (the reference generate_batch semantics,
    bench.py:66-121: k distinct edges drawn with weight ``bias`` on s-out /
    t-in edges, half decrements on positive edges and half increments on
    the rest) from O(k + |heavy|) random draws plus a few O(m) masks, for
    the 58 M-edge C4 chains.  A different random stream from fast_batch."""
    kind = KINDS[kind]
    us, vs, caps = (np.asarray(a, np.int64) for a in (us, vs, caps))
    m = us.size
    k = min(k, m)
    rng = np.random.default_rng(seed)
    heavy = np.flatnonzero((us == s) | (vs == t))
    dec_pick = np.empty(0, np.int64)
    if kind in ("dec", "mixed"):
        zero = np.flatnonzero(caps <= 0)
        excl = np.union1d(heavy, zero)
        hpos = heavy[caps[heavy] > 0]
        dec_pick = _race_smallest(rng, m, excl, hpos, bias, k if kind == "dec" else k // 2)
    if kind == "dec":
        pick = dec_pick
        new = _dec(rng, caps[pick])
    else:
        excl = np.union1d(heavy, dec_pick)
        hrest = np.setdiff1d(heavy, dec_pick, assume_unique=True)
        inc_pick = _race_smallest(rng, m, excl, hrest, bias, k - dec_pick.size)
        pick = np.concatenate([dec_pick, inc_pick])
        new = np.concatenate([_dec(rng, caps[dec_pick]), _inc(rng, caps[inc_pick])])
    order = np.lexsort((vs[pick], us[pick]))
    pick = pick[order]
    return us[pick], vs[pick], new[order], pick


# ----------------------------------------------------------------------------
# reference-signature entry points (reference bench.py:66-147)
# ----------------------------------------------------------------------------

def random_graph(n: int, m: int, seed: int, cap_lo: int = 1, cap_hi: int = 100):
    """Reference ``random_graph`` (bench.py:124-147): returns
    ``(EdgeListGraph, s, t)`` with identical draws."""
    from .graph import EdgeListGraph
    us, vs, caps, s, t = random_edges(n, m, seed, cap_lo, cap_hi)
    return EdgeListGraph(n, us, vs, caps), s, t


def generate_batch(g, s: int, t: int, spec: BatchSpec):
    """Reference ``generate_batch`` (bench.py:66-121): ``g`` is a normalized
    EdgeListGraph (e.g. ``BiCsrGraph.to_edge_list()``); returns an
    UpdateBatch, draw for draw the reference's; GraphError on a
    non-normalized list."""
    from .dynamic import UpdateBatch
    from .graph import GraphError
    try:
        bu, bv, bc, _ = batch_arrays(g.n, g.us, g.vs, g.caps, s, t, spec)
    except ValueError as e:
        if "normalized" in str(e):
            raise GraphError("generate_batch expects a normalized edge list "
                             "(unique directed pairs)") from None
        raise
    return UpdateBatch(bu, bv, bc)


def source_edges(name: str, args):
    """Edge arrays of a named generator as recorded in the golden fixtures
    (``random_graph`` there means the reference generator's draws)."""
    if name == "random_graph":
        return random_edges(*args)
    return globals()[name](*args)


def device_sample_batch(g, s: int, t: int, k: int, kind: str = "mixed", seed: int = 0,
                        bias: float = 10.0):
    """:func:`fast_batch` semantics drawn on the device from ``g``'s own
    capacities (csrc/state.cu sample_batch; the partitioned engine's sampler
    law): for graphs whose edge list is too large to sample on the host (C5:
    1.07 B edges).  Returns host arrays (us, vs, new_caps) in (u, v) order."""
    import ctypes

    from . import _lib as L
    kind_ = KINDS[kind]
    k_dec = k if kind_ == "dec" else 0 if kind_ == "inc" else k // 2
    k_inc = k - k_dec
    us, vs, cs = (np.empty(k, np.int64) for _ in range(3))
    got = ctypes.c_int64()
    L.check(L.load().mfx_sample_batch(g.handle, int(s), int(t), k_dec, k_inc, int(seed),
                                      float(bias), L.ptr64(us), L.ptr64(vs), L.ptr64(cs),
                                      ctypes.byref(got)))
    n = got.value
    order = np.lexsort((vs[:n], us[:n]))  # (the two kinds come out one after the other)
    return us[:n][order], vs[:n][order], cs[:n][order]
