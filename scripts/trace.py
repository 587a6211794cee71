"""Per-barrier trace of one static and one dynamic C2 solve (diagnostics).

    MFX_TRACE_CAP=200000 python scripts/trace.py --side 2048
Prints a histogram of phase durations by work-list size.
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("MFX_TRACE_CAP", "200000")

import paper_2511_01235_b200 as mfx  # noqa: E402
from paper_2511_01235_b200 import _lib, gen  # noqa: E402

PH = {0: "bfs", 1: "push", 2: "repair", 3: "final"}


def fetch(st, g):
    cap = int(os.environ["MFX_TRACE_CAP"])
    buf = (ctypes.c_uint64 * cap)()
    cnt = ctypes.c_int64()
    _lib.check(_lib.load().mfx_trace_fetch(st.handle, g.handle, buf, cap, ctypes.byref(cnt)))
    a = np.frombuffer(buf, dtype=np.uint64, count=cnt.value).copy()
    return (a >> np.uint64(60)).astype(int), ((a >> np.uint64(32)) & np.uint64(0xFFFFFFF)).astype(int), \
        (a & np.uint64(0xFFFFFFFF)).astype(np.int64)


def report(tag, st, g, res):
    ph, items, dt = fetch(st, g)
    raw = ph == 7
    if raw.any():
        cap = int(os.environ["MFX_TRACE_CAP"])
        buf = (ctypes.c_uint64 * cap)()
        cnt = ctypes.c_int64()
        _lib.check(_lib.load().mfx_trace_fetch(st.handle, g.handle, buf, cap, ctypes.byref(cnt)))
        a = np.frombuffer(buf, dtype=np.uint64, count=cnt.value)[raw]
        states = (a >> np.uint64(56)) & np.uint64(0xF)
        d = (a >> np.uint64(28)) & np.uint64(0xFFFFFFF)
        t = a & np.uint64(0xFFFFFFF)
        print(f"  async phases: {raw.sum()}  end states {np.bincount(states.astype(int)).tolist()}")
        for i in range(min(12, len(a))):
            print(f"    state {int(states[i])} done {int(d[i])} tail {int(t[i])}")
        keep = ~raw
        ph, items, dt = ph[keep], items[keep], dt[keep]
    keep = (ph != 6) & (ph != 5) & (ph != 4) & (ph < 8)  # epoch stats / tail waves / CTA-0 wave work (rounds_view)
    ph, items, dt = ph[keep], items[keep], dt[keep]
    print(f"== {tag}: {res.device['ms_solve']:.2f} ms, rounds {res.rounds}, "
          f"levels {res.device['bfs_levels']}, waves {res.device['waves']}, barriers {len(ph)}")
    # item count of entry i is the work of the phase that ends at entry i+1
    work = np.concatenate([[0], items[:-1]])
    for p in (0, 1):
        m = ph == p
        if not m.any():
            continue
        w, d = work[m], dt[m] / 1e3
        print(f"  {PH[p]}: n={m.sum()} total {d.sum():.2f} ms, median {np.median(d):.1f} us")
        for lo, hi in ((0, 1), (1, 100), (100, 1000), (1000, 10000), (10000, 100000), (100000, 1 << 40)):
            k = (w >= lo) & (w < hi)
            if k.any():
                print(f"    items [{lo},{hi}): {k.sum():5d} phases, {d[k].sum():8.2f} ms, "
                      f"mean {d[k].mean():7.1f} us, items/phase {w[k].mean():9.0f}")


def rounds_view(tag, st, g):
    """Per round: BFS epochs + time (+ vertices expanded: sum / max per CTA,
    from the phase-6 entries), then the push waves' item counts."""
    ph, items, dt = fetch(st, g)
    keep = (ph != 7) & (ph < 8)  # (8, 9: relabel exit inputs)
    ph, items, dt = ph[keep], items[keep], dt[keep]
    # a phase-6 entry follows its epoch's barrier entry
    xs = {}
    tails = {}  # CTA-0 tail waves (items after the wave : us), by the barrier entry that follows
    work0 = {}  # CTA 0's own work time in a grid-wide wave, by that wave's barrier entry
    out = []
    pend = []
    for q in range(len(ph)):
        if ph[q] == 6:
            xs[len(out) - 1] = (int(dt[q]), int(items[q]))
        elif ph[q] == 5:
            pend.append(f"{int(items[q])}:{dt[q] / 1e3:.0f}")
        elif ph[q] == 4:
            work0[len(out)] = int(dt[q])
        else:
            if pend:
                tails[len(out)] = pend
                pend = []
            out.append(q)
    ph, items, dt = ph[out], items[out], dt[out]
    work = np.concatenate([[0], items[:-1]])
    print(f"-- {tag}: per-round sequence")
    i, rnd = 0, 0
    while i < len(ph):
        j = i
        while j < len(ph) and ph[j] == 0:
            j += 1
        bfs_us = dt[i:j].sum() / 1e3
        k = j
        while k < len(ph) and ph[k] == 1:
            k += 1
        waves = work[j:k]
        push_us = dt[j:k].sum() / 1e3
        rep = dt[k:k + 1].sum() / 1e3 if k < len(ph) and ph[k] == 2 else 0.0
        if i in work0:
            print(f"    seeding: CTA 0 busy {work0[i] / 1e3:.1f} us of {dt[i] / 1e3:.1f} us")
        ep = " ".join(f"{int(work[q])}:{dt[q] / 1e3:.0f}"
                      + (f"[{xs[q][0]}/{xs[q][1]}]" if q in xs else "") for q in range(i, j))
        print(f"    bfs epochs (items:us) {ep}")
        print(f"  round {rnd}: bfs {j - i} epochs {bfs_us:8.1f} us | {k - j} waves {push_us:8.1f} us "
              f"items first/max/last {waves[:1].tolist()}/{int(waves.max()) if len(waves) else 0}/"
              f"{waves[-1:].tolist()} | repair {rep:6.1f} us")
        w0 = [work0[q] for q in range(j, k) if q in work0]
        if w0:
            print(f"    grid waves: CTA 0 busy {np.mean(w0) / 1e3:.1f} us of {push_us / max(1, len(w0)):.1f} us per wave")
        tw = [w for q in range(j, k + 1) for w in tails.get(q, [])]
        if tw:
            print(f"    tail waves (items:us) {len(tw)}: " + " ".join(tw[:40]) + (" ..." if len(tw) > 40 else ""))
        i = k + (1 if k < len(ph) and ph[k] == 2 else 0)
        rnd += 1
        if j == i and k == j:
            break


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=2048)
    ap.add_argument("--max-waves", type=int, default=0)
    ap.add_argument("--graph", default="grid", choices=["grid", "road"])
    ap.add_argument("--static-only", action="store_true")
    args = ap.parse_args()
    if args.graph == "road":
        us, vs, caps, s, t = gen.road_graph(args.side, args.side, 0, 0.21)
        n = args.side * args.side
    else:
        us, vs, caps, s, t = gen.grid_graph(args.side, args.side, 0)
        n = args.side * args.side + 2
    g = mfx.build_bicsr(mfx.EdgeListGraph(n, us, vs, caps))
    p = mfx.SolverParams(max_waves=args.max_waves)
    mfx.solve_static(g, s, t, p)
    r = mfx.solve_static(g, s, t, p)
    report("static", r.state, g, r)
    if args.static_only:
        rounds_view("static", r.state, g)
        return
    el = g.to_edge_list()
    bu, bv, bc, _ = gen.fast_batch(n, el.us, el.vs, el.caps, s, t, 10000, "mixed", 0)
    rr = mfx.solve_dynamic(r.state, g, mfx.UpdateBatch(bu, bv, bc), p)
    report("dynamic", rr.state, g, rr)
    rounds_view("dynamic", rr.state, g)


if __name__ == "__main__":
    main()
