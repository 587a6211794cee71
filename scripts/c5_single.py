"""C5 (R-MAT 26, ~2.1 B Bi-CSR slots) on the single-GPU engine (diagnostics):
the slot count fits the int32 layout (< 2^31 - 1), so one B200 holds the
whole graph.  Device generator -> device build -> static solve -> chained
dynamic batches (plain and push-pull) of k updates drawn on the device from
the generated edges (distinct (u, v), new caps U[0, 200]).

    python scripts/c5_single.py [--scale 26] [--batch 1000000] [--batches 3]
"""
import argparse
import ctypes
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_01235_b200 as mfx  # noqa: E402
from paper_2511_01235_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--batch", type=int, default=1_000_000)
ap.add_argument("--batches", type=int, default=3)
a = ap.parse_args()
n = 1 << a.scale
m = n * 16
lib = L.load()
e = [torch.empty(m, dtype=torch.int64, device="cuda:0") for _ in range(3)]
s, t = ctypes.c_int64(), ctypes.c_int64()
L.check(lib.mfx_rmat_device(a.scale, 16, 0, 0.57, 0.19, 0.19, 0, e[0].data_ptr(), e[1].data_ptr(),
                            e[2].data_ptr(), ctypes.byref(s), ctypes.byref(t)))
torch.cuda.synchronize()
t0 = time.perf_counter()
g = mfx.build_bicsr_device(n, e[0].data_ptr(), e[1].data_ptr(), e[2].data_ptr(), m)
torch.cuda.synchronize()
print(f"build {time.perf_counter() - t0:.1f} s: n {g.n} slots {g.m} (int32 limit 2147483647) "
      f"cap bytes {g.cap_bytes}", flush=True)
print(f"device memory in use {torch.cuda.memory_allocated() / 1e9:.1f} GB (torch)", flush=True)
for rep in range(2):
    r = mfx.solve_static(g, s.value, t.value)
    d = r.device
    print(f"static: flow {r.flow_value} rounds {r.rounds} {d['ms_total']:.1f} ms (bfs "
          f"{d['ns_bfs'] / 1e6:.1f} in {d['bfs_levels']} levels, push {d['ns_push'] / 1e6:.1f} in "
          f"{d['waves']} waves, repair {d['ns_repair'] / 1e6:.1f})", flush=True)
st = r.state
us, vs = e[0], e[1]
keep = us != vs
us, vs = us[keep], vs[keep]
gen = torch.Generator(device="cuda:0")
for mode in ("plain", "pushpull"):
    g2, st2 = g.copy(), st.copy()
    for b in range(a.batches):
        gen.manual_seed(1000 + b)
        idx = torch.randint(0, us.numel(), (2 * a.batch,), device="cuda:0", generator=gen)
        key = torch.unique(us[idx] * n + vs[idx])[: a.batch]
        key = key[torch.randperm(key.numel(), device="cuda:0", generator=gen)]
        bu, bv = key // n, key % n
        bc = torch.randint(0, 201, (key.numel(),), device="cuda:0", dtype=torch.int64, generator=gen)
        torch.cuda.synchronize()
        if mode == "plain":
            rr = mfx.solve_dynamic_device(st2, g2, key.numel(), bu.data_ptr(), bv.data_ptr(),
                                          bc.data_ptr())
        else:
            rr = mfx.solve_dynamic_pushpull(st2, g2, mfx.UpdateBatch(bu.cpu().numpy(), bv.cpu().numpy(),
                                                                      bc.cpu().numpy()))
        d = rr.device
        print(f"{mode} batch {b}: flow {rr.flow_value} rounds {rr.rounds} {d['ms_total']:.1f} ms "
              f"(update {d['ms_update']:.1f}, bfs {d['ns_bfs'] / 1e6:.1f} in {d['bfs_levels']} levels, "
              f"push {d['ns_push'] / 1e6:.1f} in {d['waves']} waves, repair {d['ns_repair'] / 1e6:.1f})",
              flush=True)
        st2 = rr.state
    rs = mfx.resolve_static(g2, mfx.init_residuals(g2, s.value, t.value))
    print(f"{mode}: static re-solve flow {rs.flow_value} {rs.device['ms_total']:.1f} ms "
          f"(agrees: {rs.flow_value == rr.flow_value})", flush=True)
