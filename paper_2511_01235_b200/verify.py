"""Device-side certificate and constraint checks (oracle.py:111-225 run as
one GPU pass; csrc/state.cu verify_kernel)."""

import ctypes
from dataclasses import dataclass

from . import _lib as L


@dataclass
class GpuReport:
    ok: bool
    problems: list
    counts: dict


def verify_gpu(st, g, claimed_flow: int | None = None) -> GpuReport:
    """Capacity (0 <= f <= cap), residual-pair conservation, excess identity
    (excess[u] == sum over u's slots of cf - cap0), sum of excess == 0, no
    active vertex, A->B saturated, B->A unloaded, s in A, t in B, and
    cut capacity == flow at the bases (== claimed_flow if given)."""
    rep = L.VerifyReport()
    L.check(L.load().mfx_verify(st.handle, g.handle, ctypes.byref(rep)))
    c = rep.as_dict()
    problems = []
    for key, label in (("negative_cf", "negative residuals"),
                       ("pair_violations", "residual-sum conservation violations"),
                       ("excess_mismatch", "excess != constructed imbalance"),
                       ("active_vertices", "active vertices remain"),
                       ("unsaturated_ab", "A->B edges not saturated"),
                       ("loaded_ba", "B->A edges carry flow"),
                       ("source_in_b", "source is not on cut side A"),
                       ("sink_in_a", "sink is not on cut side B")):
        if c[key]:
            problems.append(f"{c[key]} {label}")
    if c["excess_sum"] != 0:
        problems.append(f"sum of excess is {c['excess_sum']}, not 0")
    if c["cut_capacity"] != c["flow_at_bases"]:
        problems.append(f"cut capacity {c['cut_capacity']} != flow {c['flow_at_bases']}")
    if claimed_flow is not None and c["cut_capacity"] != claimed_flow:
        problems.append(f"cut capacity {c['cut_capacity']} != claimed flow {claimed_flow}")
    return GpuReport(not problems, problems, c)
