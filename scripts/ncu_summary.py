"""Summarise one `ncu --set full` capture of the solve kernel into
profiles/ncu_<CONFIG>_solve_kernel.json (read by bench.py as roofline.traffic
when its src_hash matches the current kernel sources) and print the key
lines.  Runs here (ncu -i needs no GPU).

    python scripts/ncu_summary.py gpurun_out/prof_C4_dyn.ncu-rep --config C4
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum": "global_atomics",
}


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
            "GB": 1e9}[unit]
    return float(v.replace(",", "")) * mult


def to_ns(v, unit):
    return float(v.replace(",", "")) * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3,
                                         "msecond": 1e6, "ms": 1e6, "second": 1e9,
                                         "s": 1e9}[unit]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--config", required=True)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(head)}
    got = {}
    for k, name in KEYS.items():
        if k in col:
            got[name] = (vals[col[k]], units[col[k]])
    dur_ns = to_ns(*got["duration"])
    rd = to_bytes(*got["dram_read"])
    wr = to_bytes(*got["dram_write"])
    from bench import kernel_source_hash
    out = {
        "config": a.config, "kernel": vals[col["Kernel Name"]] if "Kernel Name" in col else None,
        "capture": os.path.basename(a.rep),
        "selection": "first solve_kernel launch inside NVTX range 'timed' of "
                     "`bench.py --config %s --profile --steps 1 --warmup 3` "
                     "(= the first timed batch of the bench, after 3 warm-up batches)" % a.config,
        "src_hash": kernel_source_hash(),
        "duration_ms": dur_ns / 1e6,
        "dram_bytes_read": rd, "dram_bytes_write": wr,
        "dram_bytes_per_launch": rd + wr,
        "dram_gbs": (rd + wr) / dur_ns,
    }
    for name in ("achieved_occupancy_pct", "threads_per_inst", "ipc", "registers", "grid",
                 "block", "l2_hit_pct", "dram_pct_of_peak", "global_atomics"):
        if name in got:
            try:
                out[name] = float(got[name][0].replace(",", ""))
            except ValueError:
                out[name] = got[name][0]
    path = a.out or os.path.join(ROOT, "profiles", f"ncu_{a.config}_solve_kernel.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
