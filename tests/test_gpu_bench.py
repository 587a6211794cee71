"""bench.py end to end on the GPU: the single-GPU line carries the contract
keys, and ``--gpus 2`` runs the C5 vertex-range partition as two ranks
(sharing the box's GPU through CUDA IPC, gloo collectives) and reports
n_gpus = 2 with dynamic flows equal to the static re-solve."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, timeout=900):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                       capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_single_gpu_line_contract():
    d = run(["--config", "C1", "--steps", "4", "--warmup", "3", "--cpu-cap-s", "5"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "roofline", "cpu_baseline",
              "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["higher_is_better"] is False
    assert d["e2e"]["same_batches_as_value"] and d["e2e"]["h2d_bytes_per_step"] == 24 * 1000
    assert d["roofline"]["achieved"] > 0 and 0 < d["roofline"]["frac"]
    assert d["gpu_launches"] > 0
    assert len(set(d["flows"])) >= 1


def test_bench_two_ranks_run_the_c5_partition():
    d = run(["--gpus", "2", "--config", "C5", "--scale", "12", "--steps", "2", "--warmup", "1",
             "--batch", "2000"])
    assert d["n_gpus"] == 2 and d["config"]["parts"] == 2
    assert d["resolve_agrees"] and len(d["flows"]) == 2
