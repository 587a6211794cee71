"""bench.py's multi-rank plumbing: ``--gpus N`` re-launches
itself as N torchrun ranks, every rank joins the process group (gloo
without GPUs), timing is max-over-ranks, and rank 0 alone prints one JSON
line naming N.  The engine path of the same launch runs in
tests/test_gpu_bench.py on a GPU box."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_self_launch_dry_run():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "C5",
           "--scale", "12", "--dry-run"]
    p = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    if p.returncode != 0:  # one retry: the free port can be taken before torchrun binds it
        first = p.stderr[-2000:]
        p = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
        assert p.returncode == 0, (first, p.stderr[-2000:])
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"] == "C5" and d["backend"] == "gloo"
    assert d["max_over_ranks_check"] == 2.0
