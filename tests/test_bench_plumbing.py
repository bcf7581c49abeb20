"""bench.py's multi-rank plumbing on CPU (gloo): `--gpus N` outside torchrun
self-launches N ranks (torch.distributed.run, 127.0.0.1), every rank checks
WORLD_SIZE == --gpus, and the max-over-ranks reduction reaches rank 0, which
alone prints the JSON line (the GPU arm uses the same
dist_init / barrier / max_over_ranks with NCCL)."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], cwd=REPO,
                       env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return lines


def test_self_launch_two_ranks():
    lines = _run("--gpus", "2", "--plumbing-check")
    assert len(lines) == 1  # rank 0 only
    out = json.loads(lines[0])
    assert out == {"n_gpus": 2, "max_over_ranks": 2.0}


def test_single_rank_no_launch():
    lines = _run("--gpus", "1", "--plumbing-check")
    assert json.loads(lines[0]) == {"n_gpus": 1, "max_over_ranks": 1.0}
