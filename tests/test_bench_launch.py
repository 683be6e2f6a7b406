"""bench.py's multi-GPU launch path on CPU: `--gpus 2` without WORLD_SIZE re-launches itself under
torch.distributed.run (one rank per GPU, 127.0.0.1 rendezvous); every rank must see world == --gpus,
and rank 0 alone prints one JSON line with the max over ranks (`--dry-run`: gloo, no FMM)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, env=env, cwd=ROOT)


def test_bench_relaunches_one_rank_per_gpu():
    r = _run(["--gpus", "2", "--dry-run", "--steps", "3", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 2 and d["ranks_seen"] == 2 and d["steps"] == 3


def test_bench_single_rank_unchanged():
    r = _run(["--gpus", "1", "--dry-run", "--steps", "2", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["n_gpus"] == 1
