"""bench.py's multi-GPU launcher on CPU (gloo): --gpus N without WORLD_SIZE
re-launches itself under torch.distributed.run with N ranks (127.0.0.1);
the ranks shard a 256-vector batch, time with a barrier and take the max
over ranks; rank 0 alone prints the JSON line."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + list(args), capture_output=True,
                       text=True, timeout=240, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return lines


@pytest.mark.parametrize("n", [1, 2])
def test_launcher_spawns_ranks(n):
    lines = _run("--gpus", str(n), "--dry-run")
    assert len(lines) == 1, lines             # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["items"] == 256
    assert d["checksum"] == sum(range(256))


def test_launcher_rejects_world_mismatch():
    env = {k: v for k, v in os.environ.items()}
    env.update(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stdout + r.stderr)
