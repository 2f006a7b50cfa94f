"""bench.py launcher contract on CPU: `python bench.py --gpus N` outside
torchrun must re-execute itself with N ranks (gloo here, `--dry-run`: no
device work) and report n_gpus == N; the reference arm reports the same N
and runs on rank 0 only; a WORLD_SIZE that disagrees with --gpus fails."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env_extra=None, timeout=300):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    env.update(env_extra or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=timeout)
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    return p, lines


@pytest.mark.parametrize("n", [1, 2])
def test_spawn_dry_run(n):
    p, lines = run(["--gpus", str(n), "--steps", "3", "--warmup", "3", "--dry-run"])
    assert p.returncode == 0, p.stderr[-2000:]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == n and line["dry_run"] and line["ms_per_step"] >= 10.0 * n - 1.0


def test_spawn_reference_arm_reports_n():
    p, lines = run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--states", "20000"])
    assert p.returncode == 0, p.stderr[-2000:]
    assert len(lines) == 1, p.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_world_size_mismatch_fails():
    p, _ = run(["--gpus", "4", "--dry-run"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode != 0 and "WORLD_SIZE" in p.stderr
