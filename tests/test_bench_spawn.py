"""bench.py's multi-process plumbing on CPU: `bench.py --gpus N` without a
torchrun environment must start N ranks itself (one process per GPU on the
GPU box), rendezvous on 127.0.0.1, take the max over ranks and have rank 0
print the one JSON line with the real world size. The `plumbing` workload
does no GPU work, so this runs here with gloo."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("n", [1, 2])
def test_bench_spawns_n_ranks(n):
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["WF_BENCH_BACKEND"] = "gloo"
    proc = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--gpus", str(n), "--steps", "3", "--warmup", "3",
         "--workload", "plumbing"],
        capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr[-2000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, proc.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["world_size"] == n
    assert d["rank_sum"] == n * (n - 1) // 2  # every rank took part
    assert d["steps"] == 3 and d["warmup"] == 3
