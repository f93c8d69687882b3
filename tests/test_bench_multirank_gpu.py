"""The bench's N > 1 path (torchrun, cell-balanced shards, barriers, max-over-ranks timing, one
JSON line from rank 0) exercised end to end on one GPU: SW_BENCH_SHARED_GPU=1 puts both ranks on
cuda:0 over gloo.  The numbers of such a run are not measurements; the test checks the contract."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_on_one_gpu():
    """`python bench.py --gpus 2` without torchrun launches its own two ranks (self_launch); the
    workload is BASELINE configs[3] (c4, 4 M pairs) in two cell-balanced shards."""
    env = dict(os.environ, SW_BENCH_SHARED_GPU="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-extra",
           "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["warmup"] == 3 and d["scaling"] == "strong"
    assert "c4" in d["config"]["workload"] and d["config"]["pairs"] == 4_000_000
    assert d["config"]["shard_imbalance"] < 1.001 and d["status"]["bad_pairs"] == 0
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["matches_device_path"]
