"""Every-pair parity at BASELINE.json's full sizes.

c3 (50k protein pairs, ~1.4e10 cells) runs in every `-m gpu` session: the whole batch in one
sw_align_batch call, then the oracle on all host cores, all five fields of every pair.  c4 (4 M
pairs) and c5 (400k pairs up to 4096 x 16384) take minutes of oracle time: set SW_FULL_PARITY=1
(tools/parity_full.py runs the same check and records it, profiles/r08/parity_full.jsonl).
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_tool(key, tmp_path):
    out = tmp_path / f"parity_{key}.jsonl"
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "parity_full.py"), key, "--out", str(out)],
                   check=True, cwd=ROOT, timeout=3600)
    rec = json.loads(out.read_text().strip().splitlines()[-1])
    assert rec["pairs_checked"] == rec["pairs"]
    assert rec["total_mismatches"] == 0, rec
    assert rec["batch_status"] in ("SW_OK",), rec
    return rec


def test_c3_every_pair_full_size(tmp_path):
    run_tool("c3", tmp_path)


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("SW_FULL_PARITY") != "1", reason="minutes of oracle time: SW_FULL_PARITY=1")
@pytest.mark.parametrize("key", ["c4", "c5"])
def test_every_pair_full_size(key, tmp_path):
    run_tool(key, tmp_path)
