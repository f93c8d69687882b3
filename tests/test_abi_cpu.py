"""C-ABI library checks that need no GPU: it builds, loads, exports every
symbol include/sw.h declares, and its host-only helpers behave."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2208_12350_b200 import _build, sw, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sw.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sw_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ("sw_init", "sw_align_batch", "sw_free"):
        assert name in syms


def test_library_builds_and_exports_every_declared_symbol():
    path = _build.build()
    lib = ctypes.CDLL(path)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(sw.EXPORTED)


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump -lelf {_build.LIB}").read()
    assert "sm_100a" in out


def test_status_strings():
    assert sw.status_string(0) == "SW_OK"
    assert sw.status_string(2) == "SW_ERR_INVALID_SCORING"
    assert sw.status_string(7) == "SW_ERR_INTERNAL"


def test_plan_shards_balances_cells():
    b = synth.generate("c1", 0, 500)
    cuts = sw.sw_plan_shards(b.q_offsets, b.r_offsets, 4)
    assert cuts[0] == 0 and cuts[-1] == 500 and np.all(np.diff(cuts) >= 0)
    n, m = b.lengths()
    cost = n * m
    parts = [cost[cuts[k]:cuts[k + 1]].sum() for k in range(4)]
    assert max(parts) / (sum(parts) / 4) < 1.01


def test_plan_shards_degenerate():
    qo = np.array([0, 0, 0], np.int64)
    ro = np.array([0, 5, 5], np.int64)
    cuts = sw.sw_plan_shards(qo, ro, 3)
    assert cuts[0] == 0 and cuts[-1] == 2 and np.all(np.diff(cuts) >= 0)
    cuts = sw.sw_plan_shards(np.zeros(1, np.int64), np.zeros(1, np.int64), 2)
    assert list(cuts) == [0, 0, 0]
    with pytest.raises(sw.SWError):
        sw.sw_plan_shards(qo, ro, 0)


def test_init_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    st = sw.load().sw_init(ctypes.byref(h), 0)
    assert st in (sw.SW_ERR_CUDA, sw.SW_ERR_INVALID_ARGUMENT)
    assert not h.value
