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


def simcov_declared():
    text = open(os.path.join(ROOT, "include", "simcov.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(simcov_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_simcov_symbol():
    from paper_2208_12350_b200 import simcov
    lib = ctypes.CDLL(_build.build())
    missing = [s for s in simcov_declared() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(simcov_declared()) == set(simcov.EXPORTED)


def test_simcov_host_helpers():
    """Padded layout (include/simcov.h): rows on 128 B, >= 4 zero words left, room for the
    right neighbour of the last 128-column strip; no device needed."""
    from paper_2208_12350_b200 import simcov
    for W in (0, 1, 5, 120, 127, 128, 129, 2500, 16384):
        p = simcov.simcov_grid_pitch(W)
        strips = -(-W // 128) * 128
        assert p % 32 == 0 and p >= strips + 8 and p - (strips + 8) < 32
        assert simcov.simcov_grid_words(7, W) == 9 * p
    assert simcov.simcov_grid_pitch(-1) == -1 and simcov.simcov_grid_words(-1, 3) == -1
    with pytest.raises(sw.SWError):
        simcov.simcov_set_schedule(simcov.SIMCOV_MAX_TBLOCK + 1)
    simcov.simcov_set_schedule(0)
    # argument errors are returned before anything touches a device
    with pytest.raises(sw.SWError):
        simcov.simcov_diffuse(None, None, 4, 4, 1, 4096, [0], 1)
    with pytest.raises(sw.SWError):
        simcov.simcov_diffuse(1 << 20, 2 << 20, 4, 4, 0, 4096, [0], 1)
