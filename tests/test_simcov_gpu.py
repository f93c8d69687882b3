"""Parity of the CUDA diffusion stencil (include/simcov.h) with the
CPU oracle (oracle/diffusion.py, reading R22).

Everything is integer: the bar is bit-exact equality of every cell of every field.  Inputs
come from paper_2208_12350_b200.synth (no diffusion arithmetic there); the oracle is called
only here.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import diffusion as D
from paper_2208_12350_b200 import simcov, synth

pytestmark = pytest.mark.gpu

SCHEDULES = (0, 1, 2, 3, 4, 8)


@pytest.fixture(autouse=True)
def _reset_schedule():
    yield
    simcov.simcov_set_schedule(0)


def run_gpu(fields, rates, steps, schedule=0):
    H, W = fields[0].shape
    g = simcov.Grid(H, W, len(fields))
    g.upload(fields)
    simcov.simcov_set_schedule(schedule)
    g.diffuse(rates, steps)
    out = g.download()
    pad = g.padded()
    # the padding ring stays zero ("extra points of value 0")
    inner = np.zeros_like(pad, dtype=bool)
    inner[:, 1:H + 1, 4:4 + W] = True
    assert not pad[~inner].any(), "padding word written"
    return out


def assert_fields_equal(got, exp):
    for f, (a, b) in enumerate(zip(got, exp)):
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)
            y, x = bad[0]
            raise AssertionError(f"field {f}: {len(bad)} cells differ; first ({y}, {x}): gpu={a[y, x]} oracle={b[y, x]}")


@pytest.mark.parametrize("schedule", SCHEDULES)
@pytest.mark.parametrize("H,W", [(1, 1), (1, 7), (9, 1), (5, 130), (67, 121), (130, 250), (200, 371)])
def test_parity_small_grids(H, W, schedule):
    fields = synth.simcov_dense(H * 1000 + W, H, W, 2, high=1 << 30)
    rates = [simcov.rate_fixed(0.1), simcov.SIMCOV_MAX_RATE]
    for steps in (1, 2, 5):
        assert_fields_equal(run_gpu(fields, rates, steps, schedule), D.diffuse(fields, rates, steps))


@pytest.mark.parametrize("schedule", SCHEDULES)
def test_parity_step_counts(schedule):
    """Every remainder of the launch plan (k-step launches, parity split, odd-count copy back)."""
    fields = synth.simcov_fields(3, 150, 260, 2, sites=40, peak=1 << 28, background=0.05)
    rates = [simcov.rate_fixed(0.2), simcov.rate_fixed(0.05)]
    for steps in (0, 1, 2, 3, 4, 6, 7, 9, 13):
        assert_fields_equal(run_gpu(fields, rates, steps, schedule), D.diffuse(fields, rates, steps))


def test_parity_many_fields_and_rates():
    fields = synth.simcov_dense(11, 97, 301, 8, high=1 << 31)
    rates = [0, 1, 12345, simcov.rate_fixed(0.01), simcov.rate_fixed(0.125), simcov.rate_fixed(0.25) - 1,
             simcov.SIMCOV_MAX_RATE, 1 << 29]
    assert_fields_equal(run_gpu(fields, rates, 6), D.diffuse(fields, rates, 6))


def test_heldout_grid_full_parity():
    """The paper's held-out size (2500 x 2500), both fields, every cell."""
    H, W = synth.SIMCOV_HELDOUT
    fields = synth.simcov_fields(1, H, W, 2, peak=1 << 26, background=0.02)
    rates = [simcov.rate_fixed(0.2), simcov.rate_fixed(0.1)]
    assert_fields_equal(run_gpu(fields, rates, 10), D.diffuse(fields, rates, 10))


def test_large_grid_sampled_windows_and_mass_balance():
    """Bench-sized grid: windows checked against the oracle through the dependency cone
    (a cell after s steps depends only on cells within distance s), plus the closed-form
    mass balance of a single step (what leaves is exactly the edge cells' outward shares)."""
    import torch
    H, W, steps = 8192, 8192, 8
    fields = synth.simcov_fields(5, H, W, 2, peak=1 << 26, background=0.05)
    rates = [simcov.rate_fixed(0.2), simcov.rate_fixed(0.1)]
    out = run_gpu(fields, rates, steps)
    rng = np.random.default_rng(0)
    wins = [(0, 0), (H - 40, W - 40), (0, W - 40), (H - 40, 0)] + \
        [(int(rng.integers(0, H - 40)), int(rng.integers(0, W - 40))) for _ in range(8)]
    for y0, x0 in wins:
        ya, xa = max(0, y0 - steps), max(0, x0 - steps)
        yb, xb = min(H, y0 + 40 + steps), min(W, x0 + 40 + steps)
        sub = [f[ya:yb, xa:xb] for f in fields]
        exp = D.diffuse(sub, rates, steps)
        for f in range(2):
            got = out[f][y0:y0 + 40, x0:x0 + 40]
            want = exp[f][y0 - ya:y0 - ya + 40, x0 - xa:x0 - xa + 40]
            # window edges that are not grid edges are only exact `steps` cells inside
            lo_y = 0 if ya == 0 else max(0, steps - (y0 - ya))
            lo_x = 0 if xa == 0 else max(0, steps - (x0 - xa))
            hi_y = 40 if yb == H else 40 - max(0, steps - (yb - (y0 + 40)))
            hi_x = 40 if xb == W else 40 - max(0, steps - (xb - (x0 + 40)))
            assert np.array_equal(got[lo_y:hi_y, lo_x:hi_x], want[lo_y:hi_y, lo_x:hi_x]), (f, y0, x0)
    one = run_gpu(fields, rates, 1)
    for f in range(2):
        v = fields[f].astype(np.uint64)
        s = (v * np.uint64(rates[f])) >> np.uint64(32)
        leak = int(s[0, :].sum() + s[-1, :].sum() + s[:, 0].sum() + s[:, -1].sum())
        assert int(one[f].astype(np.uint64).sum()) == int(v.sum()) - leak
    del torch


def test_schedules_agree_bitwise():
    fields = synth.simcov_fields(9, 777, 1023, 2, peak=1 << 30, background=0.1)
    rates = [simcov.rate_fixed(0.24), simcov.rate_fixed(0.07)]
    ref = run_gpu(fields, rates, 11, 1)
    for sch in (0, 2, 3, 4):
        assert_fields_equal(run_gpu(fields, rates, 11, sch), ref)


def test_launch_plan_counts():
    fields = synth.simcov_fields(2, 64, 64, 1)
    g = simcov.Grid(64, 64, 1)
    g.upload(fields)
    simcov.simcov_set_schedule(4)
    g.diffuse([simcov.rate_fixed(0.1)], 16)
    assert simcov.simcov_last_launch_count() == 2 + 4  # ring zeroing x2, four 4-step launches
    g.diffuse([simcov.rate_fixed(0.1)], 5)
    assert simcov.simcov_last_launch_count() == 2 + 2  # (4, 1)
    simcov.simcov_set_schedule(0)
    g.diffuse([simcov.rate_fixed(0.1)], 16)
    assert simcov.simcov_last_launch_count() == 2 + 2  # default: (8, 8)
    g.diffuse([simcov.rate_fixed(0.1)], 5)
    assert simcov.simcov_last_launch_count() == 2 + 2  # 5 -> (2, 3): an even count ends in grid
    g.diffuse([simcov.rate_fixed(0.1)], 1)
    assert simcov.simcov_last_launch_count() == 2 + 1  # one step, then a copy back (not a kernel)


def test_argument_errors():
    g = simcov.Grid(16, 16, 1)
    with pytest.raises(simcov.sw.SWError):
        simcov.simcov_diffuse(g.grid.data_ptr(), g.scratch.data_ptr(), 16, 16, 1, g.field_stride,
                              [simcov.SIMCOV_MAX_RATE + 1], 1)
    with pytest.raises(simcov.sw.SWError):
        simcov.simcov_diffuse(g.grid.data_ptr(), g.grid.data_ptr(), 16, 16, 1, g.field_stride, [0], 1)
    with pytest.raises(simcov.sw.SWError):
        simcov.simcov_diffuse(g.grid.data_ptr(), g.scratch.data_ptr(), 16, 16, 1, g.field_stride - 4, [0], 1)
    with pytest.raises(simcov.sw.SWError):
        simcov.simcov_diffuse(g.grid.data_ptr() + 4, g.scratch.data_ptr(), 16, 16, 1, g.field_stride, [0], 1)
