"""Pins of the diffusion oracle (oracle/diffusion.py) against what the step rule and the
mathematics fix (reading R22), independent of the oracle's own code path."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import diffusion as D

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "diffusion_impulse.tsv")


def test_hand_derived_impulse_two_steps():
    rows = [l.split() for l in open(GOLDEN) if l.strip() and not l.startswith("#")]
    g = np.zeros((7, 7), np.uint32)
    g[3, 3] = 1 << 20
    for steps in (1, 2):
        exp = np.zeros((7, 7), np.int64)
        for s, dy, dx, v in rows:
            if int(s) == steps:
                exp[3 + int(dy), 3 + int(dx)] = int(v)
        got = D.diffuse([g], [1 << 30], steps)[0]
        np.testing.assert_array_equal(got.astype(np.int64), exp)


@pytest.mark.parametrize("seed", range(6))
def test_mass_balance_closed_form(seed):
    """sum(v') = sum(v) - sum over cells of share(v) x (number of its neighbours outside the grid):
    everything else a cell sends is received by an interior neighbour."""
    rng = np.random.default_rng(seed)
    h, w = int(rng.integers(1, 40)), int(rng.integers(1, 40))
    v = rng.integers(0, 1 << 31, size=(h, w), dtype=np.uint64)
    a = int(rng.integers(0, (1 << 30) + 1))
    out = D.step(v, a)
    s = (v * np.uint64(a)) >> np.uint64(32)
    outside = np.zeros((h, w), np.uint64)
    outside[0, :] += 1
    outside[-1, :] += 1
    outside[:, 0] += 1
    outside[:, -1] += 1
    assert int(out.sum()) == int(v.sum()) - int((s * outside).sum())


def test_symmetries_of_the_square_and_transpose():
    rng = np.random.default_rng(3)
    g = np.zeros((21, 21), np.uint32)
    g[10, 10] = 123456789
    out = D.diffuse([g], [D.rate_fixed(0.2)], 9)[0]
    for t in (out.T, out[::-1], out[:, ::-1], np.rot90(out)):
        np.testing.assert_array_equal(out, t)
    v = rng.integers(0, 1 << 28, size=(9, 14), dtype=np.uint64).astype(np.uint32)
    a = D.rate_fixed(0.13)
    np.testing.assert_array_equal(D.diffuse([v.T], [a], 3)[0], D.diffuse([v], [a], 3)[0].T)
    np.testing.assert_array_equal(D.diffuse([v[::-1, ::-1]], [a], 3)[0], D.diffuse([v], [a], 3)[0][::-1, ::-1])


def test_uniform_interior_is_a_fixed_point_and_degenerate_grids():
    v = np.full((12, 12), 1000, np.uint32)
    a = D.rate_fixed(0.25)
    out = D.diffuse([v], [a], 1)[0]
    assert (out[1:-1, 1:-1] == 1000).all()          # each interior cell sends and receives 4 x 250
    assert out[0, 0] == 1000 - 2 * 250 and out[0, 5] == 1000 - 250
    one = np.array([[4000]], np.uint32)              # 1 x 1: all four shares leave the grid
    assert D.diffuse([one], [a], 1)[0][0, 0] == 0
    assert D.diffuse([one], [D.rate_fixed(0.1)], 1)[0][0, 0] == 4000 - 4 * 399
    row = np.array([[0, 800, 0]], np.uint32)         # 1 x 3: up / down neighbours are padding
    np.testing.assert_array_equal(D.diffuse([row], [a], 1)[0], [[200, 0, 200]])
    assert D.diffuse([np.zeros((0, 5), np.uint32)], [a], 3)[0].shape == (0, 5)


def test_linearity_when_shares_are_exact():
    """With a = 2^30 and every value a multiple of 4, share(v) = v / 4 exactly, so one step is
    linear: D(u + w) = D(u) + D(w)."""
    rng = np.random.default_rng(5)
    u = 4 * rng.integers(0, 1 << 26, size=(10, 13), dtype=np.uint64)
    w = 4 * rng.integers(0, 1 << 26, size=(10, 13), dtype=np.uint64)
    a = 1 << 30
    np.testing.assert_array_equal(D.step(u + w, a), D.step(u, a) + D.step(w, a))


def test_rate_zero_is_identity_and_rates_are_validated():
    v = np.arange(30, dtype=np.uint32).reshape(5, 6)
    np.testing.assert_array_equal(D.diffuse([v], [0], 4)[0], v)
    with pytest.raises(ValueError):
        D.rate_fixed(0.3)
    with pytest.raises(ValueError):
        D.step(v, (1 << 30) + 1)
