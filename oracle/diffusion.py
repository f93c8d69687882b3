"""CPU oracle for the SIMCoV diffusion stencil on a zero-padded grid.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` leg may import this module; the product never imports it, and it imports
nothing from the product.

What it computes (sec. II-C task 4: "Virus and inflammatory signals diffuse from
established sites of infection to neighboring grid points"; sec. VI-D: the
neighbour reads of edge points go to "extra points of value 0" padded around the grid instead of
through boundary checks).  The paper gives neither the stencil nor its coefficients; the reading
used here is DESIGN.md R22 (after SPEC.md:437-445, "conservative stencil on the zero-padded
domain", fixed-point arithmetic, 4-neighbours):

* a field is an H x W grid of non-negative integer concentrations (uint32 on the GPU);
* the diffusion rate of a field is the fixed-point fraction a / 2^32 with 0 <= a <= 2^30
  (at most 1/4, so a cell never sends more than it holds);
* one step: every cell sends share(v) = floor(v * a / 2^32) to each of its 4 neighbours and
  keeps the rest, i.e. v' = v - 4 share(v) + sum of share over its 4 neighbours, where a
  neighbour outside the grid is a padding point of value 0 (sends nothing; what a cell sends
  to it leaves the grid -- the absorbing boundary the zero padding gives);
* the two SIMCoV fields (virions, inflammatory signal) diffuse independently, each with its
  own rate, the same step count.

Plain numpy in uint64 (no overflow: v < 2^32, a <= 2^30), one step at a time, written as the
definition above.
"""
from __future__ import annotations

import numpy as np

MAX_RATE = 1 << 30


def rate_fixed(r: float) -> int:
    """Fixed-point rate a = floor(r * 2^32) for a fraction 0 <= r <= 1/4."""
    a = int(np.floor(r * 4294967296.0))
    if not 0 <= a <= MAX_RATE:
        raise ValueError("rate must lie in [0, 1/4]")
    return a


def share(v: np.ndarray, a: int) -> np.ndarray:
    """floor(v * a / 2^32), elementwise, in uint64."""
    return (v.astype(np.uint64) * np.uint64(a)) >> np.uint64(32)


def step(v: np.ndarray, a: int) -> np.ndarray:
    """One diffusion step of one H x W field (reading R22)."""
    if not 0 <= a <= MAX_RATE:
        raise ValueError("rate must lie in [0, 2^30]")
    v = v.astype(np.uint64)
    h, w = v.shape
    s = share(v, a)
    p = np.zeros((h + 2, w + 2), dtype=np.uint64)  # the zero padding ring
    p[1:-1, 1:-1] = s
    received = p[:-2, 1:-1] + p[2:, 1:-1] + p[1:-1, :-2] + p[1:-1, 2:]  # up, down, left, right
    return v - np.uint64(4) * s + received


def diffuse(fields, rates, steps: int):
    """`steps` steps of every field (list of H x W arrays) with its rate; returns uint32 arrays."""
    out = []
    for v, a in zip(fields, rates):
        x = np.asarray(v, dtype=np.uint64)
        for _ in range(int(steps)):
            x = step(x, int(a))
        if x.size and int(x.max()) >= 1 << 32:
            raise OverflowError("a concentration left the uint32 range")
        out.append(x.astype(np.uint32))
    return out
