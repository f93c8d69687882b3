"""Brute-force enumeration of every local alignment (pin P1).

Independent of the oracle's dynamic programming: a local alignment is an
op-string over {M, I, D} that starts and ends with M; its score is the sum of
s(q_i, r_j) over the M columns plus, for every maximal run of k gap columns of
the same kind, gap_open + (k-1)*gap_extend (PAPER.md:161-163 scoring; affine
charge per PAPER.md:713-714, reading R1).  An I run directly followed
by a D run is two runs (reading R4).

For a shape (n, m) every op-string path is enumerated once; a pair's scores
are then (path x cell incidence) @ s + gap charge.  The optimal set follows the
C-6 definition:
  S     = max(0, best path score)
  end   = lexmin (r_end, q_end) over paths with score S
  start = lexmax (r_start, q_start) over paths with score S ending at `end`
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np


@lru_cache(maxsize=None)
def _paths(n: int, m: int):
    """All op-string paths in an n x m grid.

    Returns (inc, runs, gaplen, qs, rs, qe, re): inc is a (P, n*m) 0/1 matrix of
    aligned (M) cells, runs/gaplen the number of gap runs / gap columns.
    """
    rows_inc, runs_l, gap_l, qs_l, rs_l, qe_l, re_l = [], [], [], [], [], [], []

    def dfs(i, j, last, cells, runs, gaps, i0, j0):
        # state: next unconsumed query index i, reference index j; `last` op.
        if last == "M":
            rows_inc.append(tuple(cells)); runs_l.append(runs); gap_l.append(gaps)
            qs_l.append(i0); rs_l.append(j0); qe_l.append(i - 1); re_l.append(j - 1)
        if i < n and j < m:                                   # M
            cells.append(i * m + j)
            dfs(i + 1, j + 1, "M", cells, runs, gaps, i0, j0)
            cells.pop()
        if j < m:                                             # I: gap in query, consumes r_j
            dfs(i, j + 1, "I", cells, runs + (last != "I"), gaps + 1, i0, j0)
        if i < n:                                             # D: gap in reference, consumes q_i
            dfs(i + 1, j, "D", cells, runs + (last != "D"), gaps + 1, i0, j0)

    for i0 in range(n):
        for j0 in range(m):
            dfs(i0 + 1, j0 + 1, "M", [i0 * m + j0], 0, 0, i0, j0)
    P = len(rows_inc)
    inc = np.zeros((P, max(n * m, 1)), dtype=np.int64)
    for p, cells in enumerate(rows_inc):
        inc[p, list(cells)] = 1
    return (inc, np.array(runs_l, np.int64), np.array(gap_l, np.int64), np.array(qs_l, np.int64),
            np.array(rs_l, np.int64), np.array(qe_l, np.int64), np.array(re_l, np.int64))


def sigma_matrix(q: bytes, r: bytes, sigma) -> np.ndarray:
    return np.array([[sigma(a, b) for b in r] for a in q], dtype=np.int64).reshape(-1)


def optimal_set(q: bytes, r: bytes, sigma, gap_open: int, gap_extend: int):
    """(S, ends, starts_by_end) by enumeration. ends: set of (q_end, r_end) with score S."""
    n, m = len(q), len(r)
    if n == 0 or m == 0:
        return 0, set(), {}
    inc, runs, gaplen, qs, rs, qe, re = _paths(n, m)
    scores = inc @ sigma_matrix(q, r, sigma) + runs * gap_open + (gaplen - runs) * gap_extend
    best = int(scores.max())
    if best <= 0:
        return 0, set(), {}
    sel = np.nonzero(scores == best)[0]
    ends = {(int(qe[k]), int(re[k])) for k in sel}
    starts = {}
    for k in sel:
        starts.setdefault((int(qe[k]), int(re[k])), set()).add((int(qs[k]), int(rs[k])))
    return best, ends, starts


def align(q: bytes, r: bytes, sigma, gap_open: int, gap_extend: int):
    """(S, q_end, r_end, q_start, r_start) under the C-6 tie rules."""
    S, ends, starts = optimal_set(q, r, sigma, gap_open, gap_extend)
    if S == 0:
        return (0, -1, -1, -1, -1)
    qe, re = min(ends, key=lambda t: (t[1], t[0]))
    qs, rs = max(starts[(qe, re)], key=lambda t: (t[1], t[0]))
    return (S, qe, re, qs, rs)


def dna_sigma(match: int, mismatch: int):
    def s(a, b):
        return match if a == b else mismatch
    return s
