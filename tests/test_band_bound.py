"""The reverse pass's diagonal band (`rev_band` in sw_common.cuh) holds every cell
of every score-S alignment path: a CPU check by brute force, independent of the GPU.

Claim: every optimal local alignment ending at the chosen end (q_end, r_end) (reading R5) lies, in the
reversed rectangle of n2 = q_end + 1 rows and m2 = r_end + 1 columns, on diagonals d = j' - i' with
    -DI <= d <= DD,  DI = (ms n2 - S - (|o| - |e|)) / (ms + |e|),
    DD = min((ms n2 - S - (|o| - |e|)) / |e|, (ms m2 - S - (|o| - |e|)) / (ms + |e|))
(clamped at 0; ms = the largest substitution score).  Here every op-string path of small pairs is
enumerated (the cells it visits: aligned pairs and gap cells), the optimal ones ending at the oracle's end
are kept, and their cells' diagonals are checked against the bound -- on random pairs, on pairs built to
sit exactly on the bound (one gap run of maximal length) and under scorings with e = 0 and o = e.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle


def rev_band(ms, go, ge, S, n2, m2):
    """DESIGN.md sec. 5.2 (go = -gap_open, ge = -gap_extend)."""
    slack = max(0, ms * n2 - S - (go - ge))
    slack_m = max(0, ms * m2 - S - (go - ge))
    di = slack // (ms + ge)
    dd = slack_m // (ms + ge)
    if ge > 0:
        dd = min(dd, slack // ge)
    return di, dd


def optimal_path_drifts(q, r, sc, S, qe, re_):
    """Min / max of (j - i) over the cells visited by any score-S path that ends at (qe, re_) with an
    aligned pair.  Exhaustive over start cells and op strings (tiny inputs only)."""
    ma, mm, o, e = sc["match"], sc["mismatch"], sc["gap_open"], sc["gap_extend"]
    lo, hi = [10 ** 9], [-10 ** 9]
    found = [0]

    def dfs(i, j, last, score, dmin, dmax):
        # (i, j): next unconsumed query / reference index; the current cell is (i - 1, j - 1)
        if last == "M" and i - 1 == qe and j - 1 == re_ and score == S:
            found[0] += 1
            lo[0] = min(lo[0], dmin)
            hi[0] = max(hi[0], dmax)
        if i > qe + 1 or j > re_ + 1:
            return
        if i <= qe and j <= re_:
            s = ma if q[i] == r[j] else mm
            d = j - i
            dfs(i + 1, j + 1, "M", score + s, min(dmin, d), max(dmax, d))
        if j <= re_:  # reference residue against a gap: cell (i - 1, j)
            d = j - (i - 1)
            dfs(i, j + 1, "H", score + (e if last == "H" else o), min(dmin, d), max(dmax, d))
        if i <= qe:   # query residue against a gap: cell (i, j - 1)
            d = (j - 1) - i
            dfs(i + 1, j, "V", score + (e if last == "V" else o), min(dmin, d), max(dmax, d))

    for i0 in range(qe + 1):
        for j0 in range(re_ + 1):
            s0 = ma if q[i0] == r[j0] else mm
            dfs(i0 + 1, j0 + 1, "M", s0, j0 - i0, j0 - i0)
    return found[0], lo[0], hi[0]


SCORINGS = [(3, -3, -6, -1), (2, -3, -5, -2), (1, -1, -2, 0), (5, -4, -4, -4), (2, -1, -3, -1)]


def _pairs(rng, count):
    A = np.array(list(b"ACGT"))
    out = []
    for t in range(count):
        n = int(rng.integers(2, 8))
        x = rng.choice(A, n)
        kind = t % 3
        if kind == 0:   # related, one gap run
            k = int(rng.integers(1, 3))
            c = int(rng.integers(1, n))
            if rng.random() < 0.5:
                q, r = x, np.concatenate([x[:c], rng.choice(A, k), x[c:]])
            else:
                q, r = np.concatenate([x[:c], rng.choice(A, k), x[c:]]), x
        elif kind == 1:  # random
            q, r = x, rng.choice(A, int(rng.integers(2, 8)))
        else:            # low entropy (many co-optimal paths)
            q, r = rng.choice(A[:2], n), rng.choice(A[:2], int(rng.integers(2, 8)))
        out.append((bytes(q[:8].tolist()), bytes(r[:8].tolist())))
    return out


@pytest.mark.parametrize("scoring", SCORINGS)
def test_band_holds_every_optimal_path(scoring):
    ma, mm, o, e = scoring
    sc = {"alphabet": "dna", "match": ma, "mismatch": mm, "gap_open": o, "gap_extend": e}
    rng = np.random.default_rng(7000 + ma * 31 - mm * 7 - o * 3 - e)
    checked = 0
    tight_hi = tight_lo = 0
    for q, r in _pairs(rng, 60):
        S, qe, re_, qs, rs = oracle.align(q, r, sc)
        if S <= 0:
            continue
        n2, m2 = qe + 1, re_ + 1
        di, dd = rev_band(ma, -o, -e, S, n2, m2)
        found, dmin, dmax = optimal_path_drifts(q, r, sc, S, qe, re_)
        assert found >= 1, (q, r, sc)
        # reversed coordinates: d' = (r_end - j) - (q_end - i) = (re_ - qe) - (j - i)
        lo_rev, hi_rev = (re_ - qe) - dmax, (re_ - qe) - dmin
        assert -di <= lo_rev and hi_rev <= dd, (q, r, sc, S, (qe, re_), (lo_rev, hi_rev), (-di, dd))
        tight_lo += lo_rev == -di
        tight_hi += hi_rev == dd
        checked += 1
    assert checked >= 30
    if e < 0 and o < e:
        assert tight_hi + tight_lo >= 1  # the bound is reached on this set (it is not loose by construction)
