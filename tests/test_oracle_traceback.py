"""Pins of the oracle's alignment path (reading R20).

The definition: for a pair with S > 0 the path is an optimal GLOBAL affine
alignment of A = q[q_start..q_end] and B = r[r_start..r_end] (its score is S),
and among those the one whose op string read from the end is lexicographically
greatest with M > I > D (SPEC.md:395/464 diagonal > up > left; 'I' = query
residue against a gap, 'D' = reference residue against a gap).

Independent checks (no dynamic programming here): brute-force enumeration of
every global op string of the tiny substrings, an independent affine re-score,
and the consumed lengths.
"""
from __future__ import annotations

import itertools

import numpy as np
import pytest

import oracle

DNA = {"alphabet": "dna", "match": 3, "mismatch": -3, "gap_open": -6, "gap_extend": -1}
SCORINGS = [
    DNA,
    {"alphabet": "dna", "match": 2, "mismatch": -2, "gap_open": -1, "gap_extend": -1},   # linear (Fig. 2)
    {"alphabet": "dna", "match": 1, "mismatch": -1, "gap_open": -3, "gap_extend": -1},
    {"alphabet": "dna", "match": 5, "mismatch": -4, "gap_open": -10, "gap_extend": -1},
]
RANK = {"M": 2, "I": 1, "D": 0}


def sigma(sc, a: int, b: int) -> int:
    if sc["alphabet"] == "dna":
        return sc["match"] if chr(a).upper() == chr(b).upper() else sc["mismatch"]
    return oracle.blosum62(chr(a), chr(b))


def rescore(ops: str, A: bytes, B: bytes, sc) -> int:
    """Affine score of an op string (each maximal I or D run costs o + (k-1) e; reading R1/R4)."""
    i = j = 0
    total = 0
    k = 0
    while k < len(ops):
        op = ops[k]
        if op == "M":
            total += sigma(sc, A[i], B[j]); i += 1; j += 1; k += 1
            continue
        t = k
        while t < len(ops) and ops[t] == op:
            t += 1
        run = t - k
        total += sc["gap_open"] + (run - 1) * sc["gap_extend"]
        if op == "I":
            i += run
        else:
            j += run
        k = t
    assert i == len(A) and j == len(B)
    return total


def all_global(a: int, b: int):
    """Every op string aligning a query residues with b reference residues."""
    out = []

    def rec(i, j, acc):
        if i == a and j == b:
            out.append("".join(acc))
            return
        if i < a and j < b:
            acc.append("M"); rec(i + 1, j + 1, acc); acc.pop()
        if i < a:
            acc.append("I"); rec(i + 1, j, acc); acc.pop()
        if j < b:
            acc.append("D"); rec(i, j + 1, acc); acc.pop()

    rec(0, 0, [])
    return out


def brute_path(A: bytes, B: bytes, sc):
    best, chosen = None, None
    for ops in all_global(len(A), len(B)):
        s = rescore(ops, A, B, sc)
        key = [RANK[c] for c in reversed(ops)]
        if best is None or s > best or (s == best and key > [RANK[c] for c in reversed(chosen)]):
            best, chosen = s, ops
    return best, chosen


def pick(rng, letters: bytes, k: int) -> bytes:
    return np.frombuffer(letters, np.uint8)[rng.integers(0, len(letters), k)].tobytes()


def substrings(q: bytes, r: bytes, res):
    S, qe, re_, qs, rs = res
    return q[qs:qe + 1], r[rs:re_ + 1]


@pytest.mark.parametrize("sc", SCORINGS)
def test_traceback_equals_brute_force_tie_rule(sc):
    """Exhaustive tiny pairs over {A, C}, then random ACGT: the oracle path is the optimal
    global alignment of the reported interval with the reverse-lexicographic M > I > D rule."""
    pairs = []
    for n in range(1, 5):
        for m in range(1, 5):
            for q in itertools.product(b"AC", repeat=n):
                for r in itertools.product(b"AC", repeat=m):
                    pairs.append((bytes(q), bytes(r)))
    rng = np.random.default_rng(7)
    for _ in range(300):
        n, m = int(rng.integers(1, 8)), int(rng.integers(1, 8))
        pairs.append((pick(rng, b"ACGT", n), pick(rng, b"ACGT", m)))
    checked = 0
    for q, r in pairs:
        res = oracle.align(q, r, sc)
        ops = oracle.traceback(q, r, sc, res)
        if res[0] == 0:
            assert ops == ""
            continue
        A, B = substrings(q, r, res)
        if len(A) + len(B) > 12:
            continue
        best, chosen = brute_path(A, B, sc)
        assert best == res[0], (q, r, res, best)
        assert ops == chosen, (q, r, res, ops, chosen)
        checked += 1
    assert checked > 500


@pytest.mark.parametrize("alphabet", ["dna", "protein"])
def test_traceback_rescores_to_S_and_spans_the_interval(alphabet):
    """Larger random pairs (related and unrelated): the path re-scores to S, consumes exactly the
    reported interval, and starts and ends with an aligned pair."""
    rng = np.random.default_rng(11)
    letters = b"ACGT" if alphabet == "dna" else b"ARNDCQEGHILKMFPSTWYV"
    scs = [DNA, SCORINGS[1]] if alphabet == "dna" else [{"alphabet": "protein", "gap_open": -11, "gap_extend": -1},
                                                        {"alphabet": "protein", "gap_open": -5, "gap_extend": -2}]
    for sc in scs:
        for k in range(150):
            n, m = int(rng.integers(1, 70)), int(rng.integers(1, 90))
            q = pick(rng, letters, n)
            if k % 2 and m > 10:
                s0 = int(rng.integers(0, max(1, m - n)))
                mut = bytearray(q)
                for t in range(len(mut)):
                    if rng.random() < 0.1:
                        mut[t] = int(rng.choice(list(letters)))
                r = pick(rng, letters, s0) + bytes(mut)[: m - s0]
            else:
                r = pick(rng, letters, m)
            res = oracle.align(q, r, sc)
            ops = oracle.traceback(q, r, sc, res)
            if res[0] == 0:
                assert ops == ""
                continue
            A, B = substrings(q, r, res)
            assert ops.count("M") + ops.count("I") == len(A)
            assert ops.count("M") + ops.count("D") == len(B)
            assert ops[0] == "M" and ops[-1] == "M"
            assert rescore(ops, A, B, sc) == res[0]


def test_traceback_sentinels_and_cigar():
    assert oracle.traceback(b"ACGT", b"TTTT", DNA) in ("", "M")  # S = 3 (one T) or 0
    assert oracle.traceback(b"AXGT", b"ACGT", DNA) is None       # invalid symbol
    assert oracle.traceback(b"", b"ACGT", DNA) == ""
    ops = oracle.traceback(b"ACGTACGT", b"ACGTTACGT", DNA)
    assert oracle.cigar(ops) == "3M1D5M"                         # the extra T against a gap, leftmost
    assert oracle.cigar("MMMIIDM") == "3M2I1D1M"
