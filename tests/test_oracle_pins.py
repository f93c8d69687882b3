"""Pins of the CPU oracle against things other than itself (no GPU needed).

Each test names the SURVEY.md sec. 8(c) pin it implements.  Every independent
algorithm used here (brute-force enumeration, global Gotoh, linear-gap SW,
relu-form DP, Kadane, longest common substring, SPEC's traceback) is written
anew in this file or in tests/brute_force.py; none of them calls into the
oracle's arithmetic.
"""
from __future__ import annotations

import itertools
import os

import numpy as np
import pytest

import brute_force as bf
import oracle
from paper_2208_12350_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

SCORINGS_DNA = [(3, -3, -6, -1), (2, -2, -1, -1), (1, -1, -2, -1), (2, -1, -3, -1), (1, -1, -1, -1)]

BLOSUM_ORDER = "ARNDCQEGHILKMFPSTWYVBZX*"


def dna(match, mismatch, o, e):
    return oracle.scoring("dna", match, mismatch, o, e)


def prot(o=-11, e=-1):
    return oracle.scoring("protein", 0, 0, o, e)


def blosum_sigma():
    def s(a, b):
        return oracle.blosum62(chr(a), chr(b))
    return s


def rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def rand_seq(g, alpha: bytes, n: int) -> bytes:
    a = np.frombuffer(alpha, dtype=np.uint8)
    return a[g.integers(0, a.size, size=n)].tobytes()


# ----------------------------------------------------------------- goldens (P2)

def test_fig2_golden_matrix_and_score():
    lines = [l.split() for l in open(os.path.join(GOLDEN, "fig2_linear.txt")) if l.strip() and not l.startswith("#")]
    d = {}
    H = []
    for parts in lines:
        if parts[0] == "H":
            H.append([int(x) for x in parts[1:]])
        else:
            d[parts[0]] = parts[1:]
    sc = dna(*[int(x) for x in d["scoring"][1:]])
    q, r = d["query"][0], d["ref"][0]
    assert oracle.align(q, r, sc)[0] == int(d["score"][0])
    assert oracle.align(q, r, sc) == tuple(int(x) for x in d["result"])
    np.testing.assert_array_equal(oracle.fill_H(q, r, sc), np.array(H))


def _worked_rows():
    rows = []
    for l in open(os.path.join(GOLDEN, "worked_examples.tsv")):
        if l.startswith("#") or not l.strip():
            continue
        p = l.rstrip("\n").split("\t")
        rows.append((p[0], p[1], p[2], [int(x) for x in p[3:7]], tuple(int(x) for x in p[7:12])))
    return rows


@pytest.mark.parametrize("row", _worked_rows(), ids=lambda r: f"{r[0]}-{r[1]}")
def test_worked_examples(row):
    q, r, alpha, (ma, mm, o, e), expect = row
    sc = dna(ma, mm, o, e) if alpha == "dna" else prot(o, e)
    assert oracle.align(q, r, sc) == expect
    if len(q) <= 7 and len(r) <= 7:
        sigma = bf.dna_sigma(ma, mm) if alpha == "dna" else blosum_sigma()
        assert bf.align(q.encode(), r.encode(), sigma, o, e) == expect


# ------------------------------------------------------------ brute force (P1)

def _ac_strings(maxlen):
    for L in range(1, maxlen + 1):
        for t in itertools.product("AC", repeat=L):
            yield "".join(t)


@pytest.mark.parametrize("scoring", SCORINGS_DNA)
def test_bruteforce_exhaustive_two_letter(scoring):
    """All 30 x 30 pairs over {A,C}^{1..4} (P1, exhaustive part)."""
    ma, mm, o, e = scoring
    sc = dna(*scoring)
    sig = bf.dna_sigma(ma, mm)
    seqs = list(_ac_strings(4))
    for q in seqs:
        for r in seqs:
            assert oracle.align(q, r, sc) == bf.align(q.encode(), r.encode(), sig, o, e), (q, r, scoring)


def test_bruteforce_random_tiny_dna():
    """Seeded random pairs, n, m <= 6, alphabets {AC, ACG, ACGT}, five scorings (P1)."""
    g = rng(1)
    count = 0
    for alpha in (b"AC", b"ACG", b"ACGT"):
        for scoring in SCORINGS_DNA:
            ma, mm, o, e = scoring
            sc = dna(*scoring)
            sig = bf.dna_sigma(ma, mm)
            for _ in range(250):
                q = rand_seq(g, alpha, int(g.integers(1, 7)))
                r = rand_seq(g, alpha, int(g.integers(1, 7)))
                assert oracle.align(q, r, sc) == bf.align(q, r, sig, o, e), (q, r, scoring)
                count += 1
    assert count == 3750


def test_bruteforce_random_tiny_protein():
    g = rng(2)
    sig = blosum_sigma()
    for o, e in ((-11, -1), (-4, -2), (-3, -3)):
        sc = prot(o, e)
        for _ in range(200):
            q = rand_seq(g, b"ARNDCQEGHILKMFPSTWYVBZX*", int(g.integers(1, 6)))
            r = rand_seq(g, b"ARNDCQEGHILKMFPSTWYVBZX*", int(g.integers(1, 6)))
            assert oracle.align(q, r, sc) == bf.align(q, r, sig, o, e), (q, r, o, e)


def test_bruteforce_affine_vs_reopen():
    """Affine charge: a 3-gap must score o + 2e, not 3o (a dropped extend term fails this)."""
    sc = dna(10, -20, -5, -1)
    # ACGTTT vs ACG---TTT style: q = AAAAACCCCC, r = AAAAAGGGCCCCC (3 inserted Gs)
    q, r = b"AAAAACCCCC", b"AAAAAGGGCCCCC"
    S = oracle.align(q, r, sc)[0]
    assert S == 100 - 5 - 2  # ten matches, one gap run of length 3


# --------------------------------------------------------------- closed forms

def test_identity_closed_form():
    """P3: q == r -> S = sum s(a,a), end (n-1,n-1), start (0,0)."""
    g = rng(3)
    for (ma, mm, o, e) in SCORINGS_DNA:
        for n in (1, 2, 17, 150, 300):
            q = rand_seq(g, b"ACGT", n)
            assert oracle.align(q, q, dna(ma, mm, o, e)) == (ma * n, n - 1, n - 1, 0, 0)
    alpha = b"ARNDCQEGHILKMFPSTWYVBZ"  # X and * excluded
    for n in (1, 5, 64, 333):
        q = rand_seq(g, alpha, n)
        S = sum(oracle.blosum62(chr(c), chr(c)) for c in q)
        assert oracle.align(q, q, prot()) == (S, n - 1, n - 1, 0, 0)


def test_bounds_on_generated_batch():
    """P4: 0 <= S <= max_s * min(n, m); q_start <= q_end, r_start <= r_end."""
    b = synth.generate("c1", 0, 300)
    out = oracle.align_batch(b.queries, b.q_offsets, b.refs, b.r_offsets, synth.DNA_SCORING)
    n, m = b.lengths()
    assert np.all(out["score"] >= 0)
    assert np.all(out["score"] <= 3 * np.minimum(n, m))
    pos = out["score"] > 0
    assert np.all(out["q_start"][pos] <= out["q_end"][pos])
    assert np.all(out["r_start"][pos] <= out["r_end"][pos])
    assert np.all(out["q_end"][pos] < n[pos]) and np.all(out["r_end"][pos] < m[pos])


def global_gotoh(q: bytes, r: bytes, sigma, o: int, e: int) -> int:
    """Global affine alignment score (end gaps charged); independent re-scorer for P5."""
    NEG = -10 ** 9
    n, m = len(q), len(r)
    M = [[NEG] * (m + 1) for _ in range(n + 1)]
    X = [[NEG] * (m + 1) for _ in range(n + 1)]  # ends in gap consuming r
    Y = [[NEG] * (m + 1) for _ in range(n + 1)]  # ends in gap consuming q
    M[0][0] = 0
    for j in range(1, m + 1):
        X[0][j] = o + (j - 1) * e
    for i in range(1, n + 1):
        Y[i][0] = o + (i - 1) * e
    for i in range(1, n + 1):
        for j in range(1, m + 1):
            M[i][j] = max(M[i - 1][j - 1], X[i - 1][j - 1], Y[i - 1][j - 1]) + sigma(q[i - 1], r[j - 1])
            X[i][j] = max(M[i][j - 1] + o, Y[i][j - 1] + o, X[i][j - 1] + e)
            Y[i][j] = max(M[i - 1][j] + o, X[i - 1][j] + o, Y[i - 1][j] + e)
    return max(M[n][m], X[n][m], Y[n][m])


def test_global_rescore_of_reported_interval():
    """P5: global Gotoh of q[qs..qe] vs r[rs..re] equals S."""
    g = rng(5)
    for k in range(120):
        ma, mm, o, e = SCORINGS_DNA[k % len(SCORINGS_DNA)]
        q = rand_seq(g, b"ACGT", int(g.integers(5, 40)))
        r = rand_seq(g, b"ACGT", int(g.integers(5, 40)))
        if k % 2:
            r = r[:3] + q[2:-2] + r[3:]  # make it related
        S, qe, re, qs, rs = oracle.align(q, r, dna(ma, mm, o, e))
        if S == 0:
            continue
        assert global_gotoh(q[qs:qe + 1], r[rs:re + 1], bf.dna_sigma(ma, mm), o, e) == S
    sig = blosum_sigma()
    for k in range(40):
        q = rand_seq(g, b"ARNDCQEGHILKMFPSTWYV", int(g.integers(5, 30)))
        r = rand_seq(g, b"ARNDCQEGHILKMFPSTWYV", int(g.integers(5, 30)))
        r = r[:4] + q[3:] if k % 2 else r
        S, qe, re, qs, rs = oracle.align(q, r, prot())
        if S:
            assert global_gotoh(q[qs:qe + 1], r[rs:re + 1], sig, -11, -1) == S


def test_ungapped_kadane():
    """P6: with prohibitive gaps S = max over diagonals of Kadane's max-subarray of s."""
    g = rng(6)
    for _ in range(60):
        q = rand_seq(g, b"ACGT", int(g.integers(1, 50)))
        r = rand_seq(g, b"ACGT", int(g.integers(1, 50)))
        best = 0
        for d in range(-len(q) + 1, len(r)):
            run = 0
            for i in range(len(q)):
                j = i + d
                if 0 <= j < len(r):
                    run = max(0, run + (2 if q[i] == r[j] else -3))
                    best = max(best, run)
        assert oracle.align(q, r, dna(2, -3, -1000, -1000))[0] == best


def test_longest_common_substring():
    """P7: match 1, mismatch = o = e = -1000 -> S = longest common substring length."""
    g = rng(7)
    for _ in range(60):
        q = rand_seq(g, b"ACG", int(g.integers(1, 40)))
        r = rand_seq(g, b"ACG", int(g.integers(1, 40)))
        L = 0
        for i in range(len(q)):
            for j in range(len(r)):
                k = 0
                while i + k < len(q) and j + k < len(r) and q[i + k] == r[j + k]:
                    k += 1
                L = max(L, k)
        assert oracle.align(q, r, dna(1, -1000, -1000, -1000))[0] == L


COMP = bytes.maketrans(b"ACGT", b"TGCA")


def test_score_symmetries():
    """P8: S(q,r) = S(r,q) = S(rev q, rev r) = S(revcomp q, revcomp r)."""
    g = rng(8)
    for k in range(80):
        sc = dna(*SCORINGS_DNA[k % 5])
        q = rand_seq(g, b"ACGT", int(g.integers(1, 60)))
        r = rand_seq(g, b"ACGT", int(g.integers(1, 60)))
        S = oracle.align(q, r, sc)[0]
        assert oracle.align(r, q, sc)[0] == S
        assert oracle.align(q[::-1], r[::-1], sc)[0] == S
        assert oracle.align(q.translate(COMP)[::-1], r.translate(COMP)[::-1], sc)[0] == S
    for k in range(20):
        q = rand_seq(g, b"ARNDCQEGHILKMFPSTWYV", int(g.integers(1, 40)))
        r = rand_seq(g, b"ARNDCQEGHILKMFPSTWYV", int(g.integers(1, 40)))
        assert oracle.align(q, r, prot())[0] == oracle.align(r, q, prot())[0]


def spec_linear_sw(q: bytes, r: bytes, match: int, mismatch: int, gap: int):
    """SPEC.md:395 recurrence: H = max(0, diag + s, up + gap, left + gap)."""
    n, m = len(q), len(r)
    H = [[0] * (m + 1) for _ in range(n + 1)]
    for i in range(1, n + 1):
        for j in range(1, m + 1):
            s = match if q[i - 1] == r[j - 1] else mismatch
            H[i][j] = max(0, H[i - 1][j - 1] + s, H[i - 1][j] + gap, H[i][j - 1] + gap)
    return H


def test_linear_gap_matches_spec_recurrence():
    """P9: o == e reproduces SPEC's linear-gap sw_reference, whole H matrix."""
    g = rng(9)
    for k in range(60):
        ma, mm, gap = [(2, -2, -1), (3, -3, -2), (1, -1, -1)][k % 3]
        q = rand_seq(g, b"ACGT", int(g.integers(1, 30)))
        r = rand_seq(g, b"ACGT", int(g.integers(1, 30)))
        np.testing.assert_array_equal(oracle.fill_H(q, r, dna(ma, mm, gap, gap)),
                                      np.array(spec_linear_sw(q, r, ma, mm, gap)))


def test_monotonicity():
    """P10: S(q, r+x) >= S(q, r) and S(q, x+r) >= S(q, r)."""
    g = rng(10)
    sc = dna(3, -3, -6, -1)
    for _ in range(60):
        q = rand_seq(g, b"ACGT", int(g.integers(1, 40)))
        r = rand_seq(g, b"ACGT", int(g.integers(1, 40)))
        x = rand_seq(g, b"ACGT", int(g.integers(1, 10)))
        S = oracle.align(q, r, sc)[0]
        assert oracle.align(q, r + x, sc)[0] >= S
        assert oracle.align(q, x + r, sc)[0] >= S
        assert oracle.align(x + q, r, sc)[0] >= S


def test_degenerate_cases():
    """P12 and the per-pair error / S = 0 conventions (readings R7, R10, R16)."""
    sc = dna(3, -3, -6, -1)
    assert oracle.align("AAAA", "CCCC", sc) == (0, -1, -1, -1, -1)
    assert oracle.align("A", "A", sc) == (3, 0, 0, 0, 0)
    assert oracle.align("", "ACGT", sc) == (0, -1, -1, -1, -1)
    assert oracle.align("ACGT", "", sc) == (0, -1, -1, -1, -1)
    assert oracle.align("", "", sc) == (0, -1, -1, -1, -1)
    assert oracle.align("ACNT", "ACGT", sc) == (-1, -1, -1, -1, -1)
    assert oracle.align("ACGT", "ACGU", sc) == (-1, -1, -1, -1, -1)
    assert oracle.align("acgt", "ACGT", sc) == oracle.align("ACGT", "acgt", sc) == (12, 3, 3, 0, 0)
    assert oracle.align("HEAJ", "HEA", prot()) == (-1, -1, -1, -1, -1)
    assert oracle.align("heagawghee", "pawheae", prot()) == (17, 8, 4, 4, 1)


def relu_form_H(q: bytes, r: bytes, sigma, o: int, e: int, boundary: int):
    """P13: the kernel's form -- E, F relu-clamped at 0, boundary E/F = `boundary`."""
    n, m = len(q), len(r)
    H = [[0] * (m + 1) for _ in range(n + 1)]
    E = [[boundary] * (m + 1) for _ in range(n + 1)]
    F = [[boundary] * (m + 1) for _ in range(n + 1)]
    for i in range(1, n + 1):
        for j in range(1, m + 1):
            E[i][j] = max(E[i][j - 1] + e, H[i][j - 1] + o, 0)
            F[i][j] = max(F[i - 1][j] + e, H[i - 1][j] + o, 0)
            H[i][j] = max(H[i - 1][j - 1] + sigma(q[i - 1], r[j - 1]), E[i][j], F[i][j])
    return H


def test_relu_and_boundary_equivalence():
    """P13: H is unchanged under E/F relu clamping and boundary E/F in {0, o}."""
    g = rng(13)
    for k in range(60):
        ma, mm, o, e = SCORINGS_DNA[k % 5]
        q = rand_seq(g, b"ACGT", int(g.integers(1, 40)))
        r = rand_seq(g, b"ACGT", int(g.integers(1, 40)))
        H = oracle.fill_H(q, r, dna(ma, mm, o, e))
        for bnd in (0, o):
            np.testing.assert_array_equal(H, np.array(relu_form_H(q, r, bf.dna_sigma(ma, mm), o, e, bnd)))


def test_reverse_consistency_on_batches():
    """P14: max H' over the reversed prefixes equals S (the oracle raises otherwise)."""
    b = synth.random_pairs(14, 400, (0, 60), (0, 80), b"AC")
    oracle.align_batch(b.queries, b.q_offsets, b.refs, b.r_offsets, {"alphabet": "dna", "match": 1,
                       "mismatch": -1, "gap_open": -1, "gap_extend": -1})
    b = synth.generate("c3", 0, 60)
    oracle.align_batch(b.queries, b.q_offsets, b.refs, b.r_offsets, synth.PROTEIN_SCORING)


def spec_traceback_start(q: bytes, r: bytes, match: int, mismatch: int, gap: int, qe: int, re: int):
    """SPEC.md:395/464 traceback from (qe, re): ties diagonal > up > left, stop at a zero cell."""
    H = spec_linear_sw(q, r, match, mismatch, gap)
    i, j = qe + 1, re + 1
    while True:
        s = match if q[i - 1] == r[j - 1] else mismatch
        if H[i][j] == H[i - 1][j - 1] + s:
            if H[i - 1][j - 1] == 0:
                return i - 1, j - 1
            i, j = i - 1, j - 1
        elif H[i][j] == H[i - 1][j] + gap:
            i -= 1
        elif H[i][j] == H[i][j - 1] + gap:
            j -= 1
        else:  # pragma: no cover
            raise AssertionError("broken traceback")


def test_spec_traceback_start_is_a_valid_start():
    """P15: SPEC's traceback start lies in the valid-start set; equals C-5 when unique."""
    g = rng(15)
    differing = 0
    for _ in range(1500):
        ma, mm, gap = [(2, -2, -1), (1, -1, -1), (3, -3, -2)][int(g.integers(0, 3))]
        q = rand_seq(g, b"ACG", int(g.integers(1, 7)))
        r = rand_seq(g, b"ACG", int(g.integers(1, 7)))
        S, qe, re, qs, rs = oracle.align(q, r, dna(ma, mm, gap, gap))
        if S == 0:
            continue
        _, ends, starts = bf.optimal_set(q, r, bf.dna_sigma(ma, mm), gap, gap)
        valid = starts[(qe, re)]
        t = spec_traceback_start(q, r, ma, mm, gap, qe, re)
        assert t in valid
        if len(valid) == 1:
            assert t == (qs, rs)
        elif t != (qs, rs):
            differing += 1
    # documented example where the rules differ (SURVEY.md Appendix A / reading R9)
    assert spec_traceback_start(b"AAGCG", b"AAACG", 1, -1, -1, 4, 4) == (0, 0)
    assert oracle.align("AAGCG", "AAACG", dna(1, -1, -1, -1))[3:] == (0, 1)


def test_blosum62_table_properties():
    """Reading R11: the oracle's BLOSUM62 copy vs the checks listed in SURVEY.md Appendix B."""
    T = np.array([[oracle.blosum62(a, b) for b in BLOSUM_ORDER] for a in BLOSUM_ORDER])
    assert (T == T.T).all()
    diag = dict(zip(BLOSUM_ORDER, np.diag(T)))
    assert diag == dict(A=4, R=5, N=6, D=6, C=9, Q=5, E=5, G=6, H=8, I=4, L=4, K=5, M=5, F=6, P=7,
                        S=4, T=5, W=11, Y=7, V=4, B=4, Z=4, X=-1, **{"*": 1})
    assert T.min() == -4 and T.max() == 11
    assert int(T.sum()) == -726 and int(T[:20, :20].sum()) == -426
    off = T[:20, :20] - np.diag(np.diag(T[:20, :20])) - 100 * np.eye(20, dtype=int)
    assert off.max() == 3
    for a in range(22):
        for b in range(22):
            if a != b:
                assert 2 * T[a, b] < T[a, a] + T[b, b]
    # a few well-known entries
    assert oracle.blosum62("W", "F") == 1 and oracle.blosum62("C", "E") == -4 and oracle.blosum62("D", "B") == 4


def test_scoring_preconditions():
    """Reading R3: o < 0, o <= e <= 0, match > 0, mismatch < match."""
    assert oracle.check_scoring(dna(3, -3, -6, -1))
    assert oracle.check_scoring(dna(1, -1, -1, -1))
    assert not oracle.check_scoring(dna(3, -3, 0, 0))
    assert not oracle.check_scoring(dna(3, -3, -1, -4))   # e < o
    assert not oracle.check_scoring(dna(3, -3, -6, 1))    # e > 0
    assert not oracle.check_scoring(dna(0, -3, -6, -1))   # match <= 0
    assert not oracle.check_scoring(dna(3, 3, -6, -1))    # mismatch >= match
    assert oracle.check_scoring(prot(-11, -1))
    with pytest.raises(ValueError):
        oracle.align("A", "A", dna(3, -3, 0, 0))


def test_batch_equals_single_pair_calls():
    b = synth.random_pairs(16, 200, (0, 30), (0, 30), b"ACGTN")
    out = oracle.align_batch(b.queries, b.q_offsets, b.refs, b.r_offsets, synth.DNA_SCORING, threads=4)
    for p in range(b.n_pairs):
        q, r = b.pair(p)
        got = tuple(int(out[k][p]) for k in ("score", "q_end", "r_end", "q_start", "r_start"))
        assert got == oracle.align(q, r, synth.DNA_SCORING)
