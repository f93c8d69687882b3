"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Bar: every pair, all five fields, bit-exact.
Inputs are the seeded synthetic batches of paper_2208_12350_b200.synth; the
oracle is called only here, on the same bytes.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from paper_2208_12350_b200 import sw, synth

pytestmark = pytest.mark.gpu

FIELDS = ("score", "q_end", "r_end", "q_start", "r_start")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def aligner():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    # SW_MODE_POISON: every call first fills its outputs and the handle's workspace with poison,
    # so a value a call did not write in that call fails the comparison instead of passing stale
    a = sw.Aligner(0, poison=True)
    yield a
    a.close()


def oracle_batch(b: synth.Batch, threads=None):
    return oracle.align_batch(b.queries, b.q_offsets, b.refs, b.r_offsets, b.scoring, threads=threads)


def assert_parity(got: dict, exp: dict, b: synth.Batch):
    """got/exp: five int32 arrays, one entry per pair of b."""
    for f in FIELDS:
        assert len(got[f]) == len(exp[f]) == b.n_pairs
        bad = np.nonzero(got[f] != exp[f])[0]
        if bad.size:
            p = int(bad[0])
            q, r = b.pair(p)
            raise AssertionError(
                f"field {f}: {bad.size} mismatches; first pair {p} (n={len(q)}, m={len(r)}): "
                f"gpu={[int(got[k][p]) for k in FIELDS]} oracle={[int(exp[k][p]) for k in FIELDS]}\n"
                f"q={q[:80]!r}\nr={r[:80]!r}")


def run_and_compare(aligner, b: synth.Batch):
    got = aligner.align(b)
    exp = oracle_batch(b)
    assert_parity(got, exp, b)
    return got


# ----------------------------------------------------------------- goldens

def test_golden_examples(aligner):
    rows = []
    for l in open(os.path.join(GOLDEN, "worked_examples.tsv")):
        if l.startswith("#") or not l.strip():
            continue
        p = l.rstrip("\n").split("\t")
        rows.append(p)
    for alpha in ("dna", "protein"):
        sel = [p for p in rows if p[2] == alpha]
        groups = {}
        for p in sel:
            groups.setdefault(tuple(p[3:7]), []).append(p)
        for (ma, mm, o, e), ps in groups.items():
            sc = {"alphabet": alpha, "match": int(ma), "mismatch": int(mm), "gap_open": int(o), "gap_extend": int(e)}
            b = synth.from_pairs([(p[0], p[1]) for p in ps], sc)
            got = aligner.align(b)
            for k, p in enumerate(ps):
                assert tuple(int(got[f][k]) for f in FIELDS) == tuple(int(x) for x in p[7:12]), p


# ------------------------------------------------------- the five configs

def test_c1_full_parity(aligner):
    run_and_compare(aligner, synth.generate("c1"))


def test_c2_prefix_parity(aligner):
    run_and_compare(aligner, synth.generate("c2", 0, 4000))


def test_c3_protein_prefix_parity(aligner):
    run_and_compare(aligner, synth.generate("c3", 0, 1500))


def test_c5_mixed_sample_parity(aligner):
    """Length-skewed batch: multi-stripe queries up to 4 kb, references up to 16 kb."""
    cfg = synth.CONFIGS["c5"]
    n, m = synth.batch_lengths(cfg, 0, 4096)
    longs = np.nonzero(n > 150)[0]
    # a few long pairs of various sizes plus short ones, bounded oracle cost
    cost = n[longs] * m[longs]
    pick = list(longs[np.argsort(cost)][::max(1, len(longs) // 24)][:24]) + list(np.nonzero(n == 150)[0][:200])
    full = synth.generate("c5", 0, 4096)
    b = full.subset(sorted(int(p) for p in pick))
    run_and_compare(aligner, b)


def test_c2_full_size_sampled(aligner):
    """C2 at its full BASELINE size in one call; 400 sampled pairs checked against the oracle."""
    b = synth.generate("c2")
    got = aligner.align(b)
    rng = np.random.default_rng(2)
    idx = np.sort(rng.choice(b.n_pairs, size=400, replace=False))
    sub = b.subset(idx)
    exp = oracle_batch(sub)
    assert_parity({f: got[f][idx] for f in FIELDS}, exp, sub)
    assert np.all(got["score"] > 0)


def test_c3_full_size_sampled(aligner):
    """C3 (50k protein pairs, BLOSUM62, lengths up to 1,024) at its full size in one call; 300
    sampled pairs vs the oracle, and every pair's start/end consistent with its score."""
    b = synth.generate("c3")
    got = aligner.align(b)
    rng = np.random.default_rng(3)
    idx = np.sort(rng.choice(b.n_pairs, size=300, replace=False))
    sub = b.subset(idx)
    assert_parity({f: got[f][idx] for f in FIELDS}, oracle_batch(sub), sub)
    pos = got["score"] > 0
    assert np.all(got["q_start"][pos] <= got["q_end"][pos]) and np.all(got["r_start"][pos] <= got["r_end"][pos])
    assert np.all(got["q_end"][~pos] == -1)


def test_c4_per_gpu_share_sampled(aligner):
    """C4 (4M pairs) at 8 GPUs gives each GPU 500k pairs: one such call, 300 sampled pairs vs the oracle."""
    b = synth.generate("c4", 3_500_000, 4_000_000)
    got = aligner.align(b)
    rng = np.random.default_rng(4)
    idx = np.sort(rng.choice(b.n_pairs, size=300, replace=False))
    sub = b.subset(idx)
    assert_parity({f: got[f][idx] for f in FIELDS}, oracle_batch(sub), sub)


def test_c5_full_size_sampled(aligner):
    """C5 at its full size (400k pairs, references up to 16 kb, queries up to 4 kb) in one call;
    short and long sampled pairs vs the oracle (long ones bounded in oracle cost)."""
    b = synth.generate("c5")
    got = aligner.align(b)
    n = np.diff(b.q_offsets); m = np.diff(b.r_offsets)
    rng = np.random.default_rng(5)
    short = rng.choice(np.nonzero(n == 150)[0], size=150, replace=False)
    longs = np.nonzero((n > 150) & (n * m < 4e7))[0]
    long_pick = rng.choice(longs, size=min(30, longs.size), replace=False)
    idx = np.sort(np.concatenate([short, long_pick]))
    sub = b.subset(idx)
    assert_parity({f: got[f][idx] for f in FIELDS}, oracle_batch(sub), sub)


# ------------------------------------------------------------ adversarial

def test_tie_heavy_low_entropy(aligner):
    pairs = []
    rng = np.random.default_rng(11)
    for L in (1, 2, 9, 10, 11, 31, 32, 33, 150, 159, 160, 161, 250, 319, 320, 321, 480):
        pairs.append(("A" * L, "A" * (L + 7)))
        pairs.append(("AC" * (L // 2 + 1), "CA" * (L // 2 + 3)))
        pairs.append(("ACGT" * (L // 4 + 1), "ACGTACGT" * (L // 8 + 2)))
        pairs.append(("".join(rng.choice(list("AC"), L)), "".join(rng.choice(list("AC"), L + 17))))
    b = synth.from_pairs(pairs, synth.DNA_SCORING)
    run_and_compare(aligner, b)
    b = synth.from_pairs(pairs, {"alphabet": "dna", "match": 1, "mismatch": -1, "gap_open": -1, "gap_extend": -1})
    run_and_compare(aligner, b)


def test_random_small_many_scorings(aligner):
    for k, (ma, mm, o, e) in enumerate([(3, -3, -6, -1), (2, -2, -1, -1), (1, -1, -2, -1), (2, -1, -3, -1),
                                        (1, -1, -1, -1), (5, -4, -10, -2), (1, -3, -5, -2)]):
        sc = {"alphabet": "dna", "match": ma, "mismatch": mm, "gap_open": o, "gap_extend": e}
        b = synth.random_pairs(100 + k, 600, (0, 70), (0, 90), b"ACG" if k % 2 else b"ACGT", sc)
        run_and_compare(aligner, b)


def test_edge_cases_and_sentinels(aligner):
    pairs = [("", ""), ("", "ACGT"), ("ACGT", ""), ("A", "A"), ("A", "C"), ("AAAA", "CCCC"),
             ("ACNT", "ACGT"), ("ACGT", "ACGU"), ("acgt", "ACGT"), ("ACGT", "acgtacgt"), ("G" * 5000, "G" * 300)]
    b = synth.from_pairs(pairs, synth.DNA_SCORING)
    got = run_and_compare(aligner, b)
    assert tuple(got["score"][:3]) == (0, 0, 0)
    assert got["score"][6] == -1 and got["score"][7] == -1
    st, nbad = aligner.batch_status()
    assert st == sw.SW_ERR_BAD_PAIRS and nbad == 2


def test_stripe_and_lane_boundaries(aligner):
    """Queries around multiples of the 10-row lane block and the 160-row stripe."""
    rng = np.random.default_rng(12)
    pairs = []
    for n in (1, 9, 10, 11, 159, 160, 161, 319, 320, 321, 479, 481, 1000):
        for m in (1, 15, 16, 17, 200, 700):
            q = "".join(rng.choice(list("ACGT"), n))
            if m >= 10 and n >= 10:
                s = rng.integers(0, n - 5)
                r = "".join(rng.choice(list("ACGT"), m // 2)) + q[s:s + m // 2]
                r = r[:m]
            else:
                r = "".join(rng.choice(list("ACGT"), m))
            pairs.append((q, r))
    run_and_compare(aligner, synth.from_pairs(pairs, synth.DNA_SCORING))


def test_pack_vector_edges_and_bad_symbol_attribution(aligner):
    """Tiny and ragged sequences packed 32 pairs per warp (16-byte vectors straddling pairs,
    pads and warp spans), bad symbols at the start / middle / end of one pair among valid
    neighbours, and reversed prefixes ending at every column phase."""
    rng = np.random.default_rng(21)
    lens = (0, 1, 2, 3, 7, 15, 16, 17, 31, 32, 33, 47, 64, 65, 100)
    pairs = []
    for k in range(200):
        n = int(lens[k % len(lens)]); m = int(lens[(k * 7 + 3) % len(lens)])
        q = "".join(rng.choice(list("ACGT"), n)); r = "".join(rng.choice(list("ACGT"), m))
        if k % 23 == 5 and n:
            pos = (0, n // 2, n - 1)[k % 3]
            q = q[:pos] + "X" + q[pos + 1:]
        if k % 29 == 7 and m:
            pos = (0, m // 2, m - 1)[k % 3]
            r = r[:pos] + "#" + r[pos + 1:]
        pairs.append((q, r))
    # identical pairs: the alignment ends at every column phase 0..15 of the reference
    for m in range(20, 52):
        r = "".join(rng.choice(list("ACGT"), m))
        pairs.append((r[m - 18:m - 2], r))
    run_and_compare(aligner, synth.from_pairs(pairs, synth.DNA_SCORING))
    prot = [("".join(rng.choice(list("ACDEFGHIKLMNPQRSTVWY"), int(lens[k % 15]))),
             "".join(rng.choice(list("ACDEFGHIKLMNPQRSTVWY"), int(lens[(k * 5 + 1) % 15])))) for k in range(120)]
    prot[17] = (prot[17][0] + "J", prot[17][1])
    run_and_compare(aligner, synth.from_pairs(prot, synth.PROTEIN_SCORING))


def test_int32_routing_per_pair(aligner):
    """s16-eligible scoring, but pairs whose max score exceeds the int16 bound go to the s32 kernel."""
    sc = {"alphabet": "dna", "match": 30, "mismatch": -20, "gap_open": -40, "gap_extend": -5}
    rng = np.random.default_rng(13)
    pairs = []
    for L in (1100, 1200):
        q = "".join(rng.choice(list("ACGT"), L))
        pairs.append((q, q[:L - 3] + "TTT"))            # near-identity: S ~ 30 L > 32000
    for _ in range(40):
        pairs.append(("".join(rng.choice(list("ACGT"), 60)), "".join(rng.choice(list("ACGT"), 90))))
    got = run_and_compare(aligner, synth.from_pairs(pairs, sc))
    assert got["score"][0] > 32767


def test_three_routes_in_one_counting_sorted_batch(aligner):
    """TAG (max score <= 511), S16 and S32 pairs in one batch whose work keys all fit the exact
    counting-sort bins (references < 1,040, <= 8 stripes): route groups and their offsets in the
    pair order must line up for both passes."""
    sc = {"alphabet": "dna", "match": 100, "mismatch": -20, "gap_open": -25, "gap_extend": -5}
    rng = np.random.default_rng(31)
    pairs = []
    for k in range(300):
        n = int(rng.integers(1, 700)) if k % 3 else int(rng.integers(1, 6))
        m = int(rng.integers(1, 1000)) if k % 3 else int(rng.integers(1, 6))
        q = "".join(rng.choice(list("ACGT"), n))
        if k % 2 and n > 20 and m > n:
            r = "".join(rng.choice(list("ACGT"), m - n)) + q
        else:
            r = "".join(rng.choice(list("ACGT"), m))
        pairs.append((q, r))
    got = run_and_compare(aligner, synth.from_pairs(pairs, sc))
    assert got["score"].max() > 32000 and (got["score"][::3] <= 511).all()


def test_int32_routing_whole_scoring(aligner):
    """Scorings whose (s - gap_open) does not fit the int8 profile run entirely on the s32 kernel."""
    sc = {"alphabet": "dna", "match": 100, "mismatch": -90, "gap_open": -150, "gap_extend": -7}
    run_and_compare(aligner, synth.random_pairs(21, 300, (1, 400), (1, 500), b"ACGT", sc))
    psc = {"alphabet": "protein", "gap_open": -200, "gap_extend": -3}
    b = synth.generate("c3", 0, 200)
    b.scoring = psc
    run_and_compare(aligner, b)


def test_protein_small_and_case(aligner):
    pairs = [("HEAGAWGHEE", "PAWHEAE"), ("heagawghee", "pawheae"), ("MKTAYIAKQR*", "MKTAYIAKQR*"),
             ("BZX*", "BZX*"), ("ACDJ", "ACD"), ("", "ACD")]
    b = synth.from_pairs(pairs, synth.PROTEIN_SCORING)
    got = run_and_compare(aligner, b)
    assert got["score"][4] == -1


# -------------------------------------------------------- batch invariance

def test_permutation_and_shard_invariance(aligner):
    """P11: results are a pure function of the pair (order, composition, sharding)."""
    b = synth.generate("c1", 0, 600)
    ref = aligner.align(b)
    perm = np.random.default_rng(5).permutation(b.n_pairs)
    got = aligner.align(b.subset(perm))
    for f in FIELDS:
        np.testing.assert_array_equal(got[f], ref[f][perm])
    cuts = sw.sw_plan_shards(b.q_offsets, b.r_offsets, 3)
    for k in range(3):
        part = aligner.align(b.subset(range(cuts[k], cuts[k + 1])))
        for f in FIELDS:
            np.testing.assert_array_equal(part[f], ref[f][cuts[k]:cuts[k + 1]])
    again = aligner.align(b)
    for f in FIELDS:
        np.testing.assert_array_equal(again[f], ref[f])


def test_host_entry_point_matches_device_entry_point(aligner):
    import torch
    b = synth.generate("c1", 0, 300)
    ref = aligner.align(b)
    out = {f: np.zeros(b.n_pairs, np.int32) for f in FIELDS}
    qa, ra = np.ascontiguousarray(b.queries), np.ascontiguousarray(b.refs)
    qo, ro = np.ascontiguousarray(b.q_offsets), np.ascontiguousarray(b.r_offsets)
    st = sw.sw_align_batch_host(aligner.handle, qa.ctypes.data, qo.ctypes.data, ra.ctypes.data, ro.ctypes.data,
                                b.n_pairs, b.scoring, {f: out[f].ctypes.data for f in FIELDS},
                                torch.cuda.current_stream().cuda_stream)
    assert st == sw.SW_OK
    for f in FIELDS:
        np.testing.assert_array_equal(out[f], ref[f])


def test_offsets_need_not_start_at_zero(aligner):
    import torch
    b = synth.generate("c1", 0, 50)
    ref = aligner.align(b)
    q, qo, r, ro = aligner.to_device(b)
    pad = torch.zeros(100, dtype=torch.uint8, device="cuda:0")
    q2 = torch.cat([pad, q]); r2 = torch.cat([pad, r])
    out, st = aligner.align_tensors(q2, qo + 100, r2, ro + 100, b.scoring)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    for i, f in enumerate(FIELDS):
        np.testing.assert_array_equal(o[i, :50], ref[f])


# --------------------------------------------------------------- ABI errors

def test_abi_errors(aligner):
    import torch
    b = synth.generate("c1", 0, 10)
    q, qo, r, ro = aligner.to_device(b)
    bad_sc = dict(b.scoring, gap_open=1)
    out, st = aligner.align_tensors(q, qo, r, ro, bad_sc, check=False)
    assert st == sw.SW_ERR_INVALID_SCORING
    out, st = aligner.align_tensors(q, qo, r, ro, dict(b.scoring, gap_extend=-7), check=False)
    assert st == sw.SW_ERR_INVALID_SCORING
    out, st = aligner.align_tensors(q, qo, r, ro, dict(b.scoring, match=-1), check=False)
    assert st == sw.SW_ERR_INVALID_SCORING
    # decreasing offsets -> invalid argument, every field -1
    qo_bad = qo.clone(); qo_bad[3] = qo_bad[5] + 1
    out, st = aligner.align_tensors(q, qo_bad, r, ro, b.scoring, check=False)
    torch.cuda.synchronize()
    assert st == sw.SW_ERR_INVALID_ARGUMENT
    assert (out[:, :10] == -1).all()
    # zero pairs: no-op
    out, st = aligner.align_tensors(q, qo[:1], r, ro[:1], b.scoring, check=False)
    assert st == sw.SW_OK
    # the handle still works afterwards
    got = aligner.align(b)
    np.testing.assert_array_equal(got["score"], oracle_batch(b)["score"])


def test_dpx_peak_probe_runs():
    import torch
    cups = sw.sw_dpx_peak(0, 50.0, torch.cuda.current_stream().cuda_stream)
    assert 1e12 < cups < 5e13


def test_host_entry_point_chunked_pipeline(aligner):
    """The host-buffer entry point splits large batches into overlapped chunks; results must equal
    the device entry point, and per-pair errors / S = 0 sentinels must survive chunking."""
    import torch
    b = synth.generate("c2", 0, 40000)
    # sprinkle invalid symbols and empty sequences across chunk boundaries
    pairs = [b.pair(p) for p in range(b.n_pairs)]
    for p in (0, 9999, 10000, 19999, 20000, 39999):
        q, r = pairs[p]
        pairs[p] = (q[:5] + b"N" + q[6:], r) if p % 2 == 0 else (b"", r)
    b = synth.from_pairs(pairs, synth.DNA_SCORING)
    ref = aligner.align(b)
    out = {f: np.zeros(b.n_pairs, np.int32) for f in FIELDS}
    qa, ra = np.ascontiguousarray(b.queries), np.ascontiguousarray(b.refs)
    qo, ro = np.ascontiguousarray(b.q_offsets), np.ascontiguousarray(b.r_offsets)
    st = sw.sw_align_batch_host(aligner.handle, qa.ctypes.data, qo.ctypes.data, ra.ctypes.data, ro.ctypes.data,
                                b.n_pairs, b.scoring, {f: out[f].ctypes.data for f in FIELDS},
                                torch.cuda.current_stream().cuda_stream)
    assert st == sw.SW_OK
    for f in FIELDS:
        np.testing.assert_array_equal(out[f], ref[f])
    st, nbad = aligner.batch_status()
    assert st == sw.SW_ERR_BAD_PAIRS and nbad == 3
    # malformed offsets through the host entry point: every field -1, synchronous error
    qo_bad = qo.copy(); qo_bad[5] = qo_bad[7] + 1
    st = sw.sw_align_batch_host(aligner.handle, qa.ctypes.data, qo_bad.ctypes.data, ra.ctypes.data, ro.ctypes.data,
                                b.n_pairs, b.scoring, {f: out[f].ctypes.data for f in FIELDS},
                                torch.cuda.current_stream().cuda_stream)
    assert st == sw.SW_ERR_INVALID_ARGUMENT and (out["score"] == -1).all()


def test_submit_host_pipeline_of_batches(aligner):
    """Asynchronous host-buffer batches (sw_submit_host / sw_wait): several batches in flight on
    double-buffered staging, growing sizes (staging reallocation while the other slot is busy),
    DNA and protein, each result equal to the synchronous device entry point."""
    import torch
    s = torch.cuda.current_stream().cuda_stream
    batches = [synth.generate("c1", 0, 300), synth.generate("c2", 0, 3000), synth.generate("c3", 0, 500),
               synth.generate("c2", 5000, 25000), synth.generate("c1", 0, 1000)]
    keep = []
    for b in batches:
        arrs = (np.ascontiguousarray(b.queries), np.ascontiguousarray(b.q_offsets),
                np.ascontiguousarray(b.refs), np.ascontiguousarray(b.r_offsets))
        out = {f: np.full(b.n_pairs, 7, np.int32) for f in FIELDS}
        st = sw.sw_submit_host(aligner.handle, arrs[0].ctypes.data, arrs[1].ctypes.data, arrs[2].ctypes.data,
                               arrs[3].ctypes.data, b.n_pairs, b.scoring, {f: out[f].ctypes.data for f in FIELDS}, s)
        assert st == sw.SW_OK
        keep.append((b, arrs, out))
    assert sw.sw_wait(aligner.handle) == sw.SW_OK
    for b, _, out in keep:
        ref = aligner.align(b)
        for f in FIELDS:
            np.testing.assert_array_equal(out[f], ref[f])
    # validation errors come back before anything is enqueued
    b, arrs, out = keep[0]
    qo_bad = arrs[1].copy(); qo_bad[3] = qo_bad[5] + 1
    st = sw.sw_submit_host(aligner.handle, arrs[0].ctypes.data, qo_bad.ctypes.data, arrs[2].ctypes.data,
                           arrs[3].ctypes.data, b.n_pairs, b.scoring, {f: out[f].ctypes.data for f in FIELDS}, s)
    assert st == sw.SW_ERR_INVALID_ARGUMENT
    assert sw.sw_wait(aligner.handle) == sw.SW_OK


def test_end_only_mode(aligner):
    """SW_MODE_END_ONLY (forward pass only): score / q_end / r_end identical to the
    oracle, start arrays untouched, NULL start pointers accepted; FULL mode restores starts."""
    import torch
    b = synth.generate("c2", 0, 4000)
    exp = oracle_batch(b)
    q, qo, r, ro = aligner.to_device(b)
    out = torch.full((5, b.n_pairs), 12345, dtype=torch.int32, device="cuda:0")
    aligner.set_mode(sw.SW_MODE_END_ONLY)
    try:
        res = sw.sw_result_t(out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(), 0, 0)
        st = sw.load().sw_align_batch(aligner.handle, q.data_ptr(), qo.data_ptr(), r.data_ptr(), ro.data_ptr(),
                                      b.n_pairs, sw.make_scoring(b.scoring), res, torch.cuda.current_stream().cuda_stream)
        assert st == sw.SW_OK
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        for i, f in enumerate(FIELDS[:3]):
            np.testing.assert_array_equal(o[i], exp[f])
        assert (o[3] == 12345).all() and (o[4] == 12345).all()
    finally:
        aligner.set_mode(sw.SW_MODE_FULL)
    got = aligner.align(b)
    for f in FIELDS:
        np.testing.assert_array_equal(got[f], exp[f])


# ------------------------------------------------------------ alignment paths (f1)

def _oracle_paths(b: synth.Batch):
    exp = oracle_batch(b)
    out = []
    for p in range(b.n_pairs):
        q, r = b.pair(p)
        res = tuple(int(exp[f][p]) for f in FIELDS)
        out.append(oracle.traceback(q, r, b.scoring, res) if res[0] >= 0 else None)
    return out


@pytest.mark.parametrize("which", ["c1", "c2", "c3", "ties", "long", "edges"])
def test_traceback_paths_match_oracle(aligner, which):
    """sw_traceback: every pair's op string equal to the oracle's path (reading R20)."""
    rng = np.random.default_rng(17)
    if which == "c1":
        b = synth.generate("c1")
    elif which == "c2":
        b = synth.generate("c2", 0, 1500)
    elif which == "c3":
        b = synth.generate("c3", 0, 300)
    elif which == "ties":
        pairs = [("".join(rng.choice(list("AC"), int(rng.integers(1, 40)))),
                  "".join(rng.choice(list("AC"), int(rng.integers(1, 40))))) for _ in range(400)]
        b = synth.from_pairs(pairs, {"alphabet": "dna", "match": 2, "mismatch": -2, "gap_open": -1, "gap_extend": -1})
    elif which == "long":
        # multi-stripe intervals (> 160 query rows) with indels
        pairs = []
        for k in range(40):
            n = int(rng.integers(150, 700))
            q = "".join(rng.choice(list("ACGT"), n))
            mut = list(q)
            for _ in range(n // 25):
                pos = int(rng.integers(0, len(mut)))
                if rng.random() < 0.5:
                    del mut[pos]
                else:
                    mut.insert(pos, str(rng.choice(list("ACGT"))))
            pairs.append((q, "".join(rng.choice(list("ACGT"), 30)) + "".join(mut)))
        b = synth.from_pairs(pairs, synth.DNA_SCORING)
    else:
        pairs = [("", "ACGT"), ("ACGT", ""), ("A", "A"), ("A", "C"), ("ACNT", "ACGT"), ("ACGT", "ACGT" * 3),
                 ("GGGGAAAAGGGG", "GGGGGGGG"), ("ACGTACGT", "ACGTTACGT")]
        b = synth.from_pairs(pairs, synth.DNA_SCORING)
    got = aligner.traceback(b)
    exp = _oracle_paths(b)
    bad = [p for p in range(b.n_pairs) if got[p] != exp[p]]
    assert not bad, f"{len(bad)} paths differ; first pair {bad[0]}: gpu={got[bad[0]]!r} oracle={exp[bad[0]]!r}"


# ------------------------------------------------------------ linear gaps (f2)

def _rescored(b: synth.Batch, sc: dict) -> synth.Batch:
    import dataclasses
    return dataclasses.replace(b, scoring=dict(sc))


@pytest.mark.parametrize("which", ["dna_tag", "dna_s16_stripes", "protein", "ties"])
def test_linear_gap_kernels(aligner, which):
    """gap_open == gap_extend takes the two-state linear-gap kernels: all five
    fields equal to the oracle (affine recurrence with o = e) and to the affine kernels
    (SW_MODE_AFFINE_ONLY) on the same bytes."""
    rng = np.random.default_rng(31)
    if which == "dna_tag":       # 150-row reads, max_s * n <= 511: TAG route
        b = _rescored(synth.generate("c2", 0, 1500),
                      {"alphabet": "dna", "match": 2, "mismatch": -3, "gap_open": -2, "gap_extend": -2})
    elif which == "dna_s16_stripes":   # long queries: S16 route, several stripes, lane/stripe edges
        pairs = []
        for n in (1, 10, 159, 160, 161, 321, 700, 1300):
            for m in (1, 17, 300, 900):
                q = "".join(rng.choice(list("ACGT"), n))
                s0 = int(rng.integers(0, max(1, n - 5)))
                r = ("".join(rng.choice(list("ACGT"), m // 3)) + q[s0:s0 + m])[:m]
                pairs.append((q, r))
        b = synth.from_pairs(pairs, {"alphabet": "dna", "match": 3, "mismatch": -2, "gap_open": -3, "gap_extend": -3})
    elif which == "protein":
        b = _rescored(synth.generate("c3", 0, 600),
                      {"alphabet": "protein", "match": 0, "mismatch": 0, "gap_open": -4, "gap_extend": -4})
    else:
        pairs = [("AC" * L, "CA" * (L + 3)) for L in (1, 5, 16, 80, 200)]
        pairs += [("".join(rng.choice(list("AC"), L)), "".join(rng.choice(list("AC"), L + 9))) for L in (7, 60, 170, 400)]
        b = synth.from_pairs(pairs, {"alphabet": "dna", "match": 1, "mismatch": -1, "gap_open": -1, "gap_extend": -1})
    got = run_and_compare(aligner, b)
    aligner.set_mode(sw.SW_MODE_AFFINE_ONLY)
    try:
        aff = aligner.align(b)
    finally:
        aligner.set_mode(sw.SW_MODE_FULL)
    for f in FIELDS:
        np.testing.assert_array_equal(got[f], aff[f])


# ------------------------------------------------------------ one query vs a database (f2)

@pytest.mark.parametrize("alpha", ["dna", "protein"])
def test_query_db_mode(aligner, alpha):
    """sw_align_query_db: one query against many references equals the oracle on the pairs
    (query, ref_p), including empty references and a query length that is not a multiple of 16."""
    src = synth.generate("c2" if alpha == "dna" else "c3", 0, 400)
    q, _ = src.pair(7)
    refs = [src.pair(p)[1] for p in range(400)] + [b"", q, q[::-1]]
    for query in (q, q[:37], b""):
        b = synth.from_pairs([(query, r) for r in refs], src.scoring)
        got = aligner.align_query_db(query, refs, src.scoring)
        assert_parity(got, oracle_batch(b), b)


def test_speculative_extents_grow_and_rerun():
    """Device-buffer calls read the payload extents inside pack once the code buffers exist
    (sw_api.cu: speculative extents); a batch larger than the buffers must be detected there,
    grown and re-run with the same results, and a later smaller batch must reuse the buffers."""
    a = sw.Aligner(0)
    try:
        small = synth.generate("c1", 0, 50)
        big = synth.generate("c2", 0, 3000)
        for b in (small, big, small, synth.generate("c3", 0, 400), big):
            assert_parity(a.align(b), oracle_batch(b), b)
        # offsets that decrease (qN < q0 of the whole batch) on the speculative path
        import torch
        q, qo, r, ro = a.to_device(small)
        qo_bad = qo.clone()
        qo_bad[-1] = 0
        qo_bad[0] = int(qo[-1].item())
        out = a.alloc_out(small.n_pairs)
        with pytest.raises(sw.SWError):
            a.align_tensors(q, qo_bad, r, ro, small.scoring, out=out)
        torch.cuda.synchronize()
        assert (out[0, :small.n_pairs] == -1).all()
        assert_parity(a.align(small), oracle_batch(small), small)
    finally:
        a.close()


@pytest.mark.parametrize("which", ["mixed_eligibility", "c5_long"])
def test_traceback_s16x2_and_int32_kernels_agree(aligner, which):
    """DNA paths go to the s16x2 kernel (two pairs per warp) when every value fits 16 bits and to
    the int32 kernel otherwise (tb16_ok); SW_MODE_TB_INT32 forces the int32 kernel.  Both must give
    the oracle's paths; the mixed batch puts eligible and ineligible pairs in the same warp."""
    rng = np.random.default_rng(23)
    if which == "mixed_eligibility":
        # gap_extend -30: long intervals exceed the 16-bit bound (2|o| + (a+b)|e| > 16000), short ones fit
        pairs = []
        for k in range(120):
            n = int(rng.integers(5, 400)) if k % 3 else int(rng.integers(300, 420))
            q = "".join(rng.choice(list("ACGT"), n))
            mut = [c if rng.random() > 0.03 else str(rng.choice(list("ACGT"))) for c in q]
            if k % 5 == 0:
                mut.insert(len(mut) // 2, "ACG")
            pairs.append((q, "".join(rng.choice(list("ACGT"), int(rng.integers(0, 40)))) + "".join(mut)))
        b = synth.from_pairs(pairs, {"alphabet": "dna", "match": 5, "mismatch": -4, "gap_open": -40, "gap_extend": -30})
    else:
        b = synth.generate("c5", 0, 250)
    exp = _oracle_paths(b)
    got16 = aligner.traceback(b)
    aligner.set_mode(sw.SW_MODE_TB_INT32)
    try:
        got32 = aligner.traceback(b)
    finally:
        aligner.set_mode(sw.SW_MODE_FULL)
    for got in (got16, got32):
        bad = [p for p in range(b.n_pairs) if got[p] != exp[p]]
        assert not bad, f"{len(bad)} paths differ; first pair {bad[0]}: gpu={got[bad[0]]!r} oracle={exp[bad[0]]!r}"


@pytest.mark.parametrize("mismatch,gap_open", [(-1, -3), (0, -37)])
def test_reverse_multistripe_early_stop_stale_boundary(aligner, mismatch, gap_open):
    """Regression (round-2 root cause of the round-1 soak failure).  In a
    multi-stripe reverse item, a half whose start lies in stripe 1 stops the item's sweep early;
    the next stripe still sweeps up to another half's last column, and its lane 0 used to read the
    stripe boundary row up to the item's longest reversed reference -- past the columns the
    previous stripe had handed off, i.e. an earlier item's values.  On the TAG route a 4-column
    block maximum above S then hid a start in the same block (q_start = r_start = -2, the reverse
    self-check).  Half A: a 25-base exact match ending a 300 x 900 pair of C / G runs (start found
    in stripe 1 at reversed column 24, reversed reference bound 575 columns).  Half B: q == r of
    length L (S = L, start (0, 0) in the last reversed column, stripe >= 2); every L from 161 to
    479 puts that column in each lane and block phase.  Poisoned workspace (hand-off rows H = F =
    496) makes any stale read a wrong result."""
    rng = np.random.default_rng(2022)
    sc = {"alphabet": "dna", "match": 1, "mismatch": mismatch, "gap_open": gap_open, "gap_extend": -1}
    alpha = list("ACGT")
    tail = "".join(rng.choice(alpha, 25))
    qa = "C" * 275 + tail
    ra = "G" * 875 + tail
    exp_a = oracle_batch(synth.from_pairs([(qa, ra)], sc))
    assert int(exp_a["r_end"][0]) >= 600  # the long reversed reference of half A
    for L in range(161, 480):
        x = "".join(rng.choice(alpha, L))
        for pairs, ia, ib in (([(qa, ra), (x, x)], 0, 1), ([(x, x), (qa, ra), (x[:L // 2 + 1], x[:L // 2 + 1])], 1, 0)):
            b = synth.from_pairs(pairs, sc)
            got = aligner.align(b)
            assert tuple(int(got[f][ib]) for f in FIELDS) == (L, L - 1, L - 1, 0, 0), (L, [int(got[f][ib]) for f in FIELDS])
            assert tuple(int(got[f][ia]) for f in FIELDS) == tuple(int(exp_a[f][0]) for f in FIELDS), L
        st, nbad = aligner.batch_status()
        assert st == sw.SW_OK and nbad == 0, (L, st)


def test_soak_case_round1_whole_call(aligner):
    """The round-1 soak pair (tests/golden/soak_case_tb16.json: fields exact, path of a 347 x 335
    rectangle) through one sw_align_batch call whose own results feed sw_traceback, with random
    multi-stripe partners in the same reverse work item; fields, the reverse self-check and the path
    must all be the oracle's."""
    import json
    c = json.load(open(os.path.join(GOLDEN, "soak_case_tb16.json")))
    sc, q, r = c["sc"], c["q"], c["r"]
    exp_path = c["oracle"]
    rng = np.random.default_rng(7)
    for k in range(64):
        pairs = [(q, r)]
        for _ in range(int(rng.integers(1, 4))):
            n = int(rng.integers(150, 520))
            pq = "".join(rng.choice(list("ACGT"), n))
            pr = "".join(rng.choice(list("ACGT"), int(rng.integers(300, 1300))))
            pairs.append((pq, pr))
        perm = rng.permutation(len(pairs))
        pairs = [pairs[i] for i in perm]
        at = int(np.nonzero(perm == 0)[0][0])
        b = synth.from_pairs(pairs, sc)
        fields, paths = aligner.align_and_traceback(b)
        assert_parity(fields, oracle_batch(b), b)
        assert paths[at] == exp_path, k
        st, _ = aligner.batch_status()
        assert st == sw.SW_OK, (k, st)


# ------------------------------------------------- reserved (asynchronous) calls

def _reserved_aligner(b, slack=1.0):
    a = sw.Aligner(0, poison=True)
    a.reserve_for(b, slack)
    return a


@pytest.mark.parametrize("which", ["c1", "c2_prefix", "c3_prefix", "c5_mixed"])
def test_reserved_call_matches_oracle(which):
    """After sw_reserve, sw_align_batch enqueues without a host round trip (launches sized from the
    reservation, device-side counts); results are the oracle's on every config shape, including
    multi-stripe queries and long references (radix-sort path of the reservation)."""
    if which == "c1":
        b = synth.generate("c1")
    elif which == "c2_prefix":
        b = synth.generate("c2", 0, 3000)
    elif which == "c3_prefix":
        b = synth.generate("c3", 0, 800)
    else:
        full = synth.generate("c5", 0, 2048)
        n, m = full.lengths()
        idx = [int(p) for p in np.argsort(n * m)[:1900]]  # the bounded-oracle-cost part, incl. long pairs
        b = full.subset(sorted(idx))
    a = _reserved_aligner(b, 1.5)
    try:
        for _ in range(2):
            assert_parity(a.align(b), oracle_batch(b), b)
            assert a.batch_status() == (sw.SW_OK, 0)
        # a smaller batch within the same reservation
        sub = b.subset(range(0, b.n_pairs, 3))
        assert_parity(a.align(sub), oracle_batch(sub), sub)
    finally:
        a.close()


def test_reserved_call_returns_before_the_gpu_finishes():
    """Enqueue-and-return: with a reservation the call does not wait for earlier work on its stream
    (a 0.3 s device sleep is still running when it returns); without one it does."""
    import time
    import torch
    b = synth.generate("c2", 0, 2000)
    a = sw.Aligner(0)
    try:
        q, qo, r, ro = a.to_device(b)
        out = a.alloc_out(b.n_pairs)
        a.align_tensors(q, qo, r, ro, b.scoring, out=out)
        torch.cuda.synchronize()
        cycles = int(0.3 * 1.9e9)

        def timed_call():
            torch.cuda._sleep(cycles)
            t0 = time.perf_counter()
            a.align_tensors(q, qo, r, ro, b.scoring, out=out)
            dt = time.perf_counter() - t0
            torch.cuda.synchronize()
            return dt

        t_sync = timed_call()
        a.reserve_for(b)
        t_async = timed_call()
        assert t_sync > 0.1, t_sync
        assert t_async < 0.05, t_async
        got = out[:, :b.n_pairs].cpu().numpy()
        assert_parity({f: got[i] for i, f in enumerate(FIELDS)}, oracle_batch(b), b)
    finally:
        a.close()


def test_reserved_call_captured_in_cuda_graph():
    """A reserved call contains no synchronisation or allocation, so it can be captured into a CUDA
    graph; every replay rewrites the outputs with the oracle's results."""
    import torch
    b = synth.generate("c2", 0, 1500)
    a = sw.Aligner(0)
    try:
        a.reserve_for(b)
        q, qo, r, ro = a.to_device(b)
        out = a.alloc_out(b.n_pairs)
        a.align_tensors(q, qo, r, ro, b.scoring, out=out)  # warm (module load, attributes)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        with torch.cuda.graph(g, stream=cs):
            a.align_tensors(q, qo, r, ro, b.scoring, out=out)
        exp = oracle_batch(b)
        for _ in range(3):
            out.fill_(-7)
            g.replay()
            torch.cuda.synchronize()
            got = out[:, :b.n_pairs].cpu().numpy()
            assert_parity({f: got[i] for i, f in enumerate(FIELDS)}, exp, b)
    finally:
        a.close()


def test_reserved_call_rejects_batches_beyond_the_reservation():
    """Beyond the reservation (longer sequences, more payload) or with malformed offsets, a reserved
    call is rejected on the device: every output -1, reported by sw_batch_status; the handle keeps
    working for batches within the reservation."""
    import torch
    small = synth.generate("c1", 0, 200)
    a = sw.Aligner(0, poison=True)
    try:
        a.reserve_for(small)
        longer = synth.from_pairs([("ACGT" * 100, "ACGT" * 100)] + [small.pair(k) for k in range(5)], small.scoring)
        got = a.align(longer, check=False)
        assert all(np.all(got[f] == -1) for f in FIELDS)
        st, nbad = a.batch_status()
        assert st == sw.SW_ERR_INVALID_ARGUMENT and nbad == -1
        assert_parity(a.align(small), oracle_batch(small), small)
        assert a.batch_status() == (sw.SW_OK, 0)
        q, qo, r, ro = a.to_device(small)
        qo_bad = qo.clone()
        qo_bad[-1] = qo_bad[-2] - 1  # decreasing offsets at the end (no pair beyond the reserved lengths)
        out = a.alloc_out(small.n_pairs)
        a.align_tensors(q, qo_bad, r, ro, small.scoring, out=out, check=False)
        torch.cuda.synchronize()
        assert bool((out[:, :small.n_pairs] == -1).all())
        st, nbad = a.batch_status()
        assert st == sw.SW_ERR_BAD_PAIRS and nbad == -1
        assert_parity(a.align(small), oracle_batch(small), small)
    finally:
        a.close()


@pytest.mark.parametrize("kind", ["high_identity", "tandem_repeats", "protein_long"])
def test_reverse_band_multistripe(aligner, kind):
    """Reverse pass of multi-stripe pairs sweeps only the exact band min(i'+1, j'+1) + min(n2-1-i',
    m2-1-j') >= ceil(S / max_s) below its first stripe (sw_wavefront.cuh): long high-identity
    alignments (narrow band), tandem repeats (many optimal alignments on shifted diagonals: ties
    between starts at the band's edges) and long protein pairs, all five fields vs the oracle."""
    rng = np.random.default_rng({"high_identity": 31, "tandem_repeats": 32, "protein_long": 33}[kind])
    pairs = []
    if kind == "protein_long":
        alpha = list("ARNDCQEGHILKMFPSTWYV")
        sc = synth.PROTEIN_SCORING
        for _ in range(24):
            n = int(rng.integers(300, 1400))
            q = rng.choice(alpha, n)
            r = q.copy()
            mut = rng.random(n) < rng.choice([0.0, 0.05, 0.3])
            r[mut] = rng.choice(alpha, int(mut.sum()))
            pre = "".join(rng.choice(alpha, int(rng.integers(0, 300))))
            pairs.append(("".join(q), pre + "".join(r) + "".join(rng.choice(alpha, int(rng.integers(0, 300))))))
    else:
        sc = {"alphabet": "dna", "match": 2, "mismatch": -3, "gap_open": -5, "gap_extend": -2}
        for _ in range(24):
            n = int(rng.integers(330, 1500))
            if kind == "tandem_repeats":
                unit = "".join(rng.choice(list("ACGT"), int(rng.integers(1, 7))))
                q = (unit * (n // len(unit) + 1))[:n]
                r = (unit * ((n + 200) // len(unit) + 1))[: n + int(rng.integers(-50, 200))]
            else:
                qa = rng.choice(list("ACGT"), n)
                ra = qa.copy()
                mut = rng.random(n) < rng.choice([0.0, 0.01, 0.03])
                ra[mut] = rng.choice(list("ACGT"), int(mut.sum()))
                q = "".join(qa)
                r = "".join(rng.choice(list("ACGT"), int(rng.integers(0, 400)))) + "".join(ra) + \
                    "".join(rng.choice(list("ACGT"), int(rng.integers(0, 400))))
            pairs.append((q, r))
    b = synth.from_pairs(pairs, sc)
    assert_parity(aligner.align(b), oracle_batch(b), b)
    assert aligner.batch_status()[0] == sw.SW_OK


@pytest.mark.parametrize("kind", ["dna_mixed", "dna_cheap_gaps", "protein"])
def test_reverse_cooperative_items(aligner, kind):
    """Reverse items with >= SW_COOP_STRIPES (16) stripes are swept by all warps of a CTA, consecutive
    stripes on consecutive warps with published hand-off progress (sw_wavefront.cuh).  Long pairs
    (16-24 stripes) of mixed identity -- unrelated pairs whose start lies far from the origin (cheap
    gaps make their gapped score grow with length), high-identity ones, tandem repeats -- plus short
    partners in the same items; all five fields vs the oracle."""
    rng = np.random.default_rng({"dna_mixed": 41, "dna_cheap_gaps": 42, "protein": 43}[kind])
    # lengths from just above SW_COOP_STRIPES (16) stripes: 128-row protein / 160-row DNA stripes
    if kind == "protein":
        alpha, sc, lo, hi = list("ARNDCQEGHILKMFPSTWYV"), synth.PROTEIN_SCORING, 2050, 2700
    elif kind == "dna_cheap_gaps":
        alpha, lo, hi = list("ACGT"), 2570, 3300
        sc = {"alphabet": "dna", "match": 3, "mismatch": -3, "gap_open": -6, "gap_extend": -1}
    else:
        alpha, lo, hi = list("ACGT"), 2570, 3800
        sc = {"alphabet": "dna", "match": 2, "mismatch": -3, "gap_open": -5, "gap_extend": -2}
    pairs = []
    for k in range(14):
        n = int(rng.integers(lo, hi))
        q = rng.choice(alpha, n)
        u = k % 3
        if u == 0:  # unrelated
            r = rng.choice(alpha, int(rng.integers(n // 2, 2 * n)))
        elif u == 1:  # related, embedded
            r = q.copy()
            mut = rng.random(n) < 0.05
            r[mut] = rng.choice(alpha, int(mut.sum()))
            r = np.concatenate([rng.choice(alpha, int(rng.integers(0, 500))), r, rng.choice(alpha, int(rng.integers(0, 500)))])
        else:  # repeats
            unit = rng.choice(alpha, int(rng.integers(2, 9)))
            q = np.resize(unit, n)
            r = np.resize(unit, n + int(rng.integers(-100, 300)))
        pairs.append(("".join(q), "".join(r)))
        pairs.append(("".join(rng.choice(alpha, int(rng.integers(100, 600)))), "".join(rng.choice(alpha, int(rng.integers(100, 900))))))
    b = synth.from_pairs(pairs, sc)
    for _ in range(2):
        assert_parity(aligner.align(b), oracle_batch(b), b)
        assert aligner.batch_status()[0] == sw.SW_OK


@pytest.mark.parametrize("scoring", [(3, -3, -6, -1), (2, -3, -5, -2), (1, -1, -2, 0), (5, -4, -4, -4), (1, -4, -6, -3)])
def test_reverse_gap_band_edges(aligner, scoring):
    """Gap-aware reverse band (sw_wavefront.cuh): a score-S path from the reversed origin drifts at
    most DD = (ms n2 - S - (|o| - |e|)) / |e| diagonals right and DI = (ms n2 - S - (|o| - |e|)) /
    (ms + |e|) left.  Pairs whose optimal alignment carries one deletion / insertion run of length k
    sit exactly on that edge (slack = k|e| resp. k(ms + |e|)); mixed with several runs, random
    flanks, single- and multi-stripe lengths, zero-cost extension (e = 0) and linear gaps."""
    ma, mm, o, e = scoring
    sc = {"alphabet": "dna", "match": ma, "mismatch": mm, "gap_open": o, "gap_extend": e}
    rng = np.random.default_rng(1000 + ma * 7 - mm * 3 - o - e)
    A = list("ACGT")
    pairs = []
    for t in range(60):
        n = int(rng.choice([40, 150, 170, 333, 700, 1500]))
        x = rng.choice(A, n)
        k = int(rng.integers(1, 40))
        cut = int(rng.integers(1, n))
        kind = t % 4
        if kind == 0:    # deletion run of k reference residues
            q = x
            r = np.concatenate([x[:cut], rng.choice(A, k), x[cut:]])
        elif kind == 1:  # insertion run of k query residues
            q = np.concatenate([x[:cut], rng.choice(A, k), x[cut:]])
            r = x
        elif kind == 2:  # several runs of both kinds
            q, r = list(x), list(x)
            for _ in range(int(rng.integers(2, 5))):
                c, kk = int(rng.integers(1, len(q))), int(rng.integers(1, 12))
                if rng.random() < 0.5:
                    r[c:c] = list(rng.choice(A, kk))
                else:
                    q[c:c] = list(rng.choice(A, kk))
            q, r = np.array(q), np.array(r)
        else:            # substitutions plus one run
            q = x.copy()
            mut = rng.random(n) < 0.02
            q[mut] = rng.choice(A, int(mut.sum()))
            r = np.concatenate([x[:cut], rng.choice(A, k), x[cut:]])
        fl = [rng.choice(A, int(rng.integers(0, 200))), rng.choice(A, int(rng.integers(0, 200)))]
        r = np.concatenate([fl[0], r, fl[1]])
        pairs.append(("".join(q), "".join(r)))
    b = synth.from_pairs(pairs, sc)
    exp = oracle_batch(b)
    try:
        for mode in (sw.SW_MODE_FULL, sw.SW_MODE_BAND_ALWAYS):  # row-sweep and banded reverse kernels
            aligner.set_mode(mode)
            assert_parity(aligner.align(b), exp, b)
            assert aligner.batch_status()[0] == sw.SW_OK
    finally:
        aligner.set_mode(sw.SW_MODE_FULL)


@pytest.mark.parametrize("kind", ["c2", "c1_scorings", "repeats", "indels"])
def test_banded_reverse_matches_row_sweep(kind):
    """Banded reverse kernels (sw_band.cuh: lanes own diagonals of the score-S band) against the
    oracle and against the row-sweep reverse pass (SW_MODE_NO_BAND) on the same batch: all five
    fields; the banded pass sweeps far fewer reverse cells on ADEPT-shaped reads."""
    import torch
    assert torch.cuda.is_available()
    rng = np.random.default_rng({"c2": 51, "c1_scorings": 52, "repeats": 53, "indels": 54}[kind])
    batches = []
    if kind == "c2":
        batches.append(synth.generate("c2", 0, 6000))
    elif kind == "c1_scorings":
        base = synth.generate("c1")
        for sc in [(3, -3, -6, -1), (2, -3, -5, -2), (1, -1, -2, 0), (5, -4, -4, -4), (2, -8, -3, -3), (4, 2, -9, -1)]:
            s = {"alphabet": "dna", "match": sc[0], "mismatch": sc[1], "gap_open": sc[2], "gap_extend": sc[3]}
            batches.append(synth.from_pairs([base.pair(p) for p in range(base.n_pairs)], s))
    elif kind == "repeats":
        pairs = []
        for _ in range(600):
            unit = "".join(rng.choice(list("ACGT"), int(rng.integers(1, 6))))
            n = int(rng.integers(20, 176))
            q = (unit * (n // len(unit) + 2))[:n]
            r = "".join(rng.choice(list("ACGT"), int(rng.integers(0, 40)))) + (unit * 80)[: n + int(rng.integers(-10, 60))] + \
                "".join(rng.choice(list("ACGT"), int(rng.integers(0, 40))))
            pairs.append((q, r))
        batches.append(synth.from_pairs(pairs, {"alphabet": "dna", "match": 3, "mismatch": -3, "gap_open": -6, "gap_extend": -1}))
    else:
        pairs = []
        A = list("ACGT")
        for t in range(800):
            n = int(rng.integers(8, 176))
            x = rng.choice(A, n)
            q, r = list(x), list(x)
            for _ in range(int(rng.integers(0, 4))):
                c, kk = int(rng.integers(0, len(q) + 1)), int(rng.integers(1, 20))
                if rng.random() < 0.5:
                    r[c:c] = list(rng.choice(A, kk))
                else:
                    q[c:c] = list(rng.choice(A, kk))
            q = q[:176]
            fl = [rng.choice(A, int(rng.integers(0, 300))), rng.choice(A, int(rng.integers(0, 300)))]
            pairs.append(("".join(q), "".join(fl[0]) + "".join(r) + "".join(fl[1])))
        batches.append(synth.from_pairs(pairs, {"alphabet": "dna", "match": 2, "mismatch": -3, "gap_open": -5, "gap_extend": -2}))
    a = sw.Aligner(0, poison=True)
    try:
        for b in batches:
            exp = oracle_batch(b)
            a.set_mode(sw.SW_MODE_NO_BAND)
            got_rows = a.align(b)
            rev_rows = a.reverse_cells()
            a.set_mode(sw.SW_MODE_BAND_ALWAYS)  # below the 16,384-pair default threshold
            got_band = a.align(b)
            rev_band = a.reverse_cells()
            assert_parity(got_rows, exp, b)
            assert_parity(got_band, exp, b)
            assert a.batch_status()[0] == sw.SW_OK
            if kind == "c2":
                assert rev_band < 0.6 * rev_rows, (rev_band, rev_rows)
            a.set_mode(sw.SW_MODE_FULL)
            assert_parity(a.align(b), exp, b)  # default mode (row sweep for batches this small)
    finally:
        a.close()


def test_banded_reverse_edges():
    """Banded reverse kernels at their routing edges (sw_band.cuh, finish_fwd): reversed query prefixes of
    1, 175-177 rows (BAND_MAX_N2 = 176), bands of exactly 32 / 33 / 64 / 65 diagonals (one deletion run
    sized so DI + DD + 1 lands on the edge), references shorter than the query, ends in the first
    columns, identical sequences (DI = DD = 0) and odd pair counts (empty halves), on a poisoned handle with
    the band kernels forced; all five fields vs the oracle."""
    rng = np.random.default_rng(61)
    A = list("ACGT")
    sc = {"alphabet": "dna", "match": 3, "mismatch": -3, "gap_open": -6, "gap_extend": -1}
    pairs = []
    for n in (1, 2, 7, 150, 170):
        x = "".join(rng.choice(A, n))
        pairs.append((x, x))                                              # identical
        pairs.append((x, x[: max(1, n // 3)]))                            # reference shorter than the query
        pairs.append((x, x + "".join(rng.choice(A, 300))))                # end in the first columns
    for n in (175, 176, 177):                                             # n2 around BAND_MAX_N2 = 176 (max_s n2 <= 511)
        x = "".join(rng.choice(A, n))
        pairs.append((x, "".join(rng.choice(A, 50)) + x + "".join(rng.choice(A, 50))))
    for k in range(1, 70, 3):                                             # one deletion run of k: DD grows with k
        x = rng.choice(A, 150)
        c = int(rng.integers(20, 130))
        r = np.concatenate([rng.choice(A, int(rng.integers(0, 40))), x[:c], rng.choice(A, k), x[c:],
                            rng.choice(A, int(rng.integers(0, 40)))])
        pairs.append(("".join(x), "".join(r)))
    for k in range(1, 12):                                                # insertion runs: DI grows with k
        x = rng.choice(A, 150)
        c = int(rng.integers(20, 130))
        q = np.concatenate([x[:c], rng.choice(A, k), x[c:]])
        pairs.append(("".join(q), "".join(rng.choice(A, 30)) + "".join(x)))
    pairs = pairs[: len(pairs) - (1 - len(pairs) % 2)]                   # an odd count: a half stays empty
    b = synth.from_pairs(pairs, sc)
    exp = oracle_batch(b)
    a = sw.Aligner(0, poison=True)
    try:
        for mode in (sw.SW_MODE_BAND_ALWAYS, sw.SW_MODE_NO_BAND):
            a.set_mode(mode)
            assert_parity(a.align(b), exp, b)
            assert a.batch_status()[0] == sw.SW_OK
    finally:
        a.close()
