"""Small fixed workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Runs every kernel family of the library on small inputs, each result checked against the oracle:
c1 (1,000 DNA pairs, forward + reverse, paths), a c3 protein prefix, multi-stripe c5 pairs (the
stripe hand-off, incl. the early-stop regression case), tie-heavy low-entropy pairs, int32-route
scorings, linear gaps, end-only mode, query-vs-database, the host-buffer entry points, and the
diffusion stencil.  Usage: compute-sanitizer --tool <t> python tools/sanitize_run.py [poison]
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2208_12350_b200 import sw, synth  # noqa: E402

FIELDS = ("score", "q_end", "r_end", "q_start", "r_start")


def check(tag, got, b):
    exp = oracle.align_batch(b.queries, b.q_offsets, b.refs, b.r_offsets, b.scoring)
    for f in FIELDS:
        if not np.array_equal(got[f], exp[f]):
            raise SystemExit(f"{tag}: field {f} differs from the oracle")
    print(f"{tag}: {b.n_pairs} pairs ok", flush=True)


def main():
    poison = len(sys.argv) > 1 and sys.argv[1] == "poison"
    a = sw.Aligner(0, poison=poison)
    rng = np.random.default_rng(5)
    # c1 with paths
    b = synth.generate("c1")
    got, paths = a.align_and_traceback(b)
    check("c1", got, b)
    for p in range(0, b.n_pairs, 50):
        q, r = b.pair(p)
        res = tuple(int(got[f][p]) for f in FIELDS)
        assert paths[p] == oracle.traceback(q, r, b.scoring, res), p
    # protein prefix
    b = synth.generate("c3", 0, 120)
    check("c3[:120]", a.align(b), b)
    # multi-stripe long pairs (c5 shape, bounded) + the early-stop regression shape
    tail = "".join(rng.choice(list("ACGT"), 25))
    x = "".join(rng.choice(list("ACGT"), 333))
    pairs = [("C" * 275 + tail, "G" * 875 + tail), (x, x)]
    for _ in range(6):
        n = int(rng.integers(170, 900))
        q = "".join(rng.choice(list("ACGT"), n))
        pairs.append((q, "".join(rng.choice(list("ACGT"), int(rng.integers(0, 300)))) + q[: n - 7]))
    b = synth.from_pairs(pairs, {"alphabet": "dna", "match": 1, "mismatch": -1, "gap_open": -3, "gap_extend": -1})
    check("multi-stripe", a.align(b), b)
    # CTA-cooperative reverse items (>= 8 stripes): long related / unrelated pairs
    pairs = []
    for k in range(6):
        n = int(rng.integers(1300, 2000))
        q = "".join(rng.choice(list("ACGT"), n))
        r = q[: n - 11] if k % 2 == 0 else "".join(rng.choice(list("ACGT"), n + 300))
        pairs.append((q, r))
    b = synth.from_pairs(pairs, synth.DNA_SCORING)
    check("cooperative reverse", a.align(b), b)
    # tie-heavy low-entropy DNA, several scorings (TAG / S16 / S32 routes)
    for sc in ({"alphabet": "dna", "match": 1, "mismatch": 0, "gap_open": -1, "gap_extend": -1},
               {"alphabet": "dna", "match": 2, "mismatch": -1, "gap_open": -3, "gap_extend": -1},
               {"alphabet": "dna", "match": 200, "mismatch": -100, "gap_open": -300, "gap_extend": -50}):
        b = synth.random_pairs(11, 150, (0, 240), (0, 400), b"AC", sc)
        check(f"ties {sc['match']}/{sc['mismatch']}/{sc['gap_open']}/{sc['gap_extend']}", a.align(b), b)
    # linear gaps (two-state kernels)
    b = synth.generate("c1", 0, 200)
    b.scoring.update(gap_open=-4, gap_extend=-4)
    check("linear-gap", a.align(b), b)
    # end-only mode
    a.set_mode(sw.SW_MODE_END_ONLY)
    b = synth.generate("c1", 0, 200)
    q, qo, r, ro = a.to_device(b)
    out, _ = a.align_tensors(q, qo, r, ro, b.scoring)
    import torch
    torch.cuda.synchronize()
    o = out[:3, :b.n_pairs].cpu().numpy()  # END_ONLY writes score / q_end / r_end only (the start rows stay unwritten)
    exp = oracle.align_batch(b.queries, b.q_offsets, b.refs, b.r_offsets, b.scoring)
    for i, f in enumerate(FIELDS[:3]):
        assert np.array_equal(o[i], exp[f]), f
    print("end-only ok", flush=True)
    a.set_mode(sw.SW_MODE_FULL)
    # query vs database
    src = synth.generate("c1", 0, 80)
    qq = src.pair(0)[0]
    refs = [src.pair(p)[1] for p in range(80)]
    got = a.align_query_db(qq, refs, src.scoring)
    check("query-db", got, synth.from_pairs([(qq, r_) for r_ in refs], src.scoring))
    # host-buffer entry points
    b = synth.generate("c1", 0, 300)
    hout = {f: np.zeros(b.n_pairs, np.int32) for f in FIELDS}
    st = sw.sw_align_batch_host(a.handle, b.queries.ctypes.data, b.q_offsets.ctypes.data, b.refs.ctypes.data,
                                b.r_offsets.ctypes.data, b.n_pairs, b.scoring, {f: hout[f].ctypes.data for f in FIELDS})
    assert st == sw.SW_OK, st
    check("host", hout, b)
    a.close()
    # diffusion stencil
    from oracle import diffusion as D
    from paper_2208_12350_b200 import simcov
    fields = synth.simcov_fields(0, 70, 130, 2, sites=20, peak=1 << 28, background=0.05)
    rates = [simcov.rate_fixed(0.2), simcov.rate_fixed(0.05)]
    g = simcov.Grid(70, 130, 2)
    g.upload(fields)
    g.diffuse(rates, 9)
    for x_, y_ in zip(g.download(), D.diffuse(fields, rates, 9)):
        assert np.array_equal(x_, y_)
    print("diffusion ok", flush=True)
    print("sanitize workload done", flush=True)


if __name__ == "__main__":
    main()
