"""Randomised parity soak (development tool): random batches under random valid scorings, every
field and every alignment path compared with the oracle.
    python tools/soak.py [seconds] [seed]              fields + paths vs the oracle
    python tools/soak.py [seconds] invariance [seed]   batch invariance at GPU speed (+ oracle sample)
    python tools/soak.py [seconds] diffusion           the diffusion stencil vs oracle/diffusion.py"""
from __future__ import annotations

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2208_12350_b200 import sw, synth  # noqa: E402

FIELDS = ("score", "q_end", "r_end", "q_start", "r_start")


def random_scoring(rng):
    if rng.random() < 0.3:
        o = -int(rng.integers(1, 20))
        e = o if rng.random() < 0.3 else int(rng.integers(o, 1))
        return {"alphabet": "protein", "match": 0, "mismatch": 0, "gap_open": o, "gap_extend": e}
    m = int(rng.integers(1, 12))
    x = int(rng.integers(-12, m))
    o = -int(rng.integers(1, 40))
    e = o if rng.random() < 0.3 else int(rng.integers(o, 1))
    return {"alphabet": "dna", "match": m, "mismatch": x, "gap_open": o, "gap_extend": e}


def batch(rng, sc):
    alpha = "ARNDCQEGHILKMFPSTWYV" if sc["alphabet"] == "protein" else ("AC" if rng.random() < 0.3 else "ACGT")
    pairs = []
    for _ in range(int(rng.integers(1, 400))):
        u = rng.random()
        n = int(rng.integers(0, 420)) if u < 0.6 else int(rng.integers(150, 560)) if u < 0.9 else int(rng.integers(400, 1300))
        q = "".join(rng.choice(list(alpha), n))
        if rng.random() < 0.6 and n:
            mut = [c if rng.random() > 0.1 else str(rng.choice(list(alpha))) for c in q]
            r = "".join(rng.choice(list(alpha), int(rng.integers(0, 60)))) + "".join(mut)
        else:
            r = "".join(rng.choice(list(alpha), int(rng.integers(0, 420))))
        if rng.random() < 0.02:
            q = q.lower()
        pairs.append((q, r))
    return synth.from_pairs(pairs, sc)


def soak_diffusion(rng, budget):
    """Random grids / rates / step counts / schedules of simcov_diffuse vs oracle/diffusion.py."""
    from oracle import diffusion as D
    from paper_2208_12350_b200 import simcov
    t0 = time.time()
    n = 0
    while time.time() - t0 < budget:
        H, W = int(rng.integers(1, 700)), int(rng.integers(1, 700))
        nf = int(rng.integers(1, 4))
        fields = synth.simcov_dense(int(rng.integers(0, 1 << 30)), H, W, nf, high=1 << int(rng.integers(8, 31)))
        rates = [int(rng.integers(0, simcov.SIMCOV_MAX_RATE + 1)) for _ in range(nf)]
        steps = int(rng.integers(0, 20))
        sch = int(rng.choice([0, 1, 2, 3, 4, 5, 6, 7, 8]))
        g = simcov.Grid(H, W, nf)
        g.upload(fields)
        simcov.simcov_set_schedule(sch)
        g.diffuse(rates, steps)
        got = g.download()
        exp = D.diffuse(fields, rates, steps)
        for f in range(nf):
            if not np.array_equal(got[f], exp[f]):
                print("DIFFUSION MISMATCH", H, W, nf, rates, steps, sch, flush=True)
                return 1
        n += 1
    simcov.simcov_set_schedule(0)
    print(f"diffusion soak ok: {n} random grids", flush=True)
    return 0


def check_fields(tag, sc, b, got, exp, nb):
    for f in FIELDS:
        bad = np.nonzero(got[f] != exp[f])[0]
        if bad.size:
            p = int(bad[0])
            print(tag, "MISMATCH", f, sc, "batch", nb, "pair", p, b.pair(p), [int(got[k][p]) for k in FIELDS],
                  [int(exp[k][p]) for k in FIELDS], flush=True)
            return False
    return True


def save_fail(b, sc, nb, seed, p=-1):
    import json as _json
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez("gpurun_out/soak_fail.npz", queries=b.queries, q_offsets=b.q_offsets, refs=b.refs,
             r_offsets=b.r_offsets, pair=p, batch_index=nb, seed=seed)
    _json.dump(sc, open("gpurun_out/soak_fail_scoring.json", "w"))


def fast_batch(rng, sc, count):
    """A larger random batch built with numpy (invariance soak): mixed lengths including multi-stripe
    queries and long references, half of the pairs related (the query embedded with substitutions)."""
    alpha = np.frombuffer(b"ARNDCQEGHILKMFPSTWYV" if sc["alphabet"] == "protein" else b"ACGT", dtype=np.uint8)
    if sc["alphabet"] == "dna" and rng.random() < 0.3:
        alpha = alpha[:2]
    u = rng.random(count)
    n = np.where(u < 0.5, rng.integers(0, 300, count), np.where(u < 0.9, rng.integers(150, 700, count),
                                                                  rng.integers(600, 2500, count)))
    pairs = []
    for k in range(count):
        q = alpha[rng.integers(0, alpha.size, int(n[k]))]
        if rng.random() < 0.5 and n[k]:
            r = q.copy()
            mut = rng.random(r.size) < rng.choice([0.02, 0.1, 0.3])
            r[mut] = alpha[rng.integers(0, alpha.size, int(mut.sum()))]
            r = np.concatenate([alpha[rng.integers(0, alpha.size, int(rng.integers(0, 200)))], r,
                                alpha[rng.integers(0, alpha.size, int(rng.integers(0, 200)))]])
        else:
            r = alpha[rng.integers(0, alpha.size, int(rng.integers(0, 1500)))]
        pairs.append((q.tobytes(), r.tobytes()))
    return synth.from_pairs(pairs, sc)


def soak_invariance(seed, budget):
    """Batch invariance (pin P11) at GPU speed: each random batch is aligned whole, permuted and
    split into random sub-batches, on a poisoned handle; every pair's five fields must agree bit for
    bit across the calls, and a random sample is checked against the oracle."""
    rng = np.random.default_rng(seed)
    a = sw.Aligner(0, poison=True)
    t0 = time.time()
    nb = npairs = 0
    try:
        while time.time() - t0 < budget:
            sc = random_scoring(rng)
            b = fast_batch(rng, sc, int(rng.integers(500, 6000)))
            a.set_mode(sw.SW_MODE_BAND_ALWAYS)  # the whole batch on the banded reverse kernels (DNA) ...
            ref = a.align(b)
            a.set_mode(sw.SW_MODE_FULL if rng.random() < 0.5 else sw.SW_MODE_BAND_ALWAYS)  # ... the rest either way
            perm = rng.permutation(b.n_pairs)
            got = a.align(b.subset(perm))
            inv = {f: np.empty_like(ref[f]) for f in FIELDS}
            for f in FIELDS:
                inv[f][perm] = got[f]
            if not check_fields("permuted", sc, b, inv, ref, nb):
                save_fail(b, sc, nb, seed)
                return 1
            cuts = np.sort(rng.choice(np.arange(1, b.n_pairs), size=min(3, b.n_pairs - 1), replace=False))
            parts = np.split(np.arange(b.n_pairs), cuts)
            for part in parts:
                sub = b.subset(part)
                g = a.align(sub)
                if not check_fields("split", sc, sub, g, {f: ref[f][part] for f in FIELDS}, nb):
                    save_fail(b, sc, nb, seed)
                    return 1
            idx = np.sort(rng.choice(b.n_pairs, size=min(48, b.n_pairs), replace=False))
            sub = b.subset(idx)
            exp = oracle.align_batch(sub.queries, sub.q_offsets, sub.refs, sub.r_offsets, sub.scoring)
            if not check_fields("oracle-sample", sc, sub, {f: ref[f][idx] for f in FIELDS}, exp, nb):
                save_fail(b, sc, nb, seed)
                return 1
            st, _ = a.batch_status()
            if st not in (sw.SW_OK, sw.SW_ERR_BAD_PAIRS):
                print("STATUS", st, "batch", nb, flush=True)
                return 1
            nb += 1
            npairs += b.n_pairs
    finally:
        a.close()
    print(f"invariance soak ok: seed {seed}, {nb} batches, {npairs} pairs x {2 + 1} calls, {time.time() - t0:.0f} s",
          flush=True)
    return 0


def main():
    """Every batch is drawn from one seeded generator (the seed alone replays the whole batch
    history), aligned on a handle in SW_MODE_POISON; the five fields of EVERY call are compared
    with the oracle -- also of the call whose results feed sw_traceback -- and sw_batch_status
    must report no internal error after each call."""
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    if len(sys.argv) > 2 and sys.argv[2] == "diffusion":
        return soak_diffusion(np.random.default_rng(int(time.time()) & 0xffff), budget)
    if len(sys.argv) > 2 and sys.argv[2] == "invariance":
        seed = int(sys.argv[3]) if len(sys.argv) > 3 else int(time.time() * 1000) & 0xffffffff
        print(f"invariance soak seed {seed}", flush=True)
        return soak_invariance(seed, budget)
    seed = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else int(time.time() * 1000) & 0xffffffff
    print(f"soak seed {seed}", flush=True)
    rng = np.random.default_rng(seed)
    a = sw.Aligner(0, poison=True)
    t0 = time.time()
    nb = npairs = npaths = 0
    try:
        while time.time() - t0 < budget:
            sc = random_scoring(rng)
            b = batch(rng, sc)
            # half of the batches force the banded reverse kernels (DNA; batches this small use the row
            # sweep by default)
            a.set_mode(sw.SW_MODE_BAND_ALWAYS if rng.random() < 0.5 else sw.SW_MODE_FULL)
            exp = oracle.align_batch(b.queries, b.q_offsets, b.refs, b.r_offsets, b.scoring)
            with_paths = rng.random() < 0.5
            if with_paths:
                got, paths = a.align_and_traceback(b)
            else:
                got = a.align(b)
            if not check_fields("paths" if with_paths else "fields", sc, b, got, exp, nb):
                save_fail(b, sc, nb, seed)
                return 1
            st, nbad = a.batch_status()
            if st not in (sw.SW_OK, sw.SW_ERR_BAD_PAIRS) or nbad != int(np.sum(exp["score"] < 0)):
                print("STATUS", st, nbad, "batch", nb, sw.sw_last_error_message(a.handle), flush=True)
                save_fail(b, sc, nb, seed)
                return 1
            if with_paths:
                for p in range(b.n_pairs):
                    q, r = b.pair(p)
                    res = tuple(int(exp[k][p]) for k in FIELDS)
                    want = oracle.traceback(q, r, b.scoring, res) if res[0] >= 0 else None
                    if paths[p] != want:
                        print("PATH MISMATCH", sc, "batch", nb, "pair", p, (q, r), paths[p], want, flush=True)
                        save_fail(b, sc, nb, seed, p)
                        return 1
                npaths += b.n_pairs
            nb += 1
            npairs += b.n_pairs
    finally:
        a.close()
    print(f"soak ok: seed {seed}, {nb} batches, {npairs} pairs ({npaths} with paths), {time.time() - t0:.0f} s",
          flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
