"""GEVO-style search over this kernel's variants.

The paper's method: evolve program variants, keep the
ones that stay bit-exact on the test inputs, select by measured runtime.  Here a
genome is a set of compile-time tunables of the sm_100a path (rows per lane K,
lanes per segment W, code prefetch distance, column unroll, blocks per SM, loop
body length), not LLVM-IR edits.  Each generation:

  build   (CPU, this container)  python tools/gevo_search.py build GEN
          -> build_var/gevo/gGEN_*.so + build_var/gevo/gGEN.json (genomes)
  measure (GPU box)              python tools/gevo_search.py measure GEN
          -> gpurun_out/gevo_gGEN.json: per variant c2 and c3 call time, forward-kernel
             time, and the fitness gate: all five fields of 2,000 c2 pairs, 300 c3
             pairs and 400 tie-heavy pairs equal to the baseline build's, which the
             GPU parity tests tie to the oracle
  select  (CPU)                  python tools/gevo_search.py select GEN
          -> parents of GEN+1 = the fastest gated variants; next genomes by
             mutation (one tunable) and uniform crossover

Results are summarised in profiles/gevo/.
"""
from __future__ import annotations

import json
import os
import random
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "build_var", "gevo")
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles", "gevo")

# tunable -> allowed values (the first is the shipped default).  Two targets: the DNA geometry (fitness:
# c2 GCUPS) and, with GEVO_TARGET=protein, the protein path (fitness: c3 GCUPS) -- rows / lanes of the
# 25-code int8 profile, block shape, code prefetch, column unroll and the improvement-recording forms
TARGET = os.environ.get("GEVO_TARGET", "dna")
SPACE_DNA = {
    "SW_K16": [10, 8, 12, 16],
    "SW_W16": [16, 8],
    "SW_CODE_DIST": [4, 1, 2],
    "SW_UNROLL": [4, 2, 8],
    "SW_MIN_BLOCKS": [4, 3, 5],
    "SW_BODY_BLOCKS": [2, 1],
}
SPACE_PROTEIN = {
    "SW_KP": [8, 6, 4],
    "SW_WP": [16, 8],
    "SW_PROT_THREADS": [96, 64, 128, 32],
    "SW_PROT_BLOCKS": [5, 7, 3, 4, 15],
    "SW_CODE_DIST": [4, 1, 2],
    "SW_UNROLL": [4, 2, 8],
    "SW_IMPROVE_VOTE": [0, 1],
    "SW_PRED_IMPROVE": [0, 1],
    "SW_PTAG": [0, 1],
}
SPACE = SPACE_PROTEIN if TARGET == "protein" else SPACE_DNA
FIT = "c3" if TARGET == "protein" else "c2"
TAG = "p" if TARGET == "protein" else ""
POP = 10


def valid(g: dict) -> bool:
    if TARGET == "protein":
        rows = g["SW_KP"] * g["SW_WP"]
        warps = g["SW_PROT_THREADS"] // 32 * g["SW_PROT_BLOCKS"]
        if g["SW_UNROLL"] % g["SW_CODE_DIST"] or not (64 <= rows <= 128) or warps > 15 or warps < 8:
            return False        # shared memory (12.8 KB profile per warp) holds at most 15 warps per SM
        if g["SW_PTAG"] and (g["SW_KP"] != 8 or g["SW_IMPROVE_VOTE"] or g["SW_PRED_IMPROVE"]):
            return False        # the protein TAG form is the 8-row geometry and has no improvement branch
        return not (g["SW_IMPROVE_VOTE"] and g["SW_PRED_IMPROVE"])
    rows = g["SW_K16"] * g["SW_W16"]
    if g["SW_UNROLL"] % g["SW_CODE_DIST"]:
        return False            # static_assert since generations 0-1, whose parity gate rejected distance 3
    if g["SW_W16"] == 8 and g["SW_K16"] < 16:
        return False            # 8-lane segments only make sense with tall lanes
    if g["SW_K16"] > 16 and g["SW_W16"] == 16:
        return False
    return 64 <= rows <= 320


def key(g: dict) -> str:
    return "-".join(f"{k[3:].lower()}{g[k]}" for k in sorted(g)).replace("_", "")


def default() -> dict:
    return {k: v[0] for k, v in SPACE.items()}


def mutate(g: dict, rng: random.Random) -> dict:
    while True:
        c = dict(g)
        k = rng.choice(list(SPACE))
        c[k] = rng.choice([v for v in SPACE[k] if v != g[k]])
        if valid(c):
            return c


def crossover(a: dict, b: dict, rng: random.Random) -> dict:
    c = {k: (a[k] if rng.random() < 0.5 else b[k]) for k in SPACE}
    return c if valid(c) else mutate(a, rng)


def genomes_path(gen: int) -> str:
    return os.path.join(VAR, f"{TAG}g{gen}.json")


def cmd_build(gen: int):
    os.makedirs(VAR, exist_ok=True)
    rng = random.Random(1000 + gen)
    if gen == 0:
        pop = [default()]
        while len(pop) < POP:
            c = mutate(default(), rng)
            if key(c) not in {key(x) for x in pop}:
                pop.append(c)
    else:
        sel = json.load(open(os.path.join(PROF, f"select_{TAG}g{gen - 1}.json")))
        parents = sel["parents"]
        seen = set(sel["evaluated"])
        pop = [parents[0]]  # elitism
        tries = 0
        while len(pop) < POP and tries < 1000:
            tries += 1
            c = crossover(rng.choice(parents), rng.choice(parents), rng) if rng.random() < 0.5 else \
                mutate(rng.choice(parents), rng)
            if key(c) not in seen and key(c) not in {key(x) for x in pop}:
                pop.append(c)
    from paper_2208_12350_b200 import _build

    def one(g):
        out = os.path.join(VAR, f"{TAG}g{gen}_{key(g)}.so")
        if not os.path.exists(out):
            _build.build(force=True, out=out, defines=[f"{k}={v}" for k, v in g.items()])
        return out

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        libs = list(ex.map(one, pop))
    json.dump({"gen": gen, "genomes": pop, "libs": [os.path.relpath(l, ROOT) for l in libs]},
              open(genomes_path(gen), "w"), indent=1)
    print(f"generation {gen}: built {len(libs)} variants")


CHILD = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, ".")
from paper_2208_12350_b200 import sw, synth
a = sw.Aligner(0); a.enable_stage_timing(True)
res = {}
sets = {"c2": synth.generate("c2"), "c3": synth.generate("c3")}
rng = np.random.default_rng(5)
ties = synth.from_pairs([("".join(rng.choice(list("AC"), int(rng.integers(1, 300)))),
                          "".join(rng.choice(list("AC"), int(rng.integers(1, 300))))) for _ in range(400)],
                        {"alphabet": "dna", "match": 2, "mismatch": -2, "gap_open": -1, "gap_extend": -1})
for name, b in sets.items():
    q, qo, r, ro = a.to_device(b); out = a.alloc_out(b.n_pairs)
    for _ in range(2): a.align_tensors(q, qo, r, ro, b.scoring, out=out)
    torch.cuda.synchronize()
    ts, fw = [], []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); a.align_tensors(q, qo, r, ro, b.scoring, out=out); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1)); fw.append(a.stage_ms()["fwd"])
    o = out[:, :b.n_pairs].cpu().numpy()
    keep = o[:, :2000] if name == "c2" else o[:, :2000]
    res[name] = {"ms": float(np.median(ts)), "fwd_ms": float(np.median(fw)), "cells": b.cells(),
                 "gate": keep.astype(np.int64).tolist()}
o = a.align(ties)
res["ties"] = {"gate": np.stack([o[f] for f in ("score", "q_end", "r_end", "q_start", "r_start")]).astype(np.int64).tolist()}
pties = synth.from_pairs([("".join(rng.choice(list("AW"), int(rng.integers(1, 900)))),
                           "".join(rng.choice(list("AW"), int(rng.integers(1, 900))))) for _ in range(300)], synth.PROTEIN_SCORING)
o = a.align(pties)
res["pties"] = {"gate": np.stack([o[f] for f in ("score", "q_end", "r_end", "q_start", "r_start")]).astype(np.int64).tolist()}
print("RESULT " + json.dumps(res))
'''


def cmd_measure(gen: int):
    meta = json.load(open(genomes_path(gen)))
    base_lib = os.path.join(ROOT, "paper_2208_12350_b200", "libsw_b200.so")
    runs = [("baseline", base_lib, default())] + list(zip(
        [key(g) for g in meta["genomes"]], [os.path.join(ROOT, l) for l in meta["libs"]], meta["genomes"]))
    results = {}
    for name, lib, g in runs:
        env = dict(os.environ, SW_B200_LIB=lib)
        r = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True, env=env, cwd=ROOT,
                           timeout=900)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        results[name] = {"genome": g, "result": json.loads(line[-1][7:]) if line else None,
                         "error": None if line else r.stderr[-800:]}
        print(name, "ok" if line else "FAILED", flush=True)
    os.makedirs(OUT, exist_ok=True)
    json.dump(results, open(os.path.join(OUT, f"gevo_{TAG}g{gen}.json"), "w"))


def cmd_select(gen: int):
    res = json.load(open(os.path.join(OUT, f"gevo_{TAG}g{gen}.json")))
    base = res["baseline"]["result"]
    rows, evaluated = [], []
    for name, d in res.items():
        if name == "baseline":
            continue
        evaluated.append(name)
        r = d["result"]
        ok = r is not None and all(r[s]["gate"] == base[s]["gate"] for s in ("c2", "c3", "ties", "pties") if s in base)
        rows.append({"variant": name, "genome": d["genome"], "gated": ok,
                     "c2_ms": r["c2"]["ms"] if r else None, "c2_fwd_ms": r["c2"]["fwd_ms"] if r else None,
                     "c3_ms": r["c3"]["ms"] if r else None,
                     "c3_fwd_ms": r["c3"]["fwd_ms"] if r else None,
                     "fitness": (r[FIT]["cells"] / r[FIT]["ms"] / 1e6) if (r and ok) else 0.0})
    rows.sort(key=lambda x: -x["fitness"])
    prev = []
    if gen > 0:
        prev = json.load(open(os.path.join(PROF, f"select_{TAG}g{gen - 1}.json")))["evaluated"]
    parents = [x["genome"] for x in rows if x["gated"]][:3]
    os.makedirs(PROF, exist_ok=True)
    json.dump({"gen": gen, "baseline_c2_ms": base["c2"]["ms"], "baseline_c3_ms": base["c3"]["ms"],
               "rows": rows, "parents": parents or [default()], "evaluated": sorted(set(prev + evaluated))},
              open(os.path.join(PROF, f"select_{TAG}g{gen}.json"), "w"), indent=1)
    print(f"generation {gen}: baseline c2 {base['c2']['ms']:.3f} ms, c3 {base['c3']['ms']:.3f} ms")
    for x in rows:
        print(f"  {x['variant']:60s} gated={x['gated']!s:5s} c2 {x['c2_ms']} ms  fwd {x['c2_fwd_ms']}  c3 {x['c3_ms']} (fwd {x['c3_fwd_ms']})")


if __name__ == "__main__":
    cmd, gen = sys.argv[1], int(sys.argv[2])
    {"build": cmd_build, "measure": cmd_measure, "select": cmd_select}[cmd](gen)
