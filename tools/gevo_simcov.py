"""GEVO-style search over the diffusion kernel's variants (SURVEY.md sec. 8(f) f3 applied to f4).

The paper ran GEVO on SIMCoV too (1.29x on P100).  Here, as in
tools/gevo_search.py, a genome is a set of compile-time tunables of simcov_diffuse.cu -- warps
per CTA, rows per warp, the register cap (CTAs per SM), the largest steps per launch, the
persistent cp.async-prefetch variant -- and the fitness gate is bit-exact equality with the
shipped build (which tests/test_simcov_gpu.py ties to oracle/diffusion.py) on ragged grids,
full-range values and every launch-plan remainder.  Fitness: time of 24 steps of two 16384^2
fields (HBM-sized) and of the 2500^2 held-out grid.

  build   (CPU)        python tools/gevo_simcov.py build GEN
  measure (GPU box)    python tools/gevo_simcov.py measure GEN   -> gpurun_out/gevo_simcov_gGEN.json
  select  (CPU)        python tools/gevo_simcov.py select GEN    -> genomes of GEN+1 (mutation + crossover)
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
VAR = os.path.join(ROOT, "build_var", "gevo_simcov")
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles", "gevo")

SPACE = {  # first value = shipped default
    "SIMCOV_TB_WARPS": [8, 4, 16],
    "SIMCOV_TB_RPW": [20, 12, 16, 24, 10],
    "SIMCOV_TB_MINB": [2, 1, 3],
    "SIMCOV_TB_KMAX": [8, 4, 6, 7],
    "SIMCOV_TB_PIPE": [0, 1],
}
POP = 12


def valid(g):
    regs = 4 * g["SIMCOV_TB_RPW"] + 30                # tile words + working set per thread
    cap = 65536 // (32 * g["SIMCOV_TB_WARPS"] * g["SIMCOV_TB_MINB"])
    if regs > min(255, cap) + 16:                      # would spill heavily under the cap
        return False
    return g["SIMCOV_TB_WARPS"] * g["SIMCOV_TB_RPW"] > 2 * 8 + 16   # tile taller than the K=8 halo


def key(g):
    return "_".join(f"{k.split('_')[-1].lower()}{g[k]}" for k in SPACE)


def default():
    return {k: v[0] for k, v in SPACE.items()}


def genomes_path(gen):
    return os.path.join(VAR, f"g{gen}.json")


def build(gen):
    from paper_2208_12350_b200 import _build
    os.makedirs(VAR, exist_ok=True)
    if gen == 0:
        rng = random.Random(2208)
        pop = [default()]
        while len(pop) < POP:
            g = {k: rng.choice(v) for k, v in SPACE.items()}
            if valid(g) and g not in pop:
                pop.append(g)
    else:
        pop = json.load(open(genomes_path(gen)))
    pop = [default()] + [g for g in pop if g != default()]  # the shipped build is the gate's baseline
    def one(g):
        out = os.path.join(VAR, f"g{gen}_{key(g)}.so")
        _build.build(out=out, defines=[f"{k}={v}" for k, v in g.items()])
        return out
    with ThreadPoolExecutor(4) as ex:
        list(ex.map(one, pop))
    json.dump(pop, open(genomes_path(gen), "w"), indent=1)
    print(f"built {len(pop)} variants of generation {gen}")


CHILD = r'''
import json, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2208_12350_b200 import simcov, synth
res = {}
# fitness gate: outputs on ragged grids, several step counts, full-range values
outs = []
rng = np.random.default_rng(5)
for (H, W) in [(1, 1), (9, 130), (67, 121), (200, 371), (777, 1023)]:
    f = synth.simcov_dense(H * 7 + W, H, W, 2, high=1 << 30)
    g = simcov.Grid(H, W, 2)
    for steps in (1, 3, 8, 13):
        g.upload(f)
        g.diffuse([simcov.rate_fixed(0.21), simcov.SIMCOV_MAX_RATE], steps)
        outs.append(np.stack(g.download()).astype(np.uint64).sum(axis=(1, 2)).tolist()
                    + [int(np.bitwise_xor.reduce(np.stack(g.download()).ravel()))])
res["gate"] = outs
for name, (H, W) in (("g16384", (16384, 16384)), ("g2500", (2500, 2500))):
    g = simcov.Grid(H, W, 2)
    g.upload(synth.simcov_fields(5, H, W, 2, peak=1 << 26, background=0.05))
    rates = [simcov.rate_fixed(0.2), simcov.rate_fixed(0.1)]
    g.diffuse(rates, 24); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); g.diffuse(rates, 24); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    res[name] = float(np.median(ts))
    del g
print(json.dumps(res))
'''


def measure(gen):
    pop = json.load(open(genomes_path(gen)))
    base = None
    rows = []
    for g in pop:  # pop[0] is the shipped default (build())
        lib = os.path.join(VAR, f"g{gen}_{key(g)}.so")
        env = dict(os.environ, SW_B200_LIB=lib)
        r = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True, env=env, cwd=ROOT,
                           timeout=300)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
        except (IndexError, ValueError):
            rows.append({"genome": g, "error": r.stderr[-400:]})
            continue
        if base is None:
            base = d["gate"]
        d["genome"] = g
        d["gate_ok"] = d.pop("gate") == base
        rows.append(d)
        print(json.dumps({k: v for k, v in d.items()}), flush=True)
    os.makedirs(OUT, exist_ok=True)
    json.dump(rows, open(os.path.join(OUT, f"gevo_simcov_g{gen}.json"), "w"), indent=1)


def select(gen):
    rows = json.load(open(os.path.join(OUT, f"gevo_simcov_g{gen}.json")))
    ok = [r for r in rows if r.get("gate_ok")]
    ok.sort(key=lambda r: r["g16384"] + 10 * r["g2500"])
    parents = [r["genome"] for r in ok[:4]]
    rng = random.Random(gen + 1)
    nxt = [dict(parents[0])]
    while len(nxt) < POP:
        a, b = rng.sample(parents, 2) if len(parents) > 1 else (parents[0], parents[0])
        child = {k: (a[k] if rng.random() < 0.5 else b[k]) for k in SPACE}
        m = rng.choice(list(SPACE))
        child[m] = rng.choice(SPACE[m])
        if valid(child) and child not in nxt:
            nxt.append(child)
    os.makedirs(VAR, exist_ok=True)
    json.dump(nxt, open(genomes_path(gen + 1), "w"), indent=1)
    os.makedirs(PROF, exist_ok=True)
    with open(os.path.join(PROF, f"simcov_g{gen}.md"), "w") as f:
        f.write(f"# GEVO-style search over the diffusion kernel, generation {gen}\n\n"
                "| genome | gate | 16384² × 2 × 24 steps (ms) | 2500² × 2 × 24 steps (ms) |\n|---|---|---|---|\n")
        for r in sorted(rows, key=lambda r: r.get("g16384", 1e9)):
            if "error" in r:
                f.write(f"| {key(r['genome'])} | build/run error | | |\n")
            else:
                f.write(f"| {key(r['genome'])} | {'ok' if r['gate_ok'] else 'FAIL'} | {r['g16384']:.3f} | {r['g2500']:.4f} |\n")
    print("parents:", [key(p) for p in parents])


if __name__ == "__main__":
    cmd, gen = sys.argv[1], int(sys.argv[2])
    {"build": build, "measure": measure, "select": select}[cmd](gen)
