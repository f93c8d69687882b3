"""Run a small multi-stripe batch (C5-like) through the C ABI and compare with the oracle."""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle
from paper_2208_12350_b200 import sw, synth

rng = np.random.default_rng(1)
pairs = []
for n, m in [(170, 300), (400, 1200), (161, 161), (1000, 2000), (330, 50)]:
    q = "".join(rng.choice(list("ACGT"), n)); r = "".join(rng.choice(list("ACGT"), m))
    pairs.append((q, r))
b = synth.from_pairs(pairs, synth.DNA_SCORING)
a = sw.Aligner(0)
got = a.align(b)
exp = oracle.align_batch(b.queries, b.q_offsets, b.refs, b.r_offsets, b.scoring)
for f in got:
    print(f, got[f], exp[f])
