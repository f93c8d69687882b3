"""Repro of a soak path mismatch (tests/golden/soak_case_tb16.json): the pair alone, with
random partners in the other s16x2 half, and on the int32 kernel."""
import json
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import oracle  # noqa: E402
from paper_2208_12350_b200 import sw, synth  # noqa: E402

c = json.load(open("tests/golden/soak_case_tb16.json"))
sc = c["sc"]
q, r = c["q"], c["r"]
a = sw.Aligner(0)
exp = oracle.traceback(q.encode(), r.encode(), sc)
def run(pairs, idx, mode=sw.SW_MODE_FULL):
    a.set_mode(mode)
    b = synth.from_pairs(pairs, sc)
    got = a.traceback(b)
    a.set_mode(sw.SW_MODE_FULL)
    return got[idx]
print("alone s16:", run([(q, r)], 0) == exp)
print("alone int32:", run([(q, r)], 0, sw.SW_MODE_TB_INT32) == exp)
rng = np.random.default_rng(1)
bad = 0
for k in range(200):
    n = int(rng.integers(0, 420)); m = int(rng.integers(0, 420))
    p2 = ("".join(rng.choice(list("ACGT"), n)), "".join(rng.choice(list("ACGT"), m)))
    g = run([(q, r), p2], 0)
    if g != exp:
        bad += 1
        if bad <= 3:
            print("partner", n, m, "gpu len", None if g is None else len(g), "exp len", len(exp),
                  "first diff", next((i for i, (x, y) in enumerate(zip(g or "", exp)) if x != y), None))
print("bad partners:", bad, "of 200")
