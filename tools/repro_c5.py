import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2208_12350_b200 import sw, synth
cfg = synth.CONFIGS["c5"]
n, m = synth.batch_lengths(cfg, 0, 4096)
longs = np.nonzero(n > 150)[0]
cost = n[longs] * m[longs]
pick = list(longs[np.argsort(cost)][::max(1, len(longs) // 24)][:24]) + list(np.nonzero(n == 150)[0][:200])
full = synth.generate("c5", 0, 4096)
b = full.subset(sorted(int(p) for p in pick))
nn, mm = b.lengths()
print("max n", nn.max(), "max m", mm.max(), "pairs", b.n_pairs, flush=True)
a = sw.Aligner(0)
got = a.align(b)
print(got["score"][:20])
