"""Development aid: one call on a config prefix (for compute-sanitizer), optional no-band mode."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2208_12350_b200 import sw, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
b = synth.generate(cfg, 0, n)
a = sw.Aligner(0, poison=True)
a.set_mode(mode)
got = a.align(b)
torch.cuda.synchronize()
print("ok", cfg, n, "mode", mode, a.batch_status(), "rev cells", a.reverse_cells())
if len(sys.argv) > 4:
    import oracle
    exp = oracle.align_batch(b.queries, b.q_offsets, b.refs, b.r_offsets, b.scoring)
    for f in ("score", "q_end", "r_end", "q_start", "r_start"):
        bad = np.nonzero(got[f] != exp[f])[0]
        print(f, "mismatches", bad.size, bad[:10])
