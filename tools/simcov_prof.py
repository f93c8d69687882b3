"""One diffuse call per schedule on a 16384^2 x 2 grid (ncu target; development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_12350_b200 import simcov, synth  # noqa: E402

H = W = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
g = simcov.Grid(H, W, 2)
g.upload(synth.simcov_fields(5, H, W, 2, peak=1 << 26, background=0.05))
rates = [simcov.rate_fixed(0.2), simcov.rate_fixed(0.1)]
for sch, steps in ((1, 2), (4, 8)):
    simcov.simcov_set_schedule(sch)
    g.diffuse(rates, steps)
torch.cuda.synchronize()
