"""Three sw_align_batch calls on one config (for ncu: -k regex:wavefront_kernel -s 4 -c 2 captures call 3)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2208_12350_b200 import sw, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
b = synth.generate_parallel(cfg)
a = sw.Aligner(0)
q, qo, r, ro = a.to_device(b)
out = a.alloc_out(b.n_pairs)
for _ in range(3):
    a.align_tensors(q, qo, r, ro, b.scoring, out=out)
torch.cuda.synchronize()
print("done", cfg, b.n_pairs, b.cells())
