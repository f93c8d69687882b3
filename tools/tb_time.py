"""Time sw_traceback on c2 (or a config) after sw_align_batch (development tool)."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2208_12350_b200 import sw, synth  # noqa: E402
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
b = synth.generate(cfg)
a = sw.Aligner(0)
q, qo, r, ro = a.to_device(b)
out = a.alloc_out(b.n_pairs)
a.align_tensors(q, qo, r, ro, b.scoring, out=out)
ops, n_ops = a.traceback_tensors(q, qo, r, ro, b.scoring, out)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    a.traceback_tensors(q, qo, r, ro, b.scoring, out, ops, n_ops)
    e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(cfg, "traceback ms", round(float(np.median(ts)), 3), "ops", int(n_ops[:b.n_pairs].clamp(min=0).sum().item()))
