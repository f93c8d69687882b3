"""sw_align_batch then sw_traceback on c2 (ncu target for the traceback kernel; development tool)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2208_12350_b200 import sw, synth  # noqa: E402
b = synth.generate("c2")
a = sw.Aligner(0)
q, qo, r, ro = a.to_device(b)
out = a.alloc_out(b.n_pairs)
a.align_tensors(q, qo, r, ro, b.scoring, out=out)
ops, n_ops = a.traceback_tensors(q, qo, r, ro, b.scoring, out)
a.traceback_tensors(q, qo, r, ro, b.scoring, out, ops, n_ops)
torch.cuda.synchronize()
print("done")
