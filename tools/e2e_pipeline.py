"""End-to-end throughput of a stream of host-buffer batches (sw_submit_host) vs single calls."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2208_12350_b200 import sw, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
b = synth.generate(cfg)
a = sw.Aligner(0)
s = torch.cuda.current_stream()
qh = torch.from_numpy(np.ascontiguousarray(b.queries)).pin_memory()
rh = torch.from_numpy(np.ascontiguousarray(b.refs)).pin_memory()
qoh = torch.from_numpy(b.q_offsets).pin_memory()
roh = torch.from_numpy(b.r_offsets).pin_memory()
outs = [torch.empty((5, b.n_pairs), dtype=torch.int32).pin_memory() for _ in range(2)]
F = ("score", "q_end", "r_end", "q_start", "r_start")
ptrs = [{f: o[i].data_ptr() for i, f in enumerate(F)} for o in outs]


def submit(k):
    assert sw.sw_submit_host(a.handle, qh.data_ptr(), qoh.data_ptr(), rh.data_ptr(), roh.data_ptr(), b.n_pairs,
                             b.scoring, ptrs[k & 1], s.cuda_stream) == 0


for k in range(3):
    submit(k)
sw.sw_wait(a.handle)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t = time.perf_counter()
e0.record(s)
for k in range(steps):
    submit(k)
sw.sw_wait(a.handle)
e1.record(s)
e1.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"{cfg}: pipelined host batches {ms:.3f} ms/step -> {b.cells() / ms / 1e6:.1f} GCUPS "
      f"(wall {(time.perf_counter() - t) * 1e3 / steps:.3f} ms/step)")
ref = a.align(b)
o = outs[(steps - 1) & 1].numpy()
print("matches device path:", all((o[i] == ref[f]).all() for i, f in enumerate(F)))
