"""Quick timing of one config through the C ABI (development aid, not the bench contract)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2208_12350_b200 import sw, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
npairs = int(sys.argv[2]) if len(sys.argv) > 2 else None
t = time.time()
b = synth.generate_parallel(cfg, 0, npairs)
print(f"gen {cfg} {b.n_pairs} pairs cells={b.cells():.3e} in {time.time()-t:.1f}s", flush=True)
a = sw.Aligner(0)
a.enable_stage_timing(True)
q, qo, r, ro = a.to_device(b)
out = a.alloc_out(b.n_pairs)
s = torch.cuda.current_stream()
for _ in range(3):
    a.align_tensors(q, qo, r, ro, b.scoring, out=out)
torch.cuda.synchronize()
ts = []
stages = []
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    a.align_tensors(q, qo, r, ro, b.scoring, out=out)
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    stages.append(a.stage_ms())
ms = float(np.median(ts))
cells = b.cells()
fwd, swept = a.cell_counts()
print(f"{cfg}: median {ms:.3f} ms  -> {cells/ms/1e6:.1f} GCUPS (whole call)")
st = {k: float(np.median([x[k] for x in stages])) for k in stages[0]}
print("stages ms:", {k: round(v, 4) for k, v in st.items()})
print(f"fwd kernel GCUPS = {cells/st['fwd']/1e6:.1f}; swept/real = {swept/max(fwd,1):.3f}")
rsw = a.reverse_cells()
print(f"rev swept cells = {rsw:.4g} ({rsw/max(fwd,1):.3f} of fwd real); rev kernel swept GCUPS = {rsw/st['rev']/1e6:.1f}; "
      f"fwd kernel swept GCUPS = {swept/st['fwd']/1e6:.1f}")
print("launches:", a.launch_count(), "status:", a.batch_status())
print("dpx peak TCUPS:", sw.sw_dpx_peak(0, 200.0) / 1e12, "lib:", __import__("os").environ.get("SW_B200_LIB", "default"))
