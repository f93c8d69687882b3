"""Break down the host-buffer entry point: H2D bandwidth, device-only call, host call."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2208_12350_b200 import sw, synth
b = synth.generate("c2")
a = sw.Aligner(0)
s = torch.cuda.current_stream()
qh = torch.from_numpy(np.ascontiguousarray(b.queries)).pin_memory()
rh = torch.from_numpy(np.ascontiguousarray(b.refs)).pin_memory()
qoh = torch.from_numpy(b.q_offsets).pin_memory(); roh = torch.from_numpy(b.r_offsets).pin_memory()
outh = torch.empty((5, b.n_pairs), dtype=torch.int32).pin_memory()
qd = torch.empty_like(qh, device="cuda"); rd = torch.empty_like(rh, device="cuda")
def ev(): return torch.cuda.Event(enable_timing=True)
for _ in range(3):
    qd.copy_(qh, non_blocking=True); rd.copy_(rh, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = ev(), ev(); e0.record(); qd.copy_(qh, non_blocking=True); rd.copy_(rh, non_blocking=True); e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1); print(f"H2D {qh.numel()+rh.numel():,} B in {ms:.3f} ms -> {(qh.numel()+rh.numel())/ms/1e6:.1f} GB/s")
ptrs = {f: outh[i].data_ptr() for i, f in enumerate(("score", "q_end", "r_end", "q_start", "r_start"))}
def host_call():
    st = sw.sw_align_batch_host(a.handle, qh.data_ptr(), qoh.data_ptr(), rh.data_ptr(), roh.data_ptr(), b.n_pairs, b.scoring, ptrs, s.cuda_stream)
    assert st == 0, st
for _ in range(3): host_call()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t = time.perf_counter(); e0, e1 = ev(), ev(); e0.record(); host_call(); e1.record(); e1.synchronize()
    ts.append((e0.elapsed_time(e1), (time.perf_counter() - t) * 1e3))
print("host call (event ms, wall ms):", ts)
q, qo, r, ro = a.to_device(b); out = a.alloc_out(b.n_pairs)
for _ in range(3): a.align_tensors(q, qo, r, ro, b.scoring, out=out)
torch.cuda.synchronize()
e0, e1 = ev(), ev(); e0.record(); a.align_tensors(q, qo, r, ro, b.scoring, out=out); e1.record(); e1.synchronize()
print("device call ms", e0.elapsed_time(e1))
import os
if os.environ.get("SW_PROBE_CHUNKS"):
    pass
