"""GPU timeline (torch.profiler/CUPTI) of one host-buffer call: copies vs kernels on both compute streams."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2208_12350_b200 import sw, synth  # noqa: E402

b = synth.generate(sys.argv[1] if len(sys.argv) > 1 else "c2")
a = sw.Aligner(0)
s = torch.cuda.current_stream()
qh = torch.from_numpy(np.ascontiguousarray(b.queries)).pin_memory()
rh = torch.from_numpy(np.ascontiguousarray(b.refs)).pin_memory()
qoh = torch.from_numpy(b.q_offsets).pin_memory()
roh = torch.from_numpy(b.r_offsets).pin_memory()
outh = torch.empty((5, b.n_pairs), dtype=torch.int32).pin_memory()
ptrs = {f: outh[i].data_ptr() for i, f in enumerate(("score", "q_end", "r_end", "q_start", "r_start"))}


def host_call():
    assert sw.sw_align_batch_host(a.handle, qh.data_ptr(), qoh.data_ptr(), rh.data_ptr(), roh.data_ptr(),
                                  b.n_pairs, b.scoring, ptrs, s.cuda_stream) == 0


for _ in range(3):
    host_call()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        host_call()
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
ev = json.load(open("gpurun_out/e2e_trace.json"))["traceEvents"]
gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "ts" in e], key=lambda e: e["ts"])
t0 = gpu[0]["ts"]
for e in gpu:
    if e["dur"] > 8:
        print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f} s={e.get('args', {}).get('stream')} {e['name'][:60]}")
