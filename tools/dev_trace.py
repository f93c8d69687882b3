"""GPU timeline (torch.profiler/CUPTI) of one device-buffer sw_align_batch call: kernel gaps, syncs."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2208_12350_b200 import sw, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
b = synth.generate(cfg)
a = sw.Aligner(0)
q, qo, r, ro = a.to_device(b)
out = a.alloc_out(b.n_pairs)
for _ in range(3):
    a.align_tensors(q, qo, r, ro, b.scoring, out=out)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        a.align_tensors(q, qo, r, ro, b.scoring, out=out)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/dev_trace.json")
ev = json.load(open("gpurun_out/dev_trace.json"))["traceEvents"]
gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "ts" in e]
cpu = [e for e in ev if e.get("cat") == "cuda_runtime" and "ts" in e]
t0 = min(e["ts"] for e in gpu)
rows = [(e["ts"] - t0, e["dur"], "GPU", e["name"][:80]) for e in gpu]
rows += [(e["ts"] - t0, e["dur"], "CPU", e["name"][:80]) for e in cpu if e["dur"] > 5]
for t, d, k, n in sorted(rows):
    print(f"{k} {t:9.1f} {d:8.1f} {n}")
