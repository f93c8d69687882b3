"""Time several library builds (SW_B200_LIB) on one config; each variant in its own process."""
import glob, json, os, subprocess, sys

CHILD = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, ".")
from paper_2208_12350_b200 import sw, synth
cfg = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "all" else None
b = synth.generate(cfg, 0, n)
a = sw.Aligner(0); a.enable_stage_timing(True)
q, qo, r, ro = a.to_device(b); out = a.alloc_out(b.n_pairs)
for _ in range(2): a.align_tensors(q, qo, r, ro, b.scoring, out=out)
torch.cuda.synchronize()
st = []
for _ in range(5):
    a.align_tensors(q, qo, r, ro, b.scoring, out=out); torch.cuda.synchronize(); st.append(a.stage_ms())
med = {k: float(np.median([x[k] for x in st])) for k in st[0]}
res = a.batch_status()
o = out[:, :b.n_pairs].cpu().numpy()
print(json.dumps({"cfg": cfg, "cells": b.cells(), "stage_ms": med, "fwd_gcups": b.cells() / med["fwd"] / 1e6,
                  "total_ms": sum(med.values()), "status": res, "checksum": int(o.astype(np.int64).sum())}))
'''

def main():
    cfgs = sys.argv[1].split(",")
    libs = sys.argv[2:] or sorted(glob.glob("build_var/*.so"))
    for lib in libs:
        for cfg in cfgs:
            env = dict(os.environ, SW_B200_LIB=lib)
            r = subprocess.run([sys.executable, "-c", CHILD, cfg], capture_output=True, text=True, env=env)
            line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:]
            print(os.path.basename(lib), line, flush=True)

if __name__ == "__main__":
    main()
