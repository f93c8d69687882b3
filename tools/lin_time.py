"""Linear-gap kernels vs the affine kernels on c2 / c3 bytes re-scored with gap_open == gap_extend."""
import dataclasses, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2208_12350_b200 import sw, synth  # noqa: E402

for cfg, sc in (("c2", {"alphabet": "dna", "match": 3, "mismatch": -3, "gap_open": -2, "gap_extend": -2}),
                ("c3", {"alphabet": "protein", "match": 0, "mismatch": 0, "gap_open": -4, "gap_extend": -4})):
    b = dataclasses.replace(synth.generate(cfg), scoring=sc)
    a = sw.Aligner(0)
    a.enable_stage_timing(True)
    q, qo, r, ro = a.to_device(b)
    out = a.alloc_out(b.n_pairs)
    res = {}
    for mode in (sw.SW_MODE_FULL, sw.SW_MODE_AFFINE_ONLY):
        a.set_mode(mode)
        for _ in range(3):
            a.align_tensors(q, qo, r, ro, b.scoring, out=out)
        torch.cuda.synchronize()
        st = []
        for _ in range(5):
            a.align_tensors(q, qo, r, ro, b.scoring, out=out)
            torch.cuda.synchronize()
            st.append(a.stage_ms())
        med = {k: float(np.median([x[k] for x in st])) for k in st[0]}
        res[mode] = (med, out.clone())
        print(cfg, "linear" if mode == sw.SW_MODE_FULL else "affine", {k: round(v, 3) for k, v in med.items()},
              f"total {sum(med.values()):.3f} ms, fwd {b.cells() / med['fwd'] / 1e6:.0f} GCUPS", flush=True)
    assert torch.equal(res[0][1], res[2][1])
    a.close()
print("identical outputs")
