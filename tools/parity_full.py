"""Every-pair parity at BASELINE.json's full sizes ("every pair, all five
fields, bit-exact, on every config", the paper's own 100 %-accuracy regime).

For each config: the seeded batch (synth.generate_parallel, byte-identical to synth.generate), one
sw_align_batch call over the WHOLE batch on cuda:0 (the launch configuration bench.py times), then
the CPU oracle (oracle/, all host cores) on every pair, and a field-by-field comparison.  Writes one
JSON record per config (pairs, cells, mismatches per field, GPU ms, oracle s, batch SHA-256).

    python tools/parity_full.py c3 c4 c5 [--out profiles/r08/parity_full.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

FIELDS = ("score", "q_end", "r_end", "q_start", "r_start")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--out", default="gpurun_out/parity_full.jsonl")
    ap.add_argument("--threads", type=int, default=0)
    args = ap.parse_args()
    import torch

    import oracle
    from paper_2208_12350_b200 import sw, synth

    cores = args.threads or os.cpu_count() or 1
    a = sw.Aligner(0)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    for key in args.configs:
        t0 = time.time()
        b = synth.generate_parallel(key)
        t_gen = time.time() - t0
        sha = synth.batch_sha256(b)
        q, qo, r, ro = a.to_device(b)
        out = a.alloc_out(b.n_pairs)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        a.align_tensors(q, qo, r, ro, b.scoring, out=out)
        e1.record()
        e1.synchronize()
        gpu_ms = e0.elapsed_time(e1)
        st, nbad = a.batch_status()
        got = out[:, :b.n_pairs].cpu().numpy()
        del q, qo, r, ro, out
        torch.cuda.empty_cache()
        t1 = time.time()
        exp = oracle.align_batch(b.queries, b.q_offsets, b.refs, b.r_offsets, b.scoring, threads=cores)
        t_orc = time.time() - t1
        mism = {f: int(np.sum(got[i] != exp[f])) for i, f in enumerate(FIELDS)}
        first = None
        if any(mism.values()):
            bad = np.nonzero(np.any(np.stack([got[i] != exp[f] for i, f in enumerate(FIELDS)]), axis=0))[0]
            p = int(bad[0])
            first = {"pair": p, "n": int(b.q_offsets[p + 1] - b.q_offsets[p]), "m": int(b.r_offsets[p + 1] - b.r_offsets[p]),
                     "gpu": [int(got[i][p]) for i in range(5)], "oracle": [int(exp[f][p]) for f in FIELDS]}
        n, m = b.lengths()
        rec = {"config": key, "workload": synth.CONFIGS[key].name, "pairs": b.n_pairs, "cells": b.cells(),
               "max_n": int(n.max()), "max_m": int(m.max()), "batch_sha256": sha,
               "pairs_checked": b.n_pairs, "fields": list(FIELDS), "mismatches": mism,
               "total_mismatches": int(sum(mism.values())), "first_mismatch": first,
               "batch_status": sw.status_string(st), "bad_pairs": nbad,
               "gpu_call_ms": round(gpu_ms, 3), "oracle_s": round(t_orc, 1), "oracle_threads": cores,
               "oracle_gcups": round(b.cells() / t_orc / 1e9, 3), "generate_s": round(t_gen, 1),
               "gpu": torch.cuda.get_device_name(0)}
        print(json.dumps(rec), flush=True)
        with open(args.out, "a") as f:
            f.write(json.dumps(rec) + "\n")
        del b, got, exp
    a.close()


if __name__ == "__main__":
    main()
