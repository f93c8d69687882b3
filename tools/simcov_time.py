"""Time simcov_diffuse per schedule on the GPU (development tool; bench.py reports the default).

python tools/simcov_time.py [H W steps]
"""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2208_12350_b200 import simcov, synth  # noqa: E402


def time_one(g, rates, steps, reps=5):
    s = torch.cuda.current_stream()
    g.diffuse(rates, steps)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.diffuse(rates, steps)
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    H, W, steps = (int(x) for x in sys.argv[1:4]) if len(sys.argv) >= 4 else (16384, 16384, 16)
    fields = synth.simcov_fields(5, H, W, 2, peak=1 << 26, background=0.05)
    rates = [simcov.rate_fixed(0.2), simcov.rate_fixed(0.1)]
    g = simcov.Grid(H, W, 2)
    g.upload(fields)
    cells = 2 * H * W
    for sch in [int(x) for x in os.environ.get("SCHEDULES", "1,2,3,4,5,6,7,8").split(",")]:
        simcov.simcov_set_schedule(sch)
        ms = time_one(g, rates, steps)
        n = simcov.simcov_last_launch_count() - 2
        print(json.dumps({"H": H, "W": W, "steps": steps, "schedule": sch, "ms": round(ms, 4),
                          "gcell_steps_per_s": round(cells * steps / ms / 1e6, 1),
                          "launches": n,
                          "hbm_alg_GBps_per_launch": round(8 * cells * n / ms / 1e6, 1)}))
    simcov.simcov_set_schedule(0)


if __name__ == "__main__":
    main()
