"""Summarise ncu output into profiles/<round>/ (tracked): launch-list shares and the
full-capture metrics of the wavefront kernels.

    python tools/make_profiles.py r01 gpurun_out/launches_r01.csv gpurun_out/prof_c2_r01.ncu-rep
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_shares(path: str) -> str:
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(lines)))
    for r in rd:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")), r.get("Metric Unit", "")))
    agg = collections.OrderedDict()
    for name, v, unit in rows:
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        key = name.split("(")[0][:90]
        a = agg.setdefault(key, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    ours = {k: v for k, v in agg.items() if "swb::" in k or "cub::" in k}
    tot = sum(v[1] for v in ours.values()) or 1.0
    out = ["| kernel | launches | total us | share of library time |", "|---|---|---|---|"]
    for k, (n, us) in sorted(ours.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f} % |")
    other = {k: v for k, v in agg.items() if k not in ours}
    out.append("")
    out.append(f"Other kernels in the process (torch fills, L2 flush, roofline probe): {sum(v[0] for v in other.values())} launches.")
    return "\n".join(out)


def raw_metrics(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def sass_hist(rep: str, idx: int):
    """Executed-instruction histogram of the idx-th kernel in the report (0-based)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-id", f":::{idx + 1}"], capture_output=True, text=True).stdout
    blocks = out.split('"Kernel Name"')
    if len(blocks) < 2:
        return []
    body = blocks[1].split("\n", 1)[1]  # first block only (the page can repeat the kernel)
    rows = list(csv.reader(io.StringIO(body)))
    hdr = rows[0]
    cnt = collections.Counter()
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        op = d["Source"].strip().split()
        if not op or not (d.get("Instructions Executed") or "").isdigit():
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        cnt[o] += int(d["Instructions Executed"])
    return cnt.most_common(18)


KEYS = [("gpu__time_duration.sum", "duration"), ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (of 64)"),
        ("launch__registers_per_thread", "registers/thread"), ("smsp__inst_executed.sum", "warp instructions"),
        ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / instruction")]


def full_summary(rep: str) -> str:
    out = []
    for idx, (d, u) in enumerate(raw_metrics(rep)):
        out.append(f"### `{d.get('Kernel Name', '?')[:110]}`\n")
        out.append("| metric | value |\n|---|---|")
        for k, name in KEYS:
            if k in d:
                out.append(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", "") or 0)
                  for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(stalls.values()) or 1
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        out.append("\nStall samples (share of all samples): " +
                   ", ".join(f"{k} {100 * v / tot:.1f} %" for k, v in top) + "\n")
        hist = sass_hist(rep, idx)
        if hist:
            total = sum(v for _, v in hist)
            out.append("Executed SASS opcodes (top 18): " + ", ".join(f"{k} {v / 1e6:.1f}M" for k, v in hist) + "\n")
    return "\n".join(out)


def main():
    rnd, launches, rep = sys.argv[1], sys.argv[2], sys.argv[3]
    d = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "launch_shares.md"), "w") as f:
        f.write(f"# ncu launch list ({rnd}): `ncu --metrics gpu__time_duration.sum --clock-control none` over "
                f"`bench.py --steps 2 --warmup 1` (cold-cache, serialised: compare shares, not absolutes)\n\n")
        f.write(launch_shares(launches) + "\n")
    with open(os.path.join(d, "ncu_full_wavefront.md"), "w") as f:
        f.write(f"# ncu --set full ({rnd}): wavefront kernels on c2 (100k DNA pairs), "
                f"`tools/prof_one.py c2`, 3rd call (forward, then reverse)\n\n")
        f.write(full_summary(rep) + "\n")
    print("wrote", d)


if __name__ == "__main__":
    main()
