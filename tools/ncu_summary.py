"""Summarise an ncu report (raw page) for the wavefront kernels: time, pipes, stalls, DRAM traffic."""
import csv, io, subprocess, sys, json

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:]]

KEYS = ["gpu__time_duration.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]

def main(rep):
    res = []
    for d in raw(rep):
        k = {"kernel": d.get("Kernel Name", "")[:60]}
        for key in KEYS:
            if key in d:
                k[key] = d[key]
        stalls = {kk.replace("smsp__average_warp_latency_issue_stalled_", "").replace(".ratio", ""): float(v)
                  for kk, v in d.items() if kk.startswith("smsp__average_warp_latency_issue_stalled_") and kk.endswith(".ratio") and v}
        if not stalls:
            stalls = {kk.replace("smsp__warps_issue_stalled_", "").replace("_per_warp_active.pct", ""): float(v.replace(",", ""))
                      for kk, v in d.items() if kk.startswith("smsp__warps_issue_stalled_") and kk.endswith("_per_warp_active.pct") and v}
        k["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
        res.append(k)
    return res

if __name__ == "__main__":
    for r in sys.argv[1:]:
        print(r)
        for k in main(r):
            print(json.dumps(k, indent=1))
