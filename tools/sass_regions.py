"""Group a kernel's executed SASS by execution count (finds the hot loop vs per-item overhead).

    python tools/sass_regions.py rep.ncu-rep 'regex:wavefront:2'
"""
import collections, csv, io, subprocess, sys
rep, kid = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-id", "::" + kid],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out.split("\n", 1)[1])))
hdr = rows[0]
ix, isrc, istall = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
ins = [(r[isrc].strip(), int(r[ix] or 0), int(r[istall] or 0)) for r in rows[1:] if len(r) == len(hdr) and r[ix].isdigit()]
tot = sum(c for _, c, _ in ins); stot = sum(s for _, _, s in ins) or 1
print(f"total warp instr {tot/1e6:.1f}M, {len(ins)} SASS lines")
# contiguous runs with equal count = basic blocks
blocks = []
for k, (s, c, st) in enumerate(ins):
    if blocks and blocks[-1][1] == c and blocks[-1][3] == k - 1:
        b = blocks[-1]; blocks[-1] = (b[0], c, b[2] + 1, k, b[4] + st, b[5] + [s])
    else:
        blocks.append((k, c, 1, k, st, [s]))
big = sorted(blocks, key=lambda b: -b[1] * b[2])[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]
for b in sorted(big):
    ops = collections.Counter(x.split()[1] if x.startswith("@") else x.split()[0] for x in b[5] if x)
    print(f"[{b[0]:5d}-{b[3]:5d}] exec {b[1]:>10d} x {b[2]:4d} instr = {100*b[1]*b[2]/tot:5.1f}% instr, "
          f"{100*b[4]/stot:5.1f}% stalls | " + ", ".join(f"{k}:{v}" for k, v in ops.most_common(6)))
