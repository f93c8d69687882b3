"""Per-opcode executed-instruction histogram + stall samples from an ncu source page (SASS view)."""
import csv, io, subprocess, sys, collections

def load(rep, kernel_idx=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = out.split('"Kernel Name"')
    blk = blocks[1 + kernel_idx]
    lines = blk.split("\n", 1)[1]
    rows = list(csv.reader(io.StringIO(lines)))
    hdr = rows[0]
    return blocks, [dict(zip(hdr, r)) for r in rows[1:] if len(r) == len(hdr)]

ALU = ("VIADDMNMX", "VIMNMX", "VIMNMX3", "PRMT", "LOP3", "SEL", "ISETP", "SHF", "IADD3", "PLOP3", "VIADD", "LEA", "MOV", "FLO", "POPC")
FMA = ("IMAD", "VIADD.16x2")

def main(rep, kidx=0):
    blocks, rows = load(rep, kidx)
    print(blocks[1 + kidx].split("\n", 1)[0][:100])
    ex = collections.Counter(); st = collections.Counter()
    tot = 0
    for d in rows:
        op = d["Source"].strip().split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1]
        n = int(d["Instructions Executed"] or 0)
        key = o
        ex[key] += n
        tot += n
        st[key] += int(d["Warp Stall Sampling (All Samples)"] or 0)
    for k, v in ex.most_common(40):
        print(f"{k:32s} {v:14d} {100*v/tot:6.2f}%  stall-samples={st[k]}")
    print("total", tot)

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
