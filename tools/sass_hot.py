"""Per-SASS-instruction executed counts from `ncu --page source --print-source sass --csv`,
grouped into contiguous address blocks, to find where a kernel's instructions go."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia = hdr.index("Instructions Executed")
st = hdr.index("Warp Stall Sampling (All Samples)")
data = [(r[0], r[1], int(r[ia] or 0), int(r[st] or 0)) for r in rows[2:] if len(r) > ia]
tot = sum(d[2] for d in data)
tots = sum(d[3] for d in data)
print("total warp instr", tot, "stall samples", tots)
win = int(sys.argv[2]) if len(sys.argv) > 2 else 32
for i in range(0, len(data), win):
    blk = data[i:i + win]
    s = sum(d[2] for d in blk)
    ss = sum(d[3] for d in blk)
    if s > 0.01 * tot or ss > 0.02 * tots:
        print(f"{blk[0][0][-5:]}  instr {100*s/tot:5.1f}%  stall {100*ss/tots:5.1f}%  | {blk[0][1].strip()[:40]} ... {blk[-1][1].strip()[:40]}")
