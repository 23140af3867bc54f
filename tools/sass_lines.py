"""Attribute ncu per-SASS-instruction counts (--page source --print-source sass --csv) to CUDA source
lines, using the line table of `nvdisasm -g -c` for the same build.
usage: sass_lines.py NVDISASM_TXT NCU_SASS_CSV[.gz] ELEMENTS [TOP]"""
import collections
import csv
import gzip
import re
import sys

dis, src, elems = sys.argv[1], sys.argv[2], float(eval(sys.argv[3]))
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
line_of = {}
cur = None
for ln in open(dis):
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
op = gzip.open if src.endswith(".gz") else open
rows = list(csv.reader(op(src, "rt")))
h = rows[1]
ie, ist = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[0], 16), r[1].strip(), int(r[ie] or 0), int(r[ist] or 0)) for r in rows[2:] if len(r) > ie]
base = data[0][0]
agg = collections.defaultdict(lambda: [0, 0])
for a, ins, c, st in data:
    key = line_of.get(a - base, ("?", 0))
    agg[key][0] += c
    agg[key][1] += st
ti = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values()) or 1
print(f"total thread instructions per element: {32 * ti / elems:.1f}")
srcs = {}
for (f, l), (c, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    if f not in srcs:
        try:
            srcs[f] = open(next(p for p in sys.argv[5:] if p.endswith(f))).read().split("\n") if len(sys.argv) > 5 else None
        except StopIteration:
            srcs[f] = None
    text = srcs[f][l - 1].strip()[:60] if srcs.get(f) else ""
    print(f"{f}:{l:<5d} {32 * c / elems:6.1f} instr/elem {100 * st / ts:5.1f}% stall  {text}")
