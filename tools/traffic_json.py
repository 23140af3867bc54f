"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of each kernel of one C5 step,
from an ncu launch list (csv, tools/gpu_prof3.sh); lx_main launches are split into fwd / bwd by order.
Writes a small json that bench.py reports as roofline.traffic for the dominant kernel."""
import collections
import csv
import json
import sys

src, log2n, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
rows = list(csv.reader(open(src)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
per_id = collections.OrderedDict()
for r in rows[hdr + 1:]:
    d = dict(zip(h, r))
    full = d["Kernel Name"]
    name = full.split("(")[0].replace("void ", "").strip().split("<")[0].split("::")[-1]
    if name == "lx_sort_pass" and full.replace(" ", "").split("(")[0].endswith(",1>"):
        name = "lx_splan"  # the plan pass runs the sort-pass kernel with SPLAN = true
    if not name:
        continue  # input generation (torch) in the profiled script
    v = float(d["Metric Value"].replace(",", "")) if d["Metric Value"] else 0.0
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d.get("Metric Unit", ""), 1)
    e = per_id.setdefault(d["ID"], {"name": name, "bytes": 0.0})
    if d["Metric Name"].startswith("dram__bytes"):
        e["bytes"] += v * scale
agg = collections.defaultdict(list)
mains = 0
for e in per_id.values():
    name = e["name"]
    if name == "lx_main":
        name = "lx_main_fwd" if mains == 0 else "lx_main_bwd"
        mains += 1
    agg[name].append(e["bytes"])
res = {"log2n": log2n, "source": src.split("/")[-1], "unit": "bytes per launch (ncu dram read+write)",
       "kernels": {k: sum(v) / len(v) for k, v in agg.items()}}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
