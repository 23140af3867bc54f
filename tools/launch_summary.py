"""Aggregate an ncu --metrics launch list (csv) by kernel: launches, time, DRAM bytes, share of step."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
agg = collections.defaultdict(lambda: {"n": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0})
for r in rows[hdr + 1:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").strip()
    name = name.split("<")[0].split("::")[-1]
    v = float(d["Metric Value"].replace(",", "")) if d["Metric Value"] else 0.0
    unit = d.get("Metric Unit", "")
    m = d["Metric Name"]
    key = (name, d["ID"])
    if m == "gpu__time_duration.sum":
        agg[name]["n"] += 1
        agg[name]["ns"] += v * (1e6 if unit == "ms" else 1e3 if unit == "us" else 1.0)
    elif m.startswith("dram__bytes_read"):
        agg[name]["rd"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    elif m.startswith("dram__bytes_write"):
        agg[name]["wr"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
tot = sum(a["ns"] for a in agg.values())
print(f"{'kernel':28s} {'launches':>8s} {'ms':>9s} {'share':>7s} {'DRAM GB':>9s} {'GB/s':>8s}")
for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
    gb = (a["rd"] + a["wr"]) / 1e9
    print(f"{name:28s} {a['n']:8d} {a['ns']/1e6:9.3f} {100*a['ns']/tot:6.1f}% {gb:9.2f} {gb/(a['ns']/1e9) if a['ns'] else 0:8.0f}")
print(f"{'total':28s} {sum(a['n'] for a in agg.values()):8d} {tot/1e6:9.3f}")
