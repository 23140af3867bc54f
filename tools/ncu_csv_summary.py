"""Summarise ncu csv exports (tools/gpu_prof3.sh): key details metrics, instructions per element,
stall reasons and the top stalled SASS lines.  usage: ncu_csv_summary.py PREFIX ELEMENTS [PREFIX ELEMENTS ...]"""
import csv
import gzip
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "L2 Hit Rate",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Issue Slots Busy",
        "Eligible Warps Per Scheduler", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]
args = sys.argv[1:]
for pre, elems in zip(args[::2], args[1::2]):
    elems = float(eval(elems))
    rows = list(csv.reader(open(pre + ".details.csv")))
    h = rows[0]
    seen, name = {}, ""
    for r in rows[1:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", name)
        if d.get("Metric Name") in KEYS and d["Metric Name"] not in seen:
            seen[d["Metric Name"]] = f"{d['Metric Value']} {d.get('Metric Unit', '')}"
    print(f"== {pre.split('/')[-1]} :: {name[:100]}")
    for k in KEYS:
        if k in seen:
            print(f"   {k:34s} {seen[k]}")
    raw = list(csv.reader(open(pre + ".raw.csv")))
    rh, rv = raw[0], raw[2]
    rd = dict(zip(rh, rv))
    tr = sum(float(rd[k]) * (1e9 if "Gbyte" in raw[1][rh.index(k)] else 1e6 if "Mbyte" in raw[1][rh.index(k)] else 1)
             for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in rd)
    print(f"   {'DRAM bytes (read+write)':34s} {tr / 1e9:.2f} GB")
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for k, v in rd.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v}
    tot = sum(stalls.values()) or 1
    print("   stall samples: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in
                                           sorted(stalls.items(), key=lambda kv: -kv[1])[:6]))
    src = list(csv.reader(gzip.open(pre + ".sass.csv.gz", "rt")))
    sh = src[1]
    ie, ist = sh.index("Instructions Executed"), sh.index("Warp Stall Sampling (All Samples)")
    data = [(r[1].strip(), int(r[ie] or 0), int(r[ist] or 0)) for r in src[2:] if len(r) > ie]
    ti = sum(d[1] for d in data)
    ts = sum(d[2] for d in data) or 1
    print(f"   {'thread instructions per element':34s} {32 * ti / elems:.1f}")
    for ins, _, st in sorted(data, key=lambda d: -d[2])[:6]:
        print(f"      {100 * st / ts:5.1f}%  {ins[:70]}")
