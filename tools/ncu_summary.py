"""Summarise an .ncu-rep: key SOL / occupancy / DRAM metrics + top SASS stall lines."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Issue Slots Busy", "Mem Pipes Busy", "Block Limit Registers", "Block Limit Shared Mem",
        "Eligible Warps Per Scheduler", "Grid Size", "Block Size"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(io.StringIO(out))
    hdr = next(r)
    res = {}
    for row in r:
        d = dict(zip(hdr, row))
        if d.get("Metric Name") in KEYS:
            res[d["Metric Name"]] = d["Metric Value"] + " " + d.get("Metric Unit", "")
        res["_kernel"] = d.get("Kernel Name", "")
    return res


def raw(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {n: (vals[hdr.index(n)], units[hdr.index(n)]) for n in names if n in hdr}


def sass_top(rep, n=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:]]
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(float(d.get(key) or 0) for d in data) or 1
    top = sorted(data, key=lambda d: -float(d.get(key) or 0))[:n]
    return [(round(100 * float(d[key]) / tot, 1), d["Source"].strip()[:80]) for d in top]


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        d = details(rep)
        print("==", rep, "::", d.pop("_kernel")[:120])
        for k in KEYS:
            if k in d:
                print(f"   {k:32s} {d[k]}")
        r = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"])
        for k, (v, u) in r.items():
            print(f"   {k:32s} {v} {u}")
        for pct, src in sass_top(rep):
            print(f"     {pct:5.1f}%  {src}")
