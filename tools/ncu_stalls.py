"""Per-kernel key metrics and the top warp-stall reasons of an .ncu-rep (all kernels in it).
usage: ncu_stalls.py REP [REP...]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        print("==", rep.split("/")[-1], "::", d.get("Kernel Name", "")[:90])
        for k in KEYS:
            if k in d:
                print("   %-55s %s %s" % (k, d[k], units[hdr.index(k)]))
        st = {k: float(v) for k, v in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
              and v.replace(".", "", 1).isdigit()}
        top = sorted(st.items(), key=lambda kv: -kv[1])[:6]
        print("   stalls per issued instruction: " + ", ".join(
            "%s %.2f" % (k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), v)
            for k, v in top))
