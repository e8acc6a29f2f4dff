"""Key metrics of an ncu --set full report (one line per kernel launch)."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Issued Warp Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Executed Ipc Active", "Grid Size", "Block Size"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
seen = {}
for r in rows[1:]:
    d = dict(zip(h, r))
    k = (d.get("ID"), d.get("Kernel Name", "")[:50])
    seen.setdefault(k, {})
    if d.get("Metric Name") in KEYS:
        seen[k][d["Metric Name"]] = d["Metric Value"] + " " + d.get("Metric Unit", "")
for k, m in seen.items():
    print(k)
    for key in KEYS:
        if key in m:
            print(f"   {key:40s} {m[key]}")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    hh = rr[0]
    for row in rr[2:]:
        d = dict(zip(hh, row))
        rd = d.get("dram__bytes_read.sum", "?")
        wr = d.get("dram__bytes_write.sum", "?")
        print("dram read", rd, rr[1][hh.index("dram__bytes_read.sum")] if "dram__bytes_read.sum" in hh else "",
              "write", wr, rr[1][hh.index("dram__bytes_write.sum")] if "dram__bytes_write.sum" in hh else "")
