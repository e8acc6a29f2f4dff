"""Per-source-line instruction and stall shares from an ncu report (needs -lineinfo)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = collections.defaultdict(lambda: [0, 0])
hdr = None
cur_file, fn = None, None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) == 2 and r[0] == "Function Name":
        fn = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if kfilter and fn and kfilter not in fn:
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        try:
            ie = int(r[hdr.index("Instructions Executed")] or 0)
            st = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        key = (cur_file, int(r[0]), r[1][:100])
        agg[key][0] += ie
        agg[key][1] += st
tot = sum(v[0] for v in agg.values()) or 1
tots = sum(v[1] for v in agg.values()) or 1
print("total warp instructions", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:45]:
    print(f"{v[0]/tot*100:5.1f}% instr {v[1]/tots*100:5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")
