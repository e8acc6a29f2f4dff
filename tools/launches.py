"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(list)
for d in data:
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    ns = v if u in ("nsecond", "ns") else v * 1e3 if u in ("usecond", "us") else v * 1e6 if u in ("msecond", "ms") else v
    agg[d["Kernel Name"].split("(")[0][:70]].append(ns)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':70s} {'n':>4s} {'mean_us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:70s} {len(v):4d} {sum(v)/len(v)/1e3:9.2f} {sum(v)/tot*100:5.1f}%")
