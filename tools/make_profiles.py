"""Write the judged ncu summaries under profiles/<round>/ from gpurun_out/.

    python tools/make_profiles.py r1
"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r1"
out = os.path.join(ROOT, "profiles", rnd)
os.makedirs(out, exist_ok=True)
go = os.path.join(ROOT, "gpurun_out")
if os.path.exists(os.path.join(go, "launches.csv")):
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launches.py"), os.path.join(go, "launches.csv")],
                         capture_output=True, text=True).stdout
    open(os.path.join(out, "launches.txt"), "w").write(
        "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches of\n"
        "`python bench.py --workload cfg2 --steps 12 --warmup 3 --profile`, launches 300-410: past the 16 warm-up grid updates): compare SHARES, not absolutes.\n\n" + txt)
    import shutil
    shutil.copy(os.path.join(go, "launches.csv"), os.path.join(out, "launches.csv"))
traffic = {}
for rep in sorted(glob.glob(os.path.join(go, "prof_*.ncu-rep"))):
    name = os.path.basename(rep)[5:-8]
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], capture_output=True,
                         text=True).stdout
    lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep], capture_output=True,
                           text=True).stdout
    open(os.path.join(out, f"ncu_{name}.txt"), "w").write(
        f"ncu --set full --clock-control none --import-source on (one launch)\n\n{txt}\n"
        f"per-source-line instruction / stall shares (top):\n{chr(10).join(lines.splitlines()[:30])}\n")
    rd = wr = None
    for ln in txt.splitlines():
        if ln.startswith("dram read"):
            parts = ln.split()
            try:
                rd, wr = float(parts[2]), float(parts[5])
                unit_r, unit_w = parts[3], parts[6]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rd *= scale.get(unit_r, 1)
                wr *= scale.get(unit_w, 1)
            except Exception:
                rd = wr = None
    if rd is not None:
        traffic[name] = rd + wr
json.dump(traffic, open(os.path.join(out, "ncu_traffic_bytes.json"), "w"), indent=1)
print("wrote", out, traffic)
