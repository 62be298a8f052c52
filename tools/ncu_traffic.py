"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
captures made by tools/ncu_configs.sh -> profiles/ncu_traffic.json (read by
bench.py as roofline.traffic), plus one summary JSON per capture.

    python tools/ncu_traffic.py [round-tag]
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
dest = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles")  # gpurun_out/ on the box
out = {}
for rep in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "prof_*.ncu-rep"))):
    w = os.path.basename(rep)[len("prof_"):-len(".ncu-rep")]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        continue
    h, u, v = rows[0], rows[1], rows[2]
    tot = 0.0
    ok = True
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k not in h:
            ok = False
            break
        i = h.index(k)
        tot += float(v[i].replace(",", "")) * UNIT.get(u[i], 1)
    if not ok:
        continue
    out[w] = tot
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, "--json",
                    os.path.join(dest, f"prof_{w}_{tag}_summary.json")],
                   capture_output=True)
    print(f"{w:28s} {tot / 1e6:12.1f} MB per launch")
path = os.path.join(dest, "ncu_traffic.json")
old = json.load(open(path)) if os.path.exists(path) else {}
old.update(out)
json.dump(old, open(path, "w"), indent=1, sort_keys=True)
