"""Summarise tools/rate_slopes.sh: executed FP64 flops (512 per DMMA.8x8x4, 2 per DFMA,
1 per DMUL / DADD) and DRAM bytes per element for every (space, path, p), and the
log-log slope vs p over p >= 5 -- the algorithmic rate separated from the efficiency
curve of the time fits.

    python tools/rate_slopes.py gpurun_out > profiles/rate_slopes_r02.json
"""
import csv
import glob
import json
import math
import os
import re
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
E = 64
pts = {}
for f in sorted(glob.glob(os.path.join(d, "rate_c5_*.csv"))):
    m = re.search(r"rate_c5_(\w+)_p(\d+)_(\w+)\.csv", f)
    sp, p, path = m.group(1), int(m.group(2)), m.group(3)
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if len(rows) < 2:
        continue
    hdr = rows[0]
    idx = {k: i for i, k in enumerate(hdr)}
    vals = {}
    for r in rows[1:]:
        vals[r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
    fl = (512 * vals.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0)
          + 2 * vals.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0)
          + vals.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0)
          + vals.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0))
    pts.setdefault((sp, path), []).append({
        "p_test": p, "exec_dflop_per_element": fl / E,
        "dram_write_bytes_per_element": vals.get("dram__bytes_write.sum", 0) / E,
        "kernel_us": vals.get("gpu__time_duration.sum", 0) / 1e3})


def slope(xs, ys):
    lx, ly = [math.log(x) for x in xs], [math.log(y) for y in ys]
    mx, my = sum(lx) / len(lx), sum(ly) / len(ly)
    return sum((a - mx) * (b - my) for a, b in zip(lx, ly)) / sum((a - mx) ** 2 for a in lx)


out = {"note": "ncu counters on the contraction kernel, 64 elements per point; flops executed "
               "(DMMA 512/inst incl. tile padding, DFMA 2, DMUL/DADD 1); slopes over p >= 5",
       "series": []}
for (sp, path), v in sorted(pts.items()):
    v.sort(key=lambda q: q["p_test"])
    hi = [q for q in v if q["p_test"] >= 5 and q["exec_dflop_per_element"] > 0]
    s = {"space": sp, "path": path, "points": v}
    if len(hi) >= 3:
        s["slope_exec_dflop"] = slope([q["p_test"] for q in hi], [q["exec_dflop_per_element"] for q in hi])
        # the operation counts are polynomials in L = p + 1 (digit extents p + 1, rule L):
        # p^7 / p^6 of the paper are the leading powers, reached in L
        s["slope_exec_dflop_vs_L"] = slope([q["p_test"] + 1 for q in hi], [q["exec_dflop_per_element"] for q in hi])
    out["series"].append(s)
print(json.dumps(out, indent=1))
