"""Per-CUDA-source-line instruction / stall-sample totals from an ncu report
(needs -lineinfo and --import-source on).

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [topN]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
cur_file = None
hdr = None
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        idx = {k: i for i, k in enumerate(hdr)}
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        cur_line = (cur_file, int(r[0]), r[1].strip()[:70])
    try:
        n = int(r[idx["Instructions Executed"]] or 0)
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, KeyError):
        continue
    a = agg.setdefault(cur_line, [0, 0])
    a[0] += n
    a[1] += s
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]:22s}{k[1]:5d} inst {n / ti * 100:5.1f}% samples {s / ts * 100:5.1f}%  {k[2]}")
