"""Print the most-executed straight-line SASS block (the hot loop body) of an ncu report.

    python tools/ncu_hotloop.py report.ncu-rep [rank] [--ops DMMA]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 0
op = sys.argv[3] if len(sys.argv) > 3 else "DMMA"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
idx = {k: i for i, k in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        n = int(r[idx["Instructions Executed"]] or 0)
    except ValueError:
        continue
    data.append((r[idx["Address"]][-5:], r[idx["Source"]].strip(), n, int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)))
tot = sum(d[2] for d in data)
blocks = []
i = 0
while i < len(data):
    j = i
    while j + 1 < len(data) and data[j + 1][2] == data[i][2]:
        j += 1
    if data[i][2] > 0 and any(op in d[1] for d in data[i:j + 1]):
        blocks.append((sum(d[2] for d in data[i:j + 1]), i, j))
    i = j + 1
blocks.sort(reverse=True)
for k, (w, a, b) in enumerate(blocks[:8]):
    print(f"block {k}: {b - a + 1} instr x {data[a][2]} = {w / tot * 100:.1f}% of all instructions")
w, a, b = blocks[rank]
ops = collections.Counter(d[1].split()[1] if d[1].startswith("@") else d[1].split()[0] for d in data[a:b + 1])
print(ops.most_common(25))
for d in data[a:b + 1]:
    print(d[0], f"{d[3]:6d}", d[1])
