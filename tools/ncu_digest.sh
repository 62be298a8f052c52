#!/bin/bash
# On the GPU box: turn every gpurun_out/*.ncu-rep into text digests (summary JSON,
# per-source-line stall totals, hot SASS loop) and delete the report unless KEEP=1 --
# gpurun only brings back gpurun_out/ when it is under 64 MiB.
cd "$(dirname "$0")/.."
TAG=${TAG:-r02}
python tools/ncu_traffic.py $TAG gpurun_out > gpurun_out/ncu_traffic.txt 2>&1
for rep in gpurun_out/*.ncu-rep; do
  [ -f "$rep" ] || continue
  b=$(basename "$rep" .ncu-rep)
  python tools/ncu_summary.py "$rep" --json gpurun_out/${b}_${TAG}_summary.json > gpurun_out/${b}_${TAG}_summary.txt 2>&1
  python tools/ncu_lines.py "$rep" 60 > gpurun_out/${b}_${TAG}_lines.txt 2>&1
  python tools/ncu_hotloop.py "$rep" 0 > gpurun_out/${b}_${TAG}_hotloop.txt 2>&1
  [ "${KEEP:-0}" = 1 ] || rm -f "$rep"
done
du -sh gpurun_out | tail -1
