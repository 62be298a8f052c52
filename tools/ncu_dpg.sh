#!/bin/bash
# ncu --set full of the DPG-layer kernels (one launch each), after a plain run.
cd "$(dirname "$0")/.."
for wk in graph:graph_assemble condense:condense_kernel acoustics:acoustics_block; do
  w=${wk%%:*}; k=${wk##*:}
  python tools/prof_dpg.py $w > gpurun_out/plain_dpg_$w.log 2>&1 || { echo "plain failed $w"; continue; }
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_dpg_$w -f \
      python tools/prof_dpg.py $w > gpurun_out/ncu_dpg_$w.log 2>&1
  echo "$w: $(tail -1 gpurun_out/ncu_dpg_$w.log)"
done
