#!/bin/bash
# One `ncu --set full` capture of the dominant kernel of every BASELINE config
# (+ the extrusion workload); each workload first runs once without ncu.
# Writes gpurun_out/prof_<workload>.ncu-rep; tools/ncu_traffic.py summarises.
cd "$(dirname "$0")/.."
for wk in ${WLS:-c1_h1_p3_affine:affine_v2 c2_h1_p5_general:general_v3 c3_hcurl_p6_general:general_v3 c3_hcurl_p6_affine:affine_v2 c4_hdiv_p7_general:general_v3 c4_l2_p7_general:general_v3 x_hcurl_p6_extrusion:ext_v2}; do
  w=${wk%%:*}; k=${wk##*:}
  EA=""; case $w in c5_*|x5_*) EA="--elements ${ELEM:-128}";; esac
  python tools/prof_one.py $w $EA --reps 2 > gpurun_out/plain_$w.log 2>&1 || { echo "plain run failed: $w"; continue; }
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$w -f \
      python tools/prof_one.py $w $EA --reps 2 > gpurun_out/ncu_$w.log 2>&1
  echo "$w: $(tail -1 gpurun_out/ncu_$w.log)"
done
