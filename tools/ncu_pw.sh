#!/bin/bash
# ncu --set full of the general-map contraction kernel for given workloads (env WLS, ELEM)
cd "$(dirname "$0")/.."
for w in ${WLS}; do
  ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-general_} -s 1 -c 1 \
      -o gpurun_out/ncu_$w -f python tools/prof_one.py $w --elements ${ELEM:-128} --reps 2 > gpurun_out/ncu_$w.log 2>&1
  tail -2 gpurun_out/ncu_$w.log
done
