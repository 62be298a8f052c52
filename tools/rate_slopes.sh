#!/bin/bash
# Executed FP64 work and DRAM bytes per element vs test order p (the algorithmic-rate
# evidence: general ~ p^7, affine ~ p^6): one ncu metrics pass per sweep point on the
# contraction kernel, E = 64 elements.  tools/rate_slopes.py summarises the CSVs.
cd "$(dirname "$0")/.."
M=sm__inst_executed_pipe_tensor_subpipe_dmma.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum
for sp in ${SPACES:-hcurl hdiv h1}; do for path in general affine; do for p in 2 3 4 5 6 7 8 9 10; do
  w=c5_${sp}_p${p}_${path}
  k=$([ $path = general ] && echo "regex:general_" || echo "regex:affine_v2")
  ncu --metrics $M --clock-control none -k $k -c 1 --csv python tools/prof_one.py $w --elements 64 --reps 1 \
      > gpurun_out/rate_$w.csv 2> gpurun_out/rate_$w.err
done; done; done
