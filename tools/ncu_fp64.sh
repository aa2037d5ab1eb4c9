#!/bin/bash
# FP64 instruction counts of the ionic kernels (first timed step) -> gpurun_out/${R}_fp64ops_${W}.csv
R=${1:-r01}
cd "$(dirname "$0")/.."
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
for W in slab10M_tt slab10M_crn; do
  E="python bench.py --workload $W --steps 2 --warmup 3 --windows 1 --no-cpu-baseline --e2e-steps 1"
  $E > gpurun_out/${R}_plain_fp64_$W.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:"ionic_" -s 503 -c 1 --csv --log-file gpurun_out/${R}_fp64ops_$W.csv $E \
      > gpurun_out/${R}_ncu_fp64_$W.log 2>&1
done
