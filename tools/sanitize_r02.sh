#!/bin/bash
# compute-sanitizer evidence: memcheck, racecheck,
# synccheck and initcheck on the small cases of tools/sanitize_case.py.
# Output: gpurun_out/r02_sanitize_<tool>.txt (one block per case).
cd "$(dirname "$0")/.."
CS=/usr/local/cuda/bin/compute-sanitizer
CASES="grid_v0 grid_v1 grid_v4 grid_v5 crn_grid cluster_res cluster_stream cohort peer3 split3 split3_ms"
for TOOL in memcheck racecheck synccheck initcheck; do
  OUT=gpurun_out/r02_sanitize_$TOOL.txt
  : > $OUT
  for C in $CASES; do
    echo "=== $TOOL $C" >> $OUT
    timeout 600 $CS --tool $TOOL --error-exitcode 9 --print-limit 20 python tools/sanitize_case.py $C >> $OUT 2>&1
    echo "=== exit $? ($TOOL $C)" >> $OUT
  done
done
