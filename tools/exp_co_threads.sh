#!/bin/bash
# Cluster-engine CTA size (TCB_CO_THREADS 256 vs 512) on configs[0] and the cohort workload
cd "$(dirname "$0")/.."
for v in co256 co512; do
  for W in nversion_dx0.5_tt cohort100_nversion05_tt; do
    TCB200_LIB=tools/sp_$v.so python bench.py --workload $W --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $W', d['value'], d['ms_per_step'], d.get('pcg_iters_per_step'))"
  done
done
