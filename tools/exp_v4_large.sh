#!/bin/bash
# Variant 4 vs 0 on the larger surface mesh and the BiV mesh (crossover check)
cd "$(dirname "$0")/.."
for W in sphere2.6M_ms biv3M_tt; do for V in 0 4; do
  TCB200_LIB=tools/sp_bs1.so python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 --pcg-variant $V | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W v$V', d['value'], d['ms_per_step'], 'pcg_ms_it', r['pcg_ms_per_iter'], 'frac', r['frac'])"
done; done
