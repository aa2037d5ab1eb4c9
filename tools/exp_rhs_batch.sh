#!/bin/bash
# Variant 4's RHS row product: direct loop (0) vs NB slots in flight, configs[2]
cd "$(dirname "$0")/.."
for v in ${VARS:-rhs0 rhs4 rhs8 rhs16}; do
  TCB200_LIB=tools/sp_$v.so python bench.py --workload nversion_dx0.1_tt --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$v', d['config']['pcg_variant'], d['value'], d['ms_per_step'], 'pcg_ms_it', r['pcg_ms_per_iter'], 'frac', r['frac'])"
done
