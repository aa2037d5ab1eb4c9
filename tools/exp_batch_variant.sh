#!/bin/bash
# Variant 4 (latency PCG kernel) knobs on configs[2] (auto picks variant 4 there)
cd "$(dirname "$0")/.."
for v in ${VARS:-uu4 uu1 nb8uu1 uu2}; do
  TCB200_LIB=tools/sp_$v.so python bench.py --workload nversion_dx0.1_tt --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', d['config']['pcg_variant'], d['value'], d['ms_per_step'], 'pcg_ms_it', r['pcg_ms_per_iter'], 'frac', r['frac'])"
done
