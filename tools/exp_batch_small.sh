#!/bin/bash
# Variant 4 with a batch of 8 for narrow slices (TCB_BATCH_SMALL) on surface and tet meshes
cd "$(dirname "$0")/.."
for W in sphere655k_ms nversion_dx0.1_tt; do for v in ${VARS:-bs0 bs1}; do
  TCB200_LIB=tools/sp_$v.so python bench.py --workload $W --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W $v', d['config']['pcg_variant'], d['value'], d['ms_per_step'], 'pcg_ms_it', r['pcg_ms_per_iter'], 'frac', r['frac'])"
done; done
