#!/bin/bash
# Node ordering vs PCG speed: RCM (default) vs the generator's natural lexicographic order
cd "$(dirname "$0")/.."
for W in slab20M_ms slab10M_tt; do for R in "" "--no-rcm"; do
  TCB200_LIB=${LIB:-} python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 $R | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W rcm=${R:-yes}', d['value'], d['ms_per_step'], 'pcg_ms_it', r['pcg_ms_per_iter'], 'frac', r['frac'], 'iters', d['pcg_iters_per_step'], 'nnz_pad', d['config'].get('nnz'))"
done; done
