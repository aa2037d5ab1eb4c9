#!/bin/bash
# Graph engine (variant 5: init / WHILE{S, U} / final kernels) vs the persistent
# kernel (variant 0), with and without the slot-pair SELL layout
cd "$(dirname "$0")/.."
for W in ${WORKLOADS:-slab20M_ms slab10M_tt biv3M_tt sphere2.6M_ms}; do
for v in ${VARS:-gp0 gp1}; do for V in 0 5; do
  TCB200_LIB=tools/sp_$v.so python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 --pcg-variant $V | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W $v v$V', d['value'], d['ms_per_step'], 'pcg_ms_it', r['pcg_ms_per_iter'], 'frac', r['frac'], 'iters', d['pcg_iters_per_step'], 'launches', d['gpu_launches'])"
done; done; done
