#!/bin/bash
cd "$(dirname "$0")/.."
for W in slab20M_ms slab10M_tt; do
  for vv in gp0:0 gp0:5 gp1m4:5 gp1m3:5; do v=${vv%%:*}; V=${vv#*:}
  TCB200_LIB=tools/sp_$v.so python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 --pcg-variant $V | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W $v v$V', d['value'], d['ms_per_step'], 'pcg_ms_it', r['pcg_ms_per_iter'], 'frac', r['frac'], 'iters', d['pcg_iters_per_step'])"
  done
done
