#!/bin/bash
# Ionic-kernel exp variants (TCB_EXP_NOINLINE, TCB_EXP_T64) on the TT2006 / CRN 10 M slabs
cd "$(dirname "$0")/.."
for W in slab10M_tt slab10M_crn; do for v in ${VARS:-ionbase ionnoinl iont64}; do
  TCB200_LIB=tools/sp_$v.so python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 --preroll 200 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W $v', d['value'], d['ms_per_step'], 'ionic_ms', r['ionic_ms_per_step'])"
done; done
