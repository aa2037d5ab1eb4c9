#!/bin/bash
# ionic || RHS pipeline: chunks x RHS-stream priority
cd "$(dirname "$0")/.."
for W in slab10M_tt slab10M_crn biv3M_tt; do
for cfg in "0 0" "4 0" "8 0" "16 0" "8 1" "16 1" "0 0"; do
  set -- $cfg
  TCB_ION_RHS_CHUNKS=$1 TCB_RHS_PRIO=$2 python bench.py --workload $W --steps 20 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W chunks=$1 prio=$2', round(d['value']/1e9,4), round(d['ms_per_step'],4), 'ion+rhs' if $1 else 'ionic', round(r['ionic_ms_per_step'],4), 'pcg', round(r['pcg_ms_per_step'],4), 'frac', round(r['frac'],4), 'clk', d['clocks']['sm_mhz'])"
done
done
