#!/bin/bash
# cohorts of large members: members one after another (TCB_COHORT_SERIAL=1) vs sharing the GPU
cd "$(dirname "$0")/.."
for W in cohort8_nversion01_tt cohort8_sphere655k_ms; do
for mode in 1 0 1 0; do
  TCB_COHORT_SERIAL=$mode python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W serial=$mode', round(d['value']/1e9,4), round(d['ms_per_step'],4), 'frac', round(r['frac'],4), 'iters', d['pcg_iters_per_step'], 'clk', d['clocks']['sm_mhz'])"
done
done
