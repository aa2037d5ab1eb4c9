#!/bin/bash
# variant 4 with the RHS fused into the cooperative kernel (TCB_FUSE_RHS4) vs two launches
cd "$(dirname "$0")/.."
for W in nversion_dx0.1_tt sphere655k_ms; do
for v in base fuse base fuse; do
  TCB200_LIB=tools/pcg_$v.so python bench.py --workload $W --steps 50 --warmup 5 --windows 3 --no-cpu-baseline --e2e-steps 0 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W $v', round(d['value']/1e9,4), round(d['ms_per_step'],5), 'frac', round(r['frac'],4), 'clk', d['clocks']['sm_mhz'])"
done
done
