#!/bin/bash
# L2 bulk prefetch of the matrix slices D rounds ahead (TCB_XMERGE) in the direct PCG / RHS kernels
cd "$(dirname "$0")/.."
for W in slab20M_ms slab10M_tt biv3M_tt; do
for v in base xm base xm; do
  TCB200_LIB=tools/pcg_$v.so python bench.py --workload $W --steps 20 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 --no-north-star | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W $v', round(d['value']/1e9,4), round(d['ms_per_step'],4), 'pcg_ms/it', round(r['pcg_ms_per_iter'],5), 'frac', round(r['frac'],4), 'clk', d['clocks']['sm_mhz'])"
done
done
