#!/bin/bash
# PCG variants with the r02 kernel (z-form, merged x updates): 0 direct, 1 TMA-staged, 2 16-bit column offsets
cd "$(dirname "$0")/.."
for W in slab20M_ms slab10M_tt; do
for v in 0 2 1 0 2; do
  python bench.py --workload $W --steps 20 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 --no-north-star --pcg-variant $v | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W var $v', round(d['value']/1e9,4), round(d['ms_per_step'],4), 'pcg_ms/it', round(r['pcg_ms_per_iter'],5), 'frac', round(r['frac'],4), 'clk', d['clocks']['sm_mhz'])"
done
done
