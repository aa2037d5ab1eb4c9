#!/bin/bash
# PCG U phase: z-form (TCB_ZFORM=1: keep z only, 80n + 12nnz bytes per iteration)
# vs Algorithm 1's r and z (88n + 12nnz).  Libraries built by:
#   bash tools/build_variant.sh tools/pcg_zform.so -DTCB_ZFORM=1 ; bash tools/build_variant.sh tools/pcg_base.so
cd "$(dirname "$0")/.."
for W in slab20M_ms slab10M_tt; do
for v in base zform base zform; do
  TCB200_LIB=tools/pcg_$v.so python bench.py --workload $W --steps 20 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 --no-north-star | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W $v', round(d['value']/1e9,4), round(d['ms_per_step'],4), 'pcg_ms/it', round(r['pcg_ms_per_iter'],5), 'frac', round(r['frac'],4), 'iters', d['pcg_iters_per_step'], 'clk', d['clocks']['sm_mhz'])"
done
done
