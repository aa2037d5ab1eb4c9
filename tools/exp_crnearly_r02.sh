#!/bin/bash
# r02 (after the rate folding): CRN state loads before the table copy (TCB_ION_EARLY_LOADS_CRN).
cd "$(dirname "$0")/.."
VARS="late:-DTCB_ION_EARLY_LOADS_CRN=0 early:-DTCB_ION_EARLY_LOADS_CRN=1"
if [ "$1" == "build" ]; then
  for v in $VARS; do n=${v%%:*}; f=$(echo ${v#*:} | tr + ' ')
    bash tools/build_variant.sh tools/ce_$n.so $f; done; exit 0
fi
for rep in 1 2 3; do
  for v in $VARS; do
    n=${v%%:*}
    TCB200_LIB=tools/ce_$n.so python bench.py --workload slab10M_crn --steps 20 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('slab10M_crn $n', round(d['value']/1e9,4), 'ionic_ms', round(r['ionic_ms_per_step'],4), 'clk', d['clocks']['sm_mhz'], 'cyc_k', round(r['ionic_ms_per_step']*d['clocks']['sm_mhz'],1))"
  done
done
