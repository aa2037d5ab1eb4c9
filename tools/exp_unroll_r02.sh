#!/bin/bash
# r02: direct variant's slot-loop unroll (TCB_S_UNROLL) and a per-parity S phase
# (TCB_S_PARITY: p_it / p_{it-1} as kernel-parameter pointers) -- register pressure
# of the 32-register kernel (ptxas: ~100 bytes of spills).
cd "$(dirname "$0")/.."
VARS="u4:-DTCB_S_UNROLL=4 u2:-DTCB_S_UNROLL=2 u8:-DTCB_S_UNROLL=8 par:-DTCB_S_PARITY=1 paru2:-DTCB_S_PARITY=1+-DTCB_S_UNROLL=2"
if [ "$1" == "build" ]; then
  for v in $VARS; do n=${v%%:*}; f=$(echo ${v#*:} | tr + ' ')
    bash tools/build_variant.sh tools/un_$n.so $f; done; exit 0
fi
for rep in 1 2; do
for W in slab10M_tt slab20M_ms; do
for v in $VARS; do
  n=${v%%:*}
  TCB200_LIB=tools/un_$n.so python bench.py --workload $W --steps 20 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W $n', round(d['value']/1e9,4), 'frac', round(r['frac'],3), 'pcg_ms_it', round(r['pcg_ms_per_iter'],4), 'clk', d['clocks']['sm_mhz'])"
done
done
done
