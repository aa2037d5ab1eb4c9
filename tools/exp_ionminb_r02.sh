#!/bin/bash
# r02 (after the rate folding): ionic occupancy caps -- TT2006 5 vs 6 CTAs/SM
# (96 vs 80 registers, 72 B spills), CRN 4 vs 5 (128 vs 96 registers, 16 B spills).
cd "$(dirname "$0")/.."
VARS="base: tt6:-DTCB_ION_MINB=6 crn5:-DTCB_ION_MINB_CRN=5"
if [ "$1" == "build" ]; then
  for v in $VARS; do n=${v%%:*}; f=$(echo ${v#*:} | tr + ' ')
    bash tools/build_variant.sh tools/im_$n.so $f; done; exit 0
fi
for rep in 1 2 3; do
  for W in slab10M_tt:base slab10M_tt:tt6 slab10M_crn:base slab10M_crn:crn5; do
    w=${W%%:*}; n=${W##*:}
    TCB200_LIB=tools/im_$n.so python bench.py --workload $w --steps 20 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$w $n', round(d['value']/1e9,4), 'ionic_ms', round(r['ionic_ms_per_step'],4), 'clk', d['clocks']['sm_mhz'], 'cyc_k', round(r['ionic_ms_per_step']*d['clocks']['sm_mhz'],1))"
  done
done
