#!/bin/bash
# r02 ionic A/B: merged rate quotients (TCB_ION_FOLD=1, default) vs the literal
# forms (0).  Build here:  bash tools/exp_fold_r02.sh build ; run on the box:
#   bash tools/exp_fold_r02.sh   -> ionic ms/step at 10 M nodes (TT2006, CRN)
cd "$(dirname "$0")/.."
VARS="fold0:-DTCB_ION_FOLD=0 fold1:-DTCB_ION_FOLD=1"
if [ "$1" == "build" ]; then
  for v in $VARS; do n=${v%%:*}; f=$(echo ${v#*:} | tr + ' ')
    bash tools/build_variant.sh tools/ion_$n.so $f; done; exit 0
fi
for W in slab10M_tt slab10M_crn; do
for v in $VARS $VARS $VARS; do
  n=${v%%:*}
  TCB200_LIB=tools/ion_$n.so python bench.py --workload $W --steps 20 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W $n', round(d['value']/1e9,4), round(d['ms_per_step'],4), 'ionic_ms', round(r['ionic_ms_per_step'],4), 'clk', d['clocks']['sm_mhz'])"
done
done
