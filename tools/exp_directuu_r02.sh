#!/bin/bash
# r02: slices per warp pass in the direct variant's U phase (TCB_DIRECT_UU).
cd "$(dirname "$0")/.."
VARS="uu1:-DTCB_DIRECT_UU=1 uu2:-DTCB_DIRECT_UU=2"
if [ "$1" == "build" ]; then
  for v in $VARS; do n=${v%%:*}; f=$(echo ${v#*:} | tr + ' ')
    bash tools/build_variant.sh tools/du_$n.so $f; done; exit 0
fi
for rep in 1 2 3; do
  for W in slab10M_tt slab20M_ms; do
    for v in $VARS; do
      n=${v%%:*}
      TCB200_LIB=tools/du_$n.so python bench.py --workload $W --steps 20 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 --no-north-star | \
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W $n', round(d['value']/1e9,4), 'frac', round(r['frac'],3), 'pcg_ms_it', round(r['pcg_ms_per_iter'],4), 'clk', d['clocks']['sm_mhz'])"
    done
  done
done
